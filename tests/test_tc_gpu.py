"""GPU: the tcgen05 tensor-core families (F2 TF32, F3 BF16) against the CPU oracle's
float64 product (oracle/gemm_ref.c kp_ref_gemm_f64, the restatement of np.matmul on
float64 operands) of the same operands (bf16 operands are exact in fp32).

Stated tolerances (widened for TF32 truncation: tcgen05 kind::tf32
reads the top 19 bits of each fp32 operand):
    TF32: |C - C64| <= (2 * 2^-10 + 2*k*2^-24) * (|A||B|)_ij
    BF16: |C - C64| <= (2*k*2^-24) * (|A_bf16||B_bf16|)_ij  (inputs exact in bf16)
"""

import numpy as np
import pytest
import torch

from oracle import gemm_oracle as go
from paper_2008_13145_b200 import gemm
from paper_2008_13145_b200.dataset import KernelConfig

pytestmark = pytest.mark.gpu

U = 2.0 ** -24


_REF: dict = {}


def _reference(key, A, B):
    """(float64 product, |A||B|) from the CPU oracle, once per operand set."""
    if key not in _REF:
        _REF.clear()  # one shape at a time: the products of big shapes are large
        A32 = A.float().cpu().numpy()
        B32 = B.float().cpu().numpy()
        _REF[key] = go.gemm_f64(A32, B32)
    return _REF[key]


def _check(fam, cfg, m, k, n, batch, dev, bcast=False, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    A = torch.rand(batch, m, k, device=dev, generator=g) * 2 - 1
    B = torch.rand(k, n, device=dev, generator=g) * 2 - 1
    if not bcast:
        B = B.expand(batch, k, n).contiguous() + torch.rand(batch, k, n, device=dev, generator=g) * 0.1
    if fam == "bf16":
        A, B = A.bfloat16(), B.bfloat16()
        eps_in = 0.0
    else:
        eps_in = 2.0 * 2.0 ** -10
    C = gemm.matmul(A, B, cfg, fam).cpu().numpy().astype(np.float64)
    ref, mag = _reference((fam, m, k, n, batch, bcast, seed), A, B)
    bound = (eps_in + 2 * k * U) * mag.reshape(C.shape) + 1e-30
    worst = float((np.abs(C - ref.reshape(C.shape)) / bound).max())
    assert worst <= 1.0, f"{fam} {cfg.as_tuple()} {m}x{k}x{n}x{batch}: error {worst:.3f} x bound"


@pytest.mark.parametrize("fam", ["bf16", "tf32"])
def test_every_config_square(cuda_device, fam):
    for cfg in gemm.family_configs(fam):
        _check(fam, cfg, 256, 256, 256, 1, cuda_device)


@pytest.mark.parametrize("fam", ["bf16", "tf32"])
@pytest.mark.parametrize("m,k,n,batch", [(1, 64, 64, 1), (130, 72, 200, 1), (1000, 576, 64, 2), (49, 4608, 512, 1),
                                         (333, 1000, 1000, 1), (16, 8, 8, 3), (2048, 2048, 2048, 1),
                                         (4096, 512, 2048, 1), (1000, 256, 1000, 3)])
def test_ragged_and_batched(cuda_device, fam, m, k, n, batch):
    for cfg in gemm.family_configs(fam)[::3]:
        _check(fam, cfg, m, k, n, batch, cuda_device, bcast=(batch > 1), seed=m + n)


@pytest.mark.parametrize("fam", ["bf16", "tf32"])
@pytest.mark.parametrize("m,k,n,batch", [(64, 27, 64, 1), (1000, 147, 64, 1), (77, 33, 45, 2), (5, 1, 3, 1)])
@pytest.mark.parametrize("repack", ["always", "never", "auto"])
def test_unaligned_rows(cuda_device, fam, m, k, n, batch, repack):
    """Rows that TMA cannot address (k*elem or n*elem not a multiple of 16 B): copied into
    16-byte-pitched scratch for the TMA path, or staged in-kernel by the LSU loaders
    (kp_set_operand_repack); same tolerance either way (grid totality,
    dataset.py:259-264)."""
    prev = gemm.set_operand_repack(repack)
    try:
        for cfg in gemm.family_configs(fam)[::2]:
            _check(fam, cfg, m, k, n, batch, cuda_device, bcast=(batch > 1), seed=k)
    finally:
        gemm.set_operand_repack(prev)


@pytest.mark.parametrize("fam", ["bf16", "tf32"])
@pytest.mark.parametrize("m,k,n,batch", [(196, 4608, 512, 1), (32, 25088, 1024, 1), (100, 3000, 200, 2),
                                         (64, 2001, 64, 1), (128, 2048, 33, 1)])
def test_k_sliced_tensor_core(cuda_device, fam, m, k, n, batch):
    """Under-filled launches slice k over a thread-block cluster (kp_gemm_plan) and sum
    the slices through DSMEM: every config within the bound, deterministic run to run
    (k = 2001 and n = 33 rows are unaligned, so they also exercise LSU staging)."""
    from paper_2008_13145_b200.dataset import ProblemSize
    sliced = 0
    for cfg in gemm.family_configs(fam):
        s, kps = gemm.k_slice_plan(cfg, ProblemSize(m, k, n, batch), family=fam)
        sliced += s > 1
        _check(fam, cfg, m, k, n, batch, cuda_device, bcast=(batch > 1), seed=k)
    assert sliced > 0
    g = torch.Generator(device=cuda_device).manual_seed(9)
    A = torch.rand(m, k, device=cuda_device, generator=g)
    B = torch.rand(k, n, device=cuda_device, generator=g)
    if fam == "bf16":
        A, B = A.bfloat16(), B.bfloat16()
    cfg = gemm.family_configs(fam)[1]
    assert torch.equal(gemm.matmul(A, B, cfg, fam), gemm.matmul(A, B, cfg, fam))


@pytest.mark.parametrize("fam", ["bf16", "tf32"])
def test_k_sliced_epilogue(cuda_device, fam):
    """bias + ReLU applied once, after the slice sum."""
    from paper_2008_13145_b200 import _lib
    from paper_2008_13145_b200.dataset import ProblemSize
    m, k, n = 200, 4096, 256
    g = torch.Generator(device=cuda_device).manual_seed(4)
    A = torch.rand(m, k, device=cuda_device, generator=g) * 2 - 1
    B = torch.rand(k, n, device=cuda_device, generator=g) * 2 - 1
    bias = torch.rand(n, device=cuda_device, generator=g) * 2 - 1
    if fam == "bf16":
        A, B = A.bfloat16(), B.bfloat16()
    cfg = gemm.family_configs(fam)[2]
    assert gemm.k_slice_plan(cfg, ProblemSize(m, k, n, 1), family=fam)[0] > 1
    plain = gemm.matmul(A, B, cfg, fam)
    C = torch.empty(m, n, device=cuda_device)
    vid = gemm.variant_id(cfg, fam)
    _lib.check(_lib.load().kp_gemm_ex(vid, m, k, n, 1, A.data_ptr(), k, 0, B.data_ptr(), n, 0, C.data_ptr(), n, 0,
                                      bias.data_ptr(), _lib.KP_EPI_RELU, torch.cuda.current_stream().cuda_stream),
               "kp_gemm_ex")
    assert torch.equal(C, torch.relu(plain + bias))


@pytest.mark.parametrize("fam,m,k,n,batch", [("tf32", 2560, 4096, 4096, 1), ("bf16", 2560, 8192, 4096, 1),
                                              ("tf32", 640, 4096, 4096, 4)])
def test_partial_last_wave_split(cuda_device, fam, m, k, n, batch):
    """Grids of more than one wave whose last wave fills at most half the SMs run the tail
    tiles as a second, k-sliced launch: every config within the bound, deterministic."""
    from paper_2008_13145_b200.dataset import ProblemSize
    split = 0
    for cfg in gemm.family_configs(fam):
        split += gemm.k_slice_plan(cfg, ProblemSize(m, k, n, batch), family=fam)[0] > 1
        _check(fam, cfg, m, k, n, batch, cuda_device, bcast=(batch > 1), seed=n)
    assert split > 0
    g = torch.Generator(device=cuda_device).manual_seed(2)
    dt = torch.bfloat16 if fam == "bf16" else torch.float32
    A = (torch.rand(m, k, device=cuda_device, generator=g) - 0.5).to(dt)
    B = (torch.rand(k, n, device=cuda_device, generator=g) - 0.5).to(dt)
    cfg = gemm.family_configs(fam)[2]
    assert torch.equal(gemm.matmul(A, B, cfg, fam), gemm.matmul(A, B, cfg, fam))


@pytest.mark.parametrize("fam", ["bf16", "tf32"])
@pytest.mark.parametrize("m,k,n,batch", [(256, 256, 256, 1), (300, 520, 392, 1), (1000, 576, 256, 2),
                                         (2048, 2048, 2048, 1), (4096, 1024, 4096, 1), (3136, 4608, 512, 1),
                                         (700, 64, 1000, 1)])
def test_cta_pair_configs(cuda_device, fam, m, k, n, batch):
    """tile_rows = 256 configs run CTA pairs (tcgen05.mma.cta_group::2, each SM staging
    half the operands) on persistent TMA launches: within the bound on ragged m/n tails
    (a pair's second CTA partly or wholly past m), batches and long k; deterministic."""
    pairs = [c for c in gemm.family_configs(fam) if c.tile_rows == 256]
    assert len(pairs) >= 3
    for cfg in pairs:
        _check(fam, cfg, m, k, n, batch, cuda_device, bcast=(batch > 1), seed=m + k)
    g = torch.Generator(device=cuda_device).manual_seed(5)
    dt = torch.bfloat16 if fam == "bf16" else torch.float32
    A = (torch.rand(m, k, device=cuda_device, generator=g) - 0.5).to(dt)
    B = (torch.rand(k, n, device=cuda_device, generator=g) - 0.5).to(dt)
    assert torch.equal(gemm.matmul(A, B, pairs[0], fam), gemm.matmul(A, B, pairs[0], fam))
