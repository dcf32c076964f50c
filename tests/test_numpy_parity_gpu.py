"""GPU vs the reference's CPU matmul (np.matmul fp32, numpy being the reference
package's only numeric engine), as the north-star states the GEMM contract: "outputs
must match the reference's CPU matmul on the same inputs within a stated relative
tolerance".

Stated fp32 tolerance: both results lie within 2*k*u*(|A||B|) of the exact product
(u = 2^-24, any summation order), so per element
    |C_gpu - C_np| <= 4*k*u*(|A||B|)_ij
and normwise ||C_gpu - C_np||_F / ||C_np||_F <= 1e-5.

Also: GemmOperands rejects an ``out`` that the kernel could overrun or that lives on
another device."""

import numpy as np
import pytest
import torch

from paper_2008_13145_b200 import gemm, shapes
from paper_2008_13145_b200.dataset import KernelConfig, ProblemSize

pytestmark = pytest.mark.gpu

U = 2.0 ** -24
C1 = KernelConfig(4, 4, 4, 16, 16)  # BASELINE configs[0]: "one tile config" at 256^3


def _compare(C, A, B, k, what):
    ref = np.matmul(A, B)
    mag = np.matmul(np.abs(A), np.abs(B)) * (1 + 2 * k * U)  # fp32 |A||B|, rounded up
    err = np.abs(C.astype(np.float64) - ref.astype(np.float64))
    worst = float((err / (4 * k * U * mag + 1e-30)).max())
    assert worst <= 1.0, f"{what}: {worst:.3f} x the elementwise bound"
    rel = float(np.linalg.norm(C - ref) / np.linalg.norm(ref))
    assert rel <= 1e-5, f"{what}: normwise {rel:.2e}"
    return rel


@pytest.mark.parametrize("family", ["simt", "paper"])
def test_c1_256_cubed_matches_numpy(cuda_device, family):
    rng = np.random.default_rng(0)  # SURVEY 8(d) C1 inputs: U(-1, 1), seed 0
    A = rng.uniform(-1, 1, (256, 256)).astype(np.float32)
    B = rng.uniform(-1, 1, (256, 256)).astype(np.float32)
    C = gemm.matmul(torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device), C1, family)
    _compare(C.cpu().numpy(), A, B, 256, f"{family}{C1.as_tuple()} 256^3")


def test_vgg16_b16_layer_shapes_match_numpy(cuda_device):
    """Every unique VGG16 GEMM layer at batch 16 (the bench workload's shapes) with the C1
    config and with the bench's tree-dispatched variant."""
    import bench
    from paper_2008_13145_b200.dispatch import Dispatcher

    pm, subset, tree, *_ = bench.train_selector(str(bench.DEFAULT_TABLE), 4, "kmeans", "treeA")
    disp = Dispatcher(tree, subset, pm.configs, "simt")
    rng = np.random.default_rng(16)
    for layer in shapes.VGG16_LAYERS:
        p = layer.problem(16)
        A = rng.uniform(-1, 1, (p.m, p.k)).astype(np.float32)
        B = (rng.uniform(-1, 1, (p.k, p.n)) * np.sqrt(6.0 / p.k)).astype(np.float32)
        dA, dB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
        _compare(gemm.matmul(dA, dB, C1, "simt").cpu().numpy(), A, B, p.k, f"{layer.name} simt{C1.as_tuple()}")
        _compare(disp.matmul(dA, dB).cpu().numpy(), A, B, p.k, f"{layer.name} dispatched {disp.select(p).as_tuple()}")
        del dA, dB


def test_paper_sample_problems_match_numpy(cuda_device):
    """The paper's three sample problems (shapes.PAPER_SAMPLES)
    -- batched m=512 k=784 n=512 x16, rectangular 512x4608x784 and the long accumulation
    32x12321x27 (unaligned rows) -- on the row-best SIMT config of the measured table and
    the C1 config, against np.matmul fp32 per batch."""
    from paper_2008_13145_b200.dataset import parse_benchmark_csv
    import bench

    pm = parse_benchmark_csv(bench.DEFAULT_TABLE.read_text())
    rng = np.random.default_rng(284)
    for p in shapes.PAPER_SAMPLES:
        best = pm.configs[int(pm.values[list(pm.problems).index(p)].argmax())]
        A = rng.uniform(-1, 1, (p.batch, p.m, p.k)).astype(np.float32)
        B = rng.uniform(-1, 1, (p.batch, p.k, p.n)).astype(np.float32)
        dA, dB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
        for cfg in (best, C1):
            C = gemm.matmul(dA, dB, cfg, "simt").cpu().numpy()
            for b in range(p.batch):
                _compare(C[b], A[b], B[b], p.k, f"{p} simt{cfg.as_tuple()} batch {b}")


def test_out_must_not_be_overrun_or_foreign(cuda_device):
    dev = cuda_device
    A = torch.rand(3, 8, 5, device=dev)
    B = torch.rand(5, 6, device=dev)
    with pytest.raises(ValueError, match="3-D out"):
        gemm.matmul(A, B, C1, out=torch.empty(8, 6, device=dev))  # batch 3 into one (m, n) buffer
    with pytest.raises(ValueError, match="batch"):
        gemm.matmul(A, B, C1, out=torch.empty(2, 8, 6, device=dev))
    with pytest.raises(ValueError):
        gemm.matmul(A, B, C1, out=torch.empty(1, 3, 8, 6, device=dev))
    with pytest.raises(ValueError, match="CUDA"):
        gemm.matmul(A[0], B, C1, out=torch.empty(8, 6))  # host memory
    with pytest.raises(ValueError):
        gemm.matmul(A[0], B.cpu(), C1)
    good = torch.empty(3, 8, 6, device=dev)
    gemm.matmul(A, B, C1, out=good)
    assert torch.allclose(good, A @ B, rtol=1e-5, atol=1e-5)
    if torch.cuda.device_count() > 1:
        with pytest.raises(ValueError, match="CUDA tensor on"):
            gemm.matmul(A[0], B, C1, out=torch.empty(8, 6, device="cuda:1"))


def test_dispatcher_matmul_validates_out_too(cuda_device):
    import bench
    from paper_2008_13145_b200.dispatch import Dispatcher

    pm, subset, tree, *_ = bench.train_selector(str(bench.DEFAULT_TABLE), 4, "kmeans", "treeA")
    disp = Dispatcher(tree, subset, pm.configs, "simt")
    A = torch.rand(2, 16, 32, device=cuda_device)
    B = torch.rand(32, 8, device=cuda_device)
    with pytest.raises(ValueError):
        disp.matmul(A, B, out=torch.empty(16, 8, device=cuda_device))
    assert disp.matmul(A, B).shape == (2, 16, 8)
    assert ProblemSize(16, 32, 8, 2) in disp._cache
