"""GPU: the implicit-GEMM 3x3 convolution (kp_conv3x3_nhwc_ex -- TMA im2col copies
straight from the NHWC activation) equals im2col + the same GEMM variant bit for bit,
and both equal the oracle (numpy im2col + the fmaf chain of the launch's k-slice plan),
for every SIMT config that supports it; shapes whose pixel runs cross image rows and
images, ragged m tails, fused bias + ReLU."""

import numpy as np
import pytest
import torch

from oracle import gemm_oracle as go
from oracle import vgg16_ref
from paper_2008_13145_b200 import _lib, gemm
from paper_2008_13145_b200.dataset import KernelConfig, ProblemSize, enumerate_configs

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.ascontiguousarray(x).view(np.uint32)


@pytest.mark.parametrize("B,H,W,C,cout", [(2, 9, 7, 32, 64), (1, 14, 14, 64, 128), (3, 5, 6, 16, 48)])
def test_implicit_conv_all_configs_bit_exact(cuda_device, B, H, W, C, cout):
    rng = np.random.default_rng(B * 100 + C)
    x = rng.standard_normal((B, H, W, C)).astype(np.float32)
    w = (rng.standard_normal((9 * C, cout)) * 0.1).astype(np.float32)
    bias = (rng.standard_normal(cout) * 0.1).astype(np.float32)
    dx, dw, db = (torch.from_numpy(a).to(cuda_device) for a in (x, w, bias))
    cols = torch.from_numpy(vgg16_ref.im2col3x3(x)).to(cuda_device)
    prob = ProblemSize(B * H * W, 9 * C, cout, 1)
    lib = _lib.load()
    checked, bad, cache = 0, [], {}
    for cfg in enumerate_configs():
        vid = gemm.variant_id(cfg, "simt")
        if not gemm.conv3x3_supported(vid, C, cout):
            continue
        got = gemm.conv3x3(dx, dw, vid, bias=db, relu=True).cpu().numpy().reshape(-1, cout)
        ref = torch.empty(prob.m, cout, device=cuda_device)
        assert lib.kp_gemm_ex(vid, prob.m, prob.k, cout, 1, cols.data_ptr(), prob.k, 0, dw.data_ptr(), cout, 0,
                              ref.data_ptr(), cout, 0, db.data_ptr(), _lib.KP_EPI_RELU, None) == 0
        kps = gemm.k_slice_plan(vid, prob)[1]
        if kps not in cache:
            y = go.gemm_sliced(vgg16_ref.im2col3x3(x), w, kps)[0]
            cache[kps] = _bits(np.maximum(y + bias, np.float32(0.0)))
        if not (np.array_equal(_bits(got), _bits(ref.cpu().numpy())) and np.array_equal(_bits(got), cache[kps])):
            bad.append(cfg.as_tuple())
        checked += 1
    assert checked > (300 if C % 32 == 0 else 60), checked
    assert not bad, f"{len(bad)} configs differ, e.g. {bad[:5]}"


def test_implicit_conv_rejects_ineligible(cuda_device):
    lib = _lib.load()
    vid = gemm.variant_id(KernelConfig(8, 8, 8, 16, 8), "simt")
    x = torch.zeros(1, 8, 8, 3, device=cuda_device)
    w = torch.zeros(27, 64, device=cuda_device)
    out = torch.zeros(1, 8, 8, 64, device=cuda_device)
    assert not gemm.conv3x3_supported(vid, 3, 64)  # C = 3 is not a multiple of the k-tile
    assert lib.kp_conv3x3_nhwc_ex(vid, x.data_ptr(), 1, 8, 8, 3, w.data_ptr(), 64, out.data_ptr(), None, 0,
                                  None) == _lib.KP_EINVAL
    with pytest.raises(ValueError):
        gemm.conv3x3(x, w[:26], vid)


def test_implicit_conv_large_layer_matches_explicit(cuda_device):
    """VGG16 conv3_2 at batch 4 (m = 12544, k = 2304): implicit == explicit, bitwise."""
    g = torch.Generator(device=cuda_device).manual_seed(3)
    x = torch.randn(4, 56, 56, 256, device=cuda_device, generator=g)
    w = torch.randn(9 * 256, 256, device=cuda_device, generator=g) * 0.02
    lib = _lib.load()
    cols = torch.empty(4 * 56 * 56, 9 * 256, device=cuda_device)
    assert lib.kp_im2col3x3_nhwc(x.data_ptr(), 4, 56, 56, 256, cols.data_ptr(), 9 * 256, None) == 0
    for cfg in (KernelConfig(8, 8, 8, 16, 8), KernelConfig(8, 1, 8, 8, 16), KernelConfig(4, 2, 8, 16, 8)):
        vid = gemm.variant_id(cfg, "simt")
        got = gemm.conv3x3(x, w, vid).reshape(-1, 256)
        want = gemm.matmul(cols, w, cfg, "simt")
        assert torch.equal(got.view(torch.int32), want.view(torch.int32)), cfg


@pytest.mark.parametrize("B,H,W,C,cout", [(2, 9, 7, 32, 64), (1, 14, 14, 64, 128), (3, 28, 28, 256, 96),
                                         (16, 14, 14, 512, 512)])
def test_tf32_implicit_conv_equals_explicit(cuda_device, B, H, W, C, cout):
    """TF32 family: the tcgen05 producer loads 128-byte-swizzled TMA im2col boxes of 32
    channels x 128 pixels instead of the tiled A box -- the same operand tiles in shared
    memory, the same MMA sequence and k-slice plan, so the output equals im2col + the same
    TF32 variant bit for bit (fused bias + ReLU), and stays within the TF32 bound of the
    float64 product."""
    g = torch.Generator(device=cuda_device).manual_seed(B * 7 + C)
    x = torch.randn(B, H, W, C, device=cuda_device, generator=g)
    w = torch.randn(9 * C, cout, device=cuda_device, generator=g) * 0.05
    bias = torch.randn(cout, device=cuda_device, generator=g) * 0.1
    lib = _lib.load()
    m, k = B * H * W, 9 * C
    cols = torch.empty(m, k, device=cuda_device)
    assert lib.kp_im2col3x3_nhwc(x.data_ptr(), B, H, W, C, cols.data_ptr(), k, None) == 0
    c64 = cols.double() @ w.double() + bias.double()
    mag = cols.abs().double() @ w.abs().double() + bias.abs().double()
    for cfg in gemm.family_configs("tf32"):
        vid = gemm.variant_id(cfg, "tf32")
        assert gemm.conv3x3_supported(vid, C, cout)
        got = gemm.conv3x3(x, w, vid, bias=bias, relu=True).reshape(-1, cout)
        ref = torch.empty(m, cout, device=cuda_device)
        assert lib.kp_gemm_ex(vid, m, k, cout, 1, cols.data_ptr(), k, 0, w.data_ptr(), cout, 0, ref.data_ptr(), cout, 0,
                              bias.data_ptr(), _lib.KP_EPI_RELU, None) == 0
        assert torch.equal(got.view(torch.int32), ref.view(torch.int32)), (cfg.as_tuple(), gemm.k_slice_plan(vid, ProblemSize(m, k, cout, 1)))
        err = (got.double() - torch.relu(c64)).abs()
        assert bool((err <= (2 * 2.0 ** -10 + 2 * k * 2.0 ** -24) * mag + 1e-6).all()), cfg.as_tuple()


@pytest.mark.parametrize("B,H,W,C,cout", [(2, 9, 7, 64, 64), (1, 14, 14, 64, 128), (3, 28, 28, 256, 96),
                                         (16, 14, 14, 512, 512)])
def test_bf16_implicit_conv_equals_explicit(cuda_device, B, H, W, C, cout):
    """BF16 family: bf16 NHWC activations, im2col boxes of 64 channels x 128 pixels (one
    128-byte swizzled K slab) -- bit-identical to the bf16 im2col rows of the same fp32
    activations (kp_im2col3x3_nhwc_bf16 rounds to nearest even, as the bf16 cast) + the
    same BF16 variant, with fused bias + ReLU."""
    g = torch.Generator(device=cuda_device).manual_seed(B * 11 + C)
    x = torch.randn(B, H, W, C, device=cuda_device, generator=g)
    w = (torch.randn(9 * C, cout, device=cuda_device, generator=g) * 0.05).to(torch.bfloat16)
    bias = torch.randn(cout, device=cuda_device, generator=g) * 0.1
    lib = _lib.load()
    m, k = B * H * W, 9 * C
    cols = torch.empty(m, k, device=cuda_device, dtype=torch.bfloat16)
    assert lib.kp_im2col3x3_nhwc_bf16(x.data_ptr(), B, H, W, C, cols.data_ptr(), k, None) == 0
    xb = x.to(torch.bfloat16)
    for cfg in gemm.family_configs("bf16"):
        vid = gemm.variant_id(cfg, "bf16")
        assert gemm.conv3x3_supported(vid, C, cout)
        got = gemm.conv3x3(xb, w, vid, bias=bias, relu=True).reshape(-1, cout)
        ref = torch.empty(m, cout, device=cuda_device)
        assert lib.kp_gemm_ex(vid, m, k, cout, 1, cols.data_ptr(), k, 0, w.data_ptr(), cout, 0, ref.data_ptr(), cout, 0,
                              bias.data_ptr(), _lib.KP_EPI_RELU, None) == 0
        assert torch.equal(got.view(torch.int32), ref.view(torch.int32)), (cfg.as_tuple(), gemm.k_slice_plan(vid, ProblemSize(m, k, cout, 1), "bf16"))


def test_bf16_implicit_conv_contract(cuda_device):
    """BF16 variants need C % 64 == 0 and Cout % 8 == 0, and take bf16 operands only."""
    vid = gemm.variant_id(gemm.family_configs("bf16")[0], "bf16")
    assert gemm.conv3x3_supported(vid, 64, 64)
    assert not gemm.conv3x3_supported(vid, 32, 64)
    assert not gemm.conv3x3_supported(vid, 64, 12)
    x = torch.zeros(1, 4, 4, 64, device=cuda_device)
    w = torch.zeros(9 * 64, 64, device=cuda_device)
    with pytest.raises(ValueError):
        gemm.conv3x3(x, w, vid)  # fp32 operands on a BF16 variant


def test_maxpool_bf16_equals_pool_then_round(cuda_device):
    """bf16 pooling is exact: pooling the rounded activations equals rounding the fp32 pool."""
    lib = _lib.load()
    for B, H, W, C in [(2, 8, 6, 8), (3, 14, 14, 64), (1, 224, 224, 64)]:
        x = torch.randn(B, H, W, C, device=cuda_device)
        xb = x.to(torch.bfloat16)
        out = torch.empty(B, H // 2, W // 2, C, device=cuda_device, dtype=torch.bfloat16)
        assert lib.kp_maxpool2x2_nhwc_bf16(xb.data_ptr(), B, H, W, C, out.data_ptr(), None) == 0
        want = torch.nn.functional.max_pool2d(x.permute(0, 3, 1, 2), 2).permute(0, 2, 3, 1).to(torch.bfloat16)
        assert torch.equal(out.view(torch.int16), want.contiguous().view(torch.int16))
    bad = torch.empty(1, 2, 2, 4, device=cuda_device, dtype=torch.bfloat16)
    assert lib.kp_maxpool2x2_nhwc_bf16(bad.data_ptr(), 1, 2, 2, 4, out.data_ptr(), None) == _lib.KP_EINVAL
    x8 = torch.zeros(1, 2, 2, 16, device=cuda_device, dtype=torch.bfloat16)
    assert lib.kp_maxpool2x2_nhwc_bf16(x8.data_ptr() + 2, 1, 2, 2, 8, out.data_ptr(), None) == _lib.KP_EINVAL


@pytest.mark.parametrize("family", ["bf16", "tf32"])
def test_bf16_out_epilogue_equals_cast(cuda_device, family):
    """KP_EPI_BF16_OUT writes the fp32 epilogue result rounded to bf16 (nearest even) --
    equal to the fp32 output of the same variant cast afterwards -- on the persistent path
    (direct stores, TMA stores disabled), k-sliced launches (DSMEM reduction stores), the
    tail split, ragged n, and the implicit conv; SIMT variants reject the flag."""
    lib = _lib.load()
    dt = gemm.input_dtype(family)
    g = torch.Generator(device=cuda_device).manual_seed(5)
    shapes = [(1000, 512, 256), (16, 4096, 1000), (64, 25088, 512), (3000, 96, 72)]
    for ci, cfg in enumerate(gemm.family_configs(family)):
        vid = gemm.variant_id(cfg, family)
        for (m, k, n) in shapes[ci % 2::2] if ci > 1 else shapes:
            A = torch.randn(m, k, device=cuda_device, generator=g).to(dt)
            B = (torch.randn(k, n, device=cuda_device, generator=g) * 0.05).to(dt)
            bias = torch.randn(n, device=cuda_device, generator=g)
            ref = torch.empty(m, n, device=cuda_device)
            out = torch.empty(m, n, device=cuda_device, dtype=torch.bfloat16)
            assert lib.kp_gemm_ex(vid, m, k, n, 1, A.data_ptr(), k, 0, B.data_ptr(), n, 0, ref.data_ptr(), n, 0,
                                  bias.data_ptr(), _lib.KP_EPI_RELU, None) == 0
            assert lib.kp_gemm_ex(vid, m, k, n, 1, A.data_ptr(), k, 0, B.data_ptr(), n, 0, out.data_ptr(), n, 0,
                                  bias.data_ptr(), _lib.KP_EPI_RELU | _lib.KP_EPI_BF16_OUT, None) == 0
            assert torch.equal(out.view(torch.int16), ref.to(torch.bfloat16).view(torch.int16)), (cfg.as_tuple(), m, k, n)
    vid = gemm.variant_id(gemm.family_configs(family)[0], family)
    x = torch.randn(2, 14, 14, 64, device=cuda_device, generator=g).to(dt)
    w = (torch.randn(9 * 64, 128, device=cuda_device, generator=g) * 0.05).to(dt)
    ref = torch.empty(2, 14, 14, 128, device=cuda_device)
    out = torch.empty(2, 14, 14, 128, device=cuda_device, dtype=torch.bfloat16)
    assert lib.kp_conv3x3_nhwc_ex(vid, x.data_ptr(), 2, 14, 14, 64, w.data_ptr(), 128, ref.data_ptr(), None,
                                  _lib.KP_EPI_RELU, None) == 0
    assert lib.kp_conv3x3_nhwc_ex(vid, x.data_ptr(), 2, 14, 14, 64, w.data_ptr(), 128, out.data_ptr(), None,
                                  _lib.KP_EPI_RELU | _lib.KP_EPI_BF16_OUT, None) == 0
    assert torch.equal(out.view(torch.int16), ref.to(torch.bfloat16).view(torch.int16))
    py = gemm.conv3x3(x, w, vid, relu=True, out=torch.empty_like(out))  # the Python API: bf16 out
    assert torch.equal(py.view(torch.int16), out.view(torch.int16))
    sid = gemm.variant_id(KernelConfig(8, 8, 8, 16, 8), "simt")
    A = torch.zeros(8, 8, device=cuda_device)
    assert lib.kp_gemm_ex(sid, 8, 8, 8, 1, A.data_ptr(), 8, 0, A.data_ptr(), 8, 0, A.data_ptr(), 8, 0, None,
                          _lib.KP_EPI_BF16_OUT, None) == _lib.KP_EINVAL


@pytest.mark.parametrize("family,cout", [("bf16", 72), ("tf32", 68)])
def test_tensor_core_conv_writes_stay_in_bounds(cuda_device, family, cout):
    """Guard bands around the output (compute-sanitizer is unavailable on this pool):
    implicit convs with ragged m (105 pixels: a partial 128-row tile, and for CTA pairs a
    wholly out-of-range second half) and ragged Cout, fp32 and bf16 results, every config
    of the family -- nothing is written outside the (B*H*W) x Cout output."""
    dt = gemm.input_dtype(family)
    B, H, W = 3, 7, 5
    C = 64
    g = torch.Generator(device=cuda_device).manual_seed(cout)
    x = torch.randn(B, H, W, C, device=cuda_device, generator=g).to(dt)
    w = (torch.randn(9 * C, cout, device=cuda_device, generator=g) * 0.05).to(dt)
    bias = torch.randn(cout, device=cuda_device, generator=g)
    n_out, guard = B * H * W * cout, 4096
    lib = _lib.load()
    for cfg in gemm.family_configs(family):
        vid = gemm.variant_id(cfg, family)
        for odt, flags in ((torch.float32, _lib.KP_EPI_RELU), (torch.bfloat16, _lib.KP_EPI_RELU | _lib.KP_EPI_BF16_OUT)):
            buf = torch.full((guard + n_out + guard,), -3.0, device=cuda_device, dtype=odt)  # ReLU never writes < 0
            out = buf[guard:guard + n_out]
            assert lib.kp_conv3x3_nhwc_ex(vid, x.data_ptr(), B, H, W, C, w.data_ptr(), cout, out.data_ptr(),
                                          bias.data_ptr(), flags, None) == 0
            torch.cuda.synchronize()
            assert bool((buf[:guard] == -3.0).all()) and bool((buf[guard + n_out:] == -3.0).all()), (cfg.as_tuple(), odt)
            assert not bool((out == -3.0).any()), (cfg.as_tuple(), odt)  # and every element was written
