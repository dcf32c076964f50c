"""GPU: VGG16 inference (im2col + tree-dispatched GEMMs with fused bias/ReLU + max pool)
equals the CPU oracle forward (oracle/vgg16_ref.py) bit for bit, eager and as a CUDA
graph; the conv helpers match their numpy restatements exactly."""

import numpy as np
import pytest
import torch

from oracle import vgg16_ref
from paper_2008_13145_b200 import _lib, classify, dataset, selection, vgg16
from paper_2008_13145_b200.dispatch import Dispatcher
from paper_2008_13145_b200.normalize import NormScheme, normalize
from paper_2008_13145_b200.sweep import SynthTimer, benchmark_sweep

pytestmark = pytest.mark.gpu


def _dispatcher(batch):
    # a tree over a synthetic table is enough to exercise dispatch of every layer
    model = vgg16.Vgg16.__new__(vgg16.Vgg16)
    model.batch = batch
    probs = list(dict.fromkeys(vgg16.Vgg16.problems(model)))
    cfgs = tuple(dataset.enumerate_configs())
    pm = benchmark_sweep(probs, timer=SynthTimer(cfgs), configs=cfgs)
    nm = normalize(pm, NormScheme())
    sub = selection.select_subset("kmeans", nm, min(4, len(probs)), 0)
    labels = classify.label_best_in_subset(nm, sub)
    tree = classify.train_tree(classify.problem_features(pm.problems), labels, classify.TREE_PRESETS["A"],
                               n_classes=sub.k_actual)
    return Dispatcher(tree, sub, pm.configs, "simt")


def test_im2col_and_pool_exact(cuda_device):
    lib = _lib.load()
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 9, 7, 5)).astype(np.float32)
    dx = torch.from_numpy(x).to(cuda_device)
    out = torch.empty(2 * 9 * 7, 45, device=cuda_device)
    assert lib.kp_im2col3x3_nhwc(dx.data_ptr(), 2, 9, 7, 5, out.data_ptr(), 45, None) == 0
    assert np.array_equal(out.cpu().numpy(), vgg16_ref.im2col3x3(x))
    y = rng.standard_normal((2, 8, 6, 3)).astype(np.float32)
    dy = torch.from_numpy(y).to(cuda_device)
    pout = torch.empty(2, 4, 3, 3, device=cuda_device)
    assert lib.kp_maxpool2x2_nhwc(dy.data_ptr(), 2, 8, 6, 3, pout.data_ptr(), None) == 0
    assert np.array_equal(pout.cpu().numpy(), vgg16_ref.maxpool2(y))


@pytest.mark.parametrize("B,H,W,C,kpad", [(2, 9, 7, 3, 28), (1, 6, 5, 3, 32), (2, 4, 4, 8, 72)])
def test_im2col_padded_rows(cuda_device, B, H, W, C, kpad):
    """kp_im2col3x3_nhwc_pad: the 9C patch values then zeros up to kpad in every row."""
    lib = _lib.load()
    x = np.random.default_rng(kpad).standard_normal((B, H, W, C)).astype(np.float32)
    out = torch.full((B * H * W, kpad), 7.0, device=cuda_device)
    assert lib.kp_im2col3x3_nhwc_pad(torch.from_numpy(x).to(cuda_device).data_ptr(), B, H, W, C, out.data_ptr(),
                                     kpad, None) == 0
    got = out.cpu().numpy()
    assert np.array_equal(got[:, :9 * C], vgg16_ref.im2col3x3(x))
    assert not got[:, 9 * C:].any()
    assert lib.kp_im2col3x3_nhwc_pad(0, B, H, W, C, out.data_ptr(), 27, None) == _lib.KP_EINVAL


@pytest.mark.parametrize("B,H,W,C", [(2, 9, 7, 8), (3, 14, 14, 64), (1, 5, 6, 512)])
def test_im2col_and_pool_vec4_exact(cuda_device, B, H, W, C):
    """The float4 kernels (C % 4 == 0, every VGG16 layer after conv1_1), ldo > 9C too."""
    lib = _lib.load()
    rng = np.random.default_rng(C)
    x = rng.standard_normal((B, H, W, C)).astype(np.float32)
    dx = torch.from_numpy(x).to(cuda_device)
    ldo = 9 * C + 4
    out = torch.full((B * H * W, ldo), 7.0, device=cuda_device)
    assert lib.kp_im2col3x3_nhwc(dx.data_ptr(), B, H, W, C, out.data_ptr(), ldo, None) == 0
    assert np.array_equal(out[:, :9 * C].cpu().numpy(), vgg16_ref.im2col3x3(x))
    assert bool((out[:, 9 * C:] == 7.0).all())
    H2, W2 = H - H % 2, W - W % 2
    y = np.ascontiguousarray(x[:, :H2, :W2, :])
    dy = torch.from_numpy(y).to(cuda_device)
    pout = torch.empty(B, H2 // 2, W2 // 2, C, device=cuda_device)
    assert lib.kp_maxpool2x2_nhwc(dy.data_ptr(), B, H2, W2, C, pout.data_ptr(), None) == 0
    assert np.array_equal(pout.cpu().numpy(), vgg16_ref.maxpool2(y))


@pytest.mark.parametrize("batch", [1, 2])
def test_vgg16_forward_bit_exact(cuda_device, batch):
    convs, fcs = vgg16.init_weights(seed=0)
    model = vgg16.Vgg16(_dispatcher(batch), batch, cuda_device, weights=(convs, fcs))
    g = torch.Generator().manual_seed(7)
    x = torch.randn(batch, 224, 224, 3, generator=g)
    got = model.forward(x.to(cuda_device)).cpu().numpy().copy()
    plan = lambda m, k, n: model.disp.k_slice_plan(dataset.ProblemSize(m, k, n, 1))[1]  # noqa: E731
    want = vgg16_ref.forward(x.numpy(), [(w.numpy(), b.numpy()) for w, b in convs],
                             [(w.numpy(), b.numpy()) for w, b in fcs], k_per_slice=plan)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    model.capture()
    again = model.forward(x.to(cuda_device)).cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(again.view(np.uint32), want.view(np.uint32))


def test_vgg16_forward_tf32_family_within_tolerance(cuda_device):
    """VGG16 inference on the tcgen05 TF32 family (fp32 activations, tf32 products, fp32
    accumulation): logits within a stated normwise tolerance of the bit-exact fp32 oracle
    forward -- 16 layers of TF32 products (2^-11 relative operand rounding each, ReLU
    between) stay below 2e-2 relative in the 2-norm."""
    from paper_2008_13145_b200 import gemm
    from paper_2008_13145_b200.classify import TreeModel
    from paper_2008_13145_b200.selection import ConfigSubset

    cfgs = gemm.family_configs("tf32")
    leaf = TreeModel(feature=np.array([-1]), threshold=np.array([np.nan]), left=np.array([-1]),
                     right=np.array([-1]), leaf_class=np.array([0]))
    disp = Dispatcher(leaf, ConfigSubset((3,), "fixed", 1, 1), cfgs, "tf32")  # (128,32,256,4,192)
    convs, fcs = vgg16.init_weights(seed=0)
    model = vgg16.Vgg16(disp, 1, cuda_device, weights=(convs, fcs))
    x = torch.randn(1, 224, 224, 3, generator=torch.Generator().manual_seed(7))
    got = model.forward(x.to(cuda_device)).double().cpu().numpy()
    want = vgg16_ref.forward(x.numpy(), [(w.numpy(), b.numpy()) for w, b in convs],
                             [(w.numpy(), b.numpy()) for w, b in fcs]).astype(np.float64)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel < 2e-2, rel
    assert not np.array_equal(got, want)  # it really ran on the tensor cores


def test_vgg16_forward_bf16_family_within_tolerance(cuda_device):
    """VGG16 inference on the tcgen05 BF16 family: bf16 weights and im2col rows
    (kp_im2col3x3_nhwc_bf16, kp_cast_bf16 for the fc inputs), fp32 accumulation and fp32
    activations between layers; logits within 5e-2 normwise of the fp32 oracle forward
    (bf16 keeps 8 significant bits: ~2^-9 relative rounding per operand per layer)."""
    from paper_2008_13145_b200 import gemm
    from paper_2008_13145_b200.classify import TreeModel
    from paper_2008_13145_b200.selection import ConfigSubset

    cfgs = gemm.family_configs("bf16")
    leaf = TreeModel(feature=np.array([-1]), threshold=np.array([np.nan]), left=np.array([-1]),
                     right=np.array([-1]), leaf_class=np.array([0]))
    disp = Dispatcher(leaf, ConfigSubset((2,), "fixed", 1, 1), cfgs, "bf16")  # (128,64,256,4,192)
    convs, fcs = vgg16.init_weights(seed=0)
    model = vgg16.Vgg16(disp, 1, cuda_device, weights=(convs, fcs))
    x = torch.randn(1, 224, 224, 3, generator=torch.Generator().manual_seed(7))
    got = model.forward(x.to(cuda_device)).double().cpu().numpy()
    want = vgg16_ref.forward(x.numpy(), [(w.numpy(), b.numpy()) for w, b in convs],
                             [(w.numpy(), b.numpy()) for w, b in fcs]).astype(np.float64)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    print(f"bf16 VGG16 normwise relative error {rel:.3e}")
    assert rel < 5e-2, rel


def test_bf16_operand_kernels(cuda_device):
    lib = _lib.load()
    x = torch.randn(2, 5, 6, 8, device=cuda_device)
    k = 72
    out = torch.empty(2 * 5 * 6, k, device=cuda_device, dtype=torch.bfloat16)
    assert lib.kp_im2col3x3_nhwc_bf16(x.data_ptr(), 2, 5, 6, 8, out.data_ptr(), k, None) == 0
    want = torch.from_numpy(vgg16_ref.im2col3x3(x.cpu().numpy())).to(torch.bfloat16)
    assert torch.equal(out.cpu(), want)
    x3 = torch.randn(1, 4, 4, 3, device=cuda_device)
    out3 = torch.full((16, 32), 9.0, device=cuda_device, dtype=torch.bfloat16)
    assert lib.kp_im2col3x3_nhwc_bf16(x3.data_ptr(), 1, 4, 4, 3, out3.data_ptr(), 32, None) == 0
    want3 = torch.from_numpy(vgg16_ref.im2col3x3(x3.cpu().numpy())).to(torch.bfloat16)
    assert torch.equal(out3[:, :27].cpu(), want3) and not out3[:, 27:].float().any()
    v = torch.randn(64, device=cuda_device)
    c = torch.empty(64, device=cuda_device, dtype=torch.bfloat16)
    assert lib.kp_cast_bf16(v.data_ptr(), 64, c.data_ptr(), None) == 0
    assert torch.equal(c, v.to(torch.bfloat16))


@pytest.mark.parametrize("family,vid_col", [("bf16", 2), ("tf32", 3)])
def test_vgg16_tensor_core_implicit_equals_explicit(cuda_device, family, vid_col):
    """Implicit-GEMM convs on the tcgen05 families (TMA im2col boxes; BF16 with bf16
    activations end to end: KP_EPI_BF16_OUT epilogues and bf16 pools) give the same logits
    as fp32 activations + im2col + GEMM, bit for bit, eager and graph-captured, at a batch
    where conv rows cross images."""
    from paper_2008_13145_b200 import gemm
    from paper_2008_13145_b200.classify import TreeModel
    from paper_2008_13145_b200.selection import ConfigSubset

    cfgs = gemm.family_configs(family)
    leaf = TreeModel(feature=np.array([-1]), threshold=np.array([np.nan]), left=np.array([-1]),
                     right=np.array([-1]), leaf_class=np.array([0]))
    disp = Dispatcher(leaf, ConfigSubset((vid_col,), "fixed", 1, 1), cfgs, family)
    convs, fcs = vgg16.init_weights(seed=0)
    x = torch.randn(2, 224, 224, 3, generator=torch.Generator().manual_seed(3)).to(cuda_device)
    imp = vgg16.Vgg16(disp, 2, cuda_device, weights=(convs, fcs))
    exp = vgg16.Vgg16(disp, 2, cuda_device, weights=(convs, fcs), implicit=False)
    assert sum(lay[-1] for lay in imp.layers) == 12 and not any(lay[-1] for lay in exp.layers)
    assert imp.bf16_acts == (family == "bf16") and not exp.bf16_acts  # BF16: bf16 activations end to end
    a = imp.forward(x).clone()
    b = exp.forward(x).clone()
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    imp.capture()
    c = imp.forward(x).clone()
    assert torch.equal(a.view(torch.int32), c.view(torch.int32))
