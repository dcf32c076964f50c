"""GPU: the tree-dispatched GEMM (C dispatch table -> kp_gemm) launches exactly the
variant predict_tree names and produces that variant's (bit-exact) result; the CUDA
event sweep fills every cell of a small table with a positive GFLOP/s."""

import numpy as np
import pytest
import torch

from oracle import gemm_oracle as go
from paper_2008_13145_b200 import classify, dataset, gemm, selection
from paper_2008_13145_b200.codegen import export_model
from paper_2008_13145_b200.dispatch import Dispatcher
from paper_2008_13145_b200.normalize import NormScheme, normalize
from paper_2008_13145_b200.sweep import CudaEventTimer, benchmark_sweep

pytestmark = pytest.mark.gpu


def test_sweep_every_config_positive(cuda_device):
    problems = [dataset.ProblemSize(37, 27, 61, 1), dataset.ProblemSize(256, 256, 256, 1),
                dataset.ProblemSize(1, 1000, 100, 1)]
    for family in ("simt", "paper"):
        timer = CudaEventTimer(family, problems, min_ms=0.05, max_iters=20)
        pm = benchmark_sweep(problems, timer=timer)
        assert pm.n_configs == 640 and (pm.values > 0).all()
        assert pm.configs == tuple(dataset.enumerate_configs())


def test_dispatcher_matches_predict_tree_and_oracle(cuda_device):
    problems = [dataset.ProblemSize(m, k, n, 1) for m, k, n in
                ((64, 64, 64), (512, 512, 512), (1, 2048, 512), (3136, 64, 64), (49, 4608, 512), (1000, 27, 64))]
    timer = CudaEventTimer("simt", problems, min_ms=0.2)
    pm = benchmark_sweep(problems, timer=timer)
    nm = normalize(pm, NormScheme("scaled"))
    subset = selection.select_subset("kmeans", nm, 4, 0)
    labels = classify.label_best_in_subset(nm, subset)
    tree = classify.train_tree(classify.problem_features(pm.problems), labels, classify.TREE_PRESETS["A"],
                               n_classes=subset.k_actual)
    disp = Dispatcher(tree, subset, pm.configs, "simt")
    disp2 = Dispatcher.from_kptree(export_model(tree, subset, pm.configs), "simt")
    rng = np.random.default_rng(3)
    for p in problems + [dataset.ProblemSize(300, 100, 70, 1)]:
        cls = classify.predict_tree(tree, classify.problem_features([p])[0])
        want_cfg = pm.configs[subset.config_indices[cls]]
        assert disp.select(p) == want_cfg == disp2.select(p)
        assert disp.select_c_log2(p) == gemm.variant_id(want_cfg, "simt")
        A = rng.uniform(-1, 1, (p.m, p.k)).astype(np.float32)
        B = rng.uniform(-1, 1, (p.k, p.n)).astype(np.float32)
        got = disp.matmul(torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)).cpu().numpy()
        _, kps = disp.k_slice_plan(p)
        assert np.array_equal(got.view(np.uint32), go.gemm_sliced(A, B, kps)[0].view(np.uint32))


def test_bench_workload_full_size_bound(cuda_device):
    """bench.py's workload at its full size (VGG16 GEMM layer set, batch 16, dispatched by
    the committed B200 table's k-means 4 + treeA): every layer within the fp32 bound
    |C - C64| <= 2*k*u*(|A||B|) of a float64 product -- the size-independent property the
    bit-exact small-shape tests cannot cover at this scale (k-sliced layers included)."""
    import bench
    from paper_2008_13145_b200.dispatch import Dispatcher

    pm, subset, tree, *_ = bench.train_selector(str(bench.DEFAULT_TABLE), 4, "kmeans", "treeA")
    disp = Dispatcher(tree, subset, pm.configs, "simt")
    g = torch.Generator(device=cuda_device).manual_seed(5)
    sliced = 0
    for name, p in dict(bench.vgg16_layers(16)).items():
        A = torch.rand(p.m, p.k, device=cuda_device, generator=g) * 2 - 1
        W = torch.rand(p.k, p.n, device=cuda_device, generator=g) * 2 - 1
        C = disp.matmul(A, W).double()
        A64, W64 = A.double(), W.double()
        err = (C - A64 @ W64).abs()
        bound = 2 * p.k * 2.0 ** -24 * (A64.abs() @ W64.abs())
        assert bool((err <= bound).all()), name
        sliced += disp.k_slice_plan(p)[0] > 1
        del A, W, C, A64, W64, err, bound
    assert sliced > 0  # the step exercises k-sliced launches
