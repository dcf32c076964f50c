"""The reference's deployable selector, compiled: ``emit_nested_if`` output
(``select_kernel(...) -> KernelChoice``, codegen.py:185-229) is written to
``select_kernel.inc`` and built, unchanged, against include/kpgemm.h with gcc (C) and
nvcc (CUDA host code), exactly as INTEGRATION.md section 2a shows.

CPU leg: on 10^5 probe shapes the compiled selector returns the same KernelChoice as
``predict_tree`` (classify.py:230-237) and ``kp_find_variant`` maps it to the variant the
C dispatch table picks.  GPU leg: INTEGRATION 2a's ``run_gemm`` (select_kernel +
kp_find_variant + kp_gemm), compiled with nvcc, launches the selected variant
bit-exactly against the oracle; ``kp_gemm_auto(_ex)`` does the same through the table."""

import ctypes
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT
from paper_2008_13145_b200 import _lib, classify, codegen, gemm
from paper_2008_13145_b200.dataset import ProblemSize

LIB_DIR = ROOT / "paper_2008_13145_b200"
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

# INTEGRATION.md section 2a, verbatim (test_integration_doc_quotes_this_code checks it)
RUN_GEMM = r'''#include <cuda_runtime.h>
#include "kpgemm.h"            /* defines KernelChoice with the emitted field order */
#include "select_kernel.inc"   /* kernelprune codegen output, unchanged */
#include <math.h>

#ifdef __cplusplus
extern "C"                     /* C linkage when built as CUDA/C++ host code */
#endif
int run_gemm(int m, int k, int n, const float* A, const float* B, float* C, cudaStream_t s) {
  KernelChoice ch = select_kernel(log2(m), log2(k), log2(n), log2(1.0));
  int id = kp_find_variant(KP_FAMILY_SIMT, ch);          /* 5-tuple -> variant id */
  if (id < 0) return id;                                  /* KP_ENOENT, see kp_last_error() */
  return kp_gemm(id, m, k, n, 1, A, k, 0, B, n, 0, C, n, 0, s);
}
'''

# probe driver: hex-float features on stdin -> KernelChoice + variant id per line
PROBE_MAIN = r'''#include <stdio.h>
#include "kpgemm.h"
#include "select_kernel.inc"

int main(void) {
  int n = 0;
  if (scanf("%d", &n) != 1) return 2;
  for (int i = 0; i < n; ++i) {
    double f[4];
    if (scanf("%la %la %la %la", &f[0], &f[1], &f[2], &f[3]) != 4) return 3;
    KernelChoice c = select_kernel(f[0], f[1], f[2], f[3]);
    printf("%d %d %d %d %d %d\n", c.tile_rows, c.tile_acc, c.tile_cols, c.wg_rows, c.wg_cols,
           kp_find_variant(KP_FAMILY_SIMT, c));
  }
  return 0;
}
'''


@pytest.fixture(scope="module")
def selector(tmp_path_factory):
    """The bench's selector (committed VGG16 SIMT table, k-means 4, treeA), its emitted
    .inc and the C dispatch table of the same tree."""
    import bench
    from paper_2008_13145_b200.dispatch import Dispatcher

    pm, subset, tree, *_ = bench.train_selector(str(bench.DEFAULT_TABLE), 4, "kmeans", "treeA")
    work = tmp_path_factory.mktemp("emit")
    (work / "select_kernel.inc").write_text(codegen.emit_nested_if(tree, subset, pm.configs))
    return pm, subset, tree, Dispatcher(tree, subset, pm.configs, "simt"), work


def _probes(n=100_000, seed=0):
    rng = np.random.default_rng(seed)
    dims = np.exp2(rng.uniform(0, 19, size=(n, 3))).astype(np.int64) + 1
    batch = rng.choice([1, 1, 2, 4, 16, 64], size=(n, 1))
    shapes = np.concatenate([dims, batch], axis=1)
    from paper_2008_13145_b200 import shapes as net
    extra = [[p.m, p.k, p.n, p.batch] for s in ("vgg16", "resnet50") for p in net.network_problems(s)]
    return np.concatenate([shapes, np.array(extra, dtype=np.int64)])


def test_emitted_selector_compiles_and_agrees_with_predict_tree(selector):
    pm, subset, tree, disp, work = selector
    (work / "probe.c").write_text(PROBE_MAIN)
    exe = work / "probe"
    subprocess.run(["gcc", "-std=c99", "-O2", "-Wall", "-Werror", f"-I{ROOT / 'include'}", f"-I{work}",
                    str(work / "probe.c"), f"-L{LIB_DIR}", "-lkpgemm", f"-Wl,-rpath,{LIB_DIR}", "-o", str(exe)],
                   check=True, capture_output=True, text=True)
    shapes = _probes()
    feats = np.log2(shapes.astype(np.float64))  # classify.problem_features, classify.py:27-29
    stdin = f"{len(feats)}\n" + "\n".join(" ".join(float(x).hex() for x in row) for row in feats) + "\n"
    out = subprocess.run([str(exe)], input=stdin, capture_output=True, text=True, check=True).stdout.split("\n")
    got = np.array([[int(v) for v in line.split()] for line in out if line], dtype=np.int64)
    assert got.shape == (len(shapes), 6)
    want_cls = classify.predict_tree_batch(tree, feats)
    want = np.array([pm.configs[subset.config_indices[c]].as_tuple() for c in want_cls])
    assert np.array_equal(got[:, :5], want)
    vids = {c: gemm.variant_id(pm.configs[subset.config_indices[c]], "simt") for c in range(subset.k_actual)}
    assert np.array_equal(got[:, 5], [vids[c] for c in want_cls])
    for row in shapes[-50:]:  # the network shapes: the C table picks the same variants
        assert disp.variant(ProblemSize(*map(int, row))) == vids[classify.predict_tree(tree, np.log2(row.astype(float)))]


def test_emitted_selector_compiles_as_cuda_host_code(selector):
    *_, work = selector
    (work / "run_gemm.cu").write_text(RUN_GEMM)
    (work / "run_gemm.c").write_text(RUN_GEMM)
    cuda_inc = Path(NVCC).resolve().parent.parent / "include"
    subprocess.run(["gcc", "-std=c99", "-c", "-Wall", "-Werror", f"-I{cuda_inc}", f"-I{ROOT / 'include'}", f"-I{work}",
                    str(work / "run_gemm.c"), "-o", str(work / "run_gemm_c.o")], check=True, capture_output=True)
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared",
                    f"-I{ROOT / 'include'}", f"-I{work}", str(work / "run_gemm.cu"), f"-L{LIB_DIR}", "-lkpgemm",
                    f"-Xlinker", f"-rpath,{LIB_DIR}", "-o", str(work / "librun_gemm.so")],
                   check=True, capture_output=True, text=True)
    assert "run_gemm" in subprocess.run(["nm", "-D", str(work / "librun_gemm.so")], capture_output=True,
                                        text=True).stdout


def test_integration_doc_quotes_this_code():
    doc = (ROOT / "INTEGRATION.md").read_text()
    body = RUN_GEMM.strip().splitlines()
    for line in body:
        assert line in doc, f"INTEGRATION.md 2a no longer matches the compiled snippet: {line!r}"


@pytest.mark.gpu
def test_run_gemm_launches_the_selected_variant(selector, cuda_device):
    import torch

    from oracle import gemm_oracle as go

    pm, subset, tree, disp, work = selector
    so = work / "librun_gemm.so"
    if not so.exists():
        test_emitted_selector_compiles_as_cuda_host_code(selector)
    L = ctypes.CDLL(str(so))
    L.run_gemm.restype = ctypes.c_int
    L.run_gemm.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p] * 4
    rng = np.random.default_rng(1)
    for m, k, n in ((1000, 27, 64), (196, 4608, 512), (16, 4096, 1000), (333, 129, 77)):
        A = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        B = rng.uniform(-1, 1, (k, n)).astype(np.float32)
        dA, dB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
        C = torch.empty(m, n, device=cuda_device)
        rc = L.run_gemm(m, k, n, dA.data_ptr(), dB.data_ptr(), C.data_ptr(),
                        torch.cuda.current_stream().cuda_stream)
        assert rc == 0, _lib.last_error()
        p = ProblemSize(m, k, n, 1)
        kps = gemm.k_slice_plan(disp.select_c_log2(p), p)[1]
        assert np.array_equal(C.cpu().numpy().view(np.uint32), go.gemm_sliced(A, B, kps)[0].view(np.uint32))


@pytest.mark.gpu
def test_kp_gemm_auto_matches_predict_tree_and_oracle(selector, cuda_device):
    import torch

    from oracle import gemm_oracle as go

    pm, subset, tree, disp, _ = selector
    lib = _lib.load()
    rng = np.random.default_rng(2)
    stream = torch.cuda.current_stream().cuda_stream
    for m, k, n, relu in ((3136, 576, 64, 0), (32, 25088, 4096, 1), (49, 4608, 512, 1), (77, 33, 45, 0)):
        A = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        B = rng.uniform(-1, 1, (k, n)).astype(np.float32)
        bias = rng.uniform(-1, 1, n).astype(np.float32)
        dA, dB, db = (torch.from_numpy(x).to(cuda_device) for x in (A, B, bias))
        C = torch.empty(m, n, device=cuda_device)
        vid = ctypes.c_int(-1)
        if relu:
            rc = lib.kp_gemm_auto_ex(disp.handle, m, k, n, 1, dA.data_ptr(), k, 0, dB.data_ptr(), n, 0,
                                     C.data_ptr(), n, 0, db.data_ptr(), _lib.KP_EPI_RELU, stream, ctypes.byref(vid))
        else:
            rc = lib.kp_gemm_auto(disp.handle, m, k, n, 1, dA.data_ptr(), k, 0, dB.data_ptr(), n, 0,
                                  C.data_ptr(), n, 0, stream, ctypes.byref(vid))
        assert rc == 0, _lib.last_error()
        p = ProblemSize(m, k, n, 1)
        cls = classify.predict_tree(tree, classify.problem_features([p])[0])
        assert vid.value == gemm.variant_id(pm.configs[subset.config_indices[cls]], "simt")
        want = go.gemm_sliced(A, B, gemm.k_slice_plan(vid.value, p)[1])[0]
        if relu:
            want = np.maximum(want + bias, np.float32(0))
        assert np.array_equal(C.cpu().numpy().view(np.uint32), want.view(np.uint32))
