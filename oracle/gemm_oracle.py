"""ctypes wrapper of oracle/libgemmref.so (gemm_ref.c) -- TEST INFRASTRUCTURE ONLY.

Parity status: the reference (kernelprune) contains no GEMM, so
GEMM numerics are "parity unpinned" against reference outputs.  The oracle is pinned
instead by construction and by two independent restatements that must agree bit for
bit: the paper-order tiled emulation (kp_ref_gemm_tiled, dataset.py:41-46 /
dataset.py:312-316 semantics) and the row-order fmaf chain (kp_ref_gemm_chain); both
are checked against numpy float64 (the reference's numeric engine) within the fp32
bound |C - C64| <= 2*k*u*(|A||B|), u = 2^-24.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libgemmref.so"
U32 = 2.0 ** -24

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        i, i64, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
        L.kp_ref_gemm_tiled.restype = i64
        L.kp_ref_gemm_tiled.argtypes = [i] * 9 + [vp, i64, i64, vp, i64, i64, vp, i64, i64]
        L.kp_ref_gemm_chain.restype = None
        L.kp_ref_gemm_chain.argtypes = [i] * 4 + [vp, i64, i64, vp, i64, i64, vp, i64, i64]
        L.kp_ref_gemm_sliced.restype = None
        L.kp_ref_gemm_sliced.argtypes = [i] * 5 + [vp, i64, i64, vp, i64, i64, vp, i64, i64]
        L.kp_ref_threads.restype = i
        L.kp_ref_threads.argtypes = [i]
        L.kp_ref_gemm_f64.restype = None
        L.kp_ref_gemm_f64.argtypes = [i] * 4 + [vp, i64, i64, vp, i64, i64, vp, vp, i64, i64]
        _lib = L
    return _lib


def _batched(A: np.ndarray, B: np.ndarray):
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    A3 = A if A.ndim == 3 else A[None]
    B3 = B if B.ndim == 3 else B[None]
    batch = max(A3.shape[0], B3.shape[0])
    m, k = A3.shape[1:]
    n = B3.shape[2]
    sA = m * k if A3.shape[0] > 1 else 0
    sB = k * n if B3.shape[0] > 1 else 0
    return A3, B3, batch, m, k, n, sA, sB


def set_threads(n: int = 0) -> int:
    """OpenMP threads for the oracle (n <= 0: all CPUs this process may run on);
    returns the count in effect (torchrun exports OMP_NUM_THREADS=1 to each rank)."""
    import os
    if n <= 0:
        n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    return int(lib().kp_ref_threads(int(n)))


def gemm_tiled(A, B, config) -> tuple[np.ndarray, int]:
    """Paper-order emulation under a KernelConfig; returns (C, work items)."""
    A3, B3, batch, m, k, n, sA, sB = _batched(A, B)
    C = np.zeros((batch, m, n), dtype=np.float32)
    items = lib().kp_ref_gemm_tiled(config.tile_rows, config.tile_acc, config.tile_cols, config.wg_rows,
                                    config.wg_cols, m, k, n, batch, A3.ctypes.data, k, sA, B3.ctypes.data, n, sB,
                                    C.ctypes.data, n, m * n)
    return C, int(items)


def gemm_chain(A, B) -> np.ndarray:
    """Sequential fp32 fmaf chain per element (bit-exact target of F0/F1)."""
    A3, B3, batch, m, k, n, sA, sB = _batched(A, B)
    C = np.zeros((batch, m, n), dtype=np.float32)
    lib().kp_ref_gemm_chain(m, k, n, batch, A3.ctypes.data, k, sA, B3.ctypes.data, n, sB, C.ctypes.data, n, m * n)
    return C


def gemm_sliced(A, B, k_per_slice: int) -> np.ndarray:
    """k-sliced chain: fmaf chain per slice of k_per_slice, slices summed in order
    (the SIMT family's plan from kp_gemm_plan when a launch cannot fill the GPU)."""
    A3, B3, batch, m, k, n, sA, sB = _batched(A, B)
    C = np.zeros((batch, m, n), dtype=np.float32)
    lib().kp_ref_gemm_sliced(m, k, n, batch, int(k_per_slice), A3.ctypes.data, k, sA, B3.ctypes.data, n, sB,
                             C.ctypes.data, n, m * n)
    return C


def gemm_f64(A, B) -> tuple[np.ndarray, np.ndarray]:
    """(float64 product, |A||B| magnitudes) of the fp32 operands."""
    A3, B3, batch, m, k, n, sA, sB = _batched(A, B)
    C = np.zeros((batch, m, n), dtype=np.float64)
    M = np.zeros((batch, m, n), dtype=np.float64)
    lib().kp_ref_gemm_f64(m, k, n, batch, A3.ctypes.data, k, sA, B3.ctypes.data, n, sB, C.ctypes.data,
                          M.ctypes.data, n, m * n)
    return C, M


def fp32_bound(k: int, mag: np.ndarray) -> np.ndarray:
    """Per-element fp32 error bound 2*k*u*(|A||B|)."""
    return 2.0 * k * U32 * mag


def tf32_bound(k: int, mag: np.ndarray) -> np.ndarray:
    return (2.0 * 2.0 ** -11 + 2.0 * k * U32) * mag


def bf16_bound(k: int, mag: np.ndarray) -> np.ndarray:
    return (2.0 * 2.0 ** -8 + 2.0 * k * U32) * mag
