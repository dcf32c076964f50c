"""The CPU oracle itself (oracle/gemm_ref.c): the paper-order tiled emulation and the
row-order fma chain agree bit for bit, launch exactly work_items() work items
(dataset.py:312-316), and sit inside the fp32 error bound of the float64 product."""

import numpy as np
import pytest

from oracle import gemm_oracle as go
from paper_2008_13145_b200.dataset import KernelConfig, ProblemSize, enumerate_configs, work_items

SHAPES = [(1, 1, 1, 1), (7, 31, 64, 1), (37, 27, 61, 3), (64, 255, 33, 2), (129, 147, 64, 1), (1, 1000, 9, 1)]


def _inputs(m, k, n, batch, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, (batch, m, k)).astype(np.float32),
            rng.uniform(-1, 1, (batch, k, n)).astype(np.float32))


@pytest.mark.parametrize("shape", SHAPES)
def test_tiled_equals_chain_bitwise(shape):
    A, B = _inputs(*shape)
    chain = go.gemm_chain(A, B)
    for cfg in enumerate_configs()[::37]:
        tiled, items = go.gemm_tiled(A, B, cfg)
        assert np.array_equal(tiled.view(np.uint32), chain.view(np.uint32)), cfg
        assert items == work_items(ProblemSize(*shape), cfg)


@pytest.mark.parametrize("shape", SHAPES)
def test_chain_within_fp32_bound_of_float64(shape):
    m, k, n, batch = shape
    A, B = _inputs(*shape, seed=1)
    chain = go.gemm_chain(A, B).astype(np.float64)
    c64, mag = go.gemm_f64(A, B)
    np.testing.assert_allclose(c64, np.matmul(A.astype(np.float64), B.astype(np.float64)), rtol=1e-12, atol=1e-12)
    assert (np.abs(chain - c64) <= go.fp32_bound(k, mag)).all()


def test_broadcast_weights():
    rng = np.random.default_rng(2)
    A = rng.uniform(-1, 1, (3, 17, 9)).astype(np.float32)
    W = rng.uniform(-1, 1, (9, 5)).astype(np.float32)
    out = go.gemm_chain(A, W)
    for b in range(3):
        assert np.array_equal(out[b], go.gemm_chain(A[b], W)[0])


def test_zero_padding_is_exact():
    """fmaf(0, 0, acc) == acc: padded k steps cannot change a result (the GPU kernels
    zero-fill k tails)."""
    A, B = _inputs(5, 13, 7, 1, seed=3)
    ref = go.gemm_chain(A, B)
    Ap = np.concatenate([A, np.zeros((1, 5, 3), np.float32)], axis=2)
    Bp = np.concatenate([B, np.zeros((1, 3, 7), np.float32)], axis=1)
    assert np.array_equal(go.gemm_chain(Ap, Bp), ref)
