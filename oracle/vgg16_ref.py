"""CPU VGG16 forward (NHWC fp32) built from the oracle GEMM -- TEST INFRASTRUCTURE ONLY.

Mirrors paper_2008_13145_b200.vgg16 op for op: im2col of 3x3/pad-1 patches in
(dy, dx, c) order, the sequential fmaf-chain GEMM (oracle/gemm_ref.c), fp32 bias add,
ReLU, 2x2 max pooling; fc layers as GEMMs.  Every step is exact-arithmetic-equivalent
to the GPU path, so logits must match bit for bit.
"""

from __future__ import annotations

import numpy as np

from oracle import gemm_oracle as go

PLAN = ((3, 64), (64, 64), "M", (64, 128), (128, 128), "M", (128, 256), (256, 256), (256, 256), "M",
        (256, 512), (512, 512), (512, 512), "M", (512, 512), (512, 512), (512, 512), "M")
FC_RELU = (True, True, False)


def im2col3x3(x: np.ndarray) -> np.ndarray:
    B, H, W, C = x.shape
    xp = np.zeros((B, H + 2, W + 2, C), dtype=np.float32)
    xp[:, 1:-1, 1:-1, :] = x
    cols = np.empty((B, H, W, 9, C), dtype=np.float32)
    for t in range(9):
        dy, dx = divmod(t, 3)
        cols[:, :, :, t, :] = xp[:, dy:dy + H, dx:dx + W, :]
    return cols.reshape(B * H * W, 9 * C)


def maxpool2(x: np.ndarray) -> np.ndarray:
    B, H, W, C = x.shape
    return x.reshape(B, H // 2, 2, W // 2, 2, C).max(axis=(2, 4))


def _gemm(A, W, k_per_slice):
    kps = k_per_slice(A.shape[0], A.shape[1], W.shape[1]) if k_per_slice else None
    return (go.gemm_sliced(A, W, kps) if kps else go.gemm_chain(A, W))[0]


def forward(x: np.ndarray, convs, fcs, k_per_slice=None) -> np.ndarray:
    """x (B,224,224,3) fp32; convs/fcs lists of (W, b) numpy fp32 -> logits (B,1000).
    k_per_slice(m, k, n) -> int, optional: the GPU's k-slice plan for each layer GEMM
    (kp_gemm_plan), so the restatement sums the same slices in the same order."""
    B = x.shape[0]
    ci = 0
    for item in PLAN:
        if item == "M":
            x = maxpool2(x)
            continue
        w, b = convs[ci]
        ci += 1
        H = x.shape[1]
        y = _gemm(im2col3x3(x), w, k_per_slice)
        y = np.maximum(y + b, np.float32(0.0))
        x = y.reshape(B, H, H, w.shape[1])
    h = x.reshape(B, -1)
    for (w, b), relu in zip(fcs, FC_RELU):
        h = _gemm(h, w, k_per_slice) + b
        if relu:
            h = np.maximum(h, np.float32(0.0))
    return h
