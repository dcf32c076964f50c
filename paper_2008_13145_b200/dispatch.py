"""classifier-dispatch, runtime side: the decision tree as a C table inside
libkpgemm.so that maps a GEMM's shape to a kernel variant and launches it.

The reference stops at emitting ``select_kernel(log2_m, log2_k, log2_n, log2_batch)``
as C text (codegen.py:185-229) and leaves the launcher undefined.  Here the trained
TreeModel (classify.py:56-77) -- or a kptree v1 document (codegen.py:36-156) -- is
flattened into ``kp_dispatch_load`` arrays; selection walks it in C with the same
strict '<' routing as ``predict_tree`` (classify.py:230-237).

Feature parity: features are computed here with ``np.log2`` exactly as
``problem_features`` does (classify.py:27-29) and passed to
``kp_dispatch_select_feats``, because glibc ``log2`` differs from numpy's by one ulp
on a few integers; ``kp_dispatch_select`` (C log2) is offered for
C callers and agrees on the VGG16/ResNet-50 shape set.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .classify import TreeModel
from .codegen import import_model
from .dataset import KernelConfig, ProblemSize
from .gemm import GemmOperands, input_dtype, variant_id, variant_info
from .selection import ConfigSubset


def _as(arr, ctype, dtype):
    a = np.ascontiguousarray(arr, dtype=dtype)
    return a, a.ctypes.data_as(ctypes.POINTER(ctype))


class Dispatcher:
    """Tree-dispatched GEMM: ``select(problem)`` / ``matmul(A, B)``."""

    def __init__(self, model: TreeModel, subset: ConfigSubset, configs, family: str = "simt"):
        leaf = np.asarray(model.leaf_class)
        if leaf.max() >= subset.k_actual:
            raise ValueError("leaf class outside the subset")
        self.family = family
        self.model = model
        self.subset = subset
        self.choices = tuple(configs[i] for i in subset.config_indices)
        self.variants = tuple(variant_id(c, family) for c in self.choices)
        lib = _lib.load()
        keep = []
        args = []
        for arr, ct, dt in ((model.feature, ctypes.c_int32, np.int32),
                            (model.threshold, ctypes.c_double, np.float64),
                            (model.left, ctypes.c_int32, np.int32),
                            (model.right, ctypes.c_int32, np.int32),
                            (model.leaf_class, ctypes.c_int32, np.int32)):
            a, p = _as(arr, ct, dt)
            keep.append(a)
            args.append(p)
        c2v, c2v_p = _as(self.variants, ctypes.c_int32, np.int32)
        # NaN thresholds of leaves are never read; the C loader rejects NaN only on
        # internal nodes.
        self.handle = _lib.check(lib.kp_dispatch_load(model.n_nodes, *args, len(self.variants), c2v_p),
                                 "kp_dispatch_load")
        self._cache: dict[ProblemSize, int] = {}

    @classmethod
    def from_kptree(cls, doc: str, family: str = "simt") -> "Dispatcher":
        model, subset, configs = import_model(doc)
        return cls(model, subset, configs, family)

    def close(self) -> None:
        if getattr(self, "handle", None) is not None:
            _lib.check(_lib.load().kp_dispatch_free(self.handle), "kp_dispatch_free")
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    @staticmethod
    def features(problem: ProblemSize) -> np.ndarray:
        """np.log2 of (m, k, n, batch), as classify.problem_features computes it."""
        return np.log2([[problem.m, problem.k, problem.n, problem.batch]])[0]

    def select_class(self, problem: ProblemSize) -> int:
        f, fp = _as(self.features(problem), ctypes.c_double, np.float64)
        return _lib.check(_lib.load().kp_dispatch_class_feats(self.handle, fp), "kp_dispatch_class_feats")

    def variant(self, problem: ProblemSize) -> int:
        vid = self._cache.get(problem)
        if vid is None:
            f, fp = _as(self.features(problem), ctypes.c_double, np.float64)
            vid = _lib.check(_lib.load().kp_dispatch_select_feats(self.handle, fp), "kp_dispatch_select_feats")
            self._cache[problem] = vid
        return vid

    def select(self, problem: ProblemSize) -> KernelConfig:
        return variant_info(self.variant(problem))[0]

    def select_c_log2(self, problem: ProblemSize) -> int:
        """Variant chosen with the C library's log2 (kp_dispatch_select)."""
        p = problem
        return _lib.check(_lib.load().kp_dispatch_select(self.handle, p.m, p.k, p.n, p.batch),
                          "kp_dispatch_select")

    def k_slice_plan(self, problem: ProblemSize, num_sms: int = 0) -> tuple[int, int]:
        """(k_slices, k_per_slice) of the launch this dispatcher makes (kp_gemm_plan)."""
        from .gemm import k_slice_plan
        return k_slice_plan(self.variant(problem), problem, num_sms=num_sms)

    def matmul(self, A, B, out=None, stream=None):
        """C = A @ B with the tree-selected variant (device tensors)."""
        import torch

        ops = GemmOperands(A, B, out, input_dtype(self.family))
        vid = self.variant(ops.problem)
        s = (stream or torch.cuda.current_stream(ops.A.device)).cuda_stream
        _lib.check(_lib.load().kp_gemm(vid, *ops.args(), s), f"kp_gemm(variant {vid})")
        return ops.C if (A.dim() == 3 or B.dim() == 3) else ops.C[0]
