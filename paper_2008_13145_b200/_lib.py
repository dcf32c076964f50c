"""ctypes binding of libkpgemm.so (include/kpgemm.h).

The shared library is built in-tree (``make -C paper_2008_13145_b200/csrc``) and
loaded from this package directory.  There is no CPU fallback: when the library is
missing every GEMM entry point raises :class:`KernelLibraryError`.

Status codes map onto the reference's error taxonomy (errors.py:1-49):
KP_EINVAL -> ValueError, KP_ENOENT -> KeyError, KP_EIO -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_NAME = "libkpgemm.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

KP_OK = 0
KP_ENOENT = -2
KP_EIO = -5
KP_EINVAL = -22
KP_EPI_RELU = 1
KP_EPI_BF16_OUT = 2

FAMILY_PAPER = 0
FAMILY_SIMT = 1
FAMILY_TF32 = 2
FAMILY_BF16 = 3
FAMILY_NAMES = {FAMILY_PAPER: "paper", FAMILY_SIMT: "simt",
                FAMILY_TF32: "tf32", FAMILY_BF16: "bf16"}
FAMILY_IDS = {v: k for k, v in FAMILY_NAMES.items()}


class KernelLibraryError(RuntimeError):
    """libkpgemm.so is missing or failed to load; there is no fallback."""


class KernelChoice(ctypes.Structure):
    """Field order of the emitted selector's return value (codegen.py:191-192)."""

    _fields_ = [("tile_rows", ctypes.c_int32), ("tile_acc", ctypes.c_int32),
                ("tile_cols", ctypes.c_int32), ("wg_rows", ctypes.c_int32),
                ("wg_cols", ctypes.c_int32)]

    def as_tuple(self) -> tuple[int, int, int, int, int]:
        return (self.tile_rows, self.tile_acc, self.tile_cols, self.wg_rows, self.wg_cols)


_i = ctypes.c_int
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_i32p = ctypes.POINTER(ctypes.c_int32)
_vpp = ctypes.POINTER(ctypes.c_void_p)

_GEMM_ARGS = [_i, _i, _i, _i, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64]

# name -> (restype, argtypes); every symbol include/kpgemm.h declares.
SIGNATURES = {
    "kp_abi_version": (_i, []),
    "kp_last_error": (ctypes.c_char_p, []),
    "kp_num_variants": (_i, []),
    "kp_find_variant": (_i, [_i, KernelChoice]),
    "kp_variant_info": (_i, [_i, ctypes.POINTER(KernelChoice), _ip]),
    "kp_family_size": (_i, [_i]),
    "kp_family_variant": (_i, [_i, _i]),
    "kp_gemm": (_i, [_i] + _GEMM_ARGS + [_vp]),
    "kp_gemm_ex": (_i, [_i] + _GEMM_ARGS + [_vp, _i, _vp]),
    "kp_set_max_k_slices": (_i, [_i]),
    "kp_set_simt_staging": (_i, [_i]),
    "kp_set_operand_repack": (_i, [_i]),
    "kp_gemm_plan": (_i, [_i, _i, _i, _i, _i, _i, _ip, _ip]),
    "kp_bench": (_i, [_i] + _GEMM_ARGS + [_i, _i, _i, ctypes.c_double, _dp, _ip, _vp]),
    "kp_bench_sets": (_i, [_i, _i, _i, _i, _i, _i, _vpp, _i64, _i64, _vpp, _i64, _i64, _vpp, _i64, _i64,
                           _i, _i, _i, ctypes.c_double, _i, _dp, _ip, _vp]),
    "kp_ffma_peak": (_i, [_i, _dp, _vp]),
    "kp_dispatch_load": (_i, [_i, _i32p, _dp, _i32p, _i32p, _i32p, _i, _i32p]),
    "kp_dispatch_free": (_i, [_i]),
    "kp_dispatch_class_feats": (_i, [_i, _dp]),
    "kp_dispatch_select_feats": (_i, [_i, _dp]),
    "kp_dispatch_select": (_i, [_i, _i, _i, _i, _i]),
    "kp_gemm_auto": (_i, [_i] + _GEMM_ARGS + [_vp, _ip]),
    "kp_gemm_auto_ex": (_i, [_i] + _GEMM_ARGS + [_vp, _i, _vp, _ip]),
    "kp_im2col3x3_nhwc": (_i, [_vp, _i, _i, _i, _i, _vp, _i64, _vp]),
    "kp_maxpool2x2_nhwc": (_i, [_vp, _i, _i, _i, _i, _vp, _vp]),
    "kp_maxpool2x2_nhwc_bf16": (_i, [_vp, _i, _i, _i, _i, _vp, _vp]),
    "kp_conv3x3_supported": (_i, [_i, _i, _i]),
    "kp_conv3x3_nhwc_ex": (_i, [_i, _vp, _i, _i, _i, _i, _vp, _i, _vp, _vp, _i, _vp]),
    "kp_im2col3x3_nhwc_pad": (_i, [_vp, _i, _i, _i, _i, _vp, _i, _vp]),
    "kp_im2col3x3_nhwc_bf16": (_i, [_vp, _i, _i, _i, _i, _vp, _i, _vp]),
    "kp_cast_bf16": (_i, [_vp, _i64, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes handle; raises KernelLibraryError."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        # KPGEMM_LIB: development override (e.g. an experimental build); default in-tree
        p = Path(path) if path is not None else Path(os.environ.get("KPGEMM_LIB", LIB_PATH))
        if not p.exists():
            raise KernelLibraryError(
                f"{p} not found: build it with `make -C paper_2008_13145_b200/csrc -j8` "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as exc:
            raise KernelLibraryError(f"cannot load {p}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    msg = load().kp_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> int:
    """Map a negative kp_* status onto the reference's exception taxonomy."""
    if rc >= 0:
        return rc
    msg = f"{what}: {last_error()}"
    if rc == KP_EINVAL:
        raise ValueError(msg)
    if rc == KP_ENOENT:
        raise KeyError(msg)
    raise RuntimeError(msg)
