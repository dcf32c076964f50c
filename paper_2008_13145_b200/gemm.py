"""matmul-with-config: launch one variant of the sm_100a kernel family on torch
CUDA tensors through the C ABI (include/kpgemm.h, ``kp_gemm``).

The reference describes the kernel only as a contract -- a config is
``KernelConfig(R, A, C, wg_rows, wg_cols)`` (dataset.py:39-58) and the kernel
computes C = A @ B per batch.  This module is that operator.
Families (include/kpgemm.h): ``paper`` (F0, paper-faithful, no shared memory),
``simt`` (F1, B200 SIMT pipeline), ``tf32`` / ``bf16`` (tcgen05 tensor cores).
There is no CPU or library fallback: a missing kernel library raises.
"""

from __future__ import annotations

import ctypes
from functools import lru_cache

import torch

from . import _lib
from .dataset import KernelConfig, ProblemSize

FAMILIES = ("paper", "simt", "tf32", "bf16")


def _family_id(family: str | int) -> int:
    if isinstance(family, int):
        if family not in _lib.FAMILY_NAMES:
            raise ValueError(f"unknown family {family!r}")
        return family
    try:
        return _lib.FAMILY_IDS[family]
    except KeyError:
        raise ValueError(f"unknown family {family!r}, expected one of {FAMILIES}") from None


def family_list(spec: str | int) -> tuple:
    """A table spec names one family ("simt") or several joined by '+' ("simt+tf32");
    a combined table's columns are the families' config lists concatenated (their
    5-tuples are disjoint)."""
    if isinstance(spec, int):
        return (spec,)
    return tuple(spec.split("+"))


@lru_cache(maxsize=None)
def variant_id(config: KernelConfig, family: str | int = "simt") -> int:
    """Kernel-library variant id of (family, config); for a combined spec the first
    family holding the tuple wins.  KeyError if absent."""
    lib = _lib.load()
    choice = _lib.KernelChoice(*config.as_tuple())
    fams = family_list(family)
    for fam in fams[:-1]:
        rc = lib.kp_find_variant(_family_id(fam), choice)
        if rc >= 0:
            return rc
    return _lib.check(lib.kp_find_variant(_family_id(fams[-1]), choice),
                      f"kp_find_variant({family}, {config.as_tuple()})")


def variant_info(vid: int) -> tuple[KernelConfig, str]:
    lib = _lib.load()
    choice = _lib.KernelChoice()
    fam = _lib.ctypes.c_int()
    _lib.check(lib.kp_variant_info(vid, _lib.ctypes.byref(choice), _lib.ctypes.byref(fam)),
               f"kp_variant_info({vid})")
    return KernelConfig(*choice.as_tuple()), _lib.FAMILY_NAMES[fam.value]


@lru_cache(maxsize=None)
def family_configs(family: str | int) -> tuple[KernelConfig, ...]:
    """The family's canonical config list (its benchmark-table column order); for a
    combined spec, the concatenation."""
    lib = _lib.load()
    out = []
    for fam in family_list(family):
        fid = _family_id(fam)
        size = _lib.check(lib.kp_family_size(fid), "kp_family_size")
        out += [variant_info(_lib.check(lib.kp_family_variant(fid, i), "kp_family_variant"))[0]
                for i in range(size)]
    if len(set(out)) != len(out):
        raise ValueError(f"families of {family!r} share config tuples")
    return tuple(out)


def input_dtype(family: str | int) -> torch.dtype:
    dts = {torch.bfloat16 if _family_id(f) == _lib.FAMILY_BF16 else torch.float32 for f in family_list(family)}
    if len(dts) != 1:
        raise ValueError(f"families of {family!r} take different operand types; use separate tables")
    return dts.pop()


class GemmOperands:
    """Validated (batch, m, k) x (batch, k, n) operand view for the C ABI."""

    __slots__ = ("A", "B", "C", "m", "k", "n", "batch", "lda", "sA", "ldb", "sB", "ldc", "sC")

    def __init__(self, A: torch.Tensor, B: torch.Tensor, out: torch.Tensor | None, dtype: torch.dtype):
        if A.dim() not in (2, 3) or B.dim() not in (2, 3):
            raise ValueError("A and B must be 2-D (m,k)/(k,n) or 3-D batched")
        if not (A.is_cuda and B.is_cuda):
            raise ValueError("operands must be CUDA tensors (there is no CPU path)")
        if A.dtype != dtype or B.dtype != dtype:
            raise ValueError(f"operands must be {dtype}, got {A.dtype} and {B.dtype}")
        A3 = A if A.dim() == 3 else A.unsqueeze(0)
        B3 = B if B.dim() == 3 else B.unsqueeze(0)
        batch = max(A3.shape[0], B3.shape[0])
        for name, t in (("A", A3), ("B", B3)):
            if t.shape[0] not in (1, batch):
                raise ValueError(f"{name} batch {t.shape[0]} does not broadcast to {batch}")
            if t.stride(2) != 1:
                raise ValueError(f"{name} rows must be contiguous (stride(-1) == 1)")
        m, k = A3.shape[1], A3.shape[2]
        if B3.shape[1] != k:
            raise ValueError(f"inner dimensions differ: A is (.., {m}, {k}), B is (.., {B3.shape[1]}, {B3.shape[2]})")
        n = B3.shape[2]
        if A.device != B.device:
            raise ValueError(f"A is on {A.device} but B is on {B.device}")
        if out is None:
            out = torch.empty((batch, m, n), device=A.device, dtype=torch.float32)
        else:
            if not out.is_cuda or out.device != A.device:
                raise ValueError(f"out must be a CUDA tensor on {A.device}, got {out.device}")
            if out.dtype != torch.float32 or out.dim() not in (2, 3) or tuple(out.shape[-2:]) != (m, n) \
                    or out.stride(-1) != 1:
                raise ValueError("out must be float32 (m, n) or (batch, m, n) with contiguous rows")
            if out.dim() == 3 and out.shape[0] != batch:
                raise ValueError(f"out batch {out.shape[0]} != operand batch {batch}")
            if out.dim() == 2 and batch > 1:
                raise ValueError(f"a batched product (batch {batch}) needs a 3-D out")
        C3 = out if out.dim() == 3 else out.unsqueeze(0)
        self.A, self.B, self.C = A3, B3, C3
        self.m, self.k, self.n, self.batch = m, k, n, batch
        self.lda = A3.stride(1) if m > 1 else k
        self.ldb = B3.stride(1) if k > 1 else n
        self.ldc = C3.stride(1) if m > 1 else n
        self.sA = A3.stride(0) if A3.shape[0] > 1 else 0
        self.sB = B3.stride(0) if B3.shape[0] > 1 else 0
        self.sC = C3.stride(0) if batch > 1 else m * self.ldc

    def args(self):
        return (self.m, self.k, self.n, self.batch,
                self.A.data_ptr(), self.lda, self.sA,
                self.B.data_ptr(), self.ldb, self.sB,
                self.C.data_ptr(), self.ldc, self.sC)

    @property
    def problem(self) -> ProblemSize:
        return ProblemSize(self.m, self.k, self.n, self.batch)


def _squeeze_like(C3: torch.Tensor, A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    return C3 if (A.dim() == 3 or B.dim() == 3) else C3[0]


def launch(vid: int, ops: GemmOperands, stream: torch.cuda.Stream | None = None) -> None:
    lib = _lib.load()
    s = (stream or torch.cuda.current_stream(ops.A.device)).cuda_stream
    _lib.check(lib.kp_gemm(vid, *ops.args(), s), f"kp_gemm(variant {vid}, {ops.problem})")


def matmul(A: torch.Tensor, B: torch.Tensor, config: KernelConfig, family: str = "simt",
           out: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """C = A @ B with the kernel variant ``(family, config)``.

    A: (m, k) or (batch, m, k); B: (k, n) or (batch, k, n) -- a 2-D operand is
    broadcast over the batch (stride 0, e.g. conv weights).  fp32 operands for
    paper/simt/tf32, bf16 for bf16; the result is fp32.
    """
    vid = variant_id(config, family)
    ops = GemmOperands(A, B, out, input_dtype(family))
    launch(vid, ops, stream)
    return _squeeze_like(ops.C, A, B)


def conv3x3_supported(vid: int, cin: int, cout: int) -> bool:
    """Whether variant ``vid`` runs an implicit-GEMM 3x3 conv (kp_conv3x3_supported)."""
    return _lib.check(_lib.load().kp_conv3x3_supported(vid, cin, cout), "kp_conv3x3_supported") == 1


def conv3x3(x: torch.Tensor, w: torch.Tensor, vid: int, bias: torch.Tensor | None = None, relu: bool = False,
            out: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """3x3 / stride 1 / pad 1 convolution of NHWC ``x`` (B, H, W, Cin) with the (9*Cin, Cout)
    weight matrix ``w`` (k order (dy, dx, c), as kp_im2col3x3_nhwc) as an implicit GEMM on
    SIMT, TF32 or BF16 variant ``vid`` (TMA im2col copies; kp_conv3x3_nhwc_ex).  ``x`` and
    ``w`` are fp32 for SIMT/TF32 variants and bf16 for BF16 variants; the result,
    (B, H, W, Cout), is bit-identical to im2col + matmul with the same variant -- fp32, or
    rounded to bf16 when ``out`` is bf16 (tensor-core variants only, KP_EPI_BF16_OUT)."""
    dt = input_dtype(variant_info(vid)[1])
    if x.dim() != 4 or not x.is_cuda or x.dtype != dt or not x.is_contiguous():
        raise ValueError(f"x must be a contiguous (B, H, W, C) {dt} CUDA tensor for variant {vid}")
    B, H, W, C = x.shape
    if w.shape[0] != 9 * C or w.dim() != 2 or w.dtype != dt or not w.is_contiguous() \
            or w.device != x.device:
        raise ValueError(f"w must be a contiguous ({9 * C}, Cout) {dt} tensor on {x.device}")
    cout = w.shape[1]
    if out is None:
        out = torch.empty(B, H, W, cout, device=x.device)
    elif (out.shape != (B, H, W, cout) or out.dtype not in (torch.float32, torch.bfloat16)
          or not out.is_contiguous() or out.device != x.device):
        raise ValueError(f"out must be a contiguous ({B}, {H}, {W}, {cout}) fp32 (or bf16, tensor-core "
                         f"variants: KP_EPI_BF16_OUT) tensor on {x.device}")
    flags = (_lib.KP_EPI_RELU if relu else 0) | (_lib.KP_EPI_BF16_OUT if out.dtype == torch.bfloat16 else 0)
    if bias is not None and (bias.shape != (cout,) or bias.dtype != torch.float32 or bias.device != x.device):
        raise ValueError(f"bias must be a ({cout},) fp32 tensor on {x.device}")
    s = (stream or torch.cuda.current_stream(x.device)).cuda_stream
    _lib.check(_lib.load().kp_conv3x3_nhwc_ex(vid, x.data_ptr(), B, H, W, C, w.data_ptr(), cout, out.data_ptr(),
                                              bias.data_ptr() if bias is not None else None, flags, s),
               f"kp_conv3x3_nhwc_ex(variant {vid}, {tuple(x.shape)} x {cout})")
    return out


def bench(vid: int, ops: GemmOperands, warmup: int = 1, min_iters: int = 2, max_iters: int = 10000,
          min_ms: float = 2.0, stream: torch.cuda.Stream | None = None) -> tuple[float, int]:
    """Mean milliseconds per launch by CUDA events (``kp_bench``) and the loop count."""
    lib = _lib.load()
    s = (stream or torch.cuda.current_stream(ops.A.device)).cuda_stream
    mean = _lib.ctypes.c_double()
    iters = _lib.ctypes.c_int()
    _lib.check(lib.kp_bench(vid, *ops.args(), warmup, min_iters, max_iters, float(min_ms),
                            _lib.ctypes.byref(mean), _lib.ctypes.byref(iters), s),
               f"kp_bench(variant {vid}, {ops.problem})")
    return mean.value, iters.value


def bench_sets(vid: int, sets: list[GemmOperands], warmup: int = 2, min_iters: int = 1, max_iters: int = 10000,
               min_ms: float = 1.0, repeats: int = 3, stream: torch.cuda.Stream | None = None) -> tuple[float, int]:
    """Median over ``repeats`` timed loops of the per-launch mean (ms), launches rotating
    through operand ``sets`` of one shape (``kp_bench_sets``; SURVEY 8(d) protocol)."""
    lib = _lib.load()
    first = sets[0]
    s = (stream or torch.cuda.current_stream(first.A.device)).cuda_stream
    n = len(sets)
    A = (ctypes.c_void_p * n)(*[o.A.data_ptr() for o in sets])
    B = (ctypes.c_void_p * n)(*[o.B.data_ptr() for o in sets])
    C = (ctypes.c_void_p * n)(*[o.C.data_ptr() for o in sets])
    med = ctypes.c_double()
    iters = ctypes.c_int()
    _lib.check(lib.kp_bench_sets(vid, first.m, first.k, first.n, first.batch, n, A, first.lda, first.sA, B, first.ldb,
                                 first.sB, C, first.ldc, first.sC, warmup, min_iters, max_iters, float(min_ms),
                                 repeats, ctypes.byref(med), ctypes.byref(iters), s),
               f"kp_bench_sets(variant {vid}, {first.problem})")
    return med.value, iters.value


def k_slice_plan(config: KernelConfig | int, problem: ProblemSize, family: str = "simt",
                 num_sms: int = 0) -> tuple[int, int]:
    """(k_slices, k_per_slice) the library uses for this launch (kp_gemm_plan):
    SIMT launches that cannot fill the GPU sum k-slices in order; (1, k) otherwise.
    num_sms <= 0 asks the current CUDA device."""
    vid = config if isinstance(config, int) else variant_id(config, family)
    s, per = ctypes.c_int(0), ctypes.c_int(0)
    _lib.check(_lib.load().kp_gemm_plan(vid, problem.m, problem.k, problem.n, problem.batch, num_sms,
                                        ctypes.byref(s), ctypes.byref(per)), "kp_gemm_plan")
    return s.value, per.value


def set_max_k_slices(max_slices: int) -> int:
    """Cap the SIMT family's k-slicing (1 = off: every output is the single fma chain
    over k, bit-identical to the paper family); returns the previous cap."""
    return _lib.check(_lib.load().kp_set_max_k_slices(int(max_slices)), "kp_set_max_k_slices")


def set_simt_staging(mode: str) -> str:
    """SIMT operand staging: "tma" (bulk tensor copies + mbarriers wherever the rows are
    16-byte aligned; the default) or "cp.async" (per-thread copies).  Results are
    bit-identical; returns the previous mode."""
    modes = {"cp.async": 0, "tma": 1}
    if mode not in modes:
        raise ValueError(f"staging mode must be one of {sorted(modes)}, got {mode!r}")
    prev = _lib.check(_lib.load().kp_set_simt_staging(modes[mode]), "kp_set_simt_staging")
    return "tma" if prev else "cp.async"


def set_operand_repack(mode: str) -> str:
    """Operands whose rows TMA cannot address (kp_set_operand_repack): "auto" repacks them
    into 16-byte-pitched scratch when that pays (default), "always", or "never" (in-kernel
    staging); returns the previous mode.  Results are the same either way."""
    modes = {"never": 0, "auto": 1, "always": 2}
    if mode not in modes:
        raise ValueError(f"repack mode must be one of {sorted(modes)}, got {mode!r}")
    prev = _lib.check(_lib.load().kp_set_operand_repack(modes[mode]), "kp_set_operand_repack")
    return {v: k for k, v in modes.items()}[prev]


def ffma_peak_tflops(packed: bool = False, stream: torch.cuda.Stream | None = None) -> float:
    """Measured FP32 peak of the current device (kp_ffma_peak): scalar FFMA or,
    with ``packed``, sm_100 FFMA2."""
    lib = _lib.load()
    s = (stream or torch.cuda.current_stream()).cuda_stream
    out = _lib.ctypes.c_double()
    _lib.check(lib.kp_ffma_peak(int(packed), _lib.ctypes.byref(out), s), "kp_ffma_peak")
    return out.value
