#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the B200 kernel family.

Workload (BASELINE.json configs[1]): the VGG16 conv-as-GEMM layer set on one B200,
dispatched by the decision tree trained on the measured B200 sweep of the F1 (simt)
family with a k-means 4-kernel subset.  One step = every GEMM layer of one VGG16
forward pass at batch B (16 launches: 13 conv layers lowered im2col-style with the
batch folded into m, 3 fc layers), each launched through the C dispatch table
(kp_gemm with the tree-selected variant).  Inputs are synthetic U(-1,1) activations
and He-scaled weights of the VGG16 layer shapes; the per-step inputs (~4.3 GB at
B=16) exceed the 126 MB L2, so no L2 flush is needed between steps.

JSON line keys: value = GFLOP/s of the dispatched step (inputs resident in HBM);
e2e = the same layer set fed from HOST memory: every step uploads each layer's input
activation (NHWC, pinned) and reads every layer's output back, with the conv layers'
im2col done on the device (kp_im2col3x3_nhwc) inside the timed region; roofline = the
dominant launch against min(pipe peak, arithmetic intensity x HBM bandwidth);
selection = the north-star metric (geomean fraction of per-shape oracle-best GFLOP/s
of the k-means subset + tree on the held-out split, evaluate.py:71-101);
cpu_baseline = np.matmul fp32 (numpy/OpenBLAS, the reference package's numeric
engine; the reference ships no GEMM) on all host cores over the SAME layer set and
batch; cpu_port = the bit-exact fmaf-chain oracle port on the same sample.
``--impl reference`` runs the np.matmul CPU path alone on the same config.

``--gpus N`` without a torchrun environment re-launches this script under
``torch.distributed.run`` with N ranks; under torchrun WORLD_SIZE must equal N.
``--workload vgg16-infer`` is BASELINE configs[2] (images/s, data parallel);
``--workload sweep`` times the sharded benchmark sweep (configs[3], one LPT shard of
problem rows per rank, no collective) and checks the merged table's canonical order.
The default line also carries ``companions``: a short run of each of those two on the same
ranks (so a driver ``--gpus N`` scaling run times DP inference and the sharded sweep at
every N too); ``--no-companions`` skips them.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

DEFAULT_TABLE = ROOT / "data" / "sweeps" / "vgg16_simt.csv"
METRIC = "geomean % of oracle-best GFLOP/s (clustered set + tree); GFLOP/s vs FP32 peak"


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (ranks); default 1, or WORLD_SIZE under torchrun")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--batch", type=int, default=16, help="VGG16 images per step per GPU")
    ap.add_argument("--table", default=str(DEFAULT_TABLE), help="measured B200 sweep CSV")
    ap.add_argument("--family", default="simt")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--method", default="kmeans")
    ap.add_argument("--classifier", default="treeA")
    ap.add_argument("--workload", choices=("gemm-layers", "vgg16-infer", "sweep"), default="gemm-layers",
                    help="gemm-layers: BASELINE configs[1] (default); vgg16-infer: configs[2], data parallel; "
                         "sweep: the benchmark sweep sharded over the ranks")
    ap.add_argument("--sweep-set", default="vgg16", help="sweep workload: vgg16 | resnet50 | square")
    ap.add_argument("--sweep-stride", type=int, default=10,
                    help="sweep workload: every n-th config of the family (1 = the full table)")
    ap.add_argument("--sweep-min-ms", type=float, default=1.0, help="sweep workload: timed ms per cell")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-companions", action="store_true",
                    help="skip the short DP VGG16-inference and sharded-sweep measurements in the default line")
    return ap.parse_args(argv)


# ------------------------------------------------------------------ helpers --
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period: float = 0.02):
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None
        self.period = period

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nvml is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def dist_setup(args):
    """One process per GPU (torchrun env).  The process group pairs gloo for the host-side
    timing collectives (max-over-ranks, barrier) with NCCL for device tensors; the data
    path has no collective.  Returns (world, rank, device index)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours":
        import torch
        if torch.cuda.is_available():
            local = local % torch.cuda.device_count()  # ranks > GPUs share (code-path tests only)
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group(backend="cpu:gloo,cuda:nccl")
    return world, rank, local


def reduce_max(value: float, world: int, device=None) -> float:
    """Max over ranks (the contract's multi-GPU timing rule), on the host group."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.all_reduce(torch.zeros(1), op=dist.ReduceOp.SUM)  # host-group barrier


# ---------------------------------------------------------------- selection --
def train_selector(table_path: str, k: int, method: str, classifier: str):
    """Measured table -> (subset, tree, report_test, report_all, timings)."""
    from paper_2008_13145_b200 import classify, dataset, evaluate, selection
    from paper_2008_13145_b200.normalize import NormScheme, normalize

    t = {}
    t0 = time.perf_counter()
    pm = dataset.parse_benchmark_csv(Path(table_path).read_text())
    t["parse_s"] = time.perf_counter() - t0
    train, test = dataset.split(pm, dataset.SplitSpec(0.2, 0))
    t0 = time.perf_counter()
    nm = normalize(train, NormScheme("scaled"))
    subset = selection.select_subset(method, nm, k, 0, problems=train.problems)
    t["select_s"] = time.perf_counter() - t0
    labels = classify.label_best_in_subset(nm, subset)
    t0 = time.perf_counter()
    tree = classify.train_tree(classify.problem_features(train.problems), labels,
                               classify.TREE_PRESETS[classifier[-1]], n_classes=subset.k_actual)
    t["train_s"] = time.perf_counter() - t0
    predict = lambda x: classify.predict_tree(tree, x)  # noqa: E731
    rep_test = evaluate.classifier_score(test, subset, predict)
    rep_all = evaluate.classifier_score(pm, subset, predict)
    return pm, subset, tree, rep_test, rep_all, t


def selection_grid(pm, ks=(4, 8), methods=("kmeans", "spectral", "pca_kmeans", "tree")):
    """Held-out geomean fraction of oracle-best (evaluate.py:71-101) for other cells of
    the paper's grid on the same table, treeA -- reported beside the headline cell."""
    from paper_2008_13145_b200 import classify, dataset, evaluate, selection
    from paper_2008_13145_b200.normalize import NormScheme, normalize

    train, test = dataset.split(pm, dataset.SplitSpec(0.2, 0))
    nm = normalize(train, NormScheme("scaled"))
    feats = classify.problem_features(train.problems)
    out = {}
    for method in methods:
        for k in ks:
            try:
                sub = selection.select_subset(method, nm, k, 0, problems=train.problems)
            except Exception:
                continue
            labels = classify.label_best_in_subset(nm, sub)
            tree = classify.train_tree(feats, labels, classify.TREE_PRESETS["A"], n_classes=sub.k_actual)
            rep = evaluate.classifier_score(test, sub, lambda x, t=tree: classify.predict_tree(t, x))
            out[f"{method}{k}"] = {"k_actual": sub.k_actual, "achieved_test": rep.achieved, "ceiling_test": rep.ceiling}
    return out


# ----------------------------------------------------------------- workload --
def vgg16_layers(batch: int):
    from paper_2008_13145_b200 import shapes
    out = []
    for layer in shapes.VGG16_LAYERS:
        for _ in range(layer.count):
            out.append((layer.name, layer.problem(batch)))
    return out


def _layer_operands(batch: int, seed: int = 0):
    import numpy as np

    rng = np.random.default_rng(seed)
    layers = vgg16_layers(batch)
    ops = [(rng.uniform(-1, 1, (p.m, p.k)).astype(np.float32), rng.uniform(-1, 1, (p.k, p.n)).astype(np.float32))
           for _, p in layers]
    return ops, sum(p.flops for _, p in layers)


def cpu_numpy_steps(batch: int, steps: int, warmup: int = 0):
    """np.matmul fp32 (numpy -> OpenBLAS on every host core) over the VGG16 GEMM layer
    set at ``batch``: the reference package's numeric engine (SURVEY.md 8(c)/(d) CPU
    plan; the reference itself ships no GEMM).  Returns (GFLOP/s, per-step seconds,
    flops per step, cores)."""
    import numpy as np

    ops, flops = _layer_operands(batch)
    secs = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        for A, B in ops:
            np.matmul(A, B)
        dt = time.perf_counter() - t0
        if i >= warmup:
            secs.append(dt)
    return flops * len(secs) / sum(secs) / 1e9, secs, flops, _blas_threads()


def _blas_threads() -> int:
    """Threads OpenBLAS actually uses (torchrun exports OMP_NUM_THREADS=1, so the
    reference arm raises it to every host CPU before numpy is imported)."""
    try:
        from threadpoolctl import threadpool_info
        n = [d["num_threads"] for d in threadpool_info() if d.get("internal_api") == "openblas"]
        if n:
            return int(n[0])
    except Exception:
        pass
    return os.cpu_count() or 1


def cpu_port_line(batch: int):
    """The bit-exact oracle port (oracle/gemm_ref.c fmaf chain, OpenMP over every host
    CPU) on the same layer set and batch, one pass: TEST INFRASTRUCTURE used as the
    checker and a second CPU timing only."""
    from oracle import gemm_oracle as go

    threads = go.set_threads()
    ops, flops = _layer_operands(batch)
    t0 = time.perf_counter()
    for A, B in ops:
        go.gemm_chain(A, B)
    dt = time.perf_counter() - t0
    return {"value": flops / dt / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "sample": f"VGG16 GEMM layer set at batch {batch} ({flops / 1e9:.1f} GFLOP, one pass), "
                      "oracle/gemm_ref.c bit-exact fmaf chain, OpenMP over rows"}


def run_reference(args, world, rank):
    """--impl reference: the CPU path on the host cores, rank 0 only, SAME config as the
    GPU arm (VGG16 GEMM layer set at --batch): np.matmul fp32 on every host core."""
    if rank != 0:
        return 0
    gf, secs, flops, cores = cpu_numpy_steps(args.batch, args.steps, args.warmup)
    sample = (f"the full VGG16 GEMM layer set at batch {args.batch} ({flops / 1e9:.1f} GFLOP/step, "
              f"{len(secs)} steps after {args.warmup} warm-up), np.matmul fp32 -> OpenBLAS")
    line = {"metric": METRIC, "value": gf, "unit": "GFLOP/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(secs) / len(secs) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"vgg16-gemm-layers-b{args.batch}-{args.method}{args.k}-{args.classifier}",
                       "batch_per_gpu": args.batch, "same_config_as_gpu_arm": True},
            "cpu_baseline": {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                             "sample": sample,
                             "note": "the reference package has no GEMM; numpy (its only numeric engine) is "
                                     "the CPU path it would call"},
            "e2e": {"value": gf, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def c_dispatch_cost(disp, problems, reps: int = 2000) -> float:
    """Host cost of one runtime selection through the C table (kp_dispatch_select: log2
    features + tree walk + class -> variant), microseconds per call including the ctypes
    call; the Dispatcher caches the result per shape, so the timed GEMM loop never pays it."""
    from paper_2008_13145_b200 import _lib

    lib = _lib.load()
    t0 = time.perf_counter()
    for _ in range(reps):
        for p in problems:
            lib.kp_dispatch_select(disp.handle, p.m, p.k, p.n, p.batch)
    return (time.perf_counter() - t0) / (reps * len(problems)) * 1e6


# ----------------------------------------------------------------- roofline --
def measured_peaks() -> dict:
    path = ROOT / "MEASURED_PEAKS.json"
    try:
        return json.loads(path.read_text()) if path.exists() else {}
    except Exception:
        return {}


def roofline(family: str, p, ms: float, in_bytes: int, simt_peak: float | None = None) -> dict:
    """Roofline of one launch: attainable = min(pipe peak, AI x HBM bandwidth) with the
    algorithmic bytes in_bytes*(mk + kn) + 4*mn; the binding term
    decides whether the launch is reported in TFLOP/s or GB/s."""
    from paper_2008_13145_b200 import gemm

    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 0.0)) or 7700.0
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if peaks.get("hbm_gbs") else "nominal 7.7 TB/s (no MEASURED_PEAKS.json)"
    if family in ("tf32", "bf16"):
        pipe = float(peaks.get("bf16_tflops", 0.0)) or 2250.0
        pipe_src = "MEASURED_PEAKS.json bf16_tflops" if peaks.get("bf16_tflops") else "nominal 2.25 PF/s bf16"
        if family == "tf32":
            pipe, pipe_src = pipe / 2, pipe_src + " x 1/2 (tf32 rate)"
        pipe_name = f"tcgen05 {family}"
    else:
        pipe = simt_peak if simt_peak is not None else gemm.ffma_peak_tflops(packed=True)
        pipe_src = "kp_ffma_peak on this device (FFMA2 register loop; MEASURED_PEAKS.json has no FP32 figure)"
        pipe_name = "fp32 FFMA2 (SIMT)"
    flops = p.flops
    nbytes = p.batch * (in_bytes * (p.m * p.k + p.k * p.n) + 4 * p.m * p.n)
    ai = flops / nbytes
    sec = ms * 1e-3
    if ai * hbm / 1e3 < pipe:  # HBM-bound: AI x BW (GB/s -> TFLOP/s) is the lower roof
        return {"bound": "hbm", "achieved": nbytes / sec / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": nbytes / sec / 1e9 / hbm, "pipe": pipe_name, "peak_source": hbm_src,
                "algorithmic_bytes": nbytes, "flops_per_launch": flops, "arith_intensity": ai,
                "achieved_tflops": flops / sec / 1e12}
    return {"bound": "tensor" if family in ("tf32", "bf16") else "compute", "achieved": flops / sec / 1e12,
            "peak": pipe, "unit": "TFLOP/s", "frac": flops / sec / 1e12 / pipe, "pipe": pipe_name,
            "peak_source": pipe_src, "algorithmic_bytes": nbytes, "flops_per_launch": flops, "arith_intensity": ai,
            "hbm_roof_tflops": ai * hbm / 1e3}


# ---------------------------------------------------------------------- e2e --
def e2e_layers(args, world, device, stream, disp, bufs, step_flops, in_dtype):
    """The layer set through the public API from HOST memory: every step uploads each
    layer's input activation from pinned memory -- NHWC (B, H, W, Cin) for the conv
    layers, (B, k) rows for fc -- lowers the conv ones on the device (kp_im2col3x3_nhwc,
    + kp_cast_bf16 for the BF16 family), runs the dispatched GEMM and copies every
    layer's output back to pinned memory.  Uploads run on one copy stream, downloads on
    another, overlapping the compute stream layer by layer.  FLOPs counted are the GEMMs'
    only (im2col is extra work inside the timed region)."""
    import torch

    from paper_2008_13145_b200 import _lib, gemm, shapes

    lib = _lib.load()
    geo = {}
    for layer in shapes.VGG16_LAYERS:
        geo[layer.name] = None if layer.fc else (math.isqrt(layer.m_per_image), layer.k // 9)
    names = []
    for layer in shapes.VGG16_LAYERS:
        names += [layer.name] * layer.count
    gen = torch.Generator().manual_seed(99)
    host_in, dev_in = [], []
    for (name, p, A, W, C, vid), lname in zip(bufs, names):
        g = geo[lname]
        shape = (args.batch, g[0], g[0], g[1]) if g else (p.m, p.k)
        h = (torch.rand(shape, generator=gen) * 2 - 1).pin_memory()
        host_in.append(h)
        dev_in.append(torch.empty(shape, device=device))
    host_out = [torch.empty(C.shape, dtype=C.dtype, pin_memory=True) for *_, C, _ in bufs]
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(t.numel() * t.element_size() for t in host_out)
    bf16 = in_dtype == torch.bfloat16
    h2d_stream, d2h_stream = torch.cuda.Stream(device), torch.cuda.Stream(device)
    landed = [torch.cuda.Event() for _ in bufs]
    computed = [torch.cuda.Event() for _ in bufs]
    s_handle = stream.cuda_stream
    launches = [0]

    implicit = [geo[lname] is not None and gemm.conv3x3_supported(vid, geo[lname][1], p.n)
                for (name, p, A, W, C, vid), lname in zip(bufs, names)]

    def lower(i, lname, p, A):
        """Device-side operand for layer i: im2col (conv, into A's pitched rows) / cast
        (bf16 fc) into A."""
        g = geo[lname]
        x = dev_in[i]
        if g is None and not bf16:
            return x
        if g is not None:
            if bf16:
                _lib.check(lib.kp_im2col3x3_nhwc_bf16(x.data_ptr(), args.batch, g[0], g[0], g[1], A.data_ptr(),
                                                      A.stride(0), s_handle), "kp_im2col3x3_nhwc_bf16")
            else:
                _lib.check(lib.kp_im2col3x3_nhwc(x.data_ptr(), args.batch, g[0], g[0], g[1], A.data_ptr(),
                                                 A.stride(0), s_handle), "kp_im2col3x3_nhwc")
            launches[0] += 1
            return A
        _lib.check(lib.kp_cast_bf16(x.data_ptr(), p.m * p.k, A.data_ptr(), s_handle), "kp_cast_bf16")
        launches[0] += 1
        return A

    def e2e_step():
        with torch.cuda.stream(h2d_stream):
            for i in range(len(bufs)):
                dev_in[i].copy_(host_in[i], non_blocking=True)
                landed[i].record(h2d_stream)
        for i, ((name, p, A, W, C, vid), lname) in enumerate(zip(bufs, names)):
            stream.wait_event(landed[i])
            g = geo[lname]
            if g is not None and implicit[i]:
                # implicit GEMM: the dispatched variant gathers the patches from the NHWC
                # activation with TMA im2col copies (kp_conv3x3_nhwc_ex), no im2col pass
                x = dev_in[i]
                if bf16:  # BF16 family: a bf16 copy of the activation (A's rows hold m*k >= its size)
                    _lib.check(lib.kp_cast_bf16(x.data_ptr(), x.numel(), A.data_ptr(), s_handle), "kp_cast_bf16")
                    launches[0] += 1
                    x = A
                _lib.check(lib.kp_conv3x3_nhwc_ex(vid, x.data_ptr(), args.batch, g[0], g[0], g[1], W.data_ptr(), p.n,
                                                  C.data_ptr(), None, 0, s_handle), "kp_conv3x3_nhwc_ex")
            else:
                operand = lower(i, lname, p, A)
                disp.matmul(operand, W, out=C, stream=stream)
            launches[0] += 1
            computed[i].record(stream)
            d2h_stream.wait_event(computed[i])
            with torch.cuda.stream(d2h_stream):
                host_out[i].copy_(C, non_blocking=True)
        stream.wait_stream(d2h_stream)
        h2d_stream.wait_stream(stream)  # the next step's uploads may not overwrite inputs in use

    with torch.cuda.stream(stream):
        for _ in range(max(1, args.warmup)):
            e2e_step()
    torch.cuda.synchronize(device)
    barrier(world)
    launches[0] = 0
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        f0.record(stream)
        h2d_stream.wait_stream(stream)
        for _ in range(args.steps):
            e2e_step()
        f1.record(stream)
    torch.cuda.synchronize(device)
    e2e_ms = reduce_max(f0.elapsed_time(f1), world, device)
    return {"value": step_flops * args.steps * world / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps,
            "launches_per_step": launches[0] // args.steps,
            "implicit_conv_layers": sum(implicit),
            "path": "host NHWC activations -> H2D -> conv layers: kp_conv3x3_nhwc_ex (implicit GEMM, TMA im2col) "
                    "where the dispatched variant supports it" + (" on a kp_cast_bf16 copy" if bf16 else "") +
                    ", else kp_im2col3x3_nhwc" + ("_bf16" if bf16 else "") + " + Dispatcher.matmul (kp_gemm) -> D2H of every layer output"}


# --------------------------------------------------------------- companions --
def run_companions(args, world, rank, local):
    """Short measurements of the other multi-GPU rows on the same ranks, so every
    `--gpus N` run of the default line also times them at N: BASELINE configs[2] (VGG16
    inference, data parallel by batch, 16 images per GPU, CUDA graph) and the benchmark
    sweep sharded by LPT over the ranks (configs[3]-style, every ~10th config of the
    family on the VGG16 problem set, 1 ms loops).  Each is its own workload's JSON line
    (``--workload vgg16-infer`` / ``sweep``), condensed; rank 0 returns the dict."""
    import copy

    from paper_2008_13145_b200 import gemm

    a = copy.copy(args)
    a.batch, a.steps, a.warmup = 16, 10, 3
    v = run_vgg16_infer(a, world, rank, local, emit=False)
    s = copy.copy(args)
    s.sweep_set, s.sweep_min_ms, s.steps, s.warmup = "vgg16", 1.0, 1, 1
    s.sweep_stride = max(1, len(gemm.family_configs(args.family)) // 10)
    w = run_sweep(s, world, rank, local, emit=False)
    if rank != 0:
        return None
    keep = ("value", "unit", "n_gpus", "ms_per_step", "scaling", "clocks")
    return {"vgg16_infer_dp": dict({k: v[k] for k in keep}, config=v["config"], e2e=v["e2e"], gflops=v["gflops"]),
            "sweep_sharded": dict({k: w[k] for k in keep}, config=w["config"], shard_rows=w["shard_rows"],
                                  merged_canonical=w["merged_canonical"])}


# ---------------------------------------------------------------------- ours --
def run_ours(args, world, rank, local):
    import torch

    from paper_2008_13145_b200 import gemm
    from paper_2008_13145_b200.dispatch import Dispatcher

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    pm, subset, tree, rep_test, rep_all, sel_t = train_selector(args.table, args.k, args.method, args.classifier)
    disp = Dispatcher(tree, subset, pm.configs, args.family)

    layers = vgg16_layers(args.batch)
    in_dtype = gemm.input_dtype(args.family)  # fp32, or bf16 operands for the BF16 family
    sel_t["c_tree_walk_us_per_call"] = c_dispatch_cost(disp, [p for _, p in layers])
    gen = torch.Generator(device=device).manual_seed(1234 + rank)
    bufs = []
    al = 16 // in_dtype.itemsize  # rows pitched to 16 bytes, as the sweep times them (conv1_1: k = 27)
    for name, p in layers:
        A = (torch.rand(p.m, -(-p.k // al) * al, device=device, generator=gen) * 2 - 1).to(in_dtype)[:, :p.k]
        W = ((torch.rand(p.k, p.n, device=device, generator=gen) * 2 - 1) * math.sqrt(6.0 / p.k)).to(in_dtype)
        C = torch.empty(p.m, p.n, device=device)
        bufs.append((name, p, A, W, C, disp.variant(p)))
    step_flops = sum(p.flops for _, p in layers)
    stream = torch.cuda.Stream(device)

    def step(events=None):
        for i, (name, p, A, W, C, vid) in enumerate(bufs):
            if events is not None:
                events[i][0].record(stream)
            disp.matmul(A, W, out=C, stream=stream)
            if events is not None:
                events[i][1].record(stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize(device)

    per_launch = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in bufs] for _ in range(args.steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize(device)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for s in range(args.steps):
            step(per_launch[s])
        e1.record(stream)
        torch.cuda.synchronize(device)
    barrier(world)
    ms = e0.elapsed_time(e1)
    ms_max = reduce_max(ms, world, device)
    value = step_flops * args.steps * world / (ms_max * 1e-3) / 1e9

    # dominant kernel: the (variant, problem) pair with the largest summed device time
    # (conv4_2 and conv4_3 share one shape and variant, so they merge)
    layer_ms = [0.0] * len(bufs)
    for s in range(args.steps):
        for i, (a, b) in enumerate(per_launch[s]):
            layer_ms[i] += a.elapsed_time(b)
    groups: dict = {}
    for i, (name, p, _A, _W, _C, vid) in enumerate(bufs):
        g = groups.setdefault((vid, p), {"ms": 0.0, "launches": 0, "names": []})
        g["ms"] += layer_ms[i]
        g["launches"] += args.steps
        g["names"].append(name)
    (dvid, dp), dg = max(groups.items(), key=lambda kv: kv[1]["ms"])
    variant_ms = sum(g["ms"] for (v, _), g in groups.items() if v == dvid)
    dom_ms = dg["ms"] / dg["launches"]
    dom_cfg, dom_fam = gemm.variant_info(dvid)
    dname = "+".join(dg["names"])
    roof = roofline(dom_fam, dp, dom_ms, in_dtype.itemsize)
    traffic = None
    prof = ROOT / "profiles" / "dominant_kernel_traffic.json"
    if prof.exists():
        try:
            rec = json.loads(prof.read_text())
            for r in rec.get("launches", [rec]):
                if (r.get("family", "simt") == dom_fam and r.get("variant") == list(dom_cfg.as_tuple())
                        and r.get("problem") == [dp.m, dp.k, dp.n, dp.batch]):
                    traffic = r.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roof["traffic"] = traffic
    total_ms = sum(layer_ms)
    # every layer against its own roofline (the binding term of min(pipe, AI x HBM))
    simt_peak = gemm.ffma_peak_tflops(packed=True) if args.family in ("simt", "paper") else None
    per_layer = []
    for i, (name, p, _A, _W, _C, vid) in enumerate(bufs):
        cfg, fam = gemm.variant_info(vid)
        r = roofline(fam, p, layer_ms[i] / args.steps, in_dtype.itemsize, simt_peak)
        per_layer.append({"layer": name, "problem": [p.m, p.k, p.n], "variant": list(cfg.as_tuple()),
                          "ms": round(layer_ms[i] / args.steps, 4), "bound": r["bound"],
                          "achieved": round(r["achieved"], 1), "unit": r["unit"], "frac": round(r["frac"], 3)})

    e2e = None if args.no_e2e else e2e_layers(args, world, device, stream, disp, bufs, step_flops, in_dtype)

    companions = None if args.no_companions else run_companions(args, world, rank, local)

    cpu = cpu_port = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gf, secs, flops, cores = cpu_numpy_steps(args.batch, steps=1, warmup=1)
        cpu = {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": "reference",
               "sample": f"the same VGG16 GEMM layer set at batch {args.batch} ({flops / 1e9:.1f} GFLOP, one step "
                         "after one warm-up), np.matmul fp32 -> OpenBLAS (the reference package's numeric engine; "
                         "it ships no GEMM)"}
        cpu_port = cpu_port_line(args.batch)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": {"bf16": "bf16", "tf32": "tf32"}.get(args.family, "f32"),
            "data": "synthetic",
            "config": {"workload": f"vgg16-gemm-layers-b{args.batch}-{args.method}{args.k}-{args.classifier}",
                       "batch_per_gpu": args.batch, "family": args.family, "table": os.path.relpath(args.table, ROOT),
                       "table_shape": [pm.n_problems, pm.n_configs], "parallelism": f"replicas{world}",
                       "l2": "per-step inputs ~%.1f GB > 126 MB L2 (no flush needed)" %
                             (sum(A.numel() * A.element_size() for _, _, A, _, _, _ in bufs) / 1e9)},
            "selection": {"method": args.method, "k": args.k, "classifier": args.classifier,
                          "subset": [list(pm.configs[i].as_tuple()) for i in subset.config_indices],
                          "achieved_test": rep_test.achieved, "ceiling_test": rep_test.ceiling,
                          "achieved_all_rows": rep_all.achieved, "ceiling_all_rows": rep_all.ceiling,
                          "host_s": sel_t},
            "selection_grid_treeA": selection_grid(pm),
            "gpu_launches": len(bufs) * args.steps,
            "gpu_launches_e2e": e2e["launches_per_step"] * args.steps if e2e else None,
            "roofline": dict(roof, kernel=f"{dom_fam}{dom_cfg.as_tuple()} on {dname} {[dp.m, dp.k, dp.n, dp.batch]}",
                             avg_launch_ms=dom_ms, share_of_step=dg["ms"] / total_ms,
                             variant_share_of_step=variant_ms / total_ms),
            "layers": per_layer,
            "clocks": clocks.summary(),
        }
        if e2e is not None:
            line["e2e"] = e2e
        if companions is not None:
            line["companions"] = companions
        if cpu is not None:
            line["cpu_baseline"] = cpu
            line["cpu_port"] = cpu_port
        print(json.dumps(line), flush=True)
    return 0


def run_vgg16_infer(args, world, rank, local, emit=True):
    """BASELINE configs[2]: VGG16 inference, fp32, tree-dispatched GEMMs, data parallel
    by batch (each rank its own images, replicated weights, no collective).  value =
    images/s over all ranks; the forward is one CUDA graph per rank."""
    import torch

    from paper_2008_13145_b200.dispatch import Dispatcher
    from paper_2008_13145_b200.vgg16 import Vgg16

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    pm, subset, tree, rep_test, rep_all, sel_t = train_selector(args.table, args.k, args.method, args.classifier)
    disp = Dispatcher(tree, subset, pm.configs, args.family)
    model = Vgg16(disp, args.batch, device, seed=0)
    stream = torch.cuda.Stream(device)
    g = torch.Generator().manual_seed(100 + rank)
    host_x = torch.randn(args.batch, 224, 224, 3, generator=g).pin_memory()
    host_y = torch.empty(args.batch, 1000, pin_memory=True)
    model.input.copy_(host_x)
    model.capture(stream)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            model.forward(stream=stream)
    torch.cuda.synchronize(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                model.forward(stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(device)
    barrier(world)
    ms = reduce_max(e0.elapsed_time(e1), world, device)
    flops = model.flops
    value = args.batch * args.steps * world / (ms * 1e-3)
    # e2e: every step's images H2D from pinned memory and logits D2H.  The next step's
    # upload runs on a copy stream into a second staging buffer while this step's forward
    # runs (double buffering, as a serving loop would); the step then takes its images
    # with a device-to-device copy into the graph's input buffer.
    copy_stream = torch.cuda.Stream(device)
    staging = [torch.empty_like(model.input) for _ in range(2)]
    landed = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize(device)
    f0.record(stream)
    copy_stream.wait_stream(stream)

    def upload(slot):
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[slot])
            staging[slot].copy_(host_x, non_blocking=True)
            landed[slot].record(copy_stream)

    for slot in range(2):
        consumed[slot].record(stream)  # both staging buffers start free
    upload(0)
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            j = i % 2
            if i + 1 < args.steps:
                upload((i + 1) % 2)
            stream.wait_event(landed[j])
            model.input.copy_(staging[j], non_blocking=True)
            consumed[j].record(stream)
            model.forward(stream=stream)
            host_y.copy_(model.logits, non_blocking=True)
        f1.record(stream)
    torch.cuda.synchronize(device)
    e2e_ms = reduce_max(f0.elapsed_time(f1), world, device)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": {"bf16": "bf16", "tf32": "tf32"}.get(args.family, "f32"), "data": "synthetic (He-init weights)",
                "config": {"workload": f"vgg16-infer-b{args.batch}-{args.method}{args.k}-{args.classifier}",
                           "batch_per_gpu": args.batch, "family": args.family, "parallelism": f"dp{world}",
                           "table": os.path.relpath(args.table, ROOT), "cuda_graph": True},
                "gflops": flops * args.steps * world / (ms * 1e-3) / 1e9,
                "selection": {"achieved_test": rep_test.achieved, "ceiling_test": rep_test.ceiling,
                              "achieved_all_rows": rep_all.achieved},
                "gpu_launches": (16 + 13 + 5) * args.steps, "clocks": clocks.summary(),
                "e2e": {"value": args.batch * args.steps * world / (e2e_ms * 1e-3), "unit": "images/s",
                        "h2d_bytes_per_step": host_x.numel() * 4, "d2h_bytes_per_step": host_y.numel() * 4}}
        if not emit:
            return line
        print(json.dumps(line), flush=True)
    return 0 if emit else None


def run_sweep(args, world, rank, local, emit=True):
    """BASELINE configs[3]-style sweep scaling: the benchmark sweep of ``--sweep-set``
    over every ``--sweep-stride``-th config of ``--family``, problem rows sharded across
    the ranks by LPT (sweep.lpt_shards; no collective on the data path), each rank
    measuring its shard on its own GPU into a partial CSV.  Rank 0 merges canonically
    and asserts the row / column order.  value = table cells per second over the whole
    job (strong scaling: the table is fixed, more ranks finish it sooner); the time is
    each rank's shard bracketed by CUDA events on its timer stream, max over ranks."""
    import tempfile

    import torch

    from paper_2008_13145_b200 import gemm, sweep

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    problems = sweep.problem_set(args.sweep_set)
    all_cfgs = gemm.family_configs(args.family)
    cols = list(range(0, len(all_cfgs), max(1, args.sweep_stride)))
    cfgs = tuple(all_cfgs[c] for c in cols)
    shards = sweep.lpt_shards(problems, world)
    mine = shards[rank]
    timer = sweep.CudaEventTimer(args.family, [problems[r] for r in mine] or problems[:1], device=local,
                                 min_ms=args.sweep_min_ms)

    class Columns:  # the strided config subset as a timer over local column indices
        configs = cfgs

        def __call__(self, problem, ci):
            return timer(problem, cols[ci])

        def conditions(self):
            return timer.conditions()

    work = Path(os.environ.get("KP_BENCH_SWEEP_DIR") or
                Path(tempfile.gettempdir()) / f"kp_bench_sweep_{os.environ.get('MASTER_PORT', os.getpid())}")
    work.mkdir(parents=True, exist_ok=True)
    part = work / f"shard{rank}.csv"
    for w in range(args.warmup):  # warm-up: one cell per rank (module load, clocks)
        timer(problems[mine[0] if mine else 0], cols[w % len(cols)])
    torch.cuda.synchronize(device)
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(timer.stream)
        total_ms = 0.0
        for s in range(args.steps):
            if part.exists():
                part.unlink()  # each step re-measures the shard from scratch
            sweep.run_shard(problems, mine, len(cfgs), Columns(), part)
        e1.record(timer.stream)
        torch.cuda.synchronize(device)
        total_ms = e0.elapsed_time(e1)
    ms = reduce_max(total_ms, world, device)
    barrier(world)
    if rank != 0:
        return 0 if emit else None
    cells = {}
    for r in range(world):
        if shards[r]:
            cells.update(sweep._read_partial(work / f"shard{r}.csv"))
    pm = sweep.merge_cells(problems, cfgs, cells)
    assert list(pm.problems) == list(problems) and list(pm.configs) == list(cfgs), "merge is not canonical"
    n_cells = len(problems) * len(cfgs)
    flops = sum(p.flops for p in problems) * len(cfgs)
    line = {"metric": METRIC, "value": n_cells * args.steps / (ms * 1e-3), "unit": "cells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": {"bf16": "bf16", "tf32": "tf32"}.get(args.family, "f32"),
            "data": "synthetic",
            "config": {"workload": f"sweep-{args.sweep_set}-{args.family}-stride{args.sweep_stride}",
                       "table_shape": [len(problems), len(cfgs)], "min_ms_per_cell": args.sweep_min_ms,
                       "parallelism": f"lpt-shards{world}", "l2": "operands rotated over >= 2 x L2 per cell"},
            "shard_rows": [len(sh) for sh in shards], "merged_canonical": True,
            "timed_gflop_per_step": flops / 1e9, "clocks": clocks.summary(),
            "gpu_launches": None}
    if not emit:
        return line
    print(json.dumps(line), flush=True)
    return 0


def self_launch(args, argv) -> int | None:
    """--gpus N outside torchrun: re-run this script under torch.distributed.run with N
    ranks (127.0.0.1 rendezvous) and return its exit code; None when no launch is
    needed.  Under torchrun, WORLD_SIZE must match --gpus."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if args.gpus is not None and int(env_world) != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")
        return None
    if (args.gpus or 1) <= 1:
        return None
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *(argv if argv is not None else sys.argv[1:])]
    return subprocess.call(cmd)


def main(argv=None):
    args = parse_args(argv)
    rc = self_launch(args, argv)
    if rc is not None:
        return rc
    if args.impl == "reference":
        # torchrun exports OMP_NUM_THREADS=1; the CPU arm uses every host core
        n = str(os.cpu_count() or 1)
        os.environ["OMP_NUM_THREADS"] = n
        os.environ["OPENBLAS_NUM_THREADS"] = n
    world, rank, local = dist_setup(args)
    if args.gpus is None:
        args.gpus = world
    try:
        if args.impl == "reference":
            return run_reference(args, world, rank)
        if args.workload == "vgg16-infer":
            return run_vgg16_infer(args, world, rank, local)
        if args.workload == "sweep":
            return run_sweep(args, world, rank, local)
        return run_ours(args, world, rank, local)
    finally:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    raise SystemExit(main())
