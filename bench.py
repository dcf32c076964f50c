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
e2e = the same with host-pinned activations copied H2D and outputs copied D2H inside
the timed region; roofline = the dominant launch against the measured FP32 FFMA2 peak;
selection = the north-star metric (geomean fraction of per-shape oracle-best GFLOP/s
of the k-means subset + tree on the held-out split, evaluate.py:71-101);
cpu_baseline = the oracle port (oracle/gemm_ref.c fmaf chain, all host threads) on
a bounded sample (batch 1).  ``--impl reference`` runs that CPU path alone.
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
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--batch", type=int, default=16, help="VGG16 images per step per GPU")
    ap.add_argument("--table", default=str(DEFAULT_TABLE), help="measured B200 sweep CSV")
    ap.add_argument("--family", default="simt")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--method", default="kmeans")
    ap.add_argument("--classifier", default="treeA")
    ap.add_argument("--workload", choices=("gemm-layers", "vgg16-infer"), default="gemm-layers",
                    help="gemm-layers: BASELINE configs[1] (default); vgg16-infer: configs[2], data parallel")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
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


def cpu_baseline(batch: int = 1, repeats: int = 2):
    """Oracle port (oracle/gemm_ref.c, bit-exact fmaf chain, all host threads) on the
    VGG16 layer set at ``batch``: GFLOP/s.  TEST INFRASTRUCTURE used as the checker
    and CPU reference timing only."""
    import numpy as np

    from oracle import gemm_oracle as go

    threads = go.set_threads()  # all host CPUs, whatever OMP_NUM_THREADS the launcher set
    layers = vgg16_layers(batch)
    rng = np.random.default_rng(0)
    ops = [(rng.uniform(-1, 1, (p.m, p.k)).astype(np.float32), rng.uniform(-1, 1, (p.k, p.n)).astype(np.float32))
           for _, p in layers]
    flops = sum(p.flops for _, p in layers)
    best = math.inf
    for _ in range(repeats):
        t0 = time.perf_counter()
        for A, B in ops:
            go.gemm_chain(A, B)
        best = min(best, time.perf_counter() - t0)
    return flops / best / 1e9, best, flops, threads


def cpu_blas_line(batch: int = 1, repeats: int = 2):
    """Strongest CPU comparison: np.matmul fp32 (OpenBLAS, all host threads) on the same
    bounded sample -- the reference package's numeric engine; reported
    beside cpu_baseline, never a product path."""
    import numpy as np

    layers = vgg16_layers(batch)
    rng = np.random.default_rng(0)
    ops = [(rng.uniform(-1, 1, (p.m, p.k)).astype(np.float32), rng.uniform(-1, 1, (p.k, p.n)).astype(np.float32))
           for _, p in layers]
    flops = sum(p.flops for _, p in layers)
    best = math.inf
    for _ in range(repeats):
        t0 = time.perf_counter()
        for A, B in ops:
            np.matmul(A, B)
        best = min(best, time.perf_counter() - t0)
    return {"value": flops / best / 1e9, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "numpy-openblas",
            "sample": f"VGG16 GEMM layer set at batch {batch} ({flops / 1e9:.2f} GFLOP, best of {repeats}), "
                      "np.matmul fp32 (not the bit-exact fma chain)"}


def run_reference(args, world, rank):
    """--impl reference: the CPU path (oracle port) on the host cores; rank 0 only."""
    if rank != 0:
        return 0
    sample_batch = 1
    gf, secs, flops = None, [], 0
    from oracle import gemm_oracle as go
    import numpy as np
    cores = go.set_threads()  # torchrun exports OMP_NUM_THREADS=1; use every host CPU
    layers = vgg16_layers(sample_batch)
    rng = np.random.default_rng(0)
    ops = [(rng.uniform(-1, 1, (p.m, p.k)).astype(np.float32), rng.uniform(-1, 1, (p.k, p.n)).astype(np.float32))
           for _, p in layers]
    flops = sum(p.flops for _, p in layers)
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for A, B in ops:
            go.gemm_chain(A, B)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            secs.append(dt)
    total = sum(secs)
    gf = flops * len(secs) / total / 1e9
    sample = (f"VGG16 GEMM layer set at batch {sample_batch} ({flops / 1e9:.2f} GFLOP/step) instead of batch "
              f"{args.batch}; oracle/gemm_ref.c fmaf chain, OpenMP over rows")
    line = {"metric": METRIC, "value": gf, "unit": "GFLOP/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / len(secs) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"vgg16-gemm-layers-b{args.batch}-kmeans{args.k}-{args.classifier}",
                       "batch": args.batch},
            "cpu_baseline": {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": gf, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


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
    gen = torch.Generator(device=device).manual_seed(1234 + rank)
    bufs = []
    for name, p in layers:
        A = (torch.rand(p.m, p.k, device=device, generator=gen) * 2 - 1).to(in_dtype)
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
    tensor = dom_fam in ("tf32", "bf16")
    if tensor:  # tensor-pipe roofline: MEASURED_PEAKS.json dense bf16 (TF32 at half rate)
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        peak = float(peaks.get("bf16_tflops", 2250.0)) * (0.5 if dom_fam == "tf32" else 1.0)
        peak_source = ("MEASURED_PEAKS.json bf16_tflops" if peaks else "nominal 2.25 PF/s bf16") + \
            (" x 1/2 (tf32 rate)" if dom_fam == "tf32" else "")
    else:
        peak = gemm.ffma_peak_tflops(packed=True)
        peak_source = ("measured on this device by kp_ffma_peak (FFMA2 register loop); "
                       "MEASURED_PEAKS.json has no FP32 SIMT figure")
    achieved = dp.flops / (dom_ms * 1e-3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "dominant_kernel_traffic.json"
    if prof.exists():
        try:
            rec = json.loads(prof.read_text())
            for r in rec.get("launches", [rec]):
                if r.get("variant") == list(dom_cfg.as_tuple()) and r.get("problem") == [dp.m, dp.k, dp.n, dp.batch]:
                    traffic = r.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    total_ms = sum(layer_ms)

    # e2e: host-pinned activations in, outputs out, through the dispatcher
    e2e = None
    if not args.no_e2e:
        host_in = [A.cpu().pin_memory() for _, _, A, _, _, _ in bufs]
        host_out = [torch.empty(C.shape, dtype=C.dtype, pin_memory=True) for _, _, _, _, C, _ in bufs]
        dev_in = [torch.empty_like(A) for _, _, A, _, _, _ in bufs]
        h2d = sum(t.numel() * t.element_size() for t in host_in)
        d2h = sum(t.numel() * t.element_size() for t in host_out)

        # three-stage pipeline over the layers: H2D of layer i+1 (copy stream) and D2H
        # of layer i-1 (second copy engine) overlap the GEMM of layer i (compute stream)
        h2d_stream, d2h_stream = torch.cuda.Stream(device), torch.cuda.Stream(device)
        landed = [torch.cuda.Event() for _ in bufs]
        computed = [torch.cuda.Event() for _ in bufs]

        def e2e_step():
            for i, (name, p, A, W, C, vid) in enumerate(bufs):
                with torch.cuda.stream(h2d_stream):
                    dev_in[i].copy_(host_in[i], non_blocking=True)
                    landed[i].record(h2d_stream)
            for i, (name, p, A, W, C, vid) in enumerate(bufs):
                stream.wait_event(landed[i])
                disp.matmul(dev_in[i], W, out=C, stream=stream)
                computed[i].record(stream)
                d2h_stream.wait_event(computed[i])
                with torch.cuda.stream(d2h_stream):
                    host_out[i].copy_(C, non_blocking=True)
            stream.wait_stream(d2h_stream)
            h2d_stream.wait_stream(stream)  # next step's H2D may not overwrite inputs in use

        with torch.cuda.stream(stream):
            for _ in range(max(1, args.warmup)):
                e2e_step()
        torch.cuda.synchronize(device)
        barrier(world)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            f0.record(stream)
            h2d_stream.wait_stream(stream)
            for _ in range(args.steps):
                e2e_step()
            f1.record(stream)
        torch.cuda.synchronize(device)
        e2e_ms = reduce_max(f0.elapsed_time(f1), world, device)
        e2e = {"value": step_flops * args.steps * world / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps}

    cpu = cpu_blas = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gf, secs, flops, threads = cpu_baseline(batch=1)
        cpu = {"value": gf, "unit": "GFLOP/s", "cores": threads, "kind": "port",
               "sample": f"VGG16 GEMM layer set at batch 1 ({flops / 1e9:.2f} GFLOP, best of 2) with "
                         f"oracle/gemm_ref.c (bit-exact fmaf chain, OpenMP all threads)"}
        cpu_blas = cpu_blas_line(batch=1)

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
                             (sum(A.numel() * 4 for _, _, A, _, _, _ in bufs) / 1e9)},
            "selection": {"method": args.method, "k": args.k, "classifier": args.classifier,
                          "subset": [list(pm.configs[i].as_tuple()) for i in subset.config_indices],
                          "achieved_test": rep_test.achieved, "ceiling_test": rep_test.ceiling,
                          "achieved_all_rows": rep_all.achieved, "ceiling_all_rows": rep_all.ceiling,
                          "host_s": sel_t},
            "selection_grid_treeA": selection_grid(pm),
            "gpu_launches": len(bufs) * args.steps,
            "roofline": {"bound": "tensor" if tensor else "compute",
                         "pipe": f"tcgen05 {dom_fam}" if tensor else "fp32 FFMA2 (SIMT)", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes": in_dtype.itemsize * (dp.m * dp.k + dp.k * dp.n) + 4 * dp.m * dp.n,
                         "flops_per_launch": dp.flops, "avg_launch_ms": dom_ms,
                         "kernel": f"{dom_fam}{dom_cfg.as_tuple()} on {dname} {[dp.m, dp.k, dp.n, dp.batch]}",
                         "share_of_step": dg["ms"] / total_ms, "variant_share_of_step": variant_ms / total_ms,
                         "peak_source": peak_source},
            "clocks": clocks.summary(),
        }
        if e2e is not None:
            line["e2e"] = e2e
        if cpu is not None:
            line["cpu_baseline"] = cpu
            line["cpu_blas"] = cpu_blas
        print(json.dumps(line), flush=True)
    return 0


def run_vgg16_infer(args, world, rank, local):
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
        print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    args = parse_args(argv)
    world, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            return run_reference(args, world, rank)
        if args.workload == "vgg16-infer":
            return run_vgg16_infer(args, world, rank, local)
        return run_ours(args, world, rank, local)
    finally:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    raise SystemExit(main())
