"""benchmark sweep: measure every (problem, config) cell of a kernel family on B200 and
produce the reference's PerfMatrix / benchmark CSV (dataset.py:36, :206-278).

This replaces ``synth_generate`` (dataset.py:319-347) as the table producer that
``run_pipeline`` consumes (pipeline.py:149-158).  Methodology follows the paper
(PAPER.md:236-246): warm-up launches, then back-to-back launches bracketed by CUDA
events until a minimum time, mean time per launch -> GFLOP/s = 2*m*k*n*batch / t.

Timers are pluggable: :class:`CudaEventTimer` drives ``kp_bench`` (include/kpgemm.h);
:class:`SynthTimer` is the CPU-only fake hardware backend (the reference's
SynthModel, dataset.py:147-170) used to test sharding and the canonical merge
without a GPU.

Multi-GPU: the sweep is embarrassingly parallel.  Problem rows are sharded across
G worker processes -- one ``multiprocessing.Process`` per non-empty shard, its GPU
fixed with CUDA_VISIBLE_DEVICES at spawn (mapped through the parent's own device
list) -- by longest-processing-time on estimated flops; there is no collective.  Each worker
writes its shard as a partial CSV (resumable: cells already present are skipped)
and the parent merges in canonical order -- problem-list order x config order --
so the table (and hence the k-means seed path, SURVEY.md section 7 hard part 8) is
independent of scheduling.
"""

from __future__ import annotations

import csv
import heapq
import math
import multiprocessing as mp
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Iterable, Protocol

import numpy as np

from .dataset import (KernelConfig, PerfMatrix, ProblemSize, SynthModel, serialize_benchmark_csv,
                      synth_generate)
from .errors import DataError

# Per-cell record of a sweep shard (the partial / resume file).  sm_mhz and temp_c are
# the SM clock and GPU temperature sampled right after the cell's timed loop (NVML;
# empty for timers without a device), the SURVEY 8(d) per-cell conditions record.
SIDECAR_HEADER = "m,k,n,batch,config_index,mean_ms,iters,gflops,sm_mhz,temp_c"
_OLD_SIDECAR_HEADER = "m,k,n,batch,config_index,mean_ms,iters,gflops"


class Timer(Protocol):
    """Measures one cell; returns (gflops, mean_ms, iters).  gflops must be > 0."""

    def __call__(self, problem: ProblemSize, config_index: int) -> tuple[float, float, int]: ...


@dataclass
class SynthTimer:
    """CPU-only fake hardware: the reference's analytic SynthModel
    (dataset.py:147-170) evaluated per cell; noise-free so shards agree."""

    configs: tuple[KernelConfig, ...]
    model: SynthModel = field(default_factory=SynthModel)
    _rows: dict = field(default_factory=dict, repr=False)

    def __call__(self, problem: ProblemSize, config_index: int) -> tuple[float, float, int]:
        # the model's reuse term is normalised over the whole config list, so evaluate
        # a problem's full row once and serve cells from it
        row = self._rows.get(problem)
        if row is None:
            row = synth_generate(self.model, [problem], list(self.configs)).values[0]
            self._rows[problem] = row
        g = float(row[config_index])
        return g, problem.flops / (g * 1e9) * 1e3, 1


class CudaEventTimer:
    """Times kernel-library variants with CUDA events through ``kp_bench``.

    Protocol (adapted from PAPER.md:238-246): warm-up launches, then
    ``repeats`` CUDA-event loops of >= ``min_ms / repeats`` each; the cell's time is the
    median of the loops' per-launch means.  A problem whose operands total less than
    twice the L2 is timed rotating through enough copies of its operands to cover
    2 x L2, so small problems are not measured with a warm cache.  One set of buffers
    sized for the largest problem (U(-1, 1), seed 0) holds every copy.
    """

    def __init__(self, family: str, problems, warmup: int = 2, min_ms: float = 60.0,
                 max_iters: int = 100000, device: int = 0, seed: int = 0, repeats: int = 3):
        import torch  # imported lazily: CPU-only callers never need it

        from . import gemm

        self.torch = torch
        self.gemm = gemm
        self.family = family
        self.configs = gemm.family_configs(family)
        self.warmup, self.min_ms, self.max_iters, self.repeats = warmup, min_ms, max_iters, repeats
        self.l2_bytes = torch.cuda.get_device_properties(torch.device("cuda", device)).L2_cache_size
        self.device = torch.device("cuda", device)
        dtype = gemm.input_dtype(family)
        # every buffer holds at least 2 x L2 of copies (operand rotation), plus alignment slack
        floor = (2 * self.l2_bytes) // gemm.input_dtype(family).itemsize + 64 * 64
        al = 16 // dtype.itemsize  # pitched rows (operands())
        max_a = max(floor, max(p.batch * p.m * -(-p.k // al) * al for p in problems))
        max_b = max(floor, max(p.batch * p.k * -(-p.n // al) * al for p in problems))
        max_c = max(floor, max(p.batch * p.m * -(-p.n // 4) * 4 for p in problems))
        gen = torch.Generator(device=self.device).manual_seed(seed)
        self.bufA = (torch.rand(max_a, device=self.device, generator=gen) * 2 - 1).to(dtype)
        self.bufB = (torch.rand(max_b, device=self.device, generator=gen) * 2 - 1).to(dtype)
        self.bufC = torch.empty(max_c, device=self.device, dtype=torch.float32)
        self.stream = torch.cuda.Stream(self.device)
        self._ops_key = None
        self._ops = None
        self._nvml = None

    def conditions(self) -> tuple[str, str]:
        """(SM clock MHz, temperature C) of this timer's GPU now, via NVML ('' if absent)."""
        if self._nvml is None:
            try:
                import pynvml
                pynvml.nvmlInit()
                idx = self.device.index or 0
                vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
                if vis and all(v.strip().isdigit() for v in vis.split(",")):
                    idx = int(vis.split(",")[idx])  # NVML numbers physical GPUs
                self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx))
            except Exception:
                self._nvml = False
        if not self._nvml:
            return "", ""
        nv, h = self._nvml
        try:
            return (str(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                    str(nv.nvmlDeviceGetTemperature(h, nv.NVML_TEMPERATURE_GPU)))
        except Exception:
            return "", ""

    def operands(self, problem: ProblemSize):
        """Operand sets for the problem: one, or enough copies to cover 2 x L2.  Rows are
        pitched to 16 bytes (leading dimensions rounded up to 16 bytes of elements, as
        cudaMallocPitch / the VGG16 im2col writes them), so ragged k or n (27, 147, ...)
        keep the TMA operand paths; the GEMM itself is the problem's m x k x n."""
        if self._ops_key != problem:
            p = problem
            al = 16 // self.bufA.element_size()
            lda, ldb, ldc = -(-p.k // al) * al, -(-p.n // al) * al, -(-p.n // 4) * 4
            na, nb, nc = p.batch * p.m * lda, p.batch * p.k * ldb, p.batch * p.m * ldc
            foot = na * self.bufA.element_size() + nb * self.bufB.element_size() + nc * 4
            sets = 1 if foot >= 2 * self.l2_bytes else math.ceil(2 * self.l2_bytes / foot)
            pad = lambda x: (x + 63) // 64 * 64  # noqa: E731  (256-byte aligned copies)
            sets = max(1, min(sets, 64, self.bufA.numel() // pad(na), self.bufB.numel() // pad(nb),
                              self.bufC.numel() // pad(nc)))
            ops = []
            for i in range(sets):
                A = self.bufA[i * pad(na): i * pad(na) + na].view(p.batch, p.m, lda)[:, :, :p.k]
                B = self.bufB[i * pad(nb): i * pad(nb) + nb].view(p.batch, p.k, ldb)[:, :, :p.n]
                C = self.bufC[i * pad(nc): i * pad(nc) + nc].view(p.batch, p.m, ldc)[:, :, :p.n]
                ops.append(self.gemm.GemmOperands(A, B, C, A.dtype))
            self._ops = ops
            self._ops_key = problem
        return self._ops

    def __call__(self, problem: ProblemSize, config_index: int) -> tuple[float, float, int]:
        vid = self.gemm.variant_id(self.configs[config_index], self.family)
        ms, iters = self.gemm.bench_sets(vid, self.operands(problem), warmup=self.warmup, min_iters=1,
                                         max_iters=self.max_iters, min_ms=self.min_ms / self.repeats,
                                         repeats=self.repeats, stream=self.stream)
        if not (ms > 0.0 and math.isfinite(ms)):
            raise DataError(f"non-positive time for {problem} / config {config_index}")
        return problem.flops / (ms * 1e-3) / 1e9, ms, iters


# ------------------------------------------------------------------ sharding --
def lpt_shards(problems, n_shards: int, cost: Callable[[ProblemSize], float] | None = None) -> list[list[int]]:
    """Longest-processing-time assignment of problem rows to shards.  Deterministic:
    rows are taken by decreasing cost (ties by row index) and placed on the least
    loaded shard (ties by shard index); each shard lists its rows in row order."""
    if n_shards < 1:
        raise ValueError("need at least one shard")
    cost = cost or (lambda p: float(p.flops))
    order = sorted(range(len(problems)), key=lambda i: (-cost(problems[i]), i))
    heap = [(0.0, s) for s in range(n_shards)]
    shards: list[list[int]] = [[] for _ in range(n_shards)]
    for i in order:
        load, s = heapq.heappop(heap)
        shards[s].append(i)
        heapq.heappush(heap, (load + cost(problems[i]), s))
    return [sorted(rows) for rows in shards]


# ------------------------------------------------------------ partial files --
def _read_partial(path: Path) -> dict[tuple[ProblemSize, int], tuple[float, float, int]]:
    done: dict[tuple[ProblemSize, int], tuple[float, float, int]] = {}
    if not path.exists():
        return done
    with path.open() as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None or ",".join(header) not in (SIDECAR_HEADER, _OLD_SIDECAR_HEADER):
            raise DataError(f"{path}: not a sweep partial file")
        width = len(header)
        for row in reader:
            if len(row) != width:
                continue  # torn last line of an interrupted run
            m, k, n, b, ci = (int(v) for v in row[:5])
            done[(ProblemSize(m, k, n, b), ci)] = (float(row[7]), float(row[5]), int(row[6]))
    return done


def run_shard(problems, rows: Iterable[int], n_configs: int, timer: Timer, partial: Path | None = None,
              progress: Callable[[int, int], None] | None = None):
    """Measure all configs of the given problem rows; append each cell to ``partial``
    as it completes (resume: cells already in the file are not re-measured)."""
    done = _read_partial(partial) if partial is not None else {}
    out = dict(done)
    fh = None
    if partial is not None:
        new = not partial.exists()
        fh = partial.open("a", buffering=1)
        if new:
            fh.write(SIDECAR_HEADER + "\n")
    try:
        rows = list(rows)
        total = len(rows) * n_configs
        count = 0
        for r in rows:
            p = problems[r]
            for ci in range(n_configs):
                count += 1
                if (p, ci) in out:
                    continue
                g, ms, iters = timer(p, ci)
                if not (g > 0.0 and math.isfinite(g)):
                    raise DataError(f"failed measurement for {p} / config {ci}")
                out[(p, ci)] = (g, ms, iters)
                if fh is not None:
                    cond = getattr(timer, "conditions", None)
                    mhz, temp = cond() if cond is not None else ("", "")
                    fh.write(f"{p.m},{p.k},{p.n},{p.batch},{ci},{ms!r},{iters},{g!r},{mhz},{temp}\n")
                if progress is not None:
                    progress(count, total)
    finally:
        if fh is not None:
            fh.close()
    return out


def merge_cells(problems, configs, cells) -> PerfMatrix:
    """Canonical merge: rows in problem-list order, columns in config order."""
    table = np.empty((len(problems), len(configs)))
    for i, p in enumerate(problems):
        for c in range(len(configs)):
            try:
                table[i, c] = cells[(p, c)][0]
            except KeyError:
                raise DataError(f"sweep is missing {p} / {configs[c]}") from None
    return PerfMatrix(tuple(problems), tuple(configs), table)


def device_bindings(gpus: int) -> list[str]:
    """CUDA_VISIBLE_DEVICES value for each of ``gpus`` workers: the parent's own device
    list (a job given GPUs 4-7 by its scheduler sweeps 4-7), else 0..gpus-1."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis is None or vis.strip() == "":
        return [str(g) for g in range(gpus)]
    devs = [v.strip() for v in vis.split(",") if v.strip()]
    if len(devs) < gpus:
        raise ValueError(f"--gpus {gpus} but CUDA_VISIBLE_DEVICES lists only {len(devs)} devices ({vis})")
    return devs[:gpus]


def _worker(gpu_env, problems, rows, family, partial, timer_kind, timer_kw):
    # The binding is fixed before anything touches CUDA in this fresh (spawned) process,
    # and each process measures exactly one shard, so no shard can inherit another's GPU.
    os.environ["CUDA_VISIBLE_DEVICES"] = gpu_env
    Path(partial).with_suffix(".device").write_text(f"{gpu_env} {os.getpid()}\n")
    if timer_kind == "cuda":
        timer = CudaEventTimer(family, [problems[r] for r in rows], **timer_kw)
        n_configs = len(timer.configs)
    else:
        timer = SynthTimer(**timer_kw)
        n_configs = len(timer.configs)
    run_shard(problems, rows, n_configs, timer, Path(partial))


def benchmark_sweep(problems, family: str = "simt", gpus: int = 1, out_dir: str | os.PathLike | None = None,
                    timer: Timer | None = None, configs=None, timer_kind: str = "cuda",
                    timer_kw: dict | None = None, progress=None) -> PerfMatrix:
    """Measure ``family`` over ``problems`` and return the PerfMatrix.

    gpus == 1 runs in-process (``timer`` or a CudaEventTimer).  gpus > 1 spawns one
    worker per GPU on LPT shards (``timer_kind`` 'cuda' or 'synth' for the CPU fake),
    each appending to ``out_dir/shard<g>.csv``; the parent merges canonically.
    """
    problems = list(problems)
    if not problems:
        raise ValueError("no problems to sweep")
    if len(set(problems)) != len(problems):
        raise ValueError("duplicate problems in sweep")
    timer_kw = dict(timer_kw or {})
    out = Path(out_dir) if out_dir is not None else None
    if out is not None:
        out.mkdir(parents=True, exist_ok=True)
    if gpus == 1:
        if timer is None:
            timer = (CudaEventTimer(family, problems, **timer_kw) if timer_kind == "cuda"
                     else SynthTimer(**timer_kw))
        cfgs = tuple(configs) if configs is not None else tuple(timer.configs)
        cells = run_shard(problems, range(len(problems)), len(cfgs), timer,
                          out / "shard0.csv" if out is not None else None, progress)
        return merge_cells(problems, cfgs, cells)
    if out is None:
        raise ValueError("multi-GPU sweeps need out_dir for the shard files")
    shards = lpt_shards(problems, gpus)
    bindings = device_bindings(gpus)
    ctx = mp.get_context("spawn")
    procs = []
    for g in range(gpus):
        if not shards[g]:
            continue  # more GPUs than problem rows: no worker, no CUDA context
        proc = ctx.Process(target=_worker, name=f"sweep-gpu{g}",
                           args=(bindings[g], problems, shards[g], family, str(out / f"shard{g}.csv"),
                                 timer_kind, timer_kw))
        proc.start()
        procs.append(proc)
    failed = []
    for proc in procs:
        proc.join()
        if proc.exitcode != 0:
            failed.append(f"{proc.name} exit {proc.exitcode}")
    if failed:
        raise RuntimeError("sweep workers failed: " + ", ".join(failed))
    cells: dict = {}
    for g in range(gpus):
        if shards[g]:
            cells.update(_read_partial(out / f"shard{g}.csv"))
    if configs is None:
        if timer_kind == "synth":
            configs = timer_kw["configs"]
        else:
            from . import gemm
            configs = gemm.family_configs(family)
    return merge_cells(problems, tuple(configs), cells)


def write_benchmark_csv(pm: PerfMatrix, path: str | os.PathLike) -> None:
    """Reference-format CSV, written atomically (temp then rename, pipeline.py:81-84)."""
    path = Path(path)
    tmp = path.with_suffix(path.suffix + ".tmp")
    tmp.write_text(serialize_benchmark_csv(pm))
    os.replace(tmp, path)


def problem_set(name: str, batches=(1, 2, 4, 8, 16, 32, 64)) -> list[ProblemSize]:
    """Named sweep shape sets: vgg16 / resnet50 (conv-as-GEMM x batches), vgg16+paper
    (vgg16 then the paper's three sample problems, shapes.PAPER_SAMPLES), square,
    square16k."""
    from . import shapes

    if name in shapes.NETWORKS:
        return shapes.network_problems(name, batches)
    if name == "vgg16+paper":
        rows = shapes.network_problems("vgg16", batches)
        return rows + [p for p in shapes.PAPER_SAMPLES if p not in rows]
    if name == "square":  # 64..8192 squares + skinny extremes (full 640-config families)
        return shapes.square_skinny_problems(sizes=(64, 128, 256, 512, 1024, 2048, 4096, 8192))
    if name == "square16k":  # adds 16384^3 (tensor-core families)
        return shapes.square_skinny_problems()
    raise ValueError(f"unknown problem set {name!r}")


def main(argv=None) -> int:
    """python -m paper_2008_13145_b200.sweep --set vgg16 --family simt --out table.csv"""
    import argparse
    import sys
    import time

    ap = argparse.ArgumentParser(description=main.__doc__)
    ap.add_argument("--set", default="vgg16", help="vgg16 | resnet50 | square")
    ap.add_argument("--batches", default="1,2,4,8,16,32,64")
    ap.add_argument("--family", default="simt")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--out", required=True, help="benchmark CSV (reference format)")
    ap.add_argument("--work", default=None, help="shard/partial directory (default: <out>.parts)")
    ap.add_argument("--min-ms", type=float, default=60.0,
                    help="timed ms per cell, split over 3 loops (SURVEY 8(d): loops >= 20 ms)")
    args = ap.parse_args(argv)
    problems = problem_set(args.set, tuple(int(b) for b in args.batches.split(",")))
    work = Path(args.work or (args.out + ".parts"))
    t0 = time.time()
    last = [0.0]

    def progress(done, total):
        now = time.time()
        if now - last[0] > 30 or done == total:
            last[0] = now
            el = now - t0
            print(f"[sweep] {done}/{total} cells  {el:.0f}s elapsed  eta {el / max(done, 1) * (total - done):.0f}s",
                  file=sys.stderr, flush=True)

    pm = benchmark_sweep(problems, family=args.family, gpus=args.gpus, out_dir=work,
                         timer_kw={"min_ms": args.min_ms}, progress=progress)
    write_benchmark_csv(pm, args.out)
    print(f"[sweep] wrote {args.out}: {pm.n_problems} problems x {pm.n_configs} configs in {time.time() - t0:.0f}s",
          file=sys.stderr)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
