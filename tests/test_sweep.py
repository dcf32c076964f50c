"""Sweep harness host logic on CPU with the fake hardware timer (the reference's
SynthModel, dataset.py:147-170): LPT sharding, canonical merge independent of
scheduling, multi-process (G=2) == serial, resumable partial files, and the merged CSV
is the reference wire format (dataset.py:36, :206-278)."""

import numpy as np
import pytest

from paper_2008_13145_b200 import shapes, sweep
from paper_2008_13145_b200.dataset import (PerfMatrix, ProblemSize, SynthModel, enumerate_configs,
                                           parse_benchmark_csv, serialize_benchmark_csv, synth_generate)

CFGS = tuple(enumerate_configs()[:40])
PROBS = shapes.network_problems("vgg16", batches=(1, 2, 4))


def test_lpt_shards_partition_and_balance():
    shards = sweep.lpt_shards(PROBS, 3)
    flat = sorted(i for s in shards for i in s)
    assert flat == list(range(len(PROBS)))
    loads = [sum(PROBS[i].flops for i in s) for s in shards]
    assert max(loads) <= 1.6 * (sum(loads) / 3) + max(p.flops for p in PROBS)
    assert sweep.lpt_shards(PROBS, 3) == shards  # deterministic
    with pytest.raises(ValueError):
        sweep.lpt_shards(PROBS, 0)


def test_serial_sweep_equals_synth_generate():
    timer = sweep.SynthTimer(CFGS, SynthModel())
    pm = sweep.benchmark_sweep(PROBS, timer=timer, configs=CFGS)
    assert pm == synth_generate(SynthModel(), PROBS, list(CFGS))


def test_two_process_sweep_equals_serial(tmp_path):
    serial = sweep.benchmark_sweep(PROBS, timer=sweep.SynthTimer(CFGS, SynthModel()), configs=CFGS)
    par = sweep.benchmark_sweep(PROBS, gpus=2, out_dir=tmp_path, timer_kind="synth",
                                timer_kw={"configs": CFGS, "model": SynthModel()}, configs=CFGS)
    assert par == serial
    assert (tmp_path / "shard0.csv").exists() and (tmp_path / "shard1.csv").exists()
    text = serialize_benchmark_csv(par)
    assert parse_benchmark_csv(text) == par


def test_resume_skips_measured_cells(tmp_path):
    calls = []

    class Counting(sweep.SynthTimer):
        def __call__(self, problem, ci):
            calls.append((problem, ci))
            return super().__call__(problem, ci)

    first = sweep.benchmark_sweep(PROBS[:3], timer=Counting(CFGS), configs=CFGS, out_dir=tmp_path)
    n_first = len(calls)
    assert n_first == 3 * len(CFGS)
    again = sweep.benchmark_sweep(PROBS[:4], timer=Counting(CFGS), configs=CFGS, out_dir=tmp_path)
    assert len(calls) - n_first == len(CFGS)  # only the new row was measured
    assert again.take_rows(range(3)) == first


def test_failed_cell_is_fatal():
    def broken(problem, ci):
        return (0.0, 1.0, 1)
    broken.configs = CFGS
    with pytest.raises(Exception):
        sweep.benchmark_sweep(PROBS[:1], timer=broken, configs=CFGS)


def test_reference_parses_sweep_csv(kernelprune_ref, tmp_path):
    pm = sweep.benchmark_sweep(PROBS, timer=sweep.SynthTimer(CFGS, SynthModel(noise_sigma=0.0)), configs=CFGS)
    path = tmp_path / "t.csv"
    sweep.write_benchmark_csv(pm, path)
    ref = kernelprune_ref["dataset"].parse_benchmark_csv(path.read_text())
    assert [p.__dict__ for p in ref.problems] == [p.__dict__ for p in pm.problems]
    assert np.array_equal(ref.values, pm.values)


def test_shape_sets():
    vgg = shapes.network_problems("vgg16", batches=(1,))
    assert len(vgg) == 12
    assert shapes.network_flops("vgg16", 1) == pytest.approx(30.94e9, rel=0.01)
    res = shapes.network_problems("resnet50", batches=(1,))
    assert len(res) == 21
    assert shapes.network_flops("resnet50", 1) == pytest.approx(8.18e9, rel=0.02)
    allv = shapes.network_problems("vgg16")
    assert len(allv) == len(set(allv))
    assert ProblemSize(784, 4608, 512, 1) in allv  # conv4_2 @1 == conv5 @4 kept once


def test_cli_sweep_usage_and_config_keys(tmp_path, capsys):
    """CPU side of the CLI additions: flags parse, sweep keys are accepted in a run
    config, unknown keys still exit 2, usage errors exit 1 (cli.py:36-43)."""
    import json

    from paper_2008_13145_b200 import cli
    from paper_2008_13145_b200.pipeline import PipelineConfig

    args = cli.build_parser().parse_args(["sweep", "--set", "resnet50", "--batches", "1,2", "--family", "simt+tf32",
                                          "--gpus", "8", "--output", "x.csv"])
    assert args.batches == (1, 2) and args.gpus == 8 and args.func is cli.cmd_sweep
    assert cli.main(["sweep"]) == 1  # --output is required
    cfg = PipelineConfig(sweep_set="vgg16", sweep_family="bf16", sweep_gpus=2)
    assert cfg.sweep_gpus == 2
    with pytest.raises(ValueError):
        PipelineConfig(sweep_gpus=0)
    bad = tmp_path / "cfg.json"
    bad.write_text(json.dumps({"sweep_sets": "vgg16"}))
    assert cli.main(["run", "--config", str(bad), "--output-dir", str(tmp_path / "o")]) == 2


def test_multi_gpu_sweep_binds_one_distinct_device_per_shard(tmp_path, monkeypatch):
    """One process per non-empty shard, each pinned at spawn to its own device of the
    parent's CUDA_VISIBLE_DEVICES list (here '4,5,6': a scheduler-assigned range)."""
    monkeypatch.setenv("CUDA_VISIBLE_DEVICES", "4,5,6")
    probs = PROBS[:2]  # 3 GPUs, 2 rows: one shard is empty and gets no worker
    par = sweep.benchmark_sweep(probs, gpus=3, out_dir=tmp_path, timer_kind="synth",
                                timer_kw={"configs": CFGS, "model": SynthModel()}, configs=CFGS)
    assert par == synth_generate(SynthModel(), probs, list(CFGS))
    bindings = {}
    for g in range(3):
        f = tmp_path / f"shard{g}.device"
        if f.exists():
            dev, pid = f.read_text().split()
            bindings[g] = (dev, int(pid))
    assert len(bindings) == 2  # the empty shard started nothing
    devs = [d for d, _ in bindings.values()]
    pids = [p for _, p in bindings.values()]
    assert len(set(devs)) == 2 and set(devs) <= {"4", "5", "6"}
    assert len(set(pids)) == 2
    for g, (dev, _) in bindings.items():
        assert dev == "456"[g]


def test_device_bindings_respect_parent_mask(monkeypatch):
    monkeypatch.delenv("CUDA_VISIBLE_DEVICES", raising=False)
    assert sweep.device_bindings(3) == ["0", "1", "2"]
    monkeypatch.setenv("CUDA_VISIBLE_DEVICES", "GPU-a, GPU-b")
    assert sweep.device_bindings(2) == ["GPU-a", "GPU-b"]
    with pytest.raises(ValueError):
        sweep.device_bindings(3)
