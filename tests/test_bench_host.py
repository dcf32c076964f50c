"""bench.py host logic on CPU: argument defaults, the selector training path over a
benchmark table, and the multi-rank max-over-ranks timing with gloo (world_size 2)."""

import json
import os
import subprocess
import sys
import textwrap

import pytest

from conftest import ROOT


def test_defaults():
    sys.path.insert(0, str(ROOT))
    import bench
    a = bench.parse_args([])
    assert a.gpus is None and a.warmup >= 3 and a.steps >= 1 and a.impl == "ours"


def test_train_selector_on_a_table(tmp_path):
    import bench
    from paper_2008_13145_b200 import dataset, shapes, sweep
    probs = shapes.network_problems("vgg16", batches=(1, 2, 4, 8))
    cfgs = tuple(dataset.enumerate_configs())
    pm = sweep.benchmark_sweep(probs, timer=sweep.SynthTimer(cfgs), configs=cfgs)
    path = tmp_path / "t.csv"
    sweep.write_benchmark_csv(pm, path)
    pm2, subset, tree, rep_test, rep_all, t = bench.train_selector(str(path), 4, "kmeans", "treeA")
    assert pm2 == pm and 1 <= subset.k_actual <= 4
    assert 0 < rep_test.achieved <= rep_test.ceiling <= 1
    assert 0 < rep_all.achieved <= rep_all.ceiling <= 1


def test_reduce_max_two_ranks_gloo(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(textwrap.dedent(f"""
        import os, sys, json
        sys.path.insert(0, {str(ROOT)!r})
        import torch.distributed as dist
        import bench
        dist.init_process_group("gloo")
        r = dist.get_rank()
        v = bench.reduce_max(10.0 + 5.0 * r, dist.get_world_size())
        bench.barrier(dist.get_world_size())
        print(json.dumps({{"rank": r, "max": v}}))
        dist.destroy_process_group()
    """))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", str(script)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=tmp_path)
    assert out.returncode == 0, out.stderr[-3000:]
    import re
    vals = [json.loads(x) for x in re.findall(r"\{[^{}]*\}", out.stdout)]  # ranks share stdout
    assert sorted(v["rank"] for v in vals) == [0, 1]
    assert all(v["max"] == 15.0 for v in vals)


def test_reference_arm_rank_nonzero_exits_quietly(tmp_path):
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_roofline_picks_the_binding_roof():
    import bench
    from paper_2008_13145_b200.dataset import ProblemSize
    fc6 = ProblemSize(16, 25088, 4096, 1)  # AI ~ 8 FLOP/B: HBM-bound for fp32
    r = bench.roofline("simt", fc6, 0.1, 4, simt_peak=74.0)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert abs(r["achieved"] - r["algorithmic_bytes"] / 1e-4 / 1e9) < 1e-6
    conv = ProblemSize(12544, 4608, 512, 1)
    r = bench.roofline("simt", conv, 1.2, 4, simt_peak=74.0)
    assert r["bound"] == "compute" and r["unit"] == "TFLOP/s" and r["peak"] == 74.0
    conv1_1 = ProblemSize(802816, 27, 64, 1)  # bf16 k=27: far below the tensor ridge
    assert bench.roofline("bf16", conv1_1, 0.4, 2)["bound"] == "hbm"
    big = ProblemSize(8192, 8192, 8192, 1)
    assert bench.roofline("bf16", big, 1.0, 2)["bound"] == "tensor"


def test_gpus_flag_self_launches_ranks(tmp_path):
    """--gpus 2 outside torchrun re-launches under torch.distributed.run: the reference
    arm then runs on rank 0 only and reports n_gpus 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0", "--batch", "1"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=tmp_path)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
    assert lines[0]["config"]["batch_per_gpu"] == 1


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "4",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr
