"""bench.py contract checks that run without a GPU: the --impl reference arm
(oracle port on the host cores) prints exactly one JSON line with the required
keys, both alone and under torchrun with world_size 2 (gloo; rank 1 exits 0
without work)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.strip().startswith("{")]


def test_reference_arm_single_process():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg1", "--steps", "2",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = _lines(r.stdout)
    assert len(lines) == 1
    line = lines[0]
    assert KEYS <= set(line)
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    # measured, not modelled: K full-size steps whose times add up to the line's ms_per_step
    assert len(line["cpu_baseline"]["step_s"]) == 2
    assert abs(sum(line["cpu_baseline"]["step_s"]) / 2 * 1000.0 - line["ms_per_step"]) < 1e-6
    assert line["cpu_baseline"]["host"]["ram_gb"] > 0
    # the same config object as our arm prints (same_config)
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    args = argparse.Namespace(config="cfg1", mode="auto")
    assert line["config"] == bench.arm_config(args, bench.CONFIGS["cfg1"], 1, "replicas")


def test_reference_arm_under_torchrun_world2():
    env = dict(os.environ, OMP_NUM_THREADS="2")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29531", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--config", "cfg1", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2
    assert lines[0]["config"]["parallelism"].startswith("row-sharded x2")
