"""GPU: bench.py keeps the driver's contract — one JSON line with the required
keys, device-timed value, e2e with host copies, a launch count, roofline and
clocks (a small configuration, so the check is quick)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "clocks", "e2e", "gpu_launches", "roofline"]


def test_bench_emits_one_contract_line(gpu):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3", "--log2n", "22",
           "--T", "2048", "--e2e-steps", "1", "--no-cpu-baseline", "--no-euler"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in REQUIRED:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and d["roofline"]["bound"] == "fp64" and 0 < d["roofline"]["frac"] <= 1
    assert d["config"]["workload"] and d["dtype"] == "f64"


def test_bench_gpus_flag_runs_that_many_ranks(gpu):
    # `--gpus 2` outside a launcher re-executes under torch.distributed.run
    # with 2 processes (they share the device on a 1-GPU box)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--log2n", "22", "--T", "2048", "--e2e-steps", "1", "--no-cpu-baseline", "--no-euler"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ring"]["nranks"] == 2 and d["config"]["grid_size"] == 2 << 22
    assert r.stderr.count("ring connect: rank") == 2
