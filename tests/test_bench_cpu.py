"""CPU: bench.py's launcher logic. `--gpus N` outside torchrun re-executes
itself under torch.distributed.run with N processes (the flag was
parsed but unused), rank 0 alone prints the reference arm's line, and a
process count that disagrees with --gpus is refused."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["--impl", "reference", "--steps", "1", "--warmup", "0", "--log2n", "16", "--w", "64"]


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                          text=True, timeout=300, env=e)


def test_gpus_flag_launches_n_processes():
    r = _run(["--gpus", "2"] + SMALL)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["cores"] >= 2 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["block_width"] == 64 and d["config"]["steps_per_run"] == 32  # T = m = w/2


def test_world_mismatch_is_refused():
    r = _run(["--gpus", "2"] + SMALL, env={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode != 0 and "--gpus 2" in (r.stderr + r.stdout)
