"""GPU: the `s1d verify` subcommand to SPEC.md's bench-cli contract
("verify (swept vs classic vs serial oracle, prints max abs diff
and bitwise flag)", "exits non-zero on any injected kernel
perturbation of 1 ulp"). The serial-oracle leg is a dump of the compiled
reference's run_serial (oracle/dump_serial.py; the C restatement where
oracle/_ref is absent)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1811_08282_b200", "_lib", "s1d")


def dump(tmp_path, name, kv):
    out = tmp_path / name
    subprocess.run([sys.executable, os.path.join(ROOT, "oracle", "dump_serial.py"), "--out", str(out)] + kv,
                   check=True, cwd=ROOT)
    return str(out)


def verify(*args):
    return subprocess.run([CLI, "verify"] + list(args), capture_output=True, text=True, timeout=300)


@pytest.mark.parametrize("kv", [
    # the SPEC's example has n = 1024 (64 blocks, which 3 ranks cannot share:
    # the reference rejects it too); n = 960 keeps w, ranks and T
    ["equation=heat", "n=960", "w=16", "ranks=3", "steps=50"],
    ["equation=euler", "method=lengthening", "n=2048", "w=64", "ranks=2", "steps=40"],
    ["equation=euler", "method=flattening", "n=2048", "w=32", "ranks=1", "steps=33"],
], ids=["heat-spec-example", "euler-len", "euler-flat"])
def test_verify_three_way_bitwise(gpu, tmp_path, kv):
    ref = dump(tmp_path, "ref.bin", kv)
    r = verify("--against", ref, *kv)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("bitwise: true, max|diff| = 0 ") == 3 and "verify: PASS" in r.stdout


@pytest.mark.parametrize("kv", [
    ["equation=heat", "n=960", "w=16", "ranks=3", "steps=16", "fourier=0.1"],
    ["equation=euler", "method=flattening", "n=256", "w=16", "ranks=2", "steps=9"],
], ids=["heat", "euler-flat"])
def test_verify_fails_on_one_ulp_mutation(gpu, tmp_path, kv):
    # (heat at Fo = 0.1: at Fo = 0.4 FTCS damps a 1-ulp nudge below rounding
    # within a step, so no final-state check can see it; tests/test_gpu_debug.py)
    ref = dump(tmp_path, "ref.bin", kv)
    assert verify("--against", ref, *kv).returncode == 0
    r = verify("--against", ref, "--perturb-ulp", *kv)
    assert r.returncode != 0 and "bitwise: false" in r.stdout and "verify: FAIL" in r.stdout


def test_verify_rejects_wrong_oracle(gpu, tmp_path):
    other = dump(tmp_path, "other.bin", ["equation=heat", "n=1024", "steps=51"])
    kv = ["equation=heat", "n=1024", "w=16", "steps=50"]
    r = verify("--against", other, *kv)
    assert r.returncode == 1 and "swept vs serial oracle" in r.stdout and "bitwise: false" in r.stdout
    short = dump(tmp_path, "short.bin", ["equation=heat", "n=512", "steps=50"])
    r = verify("--against", short, *kv)
    assert r.returncode == 1 and "expected" in r.stderr
