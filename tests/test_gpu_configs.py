"""GPU parity at BASELINE configs[3] and configs[4] sizes, runnable on a
single-GPU box (the shards of a multi-shard run share the device; on a
multi-GPU box they spread over min(GPUs, ranks) devices):

  * configs[3]: heat nX = 2^30, w = 1024, ranks 2/4/8 == ranks 1, bit for bit
    (rank invariance, R/tests/test_decomp.cpp:81-98), at the bench's T = 6144
    and at an unaligned T (classic pad across shard seams); windows around
    every shard seam, incl. the periodic wrap, == an exact FTCS restatement on
    the window's dependency cone;
  * configs[4]: Euler Sod, 2^16 points per shard x 2/4/8 shards, both
    methods, both schemes, against the full C-oracle state (port_run_serial,
    test infrastructure) at T = 256, plus ranks 8 == ranks 1 at a long
    T = 8192 across block widths 64 / 512 / 1024;
  * one process per rank (torchrun, the bench's launch mode) at 2^27 points
    per rank, 2 ranks on this box's GPU(s): tools/mp_big_check.py.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O
from test_gpu_fullsize import _runs, bits

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEAT_SPEC = s1d.make_spec(s1d.Equation.Heat, s1d.Method.Lengthening)
N30 = 1 << 30


def ndev(ranks):
    return max(1, min(s1d.device_count(), ranks))


def heat30(ranks, steps, w=1024):
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=s1d.Scheme.Swept, grid_size=N30, block_width=w,
                           ranks=ranks, steps=steps, mode=s1d.Mode.WallClock, num_devices=ndev(ranks))
    return s1d.run(cfg).state


def ftcs_window(x0, x1, n, steps, fo=0.4):
    """Exact heat_step (inc/kernels.hpp:14-16) over the cone of [x0, x1)."""
    idx = np.arange(x0 - steps, x1 + steps) % n
    u = np.empty(idx.size)
    for a, b in _runs(idx):
        u[a:b] = s1d.initial_condition_range("heat-sine", n, HEAT_SPEC, int(idx[a]), b - a)
    for _ in range(steps):
        l, c, r = u[:-2], u[1:-1], u[2:]
        u = c + fo * ((l - 2.0 * c) + r)
    return u


@pytest.fixture(scope="module")
def heat30_ranks1():
    return heat30(1, 6144)


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_heat_2p30_rank_invariant(heat30_ranks1, ranks):
    got = heat30(ranks, 6144)
    assert np.array_equal(bits(got), bits(heat30_ranks1))
    if ranks == 8:  # every seam (k = 0 is the periodic wrap) against the exact cone
        for k in range(8):
            seam = k * (N30 // 8)
            want = ftcs_window(seam - 512, seam + 512, N30, 6144)
            assert np.array_equal(bits(got[np.arange(seam - 512, seam + 512) % N30]), bits(want)), k


def test_heat_2p30_unaligned_T_pad_across_seams():
    # T = 1000 at m = 512: one cycle + 488 classic pad substeps on 8 shards
    a = heat30(8, 1000)
    b = heat30(1, 1000)
    assert np.array_equal(bits(a), bits(b))
    seam = 3 * (N30 // 8)
    want = ftcs_window(seam - 256, seam + 256, N30, 1000)
    assert np.array_equal(bits(a[seam - 256:seam + 256]), bits(want))


EU_PER = 1 << 16
EU_T = 256


def euler_run(method, scheme, ranks, n, w, steps):
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Euler,
                           method=s1d.Method.Lengthening if method == "len" else s1d.Method.Flattening,
                           scheme=s1d.Scheme.Swept if scheme == "swept" else s1d.Scheme.Classic, grid_size=n,
                           block_width=w, ranks=ranks, steps=steps, mode=s1d.Mode.WallClock,
                           num_devices=ndev(ranks))
    return s1d.run(cfg).state


_ORACLE = {}


def euler_oracle(n):
    # flattening == lengthening bitwise in the reference, so one
    # oracle run per grid serves both methods
    if n not in _ORACLE:
        _ORACLE[n] = O.port_run_serial("euler", "lengthening", n=n, steps=EU_T)
    return _ORACLE[n]


@pytest.mark.parametrize("ranks", [2, 4, 8])
@pytest.mark.parametrize("method", ["len", "flat"])
@pytest.mark.parametrize("scheme", ["swept", "classic"])
def test_euler_2p16_per_shard_vs_oracle(ranks, method, scheme):
    n = EU_PER * ranks
    got = euler_run(method, scheme, ranks, n, 512, EU_T)
    assert np.array_equal(bits(got), bits(euler_oracle(n)))


@pytest.mark.parametrize("w", [64, 512, 1024])
@pytest.mark.parametrize("method", ["len", "flat"])
def test_euler_2p16_per_shard_long_tf_rank_invariant(w, method):
    n = EU_PER * 8
    a = euler_run(method, "swept", 8, n, w, 8192)
    b = euler_run(method, "swept", 1, n, w, 8192)
    assert np.all(np.isfinite(a))
    assert np.array_equal(bits(a), bits(b))
    rho = a.reshape(-1, 3)[:, 0]
    assert abs(rho.sum() - 0.5625 * n) <= 1e-10 * n  # mass: (1 + 0.125)/2 per point


def test_torchrun_two_ranks_2p27_per_rank():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "tools", "mp_big_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
    assert "BAD" not in r.stdout and r.stdout.count("ok ") >= 3
