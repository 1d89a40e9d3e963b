"""GPU parity at the BASELINE sizes (configs 1-2), through size-independent
properties — the CPU oracle cannot run 2^27 points x thousands of steps:

  * heat n = 2^27: linear under power-of-two scaling (bitwise) and max-norm
    non-increasing at Fo = 0.5 (test_kernels.cpp:43-74 at full size);
  * heat n = 2^27: swept (w = 1024 and the short-tile path, w = 32) ==
    classic, bit for bit; and windows of the result == an exact FTCS
    restatement run on the window's dependency cone (the value at x after T
    steps depends only on [x-T, x+T]; numpy float64 evaluates
    c + fo*((l - 2c) + r) with one IEEE rounding per operation, like the
    reference's -ffp-contract=off build);
  * Euler Sod n = 2^22: lengthening swept == flattening swept == classic,
    bit for bit, mass conserved, and windows (across both Sod jumps) == the C
    oracle run on the window's cone (4 cells per step for both methods) with
    the full problem's dt/dx.
"""
import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

pytestmark = pytest.mark.gpu

N_HEAT = 1 << 27
HEAT_SPEC = s1d.make_spec(s1d.Equation.Heat, s1d.Method.Lengthening)
T_HEAT = 1024


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def heat(scheme, w, steps=T_HEAT, n=N_HEAT):
    return s1d.run(s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=scheme, grid_size=n, block_width=w, ranks=1,
                                    steps=steps, mode=s1d.Mode.WallClock)).state


def ftcs_window(x0, x1, n, steps, fo=0.4):
    """Exact heat_step (inc/kernels.hpp:14-16) on the cone of [x0, x1)."""
    lo = x0 - steps
    idx = np.arange(lo, x1 + steps) % n
    u = np.empty(idx.size)
    # the IC restated by the library's host code (bitwise == partition.cpp, tests/test_host.py)
    for a, b in _runs(idx):
        u[a:b] = s1d.initial_condition_range("heat-sine", n, HEAT_SPEC, int(idx[a]), b - a)
    for _ in range(steps):
        l, c, r = u[:-2], u[1:-1], u[2:]
        u = c + fo * ((l - 2.0 * c) + r)
    return u  # covers [x0, x1)


def _runs(idx):
    """Split a wrapped index array into contiguous ascending runs."""
    cuts = np.nonzero(np.diff(idx) != 1)[0] + 1
    starts = np.concatenate(([0], cuts))
    ends = np.concatenate((cuts, [idx.size]))
    return zip(starts.tolist(), ends.tolist())


@pytest.fixture(scope="module")
def heat_swept_1024():
    return heat(s1d.Scheme.Swept, 1024)


def test_heat_2p27_swept_equals_classic(heat_swept_1024):
    classic = heat(s1d.Scheme.Classic, 1024)
    assert np.array_equal(bits(heat_swept_1024), bits(classic))


def test_heat_2p27_short_tiles_equal_wide(heat_swept_1024):
    assert np.array_equal(bits(heat(s1d.Scheme.Swept, 32)), bits(heat_swept_1024))


@pytest.mark.parametrize("x0", [0, N_HEAT // 2 - 700, N_HEAT - 512])
def test_heat_2p27_windows_match_exact_ftcs(heat_swept_1024, x0):
    want = ftcs_window(x0, x0 + 1024, N_HEAT, T_HEAT)
    got = heat_swept_1024[np.arange(x0, x0 + 1024) % N_HEAT]
    assert np.array_equal(bits(got), bits(want))


def euler(method, scheme, n=1 << 22, w=512, steps=512):
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Euler, method=method, scheme=scheme, grid_size=n, block_width=w,
                           ranks=1, steps=steps, mode=s1d.Mode.WallClock)
    return s1d.run(cfg).state


N_EU, T_EU = 1 << 22, 512


@pytest.fixture(scope="module")
def euler_len_swept():
    return euler(s1d.Method.Lengthening, s1d.Scheme.Swept, n=N_EU, steps=T_EU)


@pytest.mark.parametrize("method", ["lengthening", "flattening"])
@pytest.mark.parametrize("x0", [-32, N_EU // 2 - 32, N_EU // 2 + 1500])
def test_euler_2p22_windows_match_oracle(euler_len_swept, method, x0):
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Euler, grid_size=N_EU, block_width=512, ranks=1, steps=T_EU)
    cfg.finalize()  # dt/dx of the full problem (cfl / max signal speed of the whole IC)
    spec = s1d.make_spec(s1d.Equation.Euler, s1d.Method.Lengthening)
    pad, W = 4 * T_EU + 8, 64
    idx = np.arange(x0 - pad, x0 + W + pad) % N_EU
    ic = np.concatenate([s1d.initial_condition_range("euler-sod-periodic", N_EU, spec, a, b - a)
                         for a, b in ((int(idx[i]), int(idx[j - 1]) + 1) for i, j in _runs(idx))])
    want = O.port_run_state("euler", method, ic, T_EU, cfg.phys.dt_dx).reshape(-1, 3)[pad:pad + W]
    got = euler_len_swept.reshape(-1, 3)[np.arange(x0, x0 + W) % N_EU]
    assert np.array_equal(bits(got), bits(want))


def test_euler_2p22_swept_classic_flat_len_agree(euler_len_swept):
    L, F = s1d.Method.Lengthening, s1d.Method.Flattening
    ref = euler_len_swept
    assert np.array_equal(bits(euler(F, s1d.Scheme.Swept)), bits(ref))
    assert np.array_equal(bits(euler(L, s1d.Scheme.Classic)), bits(ref))
    rho = ref.reshape(-1, 3)[:, 0]
    spec = s1d.make_spec(s1d.Equation.Euler, s1d.Method.Lengthening)
    ic = s1d.initial_condition("euler-sod-periodic", 1 << 22, spec).reshape(-1, 3)
    assert abs(rho.sum() - ic[:, 0].sum()) <= 1e-12 * ic[:, 0].sum()


@pytest.mark.parametrize("method", [s1d.Method.Lengthening, s1d.Method.Flattening], ids=["len", "flat"])
def test_euler_2p26_windows_match_oracle(gpu, method):
    # the top of BASELINE configs[2] (n = 2^20 .. 2^26); windows across both Sod jumps
    n, T = 1 << 26, 256
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Euler, method=method, scheme=s1d.Scheme.Swept, grid_size=n,
                           block_width=512, ranks=1, steps=T, mode=s1d.Mode.WallClock)
    got = s1d.run(cfg).state.reshape(-1, 3)
    cfg.finalize()
    spec = s1d.make_spec(s1d.Equation.Euler, s1d.Method.Lengthening)
    name = "lengthening" if method == s1d.Method.Lengthening else "flattening"
    pad, W = 4 * T + 8, 64
    for x0 in (-32, n // 2 - 32):
        idx = np.arange(x0 - pad, x0 + W + pad) % n
        ic = np.concatenate([s1d.initial_condition_range("euler-sod-periodic", n, spec, a, b - a)
                             for a, b in ((int(idx[i]), int(idx[j - 1]) + 1) for i, j in _runs(idx))])
        want = O.port_run_state("euler", name, ic, T, cfg.phys.dt_dx).reshape(-1, 3)[pad:pad + W]
        assert np.array_equal(bits(got[np.arange(x0, x0 + W) % n]), bits(want))


def test_heat_2p27_linear_under_power_of_two_scaling(gpu):
    # test_kernels.cpp:43-48 at full size: scaling the state by 2^k is exact,
    # so solve(4 u0) == 4 solve(u0) bit for bit (swept, w = 1024)
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=s1d.Scheme.Swept, grid_size=N_HEAT, block_width=1024,
                           ranks=1, steps=T_HEAT, mode=s1d.Mode.WallClock)
    u0 = s1d.initial_condition("heat-sine", N_HEAT, HEAT_SPEC)
    with s1d.Solver(cfg) as sv:
        a, _, _ = sv.solve(u0)
        b, _, _ = sv.solve(4.0 * u0)
    assert np.array_equal(bits(b), bits(4.0 * a))


def test_heat_2p27_max_norm_non_increasing_at_fo_half(gpu):
    # test_kernels.cpp:50-74 at full size: Fo = 0.5, rough data, max-norm
    # non-increasing in T (swept)
    x = np.arange(N_HEAT, dtype=np.float64)
    u0 = np.sin(0.13 * x) + 0.2 * np.cos(0.41 * x * x)
    prev = np.abs(u0).max()
    for T in (64, 256, 1024):
        cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=s1d.Scheme.Swept, grid_size=N_HEAT,
                               block_width=1024, ranks=1, steps=T, mode=s1d.Mode.WallClock)
        cfg.phys.fourier = 0.5
        with s1d.Solver(cfg) as sv:
            u, _, _ = sv.solve(u0)
        cur = np.abs(u).max()
        assert cur <= prev + 1e-15
        prev = cur
