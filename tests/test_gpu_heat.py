"""GPU parity: heat (FTCS) classic and swept vs the CPU oracle, bitwise.

Mirrors test_decomp.cpp:81-145 (classic/swept == serial bitwise) and the
survey's fingerprints on the B200 path. All calls go through
the C ABI (libswept1d.so) via the Python mirror.
"""
import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def cfg(scheme, n, w, steps, ranks=1, wf=0, **kw):
    return s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=scheme, grid_size=n, block_width=w, ranks=ranks,
                            work_factor=wf, steps=steps, **kw)


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(got, want):
    assert got.shape == want.shape
    bad = np.nonzero(bits(got) != bits(want))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:8]}: got {got[bad[:4]]} want {want[bad[:4]]}"


@pytest.mark.parametrize("scheme", [s1d.Scheme.Swept, s1d.Scheme.Classic])
@pytest.mark.parametrize("steps,fnv", [(64, "4185347ae18fab0f"), (1000, "90d783358019c683"),
                                       (6144, "389326b8952bc813")])
def test_fingerprint_n16k_w64(gpu, scheme, steps, fnv):
    res = s1d.run(cfg(scheme, 1 << 14, 64, steps))
    assert O.fnv1a64(res.state) == fnv


# test_decomp.cpp:108-112 heat rows (n, w, ranks, wf, steps)
DECOMP = [(64, 4, 2, 0, 16), (32, 8, 2, 0, 4), (128, 8, 3, 2, 25), (64, 8, 2, 0, 21)]


@pytest.mark.parametrize("n,w,ranks,wf,steps", DECOMP)
@pytest.mark.parametrize("scheme", [s1d.Scheme.Swept, s1d.Scheme.Classic])
def test_decomp_cases(gpu, n, w, ranks, wf, steps, scheme):
    want = O.port_run_serial("heat", n=n, steps=steps)
    for r in (ranks, 1):
        got = s1d.run(cfg(scheme, n, w, steps, ranks=r, wf=wf if r > 1 else 0)).state
        assert_bitwise(got, want)


# incl. widths whose half-width the slot size does not divide (ragged last
# slot: 34, 200, 514, 1000, 2050) and beyond 256 slots (2050, 4100, 8192:
# CTAs of up to 1024 threads); the reference's check_width has no upper
# bound (R/core/src/swept.cpp:10-19)
@pytest.mark.parametrize("w", [4, 6, 8, 12, 16, 32, 34, 64, 128, 200, 256, 512, 514, 1000, 1024, 2048, 2050, 4096,
                               4100, 8192])
def test_width_sweep_unaligned(gpu, w):
    n = max(4 * w, 1 << 13)
    n -= n % w
    m = w // 2
    for steps in (m - 1, m, 2 * m, 3 * m + 5, 5 * m + 1):
        want = O.port_run_serial("heat", n=n, steps=steps)
        got = s1d.run(cfg(s1d.Scheme.Swept, n, w, steps)).state
        assert_bitwise(got, want)


def test_zero_steps_returns_ic(gpu):
    for scheme in (s1d.Scheme.Swept, s1d.Scheme.Classic):
        res = s1d.run(cfg(scheme, 64, 8, 0))
        ic = s1d.initial_condition("heat-sine", 64, s1d.make_spec(s1d.Equation.Heat, s1d.Method.Lengthening))
        assert_bitwise(res.state, ic)
        assert res.stats.exchange_rounds == 0


def test_round_counts(gpu):
    # test_decomp.cpp:147-157, 191-199
    assert s1d.run(cfg(s1d.Scheme.Swept, 64, 8, 40, ranks=2)).stats.exchange_rounds == 10
    assert s1d.run(cfg(s1d.Scheme.Classic, 64, 8, 40, ranks=2)).stats.exchange_rounds == 40
    res = s1d.run(cfg(s1d.Scheme.Swept, 128, 32, 50, ranks=2))
    assert res.stats.exchange_rounds == 5
    assert_bitwise(res.state, O.port_run_serial("heat", n=128, steps=50))


def test_uniform_fixed_point(gpu):
    res = s1d.run(cfg(s1d.Scheme.Swept, 256, 16, 37, initial="uniform"))
    assert np.all(res.state == 1.0)


def test_solver_handle_repeat_and_custom_state(gpu):
    c = cfg(s1d.Scheme.Swept, 1 << 12, 64, 100)
    with s1d.Solver(c) as sv:
        a, _, _ = sv.solve()
        b, _, t = sv.solve()
        assert_bitwise(a, b)
        assert t.loop_seconds > 0
        x = np.random.default_rng(1).standard_normal(1 << 12)
        got, _, _ = sv.solve(x)
        # classic on the same input
    with s1d.Solver(cfg(s1d.Scheme.Classic, 1 << 12, 64, 100)) as sc:
        want, _, _ = sc.solve(x)
    assert_bitwise(got, want)


def test_cli_verify_and_sweep(gpu, tmp_path):
    import os
    import subprocess
    cli = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1811_08282_b200", "_lib",
                       "s1d")
    r = subprocess.run([cli, "verify", "equation=heat", "n=960", "w=16", "ranks=3", "steps=50"], capture_output=True,
                       text=True)
    assert r.returncode == 0 and "bitwise: true" in r.stdout, r.stdout + r.stderr
    r = subprocess.run([cli, "verify", "equation=euler", "method=flattening", "n=2048", "w=32", "steps=40"],
                       capture_output=True, text=True)
    assert r.returncode == 0 and "bitwise: true" in r.stdout, r.stdout + r.stderr
    out = tmp_path / "s.csv"
    r = subprocess.run([cli, "sweep", "--n", "2^14,2^15,2^16", "--w", "32,64", "--out", str(out), "steps=64"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    recs = s1d.read_csv(str(out))
    assert len(recs) == 12 and all(x.avg_us_per_step > 0 for x in recs)
    r = subprocess.run([cli, "fit", str(out), "--scheme", "swept"], capture_output=True, text=True)
    assert r.returncode == 0 and "swept" in r.stdout


def test_measure_record(gpu):
    t = s1d.measure(cfg(s1d.Scheme.Swept, 1 << 14, 64, 128))
    assert t.avg_us_per_step > 0 and t.exchange_rounds == 4 and t.scheme == s1d.Scheme.Swept


@pytest.mark.parametrize("eq,method,n,w,steps", [("heat", "lengthening", 1 << 14, 64, 64), ("heat", "lengthening", 1 << 14, 64, 96),
                                                ("heat", "lengthening", 96 * 64, 64, 32 * 5), ("euler", "lengthening", 1 << 12, 64, 64),
                                                ("euler", "flattening", 1 << 12, 64, 48), ("euler", "lengthening", 1 << 12, 32, 8 * 3)])
def test_pipelined_solve_matches_oracle(gpu, eq, method, n, w, steps):
    # s1d_solve overlaps H2D with the UpTriangle and D2H with the DownTriangle
    # (aligned totals, both odd and even cycle counts)
    c = s1d.LaunchConfig(equation=s1d.Equation.Heat if eq == "heat" else s1d.Equation.Euler,
                         method=s1d.Method.Lengthening if method == "lengthening" else s1d.Method.Flattening,
                         scheme=s1d.Scheme.Swept, grid_size=n, block_width=w, ranks=1, steps=steps)
    want = O.port_run_serial(eq, method, n=n, steps=steps)
    with s1d.Solver(c) as sv:
        for _ in range(2):
            got, _, _ = sv.solve()
            assert_bitwise(got, want)
        x = O.port_initial_condition("uniform", n, eq)
        got, _, _ = sv.solve(x)
        assert_bitwise(got, x)


# The tile kernels' fast point update (fma(-2, c, l) for l - 2c, heat.cu
# heat_step) is exact unless 2c overflows; it runs only when every input of
# a CTA is below 2^1022 (0 < Fo <= 0.5 is guaranteed by validation), else that
# CTA's tiles are computed by the exact form. These cases drive each branch and
# compare with the oracle bit for bit (NaNs compared as NaNs: their payloads
# are platform-defined).
def _solve(u0, w, steps, fo=0.4):
    c = cfg(s1d.Scheme.Swept, u0.size, w, steps)
    c.phys.fourier = fo
    with s1d.Solver(c) as sv:
        got, _, _ = sv.solve(u0)
    return got


def _assert_same_or_both_nan(got, want):
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    assert_bitwise(got[~nan], want[~nan])


@pytest.mark.parametrize("case", ["fast", "below", "spike", "above", "overflow", "fo-0.5"])
@pytest.mark.parametrize("w", [64, 1024])
def test_fast_form_guard(gpu, case, w):
    n, steps = 1 << 16, 1500
    x = np.arange(n)
    u0 = np.sin(2 * np.pi * x / n) + 0.3 * np.cos(0.37 * x)
    fo = 0.5 if case == "fo-0.5" else 0.4  # (validate admits only 0 < Fo <= 0.5, config.cpp:45-95)
    if case == "fast":
        u0 = u0 * 2.0 ** 1000                     # large but below 2^1022: fast form throughout
    elif case == "below":
        u0 = u0 * 2.0 ** 1021                     # max 1.3 * 2^1021: still the fast form
    elif case == "spike":
        u0[12345] = 1.6 * 2.0 ** 1022             # one Up CTA flags its shard: exact from then on
    elif case == "above":
        u0 = u0 * 2.0 ** 1022                     # most CTAs see inputs >= 2^1022, no overflow anywhere
    elif case == "overflow":
        u0[777] = 1.5 * 2.0 ** 1023               # 2c overflows to inf in the reference
    want = O.port_run_state("heat", "lengthening", u0, steps, 0.0, fourier=fo)
    _assert_same_or_both_nan(_solve(u0, w, steps, fo), want)
