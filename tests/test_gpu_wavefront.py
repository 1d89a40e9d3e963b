"""GPU parity of the wavefront solve (engine.cu Solver::wavefront_phases).

s1d_solve on one shard with an aligned swept run runs the Up, the first and
last few Diamonds and the Down per chunk of tiles on two streams, overlapping
the host copies (by default for heat with m <= 128; S1D_WAVE =
"chunks,head,tail" forces a shape, which these tests use to drive every
case: odd and even cycle counts, seam-centred last cycles, the minimum of
three chunks, uneven chunks, asymmetric depths, the 512-thread P = 16 heat
build, both Euler methods, random states, the heat fast form's exact rerun,
repeated solves). Results are compared with the CPU oracle bit for bit.
"""
import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(got, want):
    assert got.shape == want.shape
    bad = np.nonzero(bits(got) != bits(want))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:8]}"


def config(eq, method, n, w, steps, min_cycles=8):
    c = s1d.LaunchConfig(equation=s1d.Equation.Heat if eq == "heat" else s1d.Equation.Euler,
                         method=s1d.Method.Lengthening if method == "lengthening" else s1d.Method.Flattening,
                         scheme=s1d.Scheme.Swept, grid_size=n, block_width=w, ranks=1, steps=steps)
    sp = c.spec()
    m = w // (2 * sp.stencil_half_width)
    total = steps * sp.substeps_per_step
    assert total % m == 0 and total // m >= min_cycles, "case must take the wavefront path"
    return c


CASES = [
    ("heat", "lengthening", 1 << 14, 32, 16 * 9),     # 9 cycles (seam-centred Down), 16 chunks
    ("heat", "lengthening", 1 << 14, 64, 32 * 10),    # 10 cycles
    ("heat", "lengthening", 5 * 64, 64, 32 * 8),      # 5 tiles: 5 chunks of one tile
    ("heat", "lengthening", 3 * 32, 32, 16 * 11),     # 3 tiles: the minimum
    ("heat", "lengthening", 37 * 64, 64, 32 * 9),     # 37 tiles: uneven chunks
    ("heat", "lengthening", 1 << 16, 256, 128 * 9),   # P = 16, 512-thread CTAs
    ("euler", "lengthening", 1 << 12, 64, 72),        # 9 cycles
    ("euler", "lengthening", 1 << 12, 32, 36),
    ("euler", "flattening", 1 << 12, 64, 80),         # 10 cycles
    ("euler", "flattening", 19 * 64, 64, 72),
]


@pytest.mark.parametrize("shape", ["16,3,3", "5,1,2", "7,2,0"])
@pytest.mark.parametrize("eq,method,n,w,steps", CASES)
def test_wavefront_solve_matches_oracle(gpu, monkeypatch, shape, eq, method, n, w, steps):
    monkeypatch.setenv("S1D_WAVE", shape)
    c = config(eq, method, n, w, steps)
    want = O.port_run_serial(eq, method, n=n, steps=steps)
    with s1d.Solver(c) as sv:
        for _ in range(2):  # events and streams reused
            got, _, _ = sv.solve()
            assert_bitwise(got, want)
        st, tm = sv.advance()  # the device-resident path is unchanged
        assert_bitwise(sv.read_state(), want)


def test_wavefront_default_shape(gpu, monkeypatch):
    # heat at m = 128 (the bench's w = 256) takes the wavefront by default
    # (3 pipelined Diamonds each side: at least 8 cycles)
    monkeypatch.delenv("S1D_WAVE", raising=False)
    n, w, steps = 1 << 16, 256, 128 * 9
    c = config("heat", "lengthening", n, w, steps, min_cycles=8)
    want = O.port_run_serial("heat", "lengthening", n=n, steps=steps)
    with s1d.Solver(c) as sv:
        got, _, tm = sv.solve()
    assert_bitwise(got, want)
    assert tm.dominant_launches == 9 - 1 - 3 - 3  # the Diamonds between the pipelined ones


@pytest.mark.parametrize("eq,method,n,w,steps", [CASES[0], CASES[5], CASES[6], CASES[8]])
def test_wavefront_random_state(gpu, monkeypatch, eq, method, n, w, steps):
    monkeypatch.setenv("S1D_WAVE", "16,3,3")
    c = config(eq, method, n, w, steps)
    r = np.random.default_rng(n + w)
    dt_dx = 0.0
    if eq == "heat":
        x = r.standard_normal(n)
    else:
        dt_dx = 0.15
        c.phys.dt_dx = dt_dx
        rho, u, p = r.uniform(0.5, 1.5, n), r.uniform(-0.5, 0.5, n), r.uniform(0.5, 1.5, n)
        st = np.empty((n, 3))
        st[:, 0], st[:, 1], st[:, 2] = rho, rho * u, p / 0.4 + 0.5 * rho * u * u
        x = st.ravel()
    want = O.port_run_state(eq, method, x, steps, dt_dx)
    with s1d.Solver(c) as sv:
        got, _, _ = sv.solve(x)
    assert_bitwise(got, want)


@pytest.mark.parametrize("w", [64, 256])
def test_wavefront_fast_form_rerun(gpu, monkeypatch, w):
    monkeypatch.setenv("S1D_WAVE", "16,3,3")
    # a value >= 2^1022 flags the fast form; the single-process solve reruns
    # the whole advance in the exact form (heat.cu heat_step)
    n, steps = 1 << 15, (w // 2) * 9
    c = config("heat", "lengthening", n, w, steps)
    x = np.arange(n)
    u0 = np.sin(2 * np.pi * x / n) + 0.3 * np.cos(0.37 * x)
    u0[n // 3] = 1.6 * 2.0 ** 1022
    want = O.port_run_state("heat", "lengthening", u0, steps, 0.0)
    with s1d.Solver(c) as sv:
        got, _, _ = sv.solve(u0)
        assert_bitwise(got, want)
        got2, _, _ = sv.solve(np.sin(2 * np.pi * x / n))  # flags re-armed: fast again, same bits as the oracle
    assert_bitwise(got2, O.port_run_state("heat", "lengthening", np.sin(2 * np.pi * x / n), steps, 0.0))
