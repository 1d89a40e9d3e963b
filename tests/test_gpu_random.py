"""GPU parity on seeded random states (custom initial state through the
handle API, s1d_set_initial), bitwise against the oracle's serial solver from
the same state (s1o_run_state). The BASELINE initial conditions are a smooth
sine and Sod plateaus (most points take the degenerate-ratio branch); random
states exercise the limiter, the reconstruction and the division paths at
every point, across unaligned totals (classic pad), several widths / points
per thread, and several shards.
"""
import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GAMMA = 1.4


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def rand_heat(n, seed):
    return np.random.default_rng(seed).standard_normal(n)


def rand_euler(n, seed):
    r = np.random.default_rng(seed)
    rho, u, p = r.uniform(0.5, 1.5, n), r.uniform(-0.5, 0.5, n), r.uniform(0.5, 1.5, n)
    st = np.empty((n, 3))
    st[:, 0], st[:, 1], st[:, 2] = rho, rho * u, p / (GAMMA - 1) + 0.5 * rho * u * u
    return st.ravel()


def solve(cfg, state):
    with s1d.Solver(cfg) as sv:
        out, _, _ = sv.solve(state)
    return out


@pytest.mark.parametrize("scheme", [s1d.Scheme.Swept, s1d.Scheme.Classic], ids=s1d.to_string)
@pytest.mark.parametrize("w,ranks", [(32, 1), (64, 3), (96, 1), (128, 2), (192, 1)])
def test_heat_random_state(gpu, scheme, w, ranks):
    n, T = 96 * 192, 333
    x = rand_heat(n, w + ranks)
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=scheme, grid_size=n, block_width=w, ranks=ranks,
                           steps=T, mode=s1d.Mode.WallClock, num_devices=1)
    want = O.port_run_state("heat", "lengthening", x, T, 0.0)
    assert np.array_equal(bits(solve(cfg, x)), bits(want))


@pytest.mark.parametrize("method", ["lengthening", "flattening"])
@pytest.mark.parametrize("scheme", [s1d.Scheme.Swept, s1d.Scheme.Classic], ids=s1d.to_string)
@pytest.mark.parametrize("w,ranks,T", [(64, 1, 150), (128, 2, 97), (32, 3, 61)])
def test_euler_random_state(gpu, method, scheme, w, ranks, T):
    n, dt_dx = 96 * 64, 0.15
    x = rand_euler(n, 7 * w + ranks)
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Euler,
                           method=s1d.Method.Lengthening if method == "lengthening" else s1d.Method.Flattening,
                           scheme=scheme, grid_size=n, block_width=w, ranks=ranks, steps=T,
                           mode=s1d.Mode.WallClock, num_devices=1)
    cfg.phys.dt_dx = dt_dx
    want = O.port_run_state("euler", method, x, T, dt_dx)
    assert np.array_equal(bits(solve(cfg, x)), bits(want))
