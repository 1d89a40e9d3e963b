"""GPU parity of the fixed-width builds (heat.cu launch_heat_tile: w = 32, 64,
128, 256, 512, 1024, 2048 with compile-time strides and the unrolled one- /
multi-slot inserts; euler.cu launch_euler_tile: w = 32, 64, 128, 256, 512,
1024, 2048 and the latency-bound w = 512 build) against the CPU oracle, bit
for bit, on seeded random states. The tile counts leave the last CTA partly
empty (tiles that are not live), and the step counts include a classic pad
and several swept cycles.
"""
import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

pytestmark = pytest.mark.gpu

# tiles per CTA of the fixed builds (heat: P = 8 at w <= 64, else P = 16)
HEAT_G = {32: 64, 64: 32, 128: 32, 256: 32, 512: 16, 1024: 8, 2048: 4}


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("w", sorted(HEAT_G))
def test_heat_fixed_width_random(gpu, monkeypatch, w):
    # the fixed build's points per thread (small grids may otherwise pick P = 8)
    monkeypatch.setenv("S1D_HEAT_P", "8" if w <= 64 else "16")
    tiles = 2 * HEAT_G[w] + 3          # last CTA holds 3 live tiles
    n = tiles * w
    steps = 2 * (w // 2) + 7            # two swept cycles and a classic pad
    x = np.random.default_rng(w).standard_normal(n)
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=s1d.Scheme.Swept, grid_size=n, block_width=w, ranks=1,
                           steps=steps)
    with s1d.Solver(cfg) as sv:
        got, _, _ = sv.solve(x)
    want = O.port_run_state("heat", "lengthening", x, steps, 0.0)
    assert np.array_equal(bits(got), bits(want))


# Euler: more CTAs than SMs take the fixed 256-thread builds (tiles per CTA
# GT = 8 / 8 or 4 / 4 at w = 32 / 64 / 128, one at 256 / 512 / 1024); fewer
# take the latency-bound builds (w = 512: the fixed 544-thread build; w = 2048
# here, whose fixed build needs more than 148 tiles, too slow for the oracle).
EULER_CASES = [(32, 8 * 150 + 3), (64, 8 * 150 + 3), (128, 4 * 150 + 3), (256, 153), (512, 153), (512, 3),
               (1024, 153), (1024, 3), (2048, 2)]


@pytest.mark.parametrize("method", ["lengthening", "flattening"])
@pytest.mark.parametrize("w,tiles", EULER_CASES)
def test_euler_fixed_width_random(gpu, method, w, tiles):
    n, dt_dx = tiles * w, 0.15
    r = np.random.default_rng(3 * w + tiles)
    rho, u, p = r.uniform(0.5, 1.5, n), r.uniform(-0.5, 0.5, n), r.uniform(0.5, 1.5, n)
    st = np.empty((n, 3))
    st[:, 0], st[:, 1], st[:, 2] = rho, rho * u, p / 0.4 + 0.5 * rho * u * u
    x = st.ravel()
    spec = s1d.make_spec(s1d.Equation.Euler,
                         s1d.Method.Lengthening if method == "lengthening" else s1d.Method.Flattening)
    m = w // (2 * spec.stencil_half_width)
    steps = (2 * m + 3) // spec.substeps_per_step + 1  # two swept cycles and a pad
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Euler,
                           method=s1d.Method.Lengthening if method == "lengthening" else s1d.Method.Flattening,
                           scheme=s1d.Scheme.Swept, grid_size=n, block_width=w, ranks=1, steps=steps)
    cfg.phys.dt_dx = dt_dx
    with s1d.Solver(cfg) as sv:
        got, _, _ = sv.solve(x)
    want = O.port_run_state("euler", method, x, steps, dt_dx)
    assert np.array_equal(bits(got), bits(want))
