"""GPU debug instrumentation (RunOptions, inc/debug.hpp): the tiling coverage
counter proves every (point, substep) is computed exactly once by the
swept/classic decomposition (SPEC.md acceptance "Tiling completeness"), and
the 1-ulp mutation hook proves the bitwise parity check is sensitive
(SPEC.md "verify exits non-zero on a 1 ulp perturbation")."""
import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

pytestmark = pytest.mark.gpu
EQ = {"heat": s1d.Equation.Heat, "euler": s1d.Equation.Euler}
ME = {"lengthening": s1d.Method.Lengthening, "flattening": s1d.Method.Flattening}

# randomized-looking but fixed valid configs: (eq, method, scheme, n, w, ranks, wf, steps)
CASES = [("heat", "lengthening", "swept", 256, 8, 1, 0, 37), ("heat", "lengthening", "swept", 384, 32, 3, 0, 50),
         ("heat", "lengthening", "swept", 128, 4, 2, 0, 16), ("heat", "lengthening", "classic", 96, 8, 2, 0, 12),
         ("heat", "lengthening", "swept", 320, 16, 3, 2, 21), ("euler", "lengthening", "swept", 192, 16, 2, 0, 13),
         ("euler", "lengthening", "swept", 96, 8, 3, 0, 10), ("euler", "flattening", "swept", 256, 16, 2, 0, 9),
         ("euler", "flattening", "swept", 128, 8, 1, 0, 5), ("euler", "lengthening", "classic", 64, 8, 1, 0, 4)]


def cfg_of(eq, me, sc, n, w, r, wf, T):
    return s1d.LaunchConfig(equation=EQ[eq], method=ME[me], scheme=s1d.Scheme.Swept if sc == "swept"
                            else s1d.Scheme.Classic, grid_size=n, block_width=w, ranks=r, work_factor=wf, steps=T)


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_coverage_exactly_once(gpu, case):
    res = s1d.run_debug(cfg_of(*case), s1d.RunOptions(coverage=True))
    assert res.defects() == []
    want = O.port_run_serial(case[0], case[1], n=case[3], steps=case[7])
    assert np.array_equal(res.result.state.view(np.uint64), want.view(np.uint64))


# A nudge can be legitimately absorbed: FTCS multiplies it by 1-2Fo per step
# (0.2 at the default Fo=0.4, rounded away after one step), so the heat cases
# run at Fo=0.1; Euler lengthening's hook nudges Pr at point 1, which is the
# NaN sentinel on the Sod plateau (reference perturb_one_ulp,
# inc/kernels.hpp:154-157), so only flattening (Q1.rho) is checked for Euler.
MUTATION_CASES = [("heat", "lengthening", "swept", 256, 8, 1, 0, 4), ("heat", "lengthening", "swept", 384, 32, 3, 0, 16),
                  ("heat", "lengthening", "classic", 96, 8, 2, 0, 3), ("euler", "flattening", "swept", 128, 8, 1, 0, 5),
                  ("euler", "flattening", "swept", 256, 16, 2, 0, 9), ("euler", "flattening", "classic", 64, 8, 1, 0, 3)]


@pytest.mark.parametrize("case", MUTATION_CASES, ids=lambda c: "-".join(map(str, c)))
def test_perturbation_is_detected(gpu, case):
    fo = 0.1 if case[0] == "heat" else 0.4
    cfg = cfg_of(*case)
    cfg.phys.fourier = fo
    clean = s1d.run_debug(cfg, s1d.RunOptions()).result.state
    want = O.port_run_serial(case[0], case[1], n=case[3], steps=case[7], fourier=fo)
    assert np.array_equal(clean.view(np.uint64), want.view(np.uint64))
    nudged = s1d.run_debug(cfg, s1d.RunOptions(perturb_ulp=True)).result.state
    assert not np.array_equal(nudged.view(np.uint64), want.view(np.uint64))
