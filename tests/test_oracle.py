"""CPU: pin the oracle. The C restatement (oracle/s1d_oracle.c) must match the
reference's golden vectors (tests/golden/golden.json, produced by the reference
compiled from source) bit for bit, and — when oracle/_ref is built — the
reference itself on fresh cases."""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def same(a, b):
    if isinstance(a, float) and isinstance(b, float) and math.isnan(a) and math.isnan(b):
        return True
    return np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64)


@pytest.mark.parametrize("fp", GOLD["fingerprints"], ids=lambda f: f"{f['equation']}-{f['method']}-{f['n']}-{f['steps']}")
def test_port_fingerprints(fp):
    st = O.port_run_serial(fp["equation"], fp["method"], n=fp["n"], steps=fp["steps"])
    assert O.fnv1a64(st) == fp["fnv1a64"]
    for i, v in fp["sample"].items():
        assert same(float(st[int(i)]), v)


@pytest.mark.parametrize("c", GOLD["decomp"], ids=lambda c: f"{c['equation']}-{c['method']}-{c['n']}-{c['w']}-{c['steps']}")
def test_port_decomp_states(c):
    st = O.port_run_serial(c["equation"], c["method"], n=c["n"], steps=c["steps"])
    assert np.array_equal(bits(st), bits(np.array(c["state"])))


def test_port_kernel_kats():
    lib = O.port()
    for l, c, r, fo, want in GOLD["kernels"]["heat_step"]:
        assert same(lib.s1o_heat_step(l, c, r, fo), want)
    for a, b, want in GOLD["kernels"]["minmod"]:
        assert same(lib.s1o_minmod(a, b), want)
    for a, b, c, want in GOLD["kernels"]["pressure_ratio"]:
        assert same(lib.s1o_pressure_ratio_value(a, b, c), want)
    for case in GOLD["kernels"]["interface_flux"]:
        out = np.empty(3)
        st = lib.s1o_interface_flux(O._ptr(np.array(case["ql"])), O._ptr(np.array(case["qr"])), case["pr_l"],
                                    case["pr_r"], 1.4, O._ptr(out))
        assert (st == 0) == (case["status"] == 0)
        if st == 0:
            assert np.array_equal(bits(out), bits(np.array(case["flux"])))


def test_sod_predictor_golden_vector():
    # test_kernels.cpp:184-197: 1e-14 relative against the frozen values
    got = GOLD["kernels"]["sod_predictor"]["q1"]
    for g, e in zip(got, GOLD["kernels"]["sod_predictor"]["expect_1e-14"]):
        assert abs(g - e) <= 1e-14 * abs(e)


def test_heat_four_point_kat():
    # test_decomp.cpp:72-79
    st = O.port_run_serial("heat", n=4, steps=1, fourier=0.25)
    assert list(st) == [0.0, 0.5, 0.0, -0.5]


def test_port_initial_conditions():
    assert np.array_equal(bits(O.port_initial_condition("heat-sine", 4)), bits(np.array(GOLD["ic"]["heat-sine-4"])))
    assert np.array_equal(bits(O.port_initial_condition("heat-sine", 12)),
                          bits(np.array(GOLD["ic"]["heat-sine-12"])))
    assert np.array_equal(bits(O.port_initial_condition("euler-sod-periodic", 4, "euler")),
                          bits(np.array(GOLD["ic"]["sod-4"])))
    assert O.fnv1a64(O.port_initial_condition("heat-sine", 1000)) == GOLD["ic"]["heat-sine-1000-fnv"]


def test_port_errors():
    with pytest.raises(O.OracleError) as ei:
        O.port_run_serial("heat", n=8, steps=1, initial="no-such-ic")
    assert ei.value.status == 2
    with pytest.raises(O.OracleError) as ei:
        O.port_run_serial("heat", n=2, steps=1)
    assert ei.value.status == 1


def test_euler_long_run_conservation():
    # long runs stay physical and conserve mass to round-off.
    st = O.port_run_serial("euler", "lengthening", n=256, steps=2000)
    ic = O.port_initial_condition("euler-sod-periodic", 256, "euler")
    for v in range(3):
        assert abs(st[v::3].sum() - ic[v::3].sum()) <= 1e-12 * max(np.abs(ic[v::3]).sum(), 1.0)


needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference sources/build not available")


@needs_ref
@pytest.mark.parametrize("eq,me,n,T", [("heat", "lengthening", 1000, 77), ("euler", "lengthening", 500, 40),
                                       ("euler", "flattening", 500, 40), ("heat", "lengthening", 10, 5),
                                       ("euler", "lengthening", 5, 3), ("euler", "flattening", 6, 9)])
def test_port_vs_reference(eq, me, n, T):
    a = O.port_run_serial(eq, me, n=n, steps=T)
    b = O.ref_run_serial(O.RefConfig(equation=eq, method=me, grid_size=n, steps=T))
    assert np.array_equal(bits(a), bits(b))


@needs_ref
def test_port_vs_reference_custom_params():
    a = O.port_run_serial("heat", n=300, steps=50, fourier=0.5)
    b = O.ref_run_serial(O.RefConfig(grid_size=300, steps=50, fourier=0.5))
    assert np.array_equal(bits(a), bits(b))
    a = O.port_run_serial("euler", "lengthening", n=200, steps=30, gamma=1.67, cfl=0.3)
    b = O.ref_run_serial(O.RefConfig(equation="euler", grid_size=200, steps=30, gamma=1.67, cfl=0.3))
    assert np.array_equal(bits(a), bits(b))
