"""CPU: the alpha-beta virtual-time model (s1d_virtual_time, host replay of
the reference's RingTransport clock) against the compiled reference's
VirtualTime mode, bit for bit, plus the reference's closed-form tests
(test_perf.cpp:111-143) and SPEC acceptance trends."""
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

EQ = {"heat": s1d.Equation.Heat, "euler": s1d.Equation.Euler}
ME = {"lengthening": s1d.Method.Lengthening, "flattening": s1d.Method.Flattening}
SC = {"swept": s1d.Scheme.Swept, "classic": s1d.Scheme.Classic}


def pair(eq, method, scheme, n, w, ranks, wf, steps, alpha, beta, cost):
    mine = s1d.LaunchConfig(equation=EQ[eq], method=ME[method], scheme=SC[scheme], grid_size=n, block_width=w,
                            ranks=ranks, work_factor=wf, steps=steps, mode=s1d.Mode.VirtualTime,
                            transport=s1d.TransportParams(alpha, beta, cost))
    ref = O.RefConfig(equation=eq, method=method, scheme=scheme, grid_size=n, block_width=w, ranks=ranks,
                      work_factor=wf, steps=steps, mode="virtual", alpha=alpha, beta=beta, compute_cost=cost)
    return mine, ref


CASES = [
    # eq, method, scheme, n, w, ranks, wf, steps, alpha, beta, compute_cost
    ("heat", "lengthening", "swept", 1024, 32, 2, 0, 64, 1e-5, 1e-9, 1e-8),
    ("heat", "lengthening", "swept", 1024, 32, 2, 0, 50, 3e-6, 2e-10, 7e-9),     # unaligned: classic pad
    ("heat", "lengthening", "classic", 1024, 32, 2, 0, 50, 3e-6, 2e-10, 7e-9),
    ("heat", "lengthening", "swept", 1536, 32, 3, 2, 96, 1e-4, 0.0, 1e-8),       # fat rank 0 (WF=2)
    ("heat", "lengthening", "classic", 1536, 32, 3, 2, 40, 1e-4, 0.0, 1e-8),
    ("heat", "lengthening", "swept", 2048, 64, 4, 0, 31, 2.5e-6, 1e-9, 3e-9),    # cycles = 0 + pad only
    ("heat", "lengthening", "swept", 2048, 64, 4, 0, 160, 2.5e-6, 1e-9, 3e-9),   # odd cycle count
    ("euler", "lengthening", "swept", 1024, 32, 2, 0, 20, 1e-5, 1e-9, 1e-8),
    ("euler", "lengthening", "swept", 1024, 32, 2, 0, 13, 1e-5, 1e-9, 1e-8),     # 52 substeps, m=16
    ("euler", "lengthening", "classic", 1024, 32, 2, 0, 13, 1e-5, 1e-9, 1e-8),
    ("euler", "flattening", "swept", 1024, 32, 2, 0, 21, 4e-6, 3e-10, 2e-8),
    ("euler", "flattening", "classic", 1024, 32, 2, 0, 21, 4e-6, 3e-10, 2e-8),
    ("euler", "flattening", "swept", 1536, 64, 3, 1, 40, 4e-6, 3e-10, 2e-8),
]


@pytest.mark.skipif(not O.ref_available(), reason="reference not compiled (oracle/_ref)")
@pytest.mark.parametrize("case", CASES)
def test_virtual_clock_matches_reference_bitwise(case):
    mine, ref = pair(*case)
    v, comm = s1d.virtual_time(mine)
    r = O.ref_run(ref)
    assert v == r.virtual_seconds, (v, r.virtual_seconds)
    assert comm == r.virtual_comm_time, (comm, r.virtual_comm_time)


@pytest.mark.skipif(not O.ref_available(), reason="reference not compiled (oracle/_ref)")
def test_comm_time_reported_in_wall_mode_too():
    # CommStats::virtual_comm_time accumulates in both modes (transport.cpp:84)
    mine, ref = pair("heat", "lengthening", "classic", 1024, 32, 2, 0, 16, 1e-5, 1e-9, 1e-8)
    ref.mode = "wall"
    _, comm = s1d.virtual_time(mine)
    assert comm == O.ref_run(ref).virtual_comm_time


def virtual_cfg(scheme, alpha):
    # test_perf.cpp:11-24
    return s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=scheme, grid_size=256, block_width=16, ranks=2,
                            steps=32, mode=s1d.Mode.VirtualTime, transport=s1d.TransportParams(alpha, 0.0, 1e-8))


def test_closed_form_classic():
    # test_perf.cpp:111-124: per substep each rank computes n/2 points then pays alpha
    v, comm = s1d.virtual_time(virtual_cfg(s1d.Scheme.Classic, 1e-5))
    per_step = (128.0 * 1e-8 + 1e-5) * 1e6
    assert v * 1e6 / 32 == pytest.approx(per_step, rel=1e-9)
    assert comm == pytest.approx(32 * 1e-5, rel=1e-12)
    c2 = virtual_cfg(s1d.Scheme.Classic, 1e-5)
    c2.steps = 64
    assert s1d.virtual_time(c2)[0] * 1e6 / 64 == pytest.approx(v * 1e6 / 32, rel=1e-12)


def test_swept_latency_scales_by_cycle_ratio():
    # test_perf.cpp:126-143: d(classic)/d(alpha) = T*S, d(swept)/d(alpha) = T*S*2h/w
    a1, a2 = 1e-6, 1e-4
    c1 = s1d.virtual_time(virtual_cfg(s1d.Scheme.Classic, a1))[0]
    c2 = s1d.virtual_time(virtual_cfg(s1d.Scheme.Classic, a2))[0]
    w1 = s1d.virtual_time(virtual_cfg(s1d.Scheme.Swept, a1))[0]
    w2 = s1d.virtual_time(virtual_cfg(s1d.Scheme.Swept, a2))[0]
    assert (c2 - c1) / 32 == pytest.approx(a2 - a1, rel=1e-9)
    assert (w2 - w1) / 32 == pytest.approx((a2 - a1) / 8.0, rel=1e-9)
    assert c2 / w2 > c1 / w1 >= 1.0


def test_spec_latency_trend():
    # beta = 0, swept speedup >= 1 and strictly increasing in
    # alpha; at large alpha it approaches w/(2h) within 10%
    prev = 0.0
    for alpha in (1e-6, 1e-5, 1e-4, 1e-3):
        c = s1d.virtual_time(virtual_cfg(s1d.Scheme.Classic, alpha))[0]
        w = s1d.virtual_time(virtual_cfg(s1d.Scheme.Swept, alpha))[0]
        sp = s1d.speedup(c, w)
        assert sp >= 1.0 and sp > prev
        prev = sp
    assert prev == pytest.approx(16 / 2, rel=0.10)


def test_spec_scaling_regularity():
    # virtual swept time per step vs n over 2^10..2^16 fits a
    # power law with R^2 > 0.99 and b in [0.9, 1.1]
    ns, ts = [], []
    for k in range(10, 17):
        c = s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=s1d.Scheme.Swept, grid_size=1 << k, block_width=64,
                             ranks=2, steps=128, mode=s1d.Mode.VirtualTime,
                             transport=s1d.TransportParams(1e-6, 1e-10, 1e-8))
        ns.append(float(1 << k))
        ts.append(s1d.virtual_time(c)[0] * 1e6 / 128)
    fit = s1d.power_law_fit(list(zip(ns, ts)))
    assert fit.r_squared > 0.99 and 0.9 <= fit.b <= 1.1


def test_virtual_time_validates():
    c = virtual_cfg(s1d.Scheme.Swept, 1e-5)
    c.block_width = 12  # 256 not divisible into w=12 blocks
    with pytest.raises(s1d.InvalidConfig):
        s1d.virtual_time(c)
