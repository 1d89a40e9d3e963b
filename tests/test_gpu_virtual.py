"""GPU: VirtualTime mode through the C ABI — the device computes the state for
real (bitwise == oracle) while timing.virtual_seconds / stats.virtual_comm_time
carry the reference's alpha-beta clock (perf.cpp:21-23 picks it for
measure()); NVLink calibration of alpha and beta (needs 2 GPUs)."""
import dataclasses

import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scheme", [s1d.Scheme.Swept, s1d.Scheme.Classic], ids=s1d.to_string)
def test_virtual_run_reports_model_and_computes_state(gpu, scheme):
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=scheme, grid_size=1 << 12, block_width=64, ranks=2,
                           steps=100, mode=s1d.Mode.VirtualTime, transport=s1d.TransportParams(2e-6, 1e-9, 1e-8))
    res = s1d.run(cfg)
    v, comm = s1d.virtual_time(cfg)
    assert res.timing.virtual_seconds == v and res.stats.virtual_comm_time == comm
    want = O.port_run_serial("heat", n=1 << 12, steps=100)
    assert np.array_equal(res.state.view(np.uint64), want.view(np.uint64))
    wall = dataclasses.replace(cfg, mode=s1d.Mode.WallClock)
    r2 = s1d.run(wall)
    assert r2.timing.virtual_seconds == 0.0 and r2.stats.virtual_comm_time == comm


def test_virtual_measure_closed_form(gpu):
    # test_perf.cpp:111-124 through measure() on the device path
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=s1d.Scheme.Classic, grid_size=256, block_width=16,
                           ranks=2, steps=32, mode=s1d.Mode.VirtualTime,
                           transport=s1d.TransportParams(1e-5, 0.0, 1e-8))
    rec = s1d.measure(cfg)
    assert rec.avg_us_per_step == pytest.approx((128.0 * 1e-8 + 1e-5) * 1e6, rel=1e-9)
    assert rec.exchange_rounds == 32
    assert rec.virtual_comm_us == pytest.approx(32 * 1e-5 * 1e6, rel=1e-12)


@pytest.mark.skipif(s1d.device_count() < 2, reason="needs >= 2 GPUs")
def test_calibrate_transport(gpu):
    tp = s1d.calibrate_transport(0, 1)
    assert 1e-7 < tp.alpha < 1e-4          # one-way NVLink flag hand-off: ~1-10 us
    assert 1.0 / 2e12 < tp.beta < 1.0 / 5e10  # 50 GB/s .. 2 TB/s peer copy
