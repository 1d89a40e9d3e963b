"""CPU: host-side logic of the B200 library (validation, geometry, initial
conditions, schedules, config parsing) against the reference's own tests
(test_partition.cpp, test_schedules.cpp, test_decomp.cpp) and golden values.
These calls never touch a GPU."""
import json
import os

import numpy as np
import pytest

import paper_1811_08282_b200 as s1d

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
HEAT = s1d.make_spec(s1d.Equation.Heat, s1d.Method.Lengthening)
LEN = s1d.make_spec(s1d.Equation.Euler, s1d.Method.Lengthening)
FLAT = s1d.make_spec(s1d.Equation.Euler, s1d.Method.Flattening)


def base(n, w, ranks, wf):
    return s1d.LaunchConfig(equation=s1d.Equation.Heat, grid_size=n, block_width=w, ranks=ranks, work_factor=wf)


def test_make_spec():
    assert (HEAT.substeps_per_step, HEAT.stencil_half_width, HEAT.state_slots) == (1, 1, 2)
    assert (LEN.substeps_per_step, LEN.stencil_half_width, LEN.state_slots) == (4, 1, 7)
    assert (FLAT.substeps_per_step, FLAT.stencil_half_width, FLAT.state_slots) == (2, 2, 6)


def test_partition_split():
    # test_partition.cpp:23-32
    assert s1d.make_partition(base(320, 32, 2, 0)).blocks == [5, 5]
    p = s1d.make_partition(base(384, 32, 3, 4))
    assert p.blocks == [8, 2, 2] and p.start_index == [0, 256, 320]
    with pytest.raises(s1d.InvalidConfig):
        s1d.make_partition(base(100, 32, 2, 0))


def test_invalid_messages():
    # test_partition.cpp:34-43 (ranks=1 is valid on the B200 path: one GPU).
    # Note: the reference test's first case (heat, w=6 -> "multiple of 2*h")
    # does not hold against the reference code itself (w=6 is valid for h=1;
    # the shipped doctest suite cannot be built, so it never ran). We check the
    # reference *code's* behaviour: heat w=6 is accepted, flattening (h=2)
    # w=10 trips the 2h rule.
    assert s1d.make_partition(base(96, 6, 2, 0)).blocks == [8, 8]
    with pytest.raises(s1d.InvalidConfig, match="multiple of 2\\*h"):
        s1d.make_partition(s1d.LaunchConfig(equation=s1d.Equation.Euler, method=s1d.Method.Flattening,
                                            grid_size=100, block_width=10, ranks=2))
    with pytest.raises(s1d.InvalidConfig, match="divisible"):
        s1d.make_partition(base(100, 32, 2, 0))
    with pytest.raises(s1d.InvalidConfig, match="rank"):
        s1d.make_partition(base(320, 32, 0, 0))
    with pytest.raises(s1d.InvalidConfig, match="shares"):
        s1d.make_partition(base(320, 32, 3, 2))
    with pytest.raises(s1d.InvalidConfig, match="even"):
        s1d.make_partition(base(320, 7, 2, 0))
    s1d.make_partition(base(320, 32, 1, 0))  # one shard is fine here


def test_ring_closure_and_coverage():
    # test_partition.cpp:45-76 (sampled)
    for w in (4, 8, 16):
        for r in (1, 2, 3, 4):
            for wf in range(0, 9, 2):
                for n in range(w, 1025, w * 7):
                    cfg = base(n, w, r, wf)
                    if (n // w) % cfg.shares():
                        continue
                    p = s1d.make_partition(cfg)
                    start = 0
                    for i in range(r):
                        assert p.start_index[i] == start
                        start += p.owned_points(i)
                    assert start == n
                    if wf > 0 and r > 1:
                        assert p.blocks[0] == wf * p.blocks[1]
                    at = 0
                    for _ in range(r):
                        at = p.left[at]
                    assert at == 0


def test_extents_and_buffer():
    # test_partition.cpp:78-112
    e = s1d.working_array_extents(4, 8, HEAT)
    assert (e.length, e.initialized) == (38, 34)
    e = s1d.working_array_extents(2, 8, FLAT)
    assert (e.ghost, e.length, e.initialized) == (2, 24, 20)
    assert s1d.swept_buffer_cells(8, HEAT) == 5
    assert s1d.swept_buffer_cells(32, HEAT) == 17
    assert s1d.swept_buffer_cells(8, FLAT) == 6


def test_initial_conditions_match_reference():
    bits = lambda a: np.asarray(a, dtype=np.float64).view(np.uint64)  # noqa: E731
    assert np.array_equal(bits(s1d.initial_condition("heat-sine", 4, HEAT)), bits(GOLD["ic"]["heat-sine-4"]))
    assert np.array_equal(bits(s1d.initial_condition("heat-sine", 12, HEAT)), bits(GOLD["ic"]["heat-sine-12"]))
    assert np.array_equal(bits(s1d.initial_condition("euler-sod-periodic", 4, LEN)), bits(GOLD["ic"]["sod-4"]))
    assert np.all(s1d.initial_condition("uniform", 6, HEAT) == 1.0)
    with pytest.raises(s1d.UnknownInitialCondition):
        s1d.initial_condition("no-such-ic", 8, HEAT)
    with pytest.raises(s1d.UnknownInitialCondition):
        s1d.initial_condition("heat-sine", 8, LEN)


def test_dt_dx_from_cfl():
    # test_partition.cpp:139-151
    sod = s1d.initial_condition("euler-sod-periodic", 8, LEN)
    assert abs(s1d.max_signal_speed(sod, 1.4) - np.sqrt(1.4)) <= 1e-14 * np.sqrt(1.4)
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Euler, grid_size=64, block_width=8, ranks=2)
    cfg.finalize()
    assert cfg.phys.dt_dx == GOLD["dt_dx_sod"]


def test_schedules_match_reference():
    for key, levels in GOLD["schedules"].items():
        kind, w, h = key.split("-")
        fn = {"triangle": s1d.triangle_schedule, "diamond": s1d.diamond_schedule,
              "down": s1d.down_triangle_schedule}[kind]
        got = [(l.substep, l.lo, l.hi) for l in fn(int(w), int(h)).levels]
        assert got == [tuple(x) for x in levels]


def test_schedule_widths_and_errors():
    # test_schedules.cpp
    w = lambda s: [l.width() for l in s.levels]  # noqa: E731
    assert w(s1d.triangle_schedule(8, 1)) == [6, 4, 2]
    assert w(s1d.diamond_schedule(8, 1)) == [2, 4, 6, 8, 6, 4, 2]
    assert w(s1d.down_triangle_schedule(8, 2)) == [4, 8]
    assert s1d.down_triangle_schedule(8, 1).substeps() == 4
    assert s1d.cycle_advance(32, 2) == 8
    for bad in ((7, 1), (4, 2), (10, 2)):
        with pytest.raises(s1d.InvalidWidth):
            s1d.triangle_schedule(*bad)


def test_validation_physics():
    with pytest.raises(s1d.InvalidConfig, match="Fourier"):
        s1d.LaunchConfig(grid_size=64, block_width=8, phys=s1d.PhysParams(fourier=0.6)).validate()
    with pytest.raises(s1d.InvalidConfig, match="gamma"):
        s1d.LaunchConfig(grid_size=64, block_width=8, phys=s1d.PhysParams(gamma=1.0)).validate()
    with pytest.raises(s1d.InvalidConfig, match="step"):
        s1d.LaunchConfig(grid_size=64, block_width=8, steps=-1).validate()
    with pytest.raises(s1d.InvalidConfig, match="small"):
        s1d.LaunchConfig(grid_size=2, block_width=8).validate(partitioned=False)
    s1d.LaunchConfig(grid_size=4, block_width=8).validate(partitioned=False)


def test_config_entries_and_file(tmp_path):
    cfg = s1d.LaunchConfig()
    for k, v in [("equation", "euler"), ("method", "flattening"), ("scheme", "classic"), ("n", "4096"),
                 ("w", "64"), ("ranks", "4"), ("wf", "2"), ("steps", "77"), ("initial", "uniform"),
                 ("mode", "wall"), ("fourier", "0.25"), ("gamma", "1.67"), ("cfl", "0.3")]:
        s1d.apply_config_entry(cfg, k, v)
    assert cfg.equation == s1d.Equation.Euler and cfg.method == s1d.Method.Flattening
    assert cfg.scheme == s1d.Scheme.Classic and cfg.grid_size == 4096 and cfg.block_width == 64
    assert cfg.ranks == 4 and cfg.work_factor == 2 and cfg.steps == 77 and cfg.initial == "uniform"
    assert cfg.mode == s1d.Mode.WallClock and cfg.phys.fourier == 0.25 and cfg.phys.gamma == 1.67
    with pytest.raises(s1d.InvalidConfig, match="unknown config key"):
        s1d.apply_config_entry(cfg, "bogus", "1")
    with pytest.raises(s1d.InvalidConfig):
        s1d.apply_config_entry(cfg, "equation", "wave")
    p = tmp_path / "c.cfg"
    p.write_text("# comment\n equation = heat \n\nn=128 # trailing\nw=8\n")
    cfg2 = s1d.LaunchConfig()
    s1d.apply_config_file(cfg2, str(p))
    assert cfg2.equation == s1d.Equation.Heat and cfg2.grid_size == 128 and cfg2.block_width == 8
    p.write_text("novalue\n")
    with pytest.raises(s1d.InvalidConfig, match="expected key=value"):
        s1d.apply_config_file(cfg2, str(p))
