"""CPU: the C-ABI library loads and exports every symbol include/swept1d.h
declares; compute entry points report NO_DEVICE (never a CPU fallback) here."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1811_08282_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "swept1d.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(s1d_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_capi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 24
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers them all
    assert set(syms) <= set(_capi.SIGNATURES), set(syms) - set(_capi.SIGNATURES)


def test_version_and_abi():
    lib = _capi.lib()
    assert lib.s1d_abi_version() == 2
    assert b"sm_100a" in lib.s1d_version()


def test_struct_sizes_match_header(tmp_path):
    # sizeof/offsetof from the real header (compiled with gcc) == the ctypes mirror
    names = ["s1d_config", "s1d_stats", "s1d_timing", "s1d_record", "s1d_debug"]
    src = tmp_path / "probe.c"
    src.write_text('#include <stdio.h>\n#include "swept1d.h"\nint main(void) {\n' +
                   "".join(f'  printf("%zu\\n", sizeof({n}));\n' for n in names) + "  return 0;\n}\n")
    exe = tmp_path / "probe"
    inc = os.path.join(os.path.dirname(__file__), "..", "include")
    subprocess.run(["gcc", "-std=c99", "-I", inc, str(src), "-o", str(exe)], check=True)
    sizes = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert sizes == [C.sizeof(getattr(_capi, n)) for n in names]


@pytest.mark.skipif(_capi.lib().s1d_device_count() > 0, reason="GPU visible")
def test_no_cpu_fallback_without_gpu():
    import paper_1811_08282_b200 as s1d
    with pytest.raises(s1d.NoDevice):
        s1d.run(s1d.LaunchConfig(grid_size=64, block_width=8, steps=2))
    with pytest.raises(s1d.NoDevice):
        s1d.Solver(s1d.LaunchConfig(grid_size=64, block_width=8, steps=2))
    with pytest.raises(s1d.NoDevice):
        s1d.calibrate_transport(0, 1)
    with pytest.raises(s1d.NoDevice):
        s1d.measure_fp64_peak(0)
    # the virtual-time model is host-only and works without a GPU
    v, comm = s1d.virtual_time(s1d.LaunchConfig(grid_size=64, block_width=8, steps=2))
    assert v > 0 and comm == 0.0


def test_defaults_mirror_reference():
    import paper_1811_08282_b200 as s1d
    c = _capi.s1d_config()
    _capi.lib().s1d_config_defaults(C.byref(c))
    d = s1d.LaunchConfig()
    assert (c.grid_size, c.block_width, c.ranks, c.work_factor, c.steps) == (1024, 32, 2, 0, 50)
    assert (c.fourier, c.gamma, c.dt_dx, c.cfl, c.compute_cost) == (0.4, 1.4, 0.0, 0.4, 1e-8)
    assert c.scheme == int(d.scheme) == 1 and c.mode == int(d.mode) == 1


def test_null_arguments_fail_loudly():
    lib = _capi.lib()
    e = C.create_string_buffer(256)
    assert lib.s1d_validate(None, 1, e, 256) == 1 and b"null" in e.value
    assert lib.s1d_run(None, None, 0, None, None, e, 256) == 1
    assert lib.s1d_virtual_time(None, None, None, e, 256) == 1
    h = C.c_void_p()
    assert lib.s1d_create(None, C.byref(h), e, 256) == 1 and not h.value
    assert lib.s1d_advance(None, None, None) == 1 and lib.s1d_read_state(None, None, 0) == 1


def test_null_outputs_fail_loudly():
    """Every pointer argument of the ABI is checked before it is dereferenced
    (no crash, S1D_INVALID_CONFIG and a message)."""
    lib = _capi.lib()
    e = C.create_string_buffer(256)
    cfg = _capi.s1d_config()
    lib.s1d_config_defaults(C.byref(cfg))
    assert lib.s1d_create(C.byref(cfg), None, e, 256) == 1 and b"null" in e.value
    assert lib.s1d_shard_create(C.byref(cfg), 0, 0, None, e, 256) == 1
    assert lib.s1d_get_config(None, C.byref(cfg)) == 1
    assert lib.s1d_shard_range(None, None, None) == 1
    assert lib.s1d_shard_connect(None, None, None) == 1
    assert lib.s1d_initial_condition(b"heat-sine", 16, 0, 1.4, None, 16, e, 256) == 1
    assert lib.s1d_initial_condition(None, 16, 0, 1.4, None, 16, e, 256) == 1
    assert lib.s1d_initial_condition_range(b"heat-sine", 16, 0, 1.4, 0, 4, None, 4, e, 256) == 1
    assert lib.s1d_max_signal_speed(None, 3, 1.4, None, e, 256) == 1
    cfg.ranks = 2
    assert lib.s1d_partition(C.byref(cfg), None, None, None, None, e, 256) == 1 and b"null" in e.value
    assert lib.s1d_csv_row(None, None, 0) == -1 * 1
    assert lib.s1d_emit_csv(None, 1, None, e, 256) == 1
    assert lib.s1d_read_csv(None, None, 0, None, e, 256) == 1
    assert lib.s1d_power_law_fit(None, None, 3, None, None, None, e, 256) == 1
    assert lib.s1d_best_config(None, 2) == -1


def test_out_buffer_validation():
    """api.py never hands the library a buffer it would overrun."""
    import numpy as np
    from paper_1811_08282_b200 import api
    assert api._out_buffer(None, 4).dtype == np.float64
    with pytest.raises(TypeError):
        api._out_buffer(np.zeros(8, np.float32), 4)
    with pytest.raises(ValueError):
        api._out_buffer(np.zeros(8)[::2], 4)
    with pytest.raises(ValueError):
        api._out_buffer(np.zeros(3), 4)
    ro = np.zeros(4)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        api._out_buffer(ro, 4)
    spec = api.make_spec(api.Equation.Heat, api.Method.Lengthening)
    with pytest.raises(TypeError):
        api.initial_condition_range("heat-sine", 16, spec, 0, 4, out=np.zeros(4, np.float32))
    got = api.initial_condition_range("heat-sine", 16, spec, 0, 4, out=np.zeros(4))
    assert got.shape == (4,)
