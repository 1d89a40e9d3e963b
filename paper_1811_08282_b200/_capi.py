"""ctypes binding of include/swept1d.h (the C ABI of libswept1d.so).

The library is built in-tree (paper_1811_08282_b200/_lib/libswept1d.so, see
csrc/Makefile). There is no fallback: importing a compute entry point without
the library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("S1D_LIB_PATH") or os.path.join(HERE, "_lib", "libswept1d.so")

S1D_HEAT, S1D_EULER = 0, 1
S1D_LENGTHENING, S1D_FLATTENING = 0, 1
S1D_CLASSIC, S1D_SWEPT = 0, 1
S1D_WALL, S1D_VIRTUAL = 0, 1


class s1d_config(C.Structure):
    _fields_ = [("equation", C.c_int), ("method", C.c_int), ("scheme", C.c_int), ("mode", C.c_int),
                ("grid_size", C.c_uint64), ("block_width", C.c_uint64), ("ranks", C.c_int),
                ("work_factor", C.c_int), ("steps", C.c_int64), ("fourier", C.c_double), ("gamma", C.c_double),
                ("dt_dx", C.c_double), ("cfl", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
                ("compute_cost", C.c_double), ("initial", C.c_char * 64), ("num_devices", C.c_int),
                ("reserved", C.c_int * 7)]


class s1d_stats(C.Structure):
    _fields_ = [("messages_sent", C.c_uint64), ("bytes_sent", C.c_uint64), ("exchange_rounds", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("edge_bytes_device", C.c_uint64),
                ("virtual_comm_seconds", C.c_double)]


class s1d_rank_stats(C.Structure):
    _fields_ = [("messages_sent", C.c_uint64), ("bytes_sent", C.c_uint64), ("exchange_rounds", C.c_uint64),
                ("virtual_comm_seconds", C.c_double)]


class s1d_message(C.Structure):
    _fields_ = [("round", C.c_uint64), ("source", C.c_int32), ("dest", C.c_int32), ("tag", C.c_uint64),
                ("bytes", C.c_uint64)]


class s1d_timing(C.Structure):
    _fields_ = [("setup_seconds", C.c_double), ("loop_seconds", C.c_double), ("virtual_seconds", C.c_double),
                ("h2d_seconds", C.c_double), ("d2h_seconds", C.c_double), ("dominant_seconds", C.c_double),
                ("dominant_launches", C.c_uint64), ("dominant_point_updates", C.c_uint64),
                ("dominant_kernel", C.c_char * 32)]


class s1d_record(C.Structure):
    _fields_ = [("equation", C.c_int), ("method", C.c_int), ("scheme", C.c_int), ("mode", C.c_int),
                ("grid_size", C.c_uint64), ("block_width", C.c_uint64), ("work_factor", C.c_int),
                ("ranks", C.c_int), ("steps", C.c_int64), ("avg_us_per_step", C.c_double),
                ("setup_us", C.c_double), ("messages_sent", C.c_uint64), ("bytes_sent", C.c_uint64),
                ("exchange_rounds", C.c_uint64), ("virtual_comm_us", C.c_double)]


class s1d_debug(C.Structure):
    _fields_ = [("coverage", C.c_int), ("perturb_ulp", C.c_int), ("coverage_out", C.POINTER(C.c_uint32)),
                ("coverage_len", C.c_size_t)]


_dp = C.POINTER(C.c_double)
_E = [C.c_char_p, C.c_size_t]

# Every symbol include/swept1d.h declares, with (restype, argtypes).
SIGNATURES = {
    "s1d_version": (C.c_char_p, []),
    "s1d_abi_version": (C.c_int, []),
    "s1d_device_count": (C.c_int, []),
    "s1d_config_defaults": (None, [C.POINTER(s1d_config)]),
    "s1d_apply_config_entry": (C.c_int, [C.POINTER(s1d_config), C.c_char_p, C.c_char_p] + _E),
    "s1d_validate": (C.c_int, [C.POINTER(s1d_config), C.c_int] + _E),
    "s1d_finalize": (C.c_int, [C.POINTER(s1d_config), C.c_int] + _E),
    "s1d_spec": (None, [C.c_int, C.c_int] + [C.POINTER(C.c_int)] * 4),
    "s1d_initial_condition": (C.c_int, [C.c_char_p, C.c_uint64, C.c_int, C.c_double, _dp, C.c_size_t] + _E),
    "s1d_initial_condition_range": (C.c_int, [C.c_char_p, C.c_uint64, C.c_int, C.c_double, C.c_uint64, C.c_uint64,
                                              _dp, C.c_size_t] + _E),
    "s1d_max_signal_speed": (C.c_int, [_dp, C.c_size_t, C.c_double, _dp] + _E),
    "s1d_partition": (C.c_int, [C.POINTER(s1d_config), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                C.POINTER(C.c_int), C.POINTER(C.c_int)] + _E),
    "s1d_cycle_advance": (C.c_int64, [C.c_uint64, C.c_uint64] + _E),
    "s1d_schedule": (C.c_int64, [C.c_int, C.c_uint64, C.c_uint64, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int64), C.c_size_t] + _E),
    "s1d_swept_buffer_cells": (C.c_uint64, [C.c_uint64, C.c_int, C.c_int]),
    "s1d_run": (C.c_int, [C.POINTER(s1d_config), _dp, C.c_size_t, C.POINTER(s1d_stats), C.POINTER(s1d_timing)]
                + _E),
    "s1d_run_debug": (C.c_int, [C.POINTER(s1d_config), C.POINTER(s1d_debug), _dp, C.c_size_t, C.POINTER(s1d_stats),
                                C.POINTER(s1d_timing)] + _E),
    "s1d_create": (C.c_int, [C.POINTER(s1d_config), C.POINTER(C.c_void_p)] + _E),
    "s1d_destroy": (None, [C.c_void_p]),
    "s1d_get_config": (C.c_int, [C.c_void_p, C.POINTER(s1d_config)]),
    "s1d_set_initial": (C.c_int, [C.c_void_p, _dp, C.c_size_t]),
    "s1d_advance": (C.c_int, [C.c_void_p, C.POINTER(s1d_stats), C.POINTER(s1d_timing)]),
    "s1d_read_state": (C.c_int, [C.c_void_p, _dp, C.c_size_t]),
    "s1d_solve": (C.c_int, [C.c_void_p, _dp, C.c_size_t, _dp, C.c_size_t, C.POINTER(s1d_stats),
                            C.POINTER(s1d_timing)]),
    "s1d_last_error": (C.c_char_p, [C.c_void_p]),
    "s1d_measure_fp64_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double)] + _E),
    "s1d_virtual_time": (C.c_int, [C.POINTER(s1d_config), _dp, _dp] + _E),
    "s1d_message_log": (C.c_int, [C.POINTER(s1d_config), C.POINTER(s1d_message), C.c_size_t,
                                  C.POINTER(C.c_size_t)] + _E),
    "s1d_comm_per_rank": (C.c_int, [C.POINTER(s1d_config), C.POINTER(s1d_rank_stats), C.c_size_t] + _E),
    "s1d_debug_wave_schedule": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int, C.POINTER(C.c_int64),
                                          C.c_size_t, C.POINTER(C.c_size_t)] + _E),
    "s1d_calibrate_transport": (C.c_int, [C.c_int, C.c_int, _dp, _dp] + _E),
    "s1d_measure": (C.c_int, [C.POINTER(s1d_config), C.POINTER(s1d_record)] + _E),
    "s1d_csv_header": (C.c_char_p, []),
    "s1d_csv_row": (C.c_int64, [C.POINTER(s1d_record), C.c_char_p, C.c_size_t]),
    "s1d_emit_csv": (C.c_int, [C.POINTER(s1d_record), C.c_size_t, C.c_char_p] + _E),
    "s1d_read_csv": (C.c_int, [C.c_char_p, C.POINTER(s1d_record), C.c_size_t, C.POINTER(C.c_size_t)] + _E),
    "s1d_power_law_fit": (C.c_int, [_dp, _dp, C.c_size_t, _dp, _dp, _dp] + _E),
    "s1d_best_config": (C.c_int64, [C.POINTER(s1d_record), C.c_size_t]),
    "s1d_shard_create": (C.c_int, [C.POINTER(s1d_config), C.c_int, C.c_int, C.POINTER(C.c_void_p)] + _E),
    "s1d_shard_blob_size": (C.c_size_t, []),
    "s1d_shard_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "s1d_shard_connect": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p]),
    "s1d_shard_range": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load libswept1d.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is missing: build it with `make -C paper_1811_08282_b200/csrc` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            # an explicit S1D_LIB_PATH (an older build variant for A/B timing)
            # may predate some symbols; the in-tree library must have them all
            if os.environ.get("S1D_LIB_PATH") and not hasattr(L, name):
                continue
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
