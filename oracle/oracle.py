"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracles.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline — never as the product path.

Two oracles:

* ``port``: oracle/_build/libs1d_oracle.so, this repo's C restatement of the
  reference serial solver (engines_impl.hpp:85-128 + src/kernels.cpp).
* ``ref``: oracle/_ref/libsweep1d_ref.so, the unmodified reference core
  compiled from /root/reference/proj/core/src by oracle/Makefile, reached
  through oracle/ref_shim.cpp. Built here (the reference is mounted in the dev
  container only); the built .so travels to the GPU box with the snapshot.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libs1d_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsweep1d_ref.so")
REF_ROOT = "/root/reference/proj"

_dp = C.POINTER(C.c_double)


def build(ref: bool | None = None) -> None:
    """Compile the port (always) and the reference (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    if ref is None:
        ref = os.path.isdir(os.path.join(REF_ROOT, "core", "src"))
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


# --------------------------------------------------------------------------
# port (C restatement)
# --------------------------------------------------------------------------
_port = None


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build(ref=False)
        lib = C.CDLL(PORT_SO)
        lib.s1o_heat_step.restype = C.c_double
        lib.s1o_heat_step.argtypes = [C.c_double] * 4
        lib.s1o_minmod.restype = C.c_double
        lib.s1o_minmod.argtypes = [C.c_double] * 2
        lib.s1o_pressure_ratio_value.restype = C.c_double
        lib.s1o_pressure_ratio_value.argtypes = [C.c_double] * 3
        lib.s1o_pressure.argtypes = [_dp, C.c_double, _dp]
        lib.s1o_interface_flux.argtypes = [_dp, _dp, C.c_double, C.c_double, C.c_double, _dp]
        lib.s1o_initial_condition.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.c_double, _dp]
        lib.s1o_max_signal_speed.argtypes = [_dp, C.c_size_t, C.c_double, _dp]
        lib.s1o_run_serial.argtypes = [C.c_int, C.c_int, C.c_size_t, C.c_long, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_char_p, _dp]
        lib.s1o_run_state.argtypes = [C.c_int, C.c_int, C.c_size_t, C.c_long, C.c_double, C.c_double, C.c_double,
                                      _dp, _dp]
        lib.s1o_fnv1a64.restype = C.c_ulonglong
        lib.s1o_fnv1a64.argtypes = [_dp, C.c_size_t]
        _port = lib
    return _port


def vpp(equation: str) -> int:
    return 1 if equation == "heat" else 3


def port_run_serial(equation="heat", method="lengthening", n=1024, steps=50, fourier=0.4, gamma=1.4,
                    dt_dx=0.0, cfl=0.4, initial="") -> np.ndarray:
    out = np.empty(n * vpp(equation), dtype=np.float64)
    st = port().s1o_run_serial(0 if equation == "heat" else 1, 0 if method == "lengthening" else 1, n, steps,
                               fourier, gamma, dt_dx, cfl, initial.encode(), _ptr(out))
    if st:
        raise OracleError(st, "port run_serial failed")
    return out


def port_run_state(equation, method, ic: np.ndarray, steps: int, dt_dx: float, fourier=0.4, gamma=1.4) -> np.ndarray:
    """serial_advance from a given periodic state (s1o_run_state)."""
    ic = np.ascontiguousarray(ic, dtype=np.float64)
    n = ic.size // vpp(equation)
    out = np.empty_like(ic)
    st = port().s1o_run_state(0 if equation == "heat" else 1, 0 if method == "lengthening" else 1, n, steps, fourier,
                              gamma, dt_dx, _ptr(ic), _ptr(out))
    if st:
        raise OracleError(st, "port run_state failed")
    return out


def port_initial_condition(initial: str, n: int, equation="heat", gamma=1.4) -> np.ndarray:
    out = np.empty(n * vpp(equation), dtype=np.float64)
    st = port().s1o_initial_condition(initial.encode(), n, 0 if equation == "heat" else 1, gamma, _ptr(out))
    if st:
        raise OracleError(st, "port initial_condition failed")
    return out


def fnv1a64(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return "%016x" % port().s1o_fnv1a64(_ptr(a), a.size)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


# --------------------------------------------------------------------------
# ref (the reference compiled from source)
# --------------------------------------------------------------------------
class RefCfg(C.Structure):
    _fields_ = [("equation", C.c_int), ("method", C.c_int), ("scheme", C.c_int), ("mode", C.c_int),
                ("grid_size", C.c_ulonglong), ("block_width", C.c_ulonglong), ("ranks", C.c_int),
                ("work_factor", C.c_int), ("steps", C.c_longlong), ("fourier", C.c_double),
                ("gamma", C.c_double), ("dt_dx", C.c_double), ("cfl", C.c_double), ("alpha", C.c_double),
                ("beta", C.c_double), ("compute_cost", C.c_double), ("initial", C.c_char * 64)]


class RefStats(C.Structure):
    _fields_ = [("messages_sent", C.c_ulonglong), ("bytes_sent", C.c_ulonglong),
                ("exchange_rounds", C.c_ulonglong), ("setup_seconds", C.c_double),
                ("loop_seconds", C.c_double), ("virtual_seconds", C.c_double),
                ("virtual_comm_time", C.c_double)]


class RefMsg(C.Structure):
    _fields_ = [("round", C.c_ulonglong), ("source", C.c_int), ("dest", C.c_int), ("tag", C.c_ulonglong),
                ("bytes", C.c_ulonglong)]


_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(os.path.join(REF_ROOT, "core", "src"))


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build(ref=True)
        lib = C.CDLL(REF_SO)
        E = [C.c_char_p, C.c_size_t]
        lib.ref_defaults.argtypes = [C.POINTER(RefCfg)]
        lib.ref_run_serial.argtypes = [C.POINTER(RefCfg), _dp, C.c_size_t] + E
        lib.ref_run.argtypes = [C.POINTER(RefCfg), _dp, C.c_size_t, C.POINTER(RefStats), C.POINTER(RefMsg),
                                C.c_size_t, C.POINTER(C.c_size_t)] + E
        lib.ref_finalize.argtypes = [C.POINTER(RefCfg), C.c_int] + E
        lib.ref_partition.argtypes = [C.POINTER(RefCfg), C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong),
                                      C.POINTER(C.c_int), C.POINTER(C.c_int)] + E
        lib.ref_working_array_extents.argtypes = [C.c_ulonglong, C.c_ulonglong, C.c_int, C.c_int,
                                                  C.POINTER(C.c_ulonglong)] + E
        lib.ref_swept_buffer_cells.restype = C.c_ulonglong
        lib.ref_swept_buffer_cells.argtypes = [C.c_ulonglong, C.c_int, C.c_int]
        lib.ref_initial_condition.argtypes = [C.c_char_p, C.c_ulonglong, C.c_int, C.c_int, C.c_double, _dp,
                                              C.c_size_t] + E
        lib.ref_max_signal_speed.argtypes = [_dp, C.c_size_t, C.c_double, _dp] + E
        lib.ref_schedule.restype = C.c_long
        lib.ref_schedule.argtypes = [C.c_int, C.c_ulonglong, C.c_ulonglong, C.POINTER(C.c_long),
                                     C.POINTER(C.c_long), C.POINTER(C.c_long), C.c_size_t] + E
        lib.ref_cycle_advance.restype = C.c_long
        lib.ref_cycle_advance.argtypes = [C.c_ulonglong, C.c_ulonglong] + E
        lib.ref_heat_step.restype = C.c_double
        lib.ref_heat_step.argtypes = [C.c_double] * 4
        lib.ref_minmod.restype = C.c_double
        lib.ref_minmod.argtypes = [C.c_double] * 2
        lib.ref_pressure_ratio_value.restype = C.c_double
        lib.ref_pressure_ratio_value.argtypes = [C.c_double] * 3
        lib.ref_pressure.argtypes = [_dp, C.c_double, _dp] + E
        lib.ref_interface_flux.argtypes = [_dp, _dp, C.c_double, C.c_double, C.c_double, _dp] + E
        lib.ref_model_apply.argtypes = [C.c_int, _dp, C.c_long, C.c_long, C.c_long, C.c_double, C.c_double,
                                        C.c_double] + E
        _ref = lib
    return _ref


_EQ = {"heat": 0, "euler": 1}
_ME = {"lengthening": 0, "flattening": 1}
_SC = {"classic": 0, "swept": 1}
_MO = {"wall": 0, "virtual": 1}


@dataclass
class RefConfig:
    """Mirror of sweep1d::LaunchConfig (inc/config.hpp:12-41) for the shim."""
    equation: str = "heat"
    method: str = "lengthening"
    scheme: str = "swept"
    grid_size: int = 1024
    block_width: int = 32
    ranks: int = 2
    work_factor: int = 0
    steps: int = 50
    initial: str = ""
    mode: str = "virtual"
    fourier: float = 0.4
    gamma: float = 1.4
    dt_dx: float = 0.0
    cfl: float = 0.4
    alpha: float = 0.0
    beta: float = 0.0
    compute_cost: float = 1e-8

    def to_c(self) -> RefCfg:
        c = RefCfg()
        c.equation = _EQ[self.equation]
        c.method = _ME[self.method]
        c.scheme = _SC[self.scheme]
        c.mode = _MO[self.mode]
        c.grid_size = self.grid_size
        c.block_width = self.block_width
        c.ranks = self.ranks
        c.work_factor = self.work_factor
        c.steps = self.steps
        c.fourier, c.gamma, c.dt_dx, c.cfl = self.fourier, self.gamma, self.dt_dx, self.cfl
        c.alpha, c.beta, c.compute_cost = self.alpha, self.beta, self.compute_cost
        c.initial = self.initial.encode()
        return c


@dataclass
class RefResult:
    state: np.ndarray
    messages_sent: int = 0
    bytes_sent: int = 0
    exchange_rounds: int = 0
    setup_seconds: float = 0.0
    loop_seconds: float = 0.0
    virtual_seconds: float = 0.0
    virtual_comm_time: float = 0.0
    log: list = field(default_factory=list)


def _err():
    return C.create_string_buffer(512)


def ref_run_serial(cfg: RefConfig) -> np.ndarray:
    out = np.empty(cfg.grid_size * vpp(cfg.equation), dtype=np.float64)
    e = _err()
    st = ref().ref_run_serial(C.byref(cfg.to_c()), _ptr(out), out.size, e, 512)
    if st:
        raise OracleError(st, e.value.decode())
    return out


def ref_run(cfg: RefConfig, keep_log: bool = False) -> RefResult:
    out = np.empty(cfg.grid_size * vpp(cfg.equation), dtype=np.float64)
    st_ = RefStats()
    e = _err()
    cap = 0
    logbuf = None
    nlog = C.c_size_t(0)
    if keep_log:
        cap = 1 << 16
        logbuf = (RefMsg * cap)()
    st = ref().ref_run(C.byref(cfg.to_c()), _ptr(out), out.size, C.byref(st_), logbuf, cap, C.byref(nlog), e, 512)
    if st:
        raise OracleError(st, e.value.decode())
    res = RefResult(out, st_.messages_sent, st_.bytes_sent, st_.exchange_rounds, st_.setup_seconds,
                    st_.loop_seconds, st_.virtual_seconds, st_.virtual_comm_time)
    if keep_log:
        res.log = [(m.round, m.source, m.dest, m.tag, m.bytes) for m in logbuf[: min(nlog.value, cap)]]
    return res


def ref_finalize(cfg: RefConfig, partitioned: bool = True) -> float:
    c = cfg.to_c()
    e = _err()
    st = ref().ref_finalize(C.byref(c), int(partitioned), e, 512)
    if st:
        raise OracleError(st, e.value.decode())
    return c.dt_dx


def ref_initial_condition(initial: str, n: int, equation="heat", method="lengthening", gamma=1.4) -> np.ndarray:
    out = np.empty(n * vpp(equation), dtype=np.float64)
    e = _err()
    st = ref().ref_initial_condition(initial.encode(), n, _EQ[equation], _ME[method], gamma, _ptr(out), out.size,
                                     e, 512)
    if st:
        raise OracleError(st, e.value.decode())
    return out


def ref_schedule(kind: str, w: int, h: int):
    k = {"triangle": 0, "diamond": 1, "down": 2}[kind]
    cap = 4096
    s, lo, hi = (C.c_long * cap)(), (C.c_long * cap)(), (C.c_long * cap)()
    e = _err()
    n = ref().ref_schedule(k, w, h, s, lo, hi, cap, e, 512)
    if n < 0:
        raise OracleError(-n, e.value.decode())
    return [(s[i], lo[i], hi[i]) for i in range(n)]


def ref_model_apply(model: int, cells: np.ndarray, i: int, counter: int, fourier=0.4, gamma=1.4, dt_dx=0.0):
    """Apply Model::apply in place on an AoS record array (2/7/6 doubles per record)."""
    width = {0: 2, 1: 7, 2: 6}[model]
    assert cells.dtype == np.float64 and cells.flags.c_contiguous
    e = _err()
    st = ref().ref_model_apply(model, _ptr(cells), cells.size // width, i, counter, fourier, gamma, dt_dx, e, 512)
    if st:
        raise OracleError(st, e.value.decode())
