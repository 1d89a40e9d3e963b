"""Python mirror of the reference `sweep1d` interface over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/core/include/sweep1d/):

    LaunchConfig, PhysParams, TransportParams   config.hpp:12-41, types.hpp:27-38
    Equation / Method / Scheme / Mode            types.hpp:8-11
    EquationSpec, make_spec                      types.hpp:15-25, kernels.cpp:7-25
    run(cfg) -> RunResult                        engine.hpp:28 (the drop-in)
    initial_condition, max_signal_speed          partition.hpp:37-47
    make_partition, working_array_extents,
    swept_buffer_cells                           partition.hpp:13-35
    cycle_advance, triangle/diamond/down_triangle_schedule  swept.hpp:27-41
    apply_config_entry / apply_config_file       config.hpp:43-46
    InvalidConfig ... TransportAborted           errors.hpp:8-47

Every compute call goes through libswept1d.so (CUDA, sm_100a); there is no CPU
fallback. Host-only helpers (validation, IC, schedules) also live in the
library so the GPU path and these checks share one implementation.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _capi
from ._capi import lib


# ---------------------------------------------------------------------------
# errors (errors.hpp:8-47)
# ---------------------------------------------------------------------------
class Sweep1dError(RuntimeError):
    status = 99


class InvalidConfig(Sweep1dError):
    status = 1


class UnknownInitialCondition(Sweep1dError):
    status = 2


class NonPhysicalState(Sweep1dError):
    status = 3


class InvalidWidth(Sweep1dError):
    status = 4


class PayloadSizeMismatch(Sweep1dError):
    status = 5


class TagMismatch(Sweep1dError):
    status = 6


class PhaseSkew(Sweep1dError):
    status = 7


class ModeMismatch(Sweep1dError):
    status = 8


class DegenerateFit(Sweep1dError):
    status = 9


class TransportAborted(Sweep1dError):
    status = 10


class CudaError(Sweep1dError):
    status = 20


class PeerUnavailable(Sweep1dError):
    status = 21


class NoDevice(Sweep1dError):
    status = 22


_BY_STATUS = {c.status: c for c in (InvalidConfig, UnknownInitialCondition, NonPhysicalState, InvalidWidth,
                                    PayloadSizeMismatch, TagMismatch, PhaseSkew, ModeMismatch, DegenerateFit,
                                    TransportAborted, CudaError, PeerUnavailable, NoDevice)}


def _raise(status: int, msg: str):
    if status == 0:
        return
    raise _BY_STATUS.get(status, Sweep1dError)(msg)


def _errbuf():
    return C.create_string_buffer(1024)


def _check(status: int, buf) -> None:
    if status:
        _raise(status, buf.value.decode(errors="replace"))


# ---------------------------------------------------------------------------
# enums and config (types.hpp, config.hpp)
# ---------------------------------------------------------------------------
class Equation(enum.IntEnum):
    Heat = 0
    Euler = 1


class Method(enum.IntEnum):
    Lengthening = 0
    Flattening = 1


class Scheme(enum.IntEnum):
    Classic = 0
    Swept = 1


class Mode(enum.IntEnum):
    WallClock = 0
    VirtualTime = 1


def to_string(v) -> str:
    names = {Equation: ("heat", "euler"), Method: ("lengthening", "flattening"), Scheme: ("classic", "swept"),
             Mode: ("wall", "virtual")}
    return names[type(v)][int(v)]


@dataclass
class EquationSpec:
    equation: Equation = Equation.Heat
    method: Method = Method.Lengthening
    substeps_per_step: int = 1
    stencil_half_width: int = 1
    state_slots: int = 2
    values_per_point: int = 1


def make_spec(eq: Equation, method: Method) -> EquationSpec:
    S, h, slots, vpp = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    lib().s1d_spec(int(eq), int(method), C.byref(S), C.byref(h), C.byref(slots), C.byref(vpp))
    return EquationSpec(Equation(eq), Method(method), S.value, h.value, slots.value, vpp.value)


@dataclass
class PhysParams:
    fourier: float = 0.4
    gamma: float = 1.4
    dt_dx: float = 0.0
    cfl: float = 0.4


@dataclass
class TransportParams:
    alpha: float = 0.0
    beta: float = 0.0
    compute_cost: float = 1e-8


@dataclass
class LaunchConfig:
    equation: Equation = Equation.Heat
    method: Method = Method.Lengthening
    scheme: Scheme = Scheme.Swept
    grid_size: int = 1024
    block_width: int = 32
    ranks: int = 2
    work_factor: int = 0
    steps: int = 50
    initial: str = ""
    mode: Mode = Mode.VirtualTime
    phys: PhysParams = field(default_factory=PhysParams)
    transport: TransportParams = field(default_factory=TransportParams)
    num_devices: int = 0  # B200 extension: 0 = all visible devices

    def spec(self) -> EquationSpec:
        return make_spec(self.equation, self.method)

    def initial_or_default(self) -> str:
        if self.initial:
            return self.initial
        return "heat-sine" if self.equation == Equation.Heat else "euler-sod-periodic"

    def shares(self) -> int:
        return self.ranks - 1 + self.work_factor if self.work_factor > 0 else self.ranks

    def to_c(self) -> _capi.s1d_config:
        c = _capi.s1d_config()
        lib().s1d_config_defaults(C.byref(c))
        c.equation, c.method, c.scheme, c.mode = int(self.equation), int(self.method), int(self.scheme), int(
            self.mode)
        c.grid_size, c.block_width, c.ranks, c.work_factor = self.grid_size, self.block_width, self.ranks, \
            self.work_factor
        c.steps = self.steps
        c.fourier, c.gamma, c.dt_dx, c.cfl = self.phys.fourier, self.phys.gamma, self.phys.dt_dx, self.phys.cfl
        c.alpha, c.beta, c.compute_cost = self.transport.alpha, self.transport.beta, self.transport.compute_cost
        enc = self.initial.encode()
        if len(enc) >= 64:
            raise InvalidConfig("initial condition id too long")
        c.initial = enc
        c.num_devices = self.num_devices
        return c

    @staticmethod
    def from_c(c: _capi.s1d_config) -> "LaunchConfig":
        return LaunchConfig(Equation(c.equation), Method(c.method), Scheme(c.scheme), c.grid_size, c.block_width,
                            c.ranks, c.work_factor, c.steps, c.initial.decode(), Mode(c.mode),
                            PhysParams(c.fourier, c.gamma, c.dt_dx, c.cfl),
                            TransportParams(c.alpha, c.beta, c.compute_cost), c.num_devices)

    def validate(self, partitioned: bool = True) -> None:
        e = _errbuf()
        _check(lib().s1d_validate(C.byref(self.to_c()), int(partitioned), e, 1024), e)

    def finalize(self, partitioned: bool = True) -> None:
        c = self.to_c()
        e = _errbuf()
        _check(lib().s1d_finalize(C.byref(c), int(partitioned), e, 1024), e)
        self.phys.dt_dx = c.dt_dx


def apply_config_entry(cfg: LaunchConfig, key: str, value: str) -> None:
    c = cfg.to_c()
    e = _errbuf()
    _check(lib().s1d_apply_config_entry(C.byref(c), key.encode(), value.encode(), e, 1024), e)
    new = LaunchConfig.from_c(c)
    cfg.__dict__.update(new.__dict__)


def apply_config_file(cfg: LaunchConfig, path: str) -> None:
    """key=value lines, # comments (config.cpp:126-148)."""
    try:
        fh = open(path)
    except OSError:
        raise InvalidConfig(f"cannot open config file '{path}'")
    with fh:
        for lineno, line in enumerate(fh, 1):
            line = line.split("#", 1)[0]
            trimmed = "".join(ch for ch in line if not ch.isspace())
            if not trimmed:
                continue
            if "=" not in trimmed:
                raise InvalidConfig(f"{path}:{lineno}: expected key=value")
            k, v = trimmed.split("=", 1)
            apply_config_entry(cfg, k, v)


# ---------------------------------------------------------------------------
# geometry / IC (partition.hpp, swept.hpp)
# ---------------------------------------------------------------------------
@dataclass
class Partition:
    block_width: int
    blocks: List[int]
    start_index: List[int]
    left: List[int]
    right: List[int]

    def ranks(self) -> int:
        return len(self.blocks)

    def owned_points(self, rank: int) -> int:
        return self.blocks[rank] * self.block_width


def make_partition(cfg: LaunchConfig) -> Partition:
    r = max(cfg.ranks, 1)
    b, s = (C.c_uint64 * r)(), (C.c_uint64 * r)()
    lft, rgt = (C.c_int * r)(), (C.c_int * r)()
    e = _errbuf()
    _check(lib().s1d_partition(C.byref(cfg.to_c()), b, s, lft, rgt, e, 1024), e)
    return Partition(cfg.block_width, list(b), list(s), list(lft), list(rgt))


@dataclass
class ArrayExtents:
    length: int
    initialized: int
    ghost: int


def working_array_extents(n_blocks: int, w: int, spec: EquationSpec) -> ArrayExtents:
    """Reference per-rank working array sizing (partition.cpp:37-44). The B200
    layout does not use it (global state + edge buffers); kept for API parity."""
    if w < 4 or (w & 1):
        raise InvalidConfig("working array requires even block width >= 4")
    h = spec.stencil_half_width
    owned = n_blocks * w
    return ArrayExtents(owned + w // 2 + 2 * h, owned + 2 * h, h)


def swept_buffer_cells(w: int, spec: EquationSpec) -> int:
    return int(lib().s1d_swept_buffer_cells(w, int(spec.equation), int(spec.method)))


def initial_condition(ident: str, n: int, spec: EquationSpec, gamma: float = 1.4) -> np.ndarray:
    out = np.empty(n * (1 if spec.equation == Equation.Heat else 3), dtype=np.float64)
    e = _errbuf()
    _check(lib().s1d_initial_condition(ident.encode(), n, int(spec.equation), gamma,
                                       out.ctypes.data_as(C.POINTER(C.c_double)), out.size, e, 1024), e)
    return out


def initial_condition_range(ident: str, n: int, spec: EquationSpec, start: int, count: int,
                            gamma: float = 1.4, out: Optional[np.ndarray] = None) -> np.ndarray:
    """Points [start, start+count) of initial_condition(ident, n, ...)."""
    vpp = 1 if spec.equation == Equation.Heat else 3
    out = _out_buffer(out, count * vpp)
    e = _errbuf()
    _check(lib().s1d_initial_condition_range(ident.encode(), n, int(spec.equation), gamma, start, count,
                                             out.ctypes.data_as(C.POINTER(C.c_double)), out.size, e, 1024), e)
    return out


def max_signal_speed(primaries: np.ndarray, gamma: float) -> float:
    a = np.ascontiguousarray(primaries, dtype=np.float64)
    out = C.c_double()
    e = _errbuf()
    _check(lib().s1d_max_signal_speed(a.ctypes.data_as(C.POINTER(C.c_double)), a.size, gamma, C.byref(out), e,
                                      1024), e)
    return out.value


def cycle_advance(w: int, h: int) -> int:
    e = _errbuf()
    m = lib().s1d_cycle_advance(w, h, e, 1024)
    if m < 0:
        _raise(-m, e.value.decode())
    return m


@dataclass
class SpanAtLevel:
    substep: int
    lo: int
    hi: int

    def width(self) -> int:
        return self.hi - self.lo


@dataclass
class PhaseSchedule:
    levels: List[SpanAtLevel]

    def substeps(self) -> int:
        return self.levels[-1].substep if self.levels else 0


def _schedule(kind: int, w: int, h: int) -> PhaseSchedule:
    cap = max(2 * w + 4, 8)
    s, lo, hi = (C.c_int64 * cap)(), (C.c_int64 * cap)(), (C.c_int64 * cap)()
    e = _errbuf()
    n = lib().s1d_schedule(kind, w, h, s, lo, hi, cap, e, 1024)
    if n < 0:
        _raise(-n, e.value.decode())
    return PhaseSchedule([SpanAtLevel(s[i], lo[i], hi[i]) for i in range(n)])


def triangle_schedule(w: int, h: int) -> PhaseSchedule:
    return _schedule(0, w, h)


def diamond_schedule(w: int, h: int) -> PhaseSchedule:
    return _schedule(1, w, h)


def down_triangle_schedule(w: int, h: int) -> PhaseSchedule:
    return _schedule(2, w, h)


# ---------------------------------------------------------------------------
# run (engine.hpp:12-28)
# ---------------------------------------------------------------------------
@dataclass
class RankCommStats:
    """RankCommStats (inc/transport.hpp:17-25)."""
    messages_sent: int = 0
    bytes_sent: int = 0
    exchange_rounds: int = 0
    virtual_comm_time: float = 0.0


@dataclass
class MessageLogEntry:
    """MessageLogEntry (inc/transport.hpp:36-42)."""
    round: int
    source: int
    dest: int
    tag: int
    bytes: int


@dataclass
class CommStats:
    messages_sent: int = 0
    bytes_sent: int = 0
    exchange_rounds: int = 0
    kernel_launches: int = 0
    edge_bytes_device: int = 0
    setup_seconds: float = 0.0
    virtual_comm_time: float = 0.0  # CommStats::virtual_comm_time (transport.hpp:20-30)
    per_rank: list = field(default_factory=list)  # [RankCommStats] (transport.cpp:190-196)


@dataclass
class EngineTiming:
    setup_seconds: float = 0.0
    loop_seconds: float = 0.0
    virtual_seconds: float = 0.0
    h2d_seconds: float = 0.0
    d2h_seconds: float = 0.0
    dominant_seconds: float = 0.0
    dominant_launches: int = 0
    dominant_point_updates: int = 0
    dominant_kernel: str = ""


@dataclass
class RunResult:
    state: np.ndarray
    stats: CommStats
    timing: EngineTiming
    log: list = field(default_factory=list)


def _stats(s: _capi.s1d_stats, setup: float = 0.0) -> CommStats:
    return CommStats(s.messages_sent, s.bytes_sent, s.exchange_rounds, s.kernel_launches, s.edge_bytes_device,
                     setup, s.virtual_comm_seconds)


def _timing(t: _capi.s1d_timing) -> EngineTiming:
    return EngineTiming(t.setup_seconds, t.loop_seconds, t.virtual_seconds, t.h2d_seconds, t.d2h_seconds,
                        t.dominant_seconds, t.dominant_launches, t.dominant_point_updates,
                        t.dominant_kernel.decode())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _out_buffer(out: Optional[np.ndarray], n: int) -> np.ndarray:
    """A caller-supplied output array is written through its raw pointer by the
    library, so it must be exactly what the C ABI assumes: float64,
    C-contiguous, writeable, at least n elements."""
    if out is None:
        return np.empty(n, dtype=np.float64)
    if not isinstance(out, np.ndarray):
        raise TypeError("out must be a numpy.ndarray")
    if out.dtype != np.float64:
        raise TypeError(f"out must be float64, got {out.dtype}")
    if not out.flags.c_contiguous:
        raise ValueError("out must be C-contiguous")
    if not out.flags.writeable:
        raise ValueError("out must be writeable")
    if out.size < n:
        raise ValueError(f"out holds {out.size} values, {n} needed")
    return out


def run(cfg: LaunchConfig, opts: Optional["RunOptions"] = None) -> RunResult:
    """The drop-in for sweep1d::run(cfg, opts) (src/engine.cpp:40-47) on B200
    GPUs. stats.per_rank and (opts.keep_message_log) the log are the
    reference transport's, replayed on the host (rank_stats, message_log)."""
    if opts is not None and (opts.coverage or opts.perturb_ulp):
        res = run_debug(cfg, opts).result
    else:
        spec = cfg.spec()
        out = np.empty(cfg.grid_size * spec.values_per_point, dtype=np.float64)
        st, tm = _capi.s1d_stats(), _capi.s1d_timing()
        e = _errbuf()
        _check(lib().s1d_run(C.byref(cfg.to_c()), _dptr(out), out.size, C.byref(st), C.byref(tm), e, 1024), e)
        res = RunResult(out, _stats(st, tm.setup_seconds), _timing(tm))
    res.stats.per_rank = rank_stats(cfg)
    if opts is not None and opts.keep_message_log:
        res.log = message_log(cfg)
    return res


def rank_stats(cfg: LaunchConfig) -> list:
    """CommStats::per_rank for cfg (transport.cpp:190-196), host-only."""
    arr = (_capi.s1d_rank_stats * max(cfg.ranks, 1))()
    e = _errbuf()
    _check(lib().s1d_comm_per_rank(C.byref(cfg.to_c()), arr, len(arr), e, 1024), e)
    return [RankCommStats(a.messages_sent, a.bytes_sent, a.exchange_rounds, a.virtual_comm_seconds) for a in arr]


def message_log(cfg: LaunchConfig) -> list:
    """The reference transport's sorted message log for cfg
    (RunOptions::keep_message_log; transport.cpp:66-110, 197-206), host-only."""
    n = C.c_size_t(0)
    e = _errbuf()
    _check(lib().s1d_message_log(C.byref(cfg.to_c()), None, 0, C.byref(n), e, 1024), e)
    arr = (_capi.s1d_message * max(n.value, 1))()
    _check(lib().s1d_message_log(C.byref(cfg.to_c()), arr, n.value, C.byref(n), e, 1024), e)
    return [MessageLogEntry(m.round, m.source, m.dest, m.tag, m.bytes) for m in arr[:n.value]]


def wave_schedule(chunks: int, head: int, tail: int, cycles: int, multi_process: bool = False) -> list:
    """Issue order of the wavefront solve (test hook, host-only):
    tuples (kind, phase, chunk), kind "chunk" / "signal" / "middle"."""
    n = C.c_size_t(0)
    e = _errbuf()
    _check(lib().s1d_debug_wave_schedule(chunks, head, tail, cycles, int(multi_process), None, 0, C.byref(n), e,
                                         1024), e)
    buf = (C.c_int64 * (3 * max(n.value, 1)))()
    _check(lib().s1d_debug_wave_schedule(chunks, head, tail, cycles, int(multi_process), buf, n.value, C.byref(n), e,
                                         1024), e)
    kinds = ("chunk", "signal", "middle")
    return [(kinds[buf[3 * i]], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n.value)]


@dataclass
class RunOptions:
    """sweep1d::RunOptions subset (inc/debug.hpp:17-24)."""
    keep_message_log: bool = False
    coverage: bool = False
    perturb_ulp: bool = False


@dataclass
class DebugResult:
    result: RunResult
    coverage: Optional[np.ndarray]  # [steps*S, n] counts, or None

    def defects(self):
        """(substep, point) pairs not computed exactly once (CoverageCounter::defects)."""
        if self.coverage is None:
            return []
        bad = np.argwhere(self.coverage != 1)
        return [(int(lv) + 1, int(x), int(self.coverage[lv, x])) for lv, x in bad[:100]]


def run_debug(cfg: LaunchConfig, opts: RunOptions) -> DebugResult:
    """s1d_run with the instrumented kernels (tiling coverage counter, 1-ulp
    mutation hook)."""
    spec = cfg.spec()
    out = np.empty(cfg.grid_size * spec.values_per_point, dtype=np.float64)
    total = cfg.steps * spec.substeps_per_step
    cov = np.zeros((total, cfg.grid_size), dtype=np.uint32) if opts.coverage else None
    d = _capi.s1d_debug()
    d.coverage = int(opts.coverage)
    d.perturb_ulp = int(opts.perturb_ulp)
    if cov is not None:
        d.coverage_out = cov.ctypes.data_as(C.POINTER(C.c_uint32))
        d.coverage_len = cov.size
    st, tm = _capi.s1d_stats(), _capi.s1d_timing()
    e = _errbuf()
    _check(lib().s1d_run_debug(C.byref(cfg.to_c()), C.byref(d), _dptr(out), out.size, C.byref(st), C.byref(tm), e,
                               1024), e)
    return DebugResult(RunResult(out, _stats(st, tm.setup_seconds), _timing(tm)), cov)


class Solver:
    """Reusable device-resident solver (s1d_create/s1d_solve/...)."""

    def __init__(self, cfg: LaunchConfig):
        self._h = C.c_void_p()
        e = _errbuf()
        _check(lib().s1d_create(C.byref(cfg.to_c()), C.byref(self._h), e, 1024), e)
        self._post_init()

    def _post_init(self):
        c = _capi.s1d_config()
        lib().s1d_get_config(self._h, C.byref(c))
        self.cfg = LaunchConfig.from_c(c)
        self.spec = self.cfg.spec()
        start, count = C.c_uint64(), C.c_uint64()
        lib().s1d_shard_range(self._h, C.byref(start), C.byref(count))
        self.start, self.count = start.value, count.value
        self.state_len = self.count * self.spec.values_per_point

    def _chk(self, status: int):
        if status:
            _raise(status, lib().s1d_last_error(self._h).decode(errors="replace"))

    def close(self):
        if self._h:
            lib().s1d_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_initial(self, state: Optional[np.ndarray] = None) -> None:
        if state is None:
            self._chk(lib().s1d_set_initial(self._h, None, 0))
        else:
            a = np.ascontiguousarray(state, dtype=np.float64)
            self._chk(lib().s1d_set_initial(self._h, _dptr(a), a.size))

    def advance(self):
        st, tm = _capi.s1d_stats(), _capi.s1d_timing()
        self._chk(lib().s1d_advance(self._h, C.byref(st), C.byref(tm)))
        return _stats(st), _timing(tm)

    def read_state(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        out = _out_buffer(out, self.state_len)
        self._chk(lib().s1d_read_state(self._h, _dptr(out), out.size))
        return out

    def solve_ptr(self, in_ptr: int, in_len: int, out_ptr: int, out_len: int):
        """End to end through caller-owned host buffers (raw addresses, e.g. pinned)."""
        st, tm = _capi.s1d_stats(), _capi.s1d_timing()
        self._chk(lib().s1d_solve(self._h, C.cast(in_ptr, C.POINTER(C.c_double)) if in_ptr else None, in_len,
                                  C.cast(out_ptr, C.POINTER(C.c_double)), out_len, C.byref(st), C.byref(tm)))
        return _stats(st), _timing(tm)

    def solve(self, state_in: Optional[np.ndarray] = None, out: Optional[np.ndarray] = None):
        out = _out_buffer(out, self.state_len)
        st, tm = _capi.s1d_stats(), _capi.s1d_timing()
        if state_in is not None:
            a = np.ascontiguousarray(state_in, dtype=np.float64)
            status = lib().s1d_solve(self._h, _dptr(a), a.size, _dptr(out), out.size, C.byref(st), C.byref(tm))
        else:
            status = lib().s1d_solve(self._h, None, 0, _dptr(out), out.size, C.byref(st), C.byref(tm))
        self._chk(status)
        return out, _stats(st), _timing(tm)


class Shard(Solver):
    """One shard of the ring owned by this process (one process per GPU).

    Usage (e.g. under torchrun):
        sh = Shard(cfg, rank, device)
        blobs = all_gather(sh.export())            # any transport
        sh.connect(blobs[left], blobs[right])
        sh.advance()                               # lockstep with the neighbours
    Host I/O covers the local slice [sh.start, sh.start + sh.count)."""

    def __init__(self, cfg: LaunchConfig, rank: int, device: int):
        self._h = C.c_void_p()
        e = _errbuf()
        _check(lib().s1d_shard_create(C.byref(cfg.to_c()), rank, device, C.byref(self._h), e, 1024), e)
        self.rank = rank
        self._post_init()

    def export(self) -> bytes:
        n = lib().s1d_shard_blob_size()
        buf = C.create_string_buffer(n)
        self._chk(lib().s1d_shard_export(self._h, buf, n))
        return buf.raw

    def connect(self, left_blob: bytes, right_blob: bytes) -> None:
        self._chk(lib().s1d_shard_connect(self._h, left_blob, right_blob))


def virtual_time(cfg: LaunchConfig) -> Tuple[float, float]:
    """The reference's alpha-beta virtual clock for `cfg` (host replay, no GPU):
    (virtual_seconds, virtual_comm_seconds) — what sweep1d::run reports in
    VirtualTime mode (engines_impl.hpp:413) and CommStats::virtual_comm_time."""
    v, c = C.c_double(), C.c_double()
    e = _errbuf()
    _check(lib().s1d_virtual_time(C.byref(cfg.to_c()), C.byref(v), C.byref(c), e, 1024), e)
    return v.value, c.value


def calibrate_transport(dev_a: int = 0, dev_b: int = 1, compute_cost: float = 1e-8) -> TransportParams:
    """Measured NVLink alpha (one-way device flag hand-off latency, s) and beta
    (s/byte of a large peer copy) between two devices, as TransportParams."""
    a, b = C.c_double(), C.c_double()
    e = _errbuf()
    _check(lib().s1d_calibrate_transport(dev_a, dev_b, C.byref(a), C.byref(b), e, 1024), e)
    return TransportParams(a.value, b.value, compute_cost)


def measure_fp64_peak(device: int = 0) -> float:
    """Sustained FP64 DADD/DMUL instruction rate (ops/s) of one device."""
    out = C.c_double()
    e = _errbuf()
    _check(lib().s1d_measure_fp64_peak(device, C.byref(out), e, 1024), e)
    return out.value


def device_count() -> int:
    return int(lib().s1d_device_count())


def version() -> str:
    return lib().s1d_version().decode()


# ---------------------------------------------------------------------------
# measurement records, CSV, fits (inc/perf.hpp, inc/csv.hpp)
# ---------------------------------------------------------------------------
@dataclass
class TimingRecord:
    """sweep1d::TimingRecord (inc/perf.hpp:16-29)."""
    equation: Equation = Equation.Heat
    method: Method = Method.Lengthening
    scheme: Scheme = Scheme.Classic
    grid_size: int = 0
    block_width: int = 0
    work_factor: int = 0
    ranks: int = 0
    steps: int = 0
    mode: Mode = Mode.VirtualTime
    avg_us_per_step: float = 0.0
    setup_us: float = 0.0
    messages_sent: int = 0
    bytes_sent: int = 0
    exchange_rounds: int = 0
    virtual_comm_us: float = 0.0

    def to_c(self) -> _capi.s1d_record:
        r = _capi.s1d_record()
        r.equation, r.method, r.scheme, r.mode = int(self.equation), int(self.method), int(self.scheme), int(
            self.mode)
        r.grid_size, r.block_width, r.work_factor, r.ranks, r.steps = (self.grid_size, self.block_width,
                                                                       self.work_factor, self.ranks, self.steps)
        r.avg_us_per_step, r.setup_us = self.avg_us_per_step, self.setup_us
        r.messages_sent, r.bytes_sent, r.exchange_rounds = self.messages_sent, self.bytes_sent, self.exchange_rounds
        r.virtual_comm_us = self.virtual_comm_us
        return r

    @staticmethod
    def from_c(r: _capi.s1d_record) -> "TimingRecord":
        return TimingRecord(Equation(r.equation), Method(r.method), Scheme(r.scheme), r.grid_size, r.block_width,
                            r.work_factor, r.ranks, r.steps, Mode(r.mode), r.avg_us_per_step, r.setup_us,
                            r.messages_sent, r.bytes_sent, r.exchange_rounds, r.virtual_comm_us)


@dataclass
class FitResult:
    A: float
    b: float
    r_squared: float


def measure(cfg: LaunchConfig) -> TimingRecord:
    """sweep1d::measure (src/perf.cpp:29-32) on the B200."""
    rec = _capi.s1d_record()
    e = _errbuf()
    _check(lib().s1d_measure(C.byref(cfg.to_c()), C.byref(rec), e, 1024), e)
    return TimingRecord.from_c(rec)


CSV_HEADER = None


def csv_header() -> str:
    return lib().s1d_csv_header().decode()


def csv_row(rec: TimingRecord) -> str:
    buf = C.create_string_buffer(1024)
    n = lib().s1d_csv_row(C.byref(rec.to_c()), buf, 1024)
    if n < 0:
        raise Sweep1dError("csv row too long")
    return buf.value.decode()


def emit_csv(records: List[TimingRecord], path: str) -> None:
    arr = (_capi.s1d_record * max(len(records), 1))(*[r.to_c() for r in records])
    e = _errbuf()
    _check(lib().s1d_emit_csv(arr, len(records), path.encode(), e, 1024), e)


def read_csv(path: str) -> List[TimingRecord]:
    n = C.c_size_t(0)
    e = _errbuf()
    _check(lib().s1d_read_csv(path.encode(), None, 0, C.byref(n), e, 1024), e)
    arr = (_capi.s1d_record * max(n.value, 1))()
    _check(lib().s1d_read_csv(path.encode(), arr, n.value, C.byref(n), e, 1024), e)
    return [TimingRecord.from_c(arr[i]) for i in range(n.value)]


def power_law_fit(points) -> FitResult:
    """Least-squares fit of log(time) vs log(n) (src/perf.cpp:42-82)."""
    xs = np.ascontiguousarray([p[0] for p in points], dtype=np.float64)
    ys = np.ascontiguousarray([p[1] for p in points], dtype=np.float64)
    A, b, r2 = C.c_double(), C.c_double(), C.c_double()
    e = _errbuf()
    _check(lib().s1d_power_law_fit(_dptr(xs), _dptr(ys), xs.size, C.byref(A), C.byref(b), C.byref(r2), e, 1024), e)
    return FitResult(A.value, b.value, r2.value)


def best_config(records: List[TimingRecord]) -> TimingRecord:
    """Fastest record; ties: smaller w, then smaller WF (src/perf.cpp:84-97)."""
    arr = (_capi.s1d_record * max(len(records), 1))(*[r.to_c() for r in records])
    i = lib().s1d_best_config(arr, len(records))
    if i < 0:
        _raise(-i, "best_config over an empty record set")
    return records[i]


def speedup(time_classic: float, time_swept: float) -> float:
    return time_classic / time_swept


def flattening_speedup(time_lengthening: float, time_flattening: float) -> float:
    return time_lengthening / time_flattening
