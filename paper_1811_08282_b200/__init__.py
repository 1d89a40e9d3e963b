"""swept1d-b200: B200-native (sm_100a, FP64) swept time-space decomposition for
1-D explicit PDEs — a drop-in for the reference `sweep1d` engine path.

The product is the C-ABI library `_lib/libswept1d.so` (include/swept1d.h);
this package is its Python mirror of the reference interface (api.py).
"""
from .api import (  # noqa: F401
    ArrayExtents, CommStats, CudaError, DegenerateFit, EngineTiming, Equation, EquationSpec, InvalidConfig,
    InvalidWidth, LaunchConfig, Method, Mode, ModeMismatch, NoDevice, NonPhysicalState, Partition,
    PayloadSizeMismatch, PeerUnavailable, PhaseSchedule, PhaseSkew, PhysParams, RunResult, Scheme, Shard, Solver,
    SpanAtLevel, Sweep1dError, TagMismatch, TransportAborted, TransportParams, UnknownInitialCondition,
    apply_config_entry, apply_config_file, cycle_advance, device_count, diamond_schedule, down_triangle_schedule,
    initial_condition, initial_condition_range, make_partition, make_spec, max_signal_speed, measure_fp64_peak, run, swept_buffer_cells, to_string,
    triangle_schedule, version, working_array_extents)
from .api import (  # noqa: F401
    FitResult, TimingRecord, best_config, csv_header, csv_row, emit_csv, flattening_speedup, measure, power_law_fit,
    read_csv, speedup)
from .api import DebugResult, RunOptions, run_debug  # noqa: F401
from .api import calibrate_transport, virtual_time  # noqa: F401
from .api import MessageLogEntry, RankCommStats, message_log, rank_stats  # noqa: F401
from .api import wave_schedule  # noqa: F401
