/*
 * swept1d.h — C ABI of the B200-native swept 1-D explicit-PDE solver.
 *
 * Drop-in boundary for the reference `sweep1d` engine entry points
 * (/root/reference/proj/core):
 *
 *   s1d_run            replaces  RunResult sweep1d::run(const LaunchConfig&, ...)
 *                                inc/engine.hpp:28, src/engine.cpp:40-47
 *   s1d_config         mirrors   sweep1d::LaunchConfig  inc/config.hpp:12-41
 *                                (+ PhysParams/TransportParams inc/types.hpp:27-38)
 *   s1d_config_defaults          LaunchConfig member initialisers inc/config.hpp:13-24
 *   s1d_validate       replaces  LaunchConfig::validate  src/config.cpp:45-95
 *   s1d_finalize       replaces  LaunchConfig::finalize  src/config.cpp:97-103
 *   s1d_apply_config_entry       apply_config_entry      src/config.cpp:105-124
 *   s1d_initial_condition        initial_condition       src/partition.cpp:67-102
 *   s1d_max_signal_speed         max_signal_speed        src/partition.cpp:104-113
 *   s1d_partition      replaces  make_partition          src/partition.cpp:10-35
 *   s1d_cycle_advance  replaces  cycle_advance           src/swept.cpp:23-26
 *   s1d_schedule       replaces  triangle/diamond/down_triangle_schedule
 *                                                        src/swept.cpp:28-64
 *   s1d_swept_buffer_cells       swept_buffer_cells      src/partition.cpp:46-48
 *   s1d_create/s1d_solve/...     (new) a reusable solver handle so repeated
 *                                timed runs do not re-allocate device memory.
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * Exceptions of the reference (inc/errors.hpp:8-47) become status codes with
 * a message written to a caller buffer. Functions marked [host] never touch a
 * GPU and work on machines without one.
 */
#ifndef SWEPT1D_H
#define SWEPT1D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S1D_ABI_VERSION 2

/* Status codes. 1..10 map one-to-one onto the reference exception types
 * (inc/errors.hpp:8-47); 20+ are device-side conditions. */
typedef enum s1d_status {
    S1D_OK = 0,
    S1D_INVALID_CONFIG = 1,        /* InvalidConfig */
    S1D_UNKNOWN_IC = 2,            /* UnknownInitialCondition */
    S1D_NONPHYSICAL = 3,           /* NonPhysicalState */
    S1D_INVALID_WIDTH = 4,         /* InvalidWidth */
    S1D_PAYLOAD_SIZE_MISMATCH = 5, /* PayloadSizeMismatch */
    S1D_TAG_MISMATCH = 6,          /* TagMismatch */
    S1D_PHASE_SKEW = 7,            /* PhaseSkew */
    S1D_MODE_MISMATCH = 8,         /* ModeMismatch */
    S1D_DEGENERATE_FIT = 9,        /* DegenerateFit */
    S1D_TRANSPORT_ABORTED = 10,    /* TransportAborted */
    S1D_CUDA_ERROR = 20,           /* a CUDA runtime call failed */
    S1D_PEER_UNAVAILABLE = 21,     /* ranks on distinct GPUs without P2P access */
    S1D_NO_DEVICE = 22,            /* no CUDA device visible */
    S1D_INTERNAL = 99
} s1d_status;

/* Enumerations: inc/types.hpp:8-11. */
enum { S1D_HEAT = 0, S1D_EULER = 1 };
enum { S1D_LENGTHENING = 0, S1D_FLATTENING = 1 };
enum { S1D_CLASSIC = 0, S1D_SWEPT = 1 };
enum { S1D_WALL = 0, S1D_VIRTUAL = 1 };

/* sweep1d::LaunchConfig. `ranks` is the number of shards of the periodic
 * ring; shard r runs on visible device (r % num_devices). The reference
 * requires ranks >= 2 (config.cpp:79-81); results are rank-invariant
 * (test_decomp.cpp:81-98), so ranks = 1 is accepted here. `mode` and the
 * transport cost parameters are accepted for drop-in compatibility; timing is
 * always measured (CUDA events) and never virtual. */
typedef struct s1d_config {
    int equation;           /* S1D_HEAT | S1D_EULER            (default heat) */
    int method;             /* S1D_LENGTHENING | S1D_FLATTENING (default lengthening) */
    int scheme;             /* S1D_CLASSIC | S1D_SWEPT          (default swept) */
    int mode;               /* S1D_WALL | S1D_VIRTUAL           (default virtual) */
    uint64_t grid_size;     /* n   (default 1024) */
    uint64_t block_width;   /* w   (default 32) */
    int ranks;              /* R   (default 2) */
    int work_factor;        /* WF  (default 0) */
    int64_t steps;          /* T   (default 50) */
    double fourier;         /* Fo  (default 0.4) */
    double gamma;           /*     (default 1.4) */
    double dt_dx;           /* 0 = derived from cfl at finalize (Euler) */
    double cfl;             /*     (default 0.4) */
    double alpha, beta, compute_cost; /* transport cost model (virtual mode, CommStats::virtual_comm_time) */
    char initial[64];       /* "" = per-equation default */
    int num_devices;        /* 0 = all visible devices */
    int reserved[7];
} s1d_config;

/* CommStats subset (inc/transport.hpp:27-34), counted by the host
 * orchestrator with the reference's formulas (transport.cpp:48-110) so the
 * round/message/byte tests apply unchanged. `edge_bytes_device` is what the
 * B200 path actually moved between shards (peer reads of triangle edges). */
typedef struct s1d_stats {
    uint64_t messages_sent;
    uint64_t bytes_sent;
    uint64_t exchange_rounds;
    uint64_t kernel_launches;   /* device kernels launched by the stepping loop */
    uint64_t edge_bytes_device; /* bytes read across shard boundaries */
    double virtual_comm_seconds; /* CommStats::virtual_comm_time: per-rank sum of
                                    alpha + beta*bytes over rounds (any mode) */
} s1d_stats;

/* RankCommStats (inc/transport.hpp:17-25): one rank's counters. */
typedef struct s1d_rank_stats {
    uint64_t messages_sent;
    uint64_t bytes_sent;
    uint64_t exchange_rounds;
    double virtual_comm_seconds;
} s1d_rank_stats;

/* MessageLogEntry (inc/transport.hpp:36-42): one message of the reference
 * transport's log (RunOptions::keep_message_log). */
typedef struct s1d_message {
    uint64_t round;
    int32_t source;
    int32_t dest;
    uint64_t tag;
    uint64_t bytes;
} s1d_message;

/* EngineTiming (inc/engine.hpp:12-16). loop_seconds = max over shards of the
 * CUDA-event time of the stepping loop (setup and host copies excluded);
 * h2d/d2h seconds are reported separately. */
typedef struct s1d_timing {
    double setup_seconds;
    double loop_seconds;
    double virtual_seconds; /* virtual mode: the reference's alpha-beta clock (s1d_virtual_time) */
    double h2d_seconds;
    double d2h_seconds;
    /* The dominant kernel of the run (swept: the Diamond phases; classic: the
     * per-substep kernel), timed with CUDA events on its own stream around the
     * contiguous run of those launches (max over shards). */
    double dominant_seconds;
    uint64_t dominant_launches;
    uint64_t dominant_point_updates; /* point-substeps those launches computed (all shards) */
    char dominant_kernel[32];
} s1d_timing;

/* ---- library ------------------------------------------------------------ */
const char* s1d_version(void);                 /* [host] */
int s1d_abi_version(void);                     /* [host] */
int s1d_device_count(void);                    /* visible CUDA devices (0 if none) */

/* ---- configuration & host helpers [host] -------------------------------- */
void s1d_config_defaults(s1d_config* cfg);
int s1d_apply_config_entry(s1d_config* cfg, const char* key, const char* value, char* err, size_t errlen);
int s1d_validate(const s1d_config* cfg, int partitioned, char* err, size_t errlen);
int s1d_finalize(s1d_config* cfg, int partitioned, char* err, size_t errlen);
/* (substeps S, half width h, state slots, values per point) — make_spec, kernels.cpp:7-25 */
void s1d_spec(int equation, int method, int* substeps, int* half_width, int* slots, int* values_per_point);
int s1d_initial_condition(const char* id, uint64_t n, int equation, double gamma, double* out, size_t out_len,
                          char* err, size_t errlen);
/* Points [j0, j0+count) of the same initial condition (no full-grid array). */
int s1d_initial_condition_range(const char* id, uint64_t n, int equation, double gamma, uint64_t j0, uint64_t count,
                                double* out, size_t out_len, char* err, size_t errlen);
int s1d_max_signal_speed(const double* prim, size_t len, double gamma, double* out, char* err, size_t errlen);
/* arrays of length cfg->ranks */
int s1d_partition(const s1d_config* cfg, uint64_t* blocks, uint64_t* start_index, int* left, int* right,
                  char* err, size_t errlen);
int64_t s1d_cycle_advance(uint64_t w, uint64_t h, char* err, size_t errlen); /* <0: -status */
/* The message log RunResult::log holds for cfg with keep_message_log
 * (RingTransport::sorted_log, transport.cpp:197-206): *count = its length, up
 * to cap entries written. Payload sizes are the reference's Cell bytes. */
int s1d_message_log(const s1d_config* cfg, s1d_message* out, size_t cap, size_t* count, char* err, size_t errlen);
/* CommStats::per_rank for cfg (transport.cpp:190-196); arrays of cfg->ranks. */
int s1d_comm_per_rank(const s1d_config* cfg, s1d_rank_stats* out, size_t cap, char* err, size_t errlen);

/* Test hook (no reference counterpart, no CUDA): the issue order of the
 * wavefront solve that s1d_solve uses to overlap the host copies (DESIGN.md
 * §12) for `chunks` chunks, `head` / `tail` pipelined Diamonds, `cycles`
 * swept cycles, one process per GPU or not. `out` receives *count triples
 * (kind, phase, chunk) up to `cap` triples; kind 0 = chunk launch,
 * 1 = round signal (multi-process only), 2 = the whole-shard middle
 * Diamonds. */
int s1d_debug_wave_schedule(int chunks, int head, int tail, int64_t cycles, int multi_process, int64_t* out,
                            size_t cap, size_t* count, char* err, size_t errlen);
/* kind 0 triangle, 1 diamond, 2 down-triangle. Returns the level count (or
 * -status); fills up to cap (substep, lo, hi) triples. */
int64_t s1d_schedule(int kind, uint64_t w, uint64_t h, int64_t* substep, int64_t* lo, int64_t* hi, size_t cap,
                     char* err, size_t errlen);
uint64_t s1d_swept_buffer_cells(uint64_t w, int equation, int method);

/* ---- one-shot run (the drop-in for sweep1d::run) ------------------------- */
/* Finalizes a copy of cfg, builds the initial condition on the host, runs the
 * configured scheme on the GPU(s) and writes n*vpp doubles in global order to
 * state_out. stats/timing may be NULL. */
int s1d_run(const s1d_config* cfg, double* state_out, size_t state_len, s1d_stats* stats, s1d_timing* timing,
            char* err, size_t errlen);

/* ---- debug run (RunOptions, inc/debug.hpp:17-62) ------------------------- */
typedef struct s1d_debug {
    int coverage;            /* count every (point, substep) the kernels compute */
    int perturb_ulp;         /* nudge the run's first computed value by one ulp (shard 0) */
    uint32_t* coverage_out;  /* host [steps*S][n] counts, index (substep-1)*n + point */
    size_t coverage_len;
} s1d_debug;
/* s1d_run with instrumented kernels (same geometry and arithmetic; slower).
 * A correct tiling computes every (point, substep) exactly once
 * (CoverageCounter::defects() empty). */
int s1d_run_debug(const s1d_config* cfg, const s1d_debug* dbg, double* state_out, size_t state_len,
                  s1d_stats* stats, s1d_timing* timing, char* err, size_t errlen);

/* ---- reusable solver handle -------------------------------------------- */
typedef struct s1d_solver s1d_solver;
int s1d_create(const s1d_config* cfg, s1d_solver** out, char* err, size_t errlen);
void s1d_destroy(s1d_solver* s);
/* Effective (finalized) configuration of the handle. */
int s1d_get_config(const s1d_solver* s, s1d_config* out);
/* Upload n*vpp doubles (global order) as the initial state; NULL = the
 * configured initial condition (already resident since s1d_create). */
int s1d_set_initial(s1d_solver* s, const double* host_state, size_t len);
/* Run cfg.steps time steps from the resident initial state, on the device
 * only (no host copies). */
int s1d_advance(s1d_solver* s, s1d_stats* stats, s1d_timing* timing);
/* Copy the resident final state (n*vpp doubles, global order) to the host. */
int s1d_read_state(s1d_solver* s, double* host_out, size_t len);
/* End to end through host buffers: H2D of host_in (NULL = configured IC),
 * advance, D2H into host_out. timing splits h2d / loop / d2h. */
int s1d_solve(s1d_solver* s, const double* host_in, size_t in_len, double* host_out, size_t out_len,
              s1d_stats* stats, s1d_timing* timing);
const char* s1d_last_error(const s1d_solver* s);

/* ---- one process per GPU (e.g. under torchrun) -------------------------- */
/* Create shard `rank` (0 <= rank < cfg->ranks, partition as s1d_partition) on
 * visible device `device`. The process owns only that shard; its ring
 * neighbours live in other processes. Host I/O of the handle (set_initial,
 * solve, read_state) covers the local slice [start, start+count) only. */
int s1d_shard_create(const s1d_config* cfg, int rank, int device, s1d_solver** out, char* err, size_t errlen);
/* Size of the opaque blob (CUDA IPC handles of the shard's device buffers). */
size_t s1d_shard_blob_size(void);
int s1d_shard_export(s1d_solver* s, void* blob, size_t blob_len);
/* Map the ring neighbours' buffers (their blobs, exchanged by the caller's
 * transport). Afterwards every s1d_advance runs in lockstep with them:
 * boundary tiles read the neighbour's edges in place over NVLink, rounds are
 * ordered by device-side flags (no host round trip). */
int s1d_shard_connect(s1d_solver* s, const void* left_blob, const void* right_blob);
int s1d_shard_range(const s1d_solver* s, uint64_t* start, uint64_t* count);

/* ---- measurement records, CSV, fits (inc/perf.hpp, inc/csv.hpp) --------- */
/* TimingRecord (inc/perf.hpp:16-29). avg_us_per_step = loop time / steps
 * (CUDA events; the reference's WallClock branch of make_record). */
typedef struct s1d_record {
    int equation, method, scheme, mode;
    uint64_t grid_size, block_width;
    int work_factor, ranks;
    int64_t steps;
    double avg_us_per_step;
    double setup_us;
    uint64_t messages_sent, bytes_sent, exchange_rounds;
    double virtual_comm_us; /* CommStats::virtual_comm_time in microseconds (the alpha-beta model) */
} s1d_record;
/* measure (src/perf.cpp:29-32): one run of cfg, reduced to a record. */
int s1d_measure(const s1d_config* cfg, s1d_record* out, char* err, size_t errlen);
/* The reference's fixed 15-column header (inc/csv.hpp:11-13). [host] */
const char* s1d_csv_header(void);
/* csv_row (src/csv.cpp:69-78): writes the row (no newline); returns its
 * length, or -1 if buf is too small. [host] */
int64_t s1d_csv_row(const s1d_record* r, char* buf, size_t len);
/* emit_csv (src/csv.cpp:80-99): header + rows in config-lexicographic order. [host] */
int s1d_emit_csv(const s1d_record* recs, size_t n, const char* path, char* err, size_t errlen);
/* read_csv (src/csv.cpp:101-136). [host] */
int s1d_read_csv(const char* path, s1d_record* out, size_t cap, size_t* count, char* err, size_t errlen);
/* power_law_fit (src/perf.cpp:42-82): y = A x^b by log-log OLS. [host] */
int s1d_power_law_fit(const double* n, const double* t, size_t count, double* A, double* b, double* r2, char* err,
                      size_t errlen);
/* best_config (src/perf.cpp:84-97): index of the fastest record (ties: smaller
 * w, then smaller WF), or -status. [host] */
int64_t s1d_best_config(const s1d_record* recs, size_t n);

/* ---- alpha-beta virtual-time model -------------------------------------- */
/* The reference's VirtualTime clock for cfg's run (RingTransport
 * advance_clock/round cost, transport.cpp:73-90, 173-182; advance points
 * engines_impl.hpp:201-213, 249-321; result engines_impl.hpp:413), replayed
 * without running the stencil: *virtual_seconds = the final max rank clock
 * (RunResult.timing.virtual_seconds in virtual mode), *comm_seconds = the
 * per-rank sum of round costs (CommStats::virtual_comm_time, any mode).
 * Uses cfg->alpha, beta, compute_cost; cfg is copied and finalized. s1d_run
 * and s1d_measure report the same values. [host] */
int s1d_virtual_time(const s1d_config* cfg, double* virtual_seconds, double* comm_seconds, char* err,
                     size_t errlen);
/* Measured transport parameters between two devices for the model above:
 * *alpha = one-way latency (s) of a device-side flag hand-off over NVLink (the
 * swept round's synchronisation), *beta = s/byte of a 256 MiB peer copy. */
int s1d_calibrate_transport(int dev_a, int dev_b, double* alpha, double* beta, char* err, size_t errlen);

/* ---- measurement helpers (not part of the reference interface) --------- */
/* Sustained FP64 DADD/DMUL instruction rate of `device` (ops/s), measured by
 * a dependent-chain-free microkernel: the roofline denominator for the
 * FP64-pipe-bound swept kernels. */
int s1d_measure_fp64_peak(int device, double* ops_per_second, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
#endif /* SWEPT1D_H */
