// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference `sweep1d` core, compiled from
// the sources where they lie under /root/reference/proj/core (see
// oracle/Makefile). The shim is this repo's own code; it only translates
// plain C structs into the reference's LaunchConfig and exceptions into status
// codes so pytest (ctypes) and bench.py's reference arm can drive:
//   sweep1d::run_serial   inc/engine.hpp:32, src/serial.cpp:5-12
//   sweep1d::run          inc/engine.hpp:28, src/engine.cpp:40-47
// plus the per-point kernels and host helpers the parity tests pin
// (inc/kernels.hpp, src/kernels.cpp, src/partition.cpp, src/swept.cpp,
// src/config.cpp).
//
// Status codes match include/swept1d.h (S1D_*), so tests can compare error
// behaviour of the reference and the B200 library one-to-one.

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "sweep1d/config.hpp"
#include "sweep1d/csv.hpp"
#include "sweep1d/perf.hpp"
#include "sweep1d/engine.hpp"
#include "sweep1d/errors.hpp"
#include "sweep1d/kernels.hpp"
#include "sweep1d/partition.hpp"
#include "sweep1d/swept.hpp"

using namespace sweep1d;

extern "C" {

struct ref_cfg {
    int equation;  // 0 heat, 1 euler
    int method;    // 0 lengthening, 1 flattening
    int scheme;    // 0 classic, 1 swept
    int mode;      // 0 wall, 1 virtual
    unsigned long long grid_size;
    unsigned long long block_width;
    int ranks;
    int work_factor;
    long long steps;
    double fourier, gamma, dt_dx, cfl;
    double alpha, beta, compute_cost;
    char initial[64];  // "" = per-equation default
};

struct ref_stats {
    unsigned long long messages_sent, bytes_sent, exchange_rounds;
    double setup_seconds, loop_seconds, virtual_seconds;
    double virtual_comm_time;  // CommStats::virtual_comm_time (transport.hpp:20-30)
};

struct ref_msg {
    unsigned long long round;
    int source, dest;
    unsigned long long tag, bytes;
};

}  // extern "C"

namespace {

enum : int {
    kOk = 0,
    kInvalidConfig = 1,
    kUnknownIc = 2,
    kNonPhysical = 3,
    kInvalidWidth = 4,
    kPayloadSize = 5,
    kTagMismatch = 6,
    kPhaseSkew = 7,
    kModeMismatch = 8,
    kDegenerateFit = 9,
    kTransportAborted = 10,
    kOther = 99,
};

void put_err(char* err, size_t errlen, const char* what) {
    if (!err || errlen == 0) return;
    std::strncpy(err, what, errlen - 1);
    err[errlen - 1] = '\0';
}

template <class Fn>
int guarded(char* err, size_t errlen, Fn&& fn) {
    try {
        fn();
        put_err(err, errlen, "");
        return kOk;
    } catch (const InvalidConfig& e) { put_err(err, errlen, e.what()); return kInvalidConfig; }
    catch (const UnknownInitialCondition& e) { put_err(err, errlen, e.what()); return kUnknownIc; }
    catch (const NonPhysicalState& e) { put_err(err, errlen, e.what()); return kNonPhysical; }
    catch (const InvalidWidth& e) { put_err(err, errlen, e.what()); return kInvalidWidth; }
    catch (const PayloadSizeMismatch& e) { put_err(err, errlen, e.what()); return kPayloadSize; }
    catch (const TagMismatch& e) { put_err(err, errlen, e.what()); return kTagMismatch; }
    catch (const PhaseSkew& e) { put_err(err, errlen, e.what()); return kPhaseSkew; }
    catch (const ModeMismatch& e) { put_err(err, errlen, e.what()); return kModeMismatch; }
    catch (const DegenerateFit& e) { put_err(err, errlen, e.what()); return kDegenerateFit; }
    catch (const TransportAborted& e) { put_err(err, errlen, e.what()); return kTransportAborted; }
    catch (const std::exception& e) { put_err(err, errlen, e.what()); return kOther; }
}

LaunchConfig to_cfg(const ref_cfg* c) {
    LaunchConfig cfg;
    cfg.equation = c->equation ? Equation::Euler : Equation::Heat;
    cfg.method = c->method ? Method::Flattening : Method::Lengthening;
    cfg.scheme = c->scheme ? Scheme::Swept : Scheme::Classic;
    cfg.mode = c->mode ? Mode::VirtualTime : Mode::WallClock;
    cfg.grid_size = c->grid_size;
    cfg.block_width = c->block_width;
    cfg.ranks = c->ranks;
    cfg.work_factor = c->work_factor;
    cfg.steps = static_cast<long>(c->steps);
    cfg.phys.fourier = c->fourier;
    cfg.phys.gamma = c->gamma;
    cfg.phys.dt_dx = c->dt_dx;
    cfg.phys.cfl = c->cfl;
    cfg.transport.alpha = c->alpha;
    cfg.transport.beta = c->beta;
    cfg.transport.compute_cost = c->compute_cost;
    cfg.initial = std::string(c->initial, strnlen(c->initial, sizeof(c->initial)));
    return cfg;
}

EulerCell len_cell(const double* v) {
    EulerCell c;
    c.Q[0] = Cons{v[0], v[1], v[2]};
    c.Q[1] = Cons{v[3], v[4], v[5]};
    c.Pr = v[6];
    return c;
}

}  // namespace

extern "C" {

int ref_defaults(ref_cfg* out) {
    LaunchConfig cfg;
    out->equation = 0;
    out->method = 0;
    out->scheme = cfg.scheme == Scheme::Swept ? 1 : 0;
    out->mode = cfg.mode == Mode::VirtualTime ? 1 : 0;
    out->grid_size = cfg.grid_size;
    out->block_width = cfg.block_width;
    out->ranks = cfg.ranks;
    out->work_factor = cfg.work_factor;
    out->steps = cfg.steps;
    out->fourier = cfg.phys.fourier;
    out->gamma = cfg.phys.gamma;
    out->dt_dx = cfg.phys.dt_dx;
    out->cfl = cfg.phys.cfl;
    out->alpha = cfg.transport.alpha;
    out->beta = cfg.transport.beta;
    out->compute_cost = cfg.transport.compute_cost;
    out->initial[0] = '\0';
    return 0;
}

int ref_run_serial(const ref_cfg* c, double* out, size_t cap, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const auto v = run_serial(to_cfg(c));
        if (v.size() > cap) throw std::runtime_error("output buffer too small");
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int ref_run(const ref_cfg* c, double* out, size_t cap, ref_stats* st, ref_msg* log, size_t log_cap,
            size_t* log_len, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        RunOptions opts;
        opts.keep_message_log = log != nullptr;
        const auto res = run(to_cfg(c), opts);
        if (res.state.size() > cap) throw std::runtime_error("output buffer too small");
        if (out) std::memcpy(out, res.state.data(), res.state.size() * sizeof(double));
        if (st) {
            st->messages_sent = res.stats.messages_sent;
            st->bytes_sent = res.stats.bytes_sent;
            st->exchange_rounds = res.stats.exchange_rounds;
            st->setup_seconds = res.timing.setup_seconds;
            st->loop_seconds = res.timing.loop_seconds;
            st->virtual_seconds = res.timing.virtual_seconds;
            st->virtual_comm_time = res.stats.virtual_comm_time;
        }
        if (log) {
            const size_t n = res.log.size() < log_cap ? res.log.size() : log_cap;
            for (size_t i = 0; i < n; ++i) {
                log[i].round = res.log[i].round;
                log[i].source = res.log[i].source;
                log[i].dest = res.log[i].dest;
                log[i].tag = res.log[i].tag;
                log[i].bytes = res.log[i].bytes;
            }
            if (log_len) *log_len = res.log.size();
        }
    });
}

int ref_finalize(ref_cfg* c, int partitioned, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        LaunchConfig cfg = to_cfg(c);
        cfg.finalize(partitioned != 0);
        c->dt_dx = cfg.phys.dt_dx;
    });
}

int ref_partition(const ref_cfg* c, unsigned long long* blocks, unsigned long long* starts, int* left,
                  int* right, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const Partition p = make_partition(to_cfg(c));
        for (int r = 0; r < p.ranks(); ++r) {
            blocks[r] = p.blocks[static_cast<size_t>(r)];
            starts[r] = p.start_index[static_cast<size_t>(r)];
            left[r] = p.left[static_cast<size_t>(r)];
            right[r] = p.right[static_cast<size_t>(r)];
        }
    });
}

int ref_working_array_extents(unsigned long long n_blocks, unsigned long long w, int equation, int method,
                              unsigned long long* out3, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const auto e = working_array_extents(n_blocks, w,
                                             make_spec(equation ? Equation::Euler : Equation::Heat,
                                                       method ? Method::Flattening : Method::Lengthening));
        out3[0] = e.length;
        out3[1] = e.initialized;
        out3[2] = e.ghost;
    });
}

unsigned long long ref_swept_buffer_cells(unsigned long long w, int equation, int method) {
    return swept_buffer_cells(w, make_spec(equation ? Equation::Euler : Equation::Heat,
                                           method ? Method::Flattening : Method::Lengthening));
}

int ref_initial_condition(const char* id, unsigned long long n, int equation, int method, double gamma,
                          double* out, size_t cap, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const auto v = initial_condition(id, n,
                                         make_spec(equation ? Equation::Euler : Equation::Heat,
                                                   method ? Method::Flattening : Method::Lengthening),
                                         gamma);
        if (v.size() > cap) throw std::runtime_error("output buffer too small");
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int ref_max_signal_speed(const double* v, size_t len, double gamma, double* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { *out = max_signal_speed(std::vector<double>(v, v + len), gamma); });
}

// schedule kind: 0 triangle, 1 diamond, 2 down-triangle. Returns level count
// (or -status on error, message in err).
long ref_schedule(int kind, unsigned long long w, unsigned long long h, long* substep, long* lo, long* hi,
                  size_t cap, char* err, size_t errlen) {
    PhaseSchedule s;
    const int rc = guarded(err, errlen, [&] {
        s = kind == 0 ? triangle_schedule(w, h) : kind == 1 ? diamond_schedule(w, h) : down_triangle_schedule(w, h);
    });
    if (rc != kOk) return -rc;
    for (size_t i = 0; i < s.levels.size() && i < cap; ++i) {
        substep[i] = s.levels[i].substep;
        lo[i] = static_cast<long>(s.levels[i].lo);
        hi[i] = static_cast<long>(s.levels[i].hi);
    }
    return static_cast<long>(s.levels.size());
}

long ref_cycle_advance(unsigned long long w, unsigned long long h, char* err, size_t errlen) {
    size_t m = 0;
    const int rc = guarded(err, errlen, [&] { m = cycle_advance(w, h); });
    return rc == kOk ? static_cast<long>(m) : -rc;
}

// ---- per-point kernels (inc/kernels.hpp, src/kernels.cpp) -------------------

double ref_heat_step(double l, double c, double r, double fo) { return heat_step(l, c, r, fo); }
double ref_minmod(double a, double b) { return minmod(a, b); }
double ref_pressure_ratio_value(double pl, double pc, double pr) { return pressure_ratio_value(pl, pc, pr); }

int ref_pressure(const double* q, double gamma, double* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { *out = pressure(Cons{q[0], q[1], q[2]}, gamma); });
}

int ref_interface_flux(const double* ql, const double* qr, double pr_l, double pr_r, double gamma, double* out,
                       char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const Cons f = interface_flux(Cons{ql[0], ql[1], ql[2]}, Cons{qr[0], qr[1], qr[2]}, pr_l, pr_r, gamma);
        out[0] = f.rho;
        out[1] = f.mom;
        out[2] = f.ene;
    });
}

// Apply Model::apply at index i of an AoS array of ncells records. Records:
// heat 2 doubles {T0,T1}; lengthening 7 {Q0,Q1,Pr}; flattening 6 {Q0,Q1}.
int ref_model_apply(int model, double* cells, long ncells, long i, long counter, double fourier, double gamma,
                    double dt_dx, char* err, size_t errlen) {
    PhysParams phys;
    phys.fourier = fourier;
    phys.gamma = gamma;
    phys.dt_dx = dt_dx;
    return guarded(err, errlen, [&] {
        if (model == 0) {
            std::vector<HeatCell> v(static_cast<size_t>(ncells));
            std::memcpy(v.data(), cells, sizeof(HeatCell) * v.size());
            HeatModel::apply(v.data(), i, counter, phys);
            std::memcpy(cells, v.data(), sizeof(HeatCell) * v.size());
        } else if (model == 1) {
            std::vector<EulerCell> v;
            for (long k = 0; k < ncells; ++k) v.push_back(len_cell(cells + 7 * k));
            EulerLenModel::apply(v.data(), i, counter, phys);
            for (long k = 0; k < ncells; ++k) {
                double* o = cells + 7 * k;
                const EulerCell& e = v[static_cast<size_t>(k)];
                o[0] = e.Q[0].rho; o[1] = e.Q[0].mom; o[2] = e.Q[0].ene;
                o[3] = e.Q[1].rho; o[4] = e.Q[1].mom; o[5] = e.Q[1].ene;
                o[6] = e.Pr;
            }
        } else {
            std::vector<FlatEulerCell> v(static_cast<size_t>(ncells));
            for (long k = 0; k < ncells; ++k) {
                const double* s = cells + 6 * k;
                v[static_cast<size_t>(k)].Q[0] = Cons{s[0], s[1], s[2]};
                v[static_cast<size_t>(k)].Q[1] = Cons{s[3], s[4], s[5]};
            }
            EulerFlatModel::apply(v.data(), i, counter, phys);
            for (long k = 0; k < ncells; ++k) {
                double* o = cells + 6 * k;
                const FlatEulerCell& e = v[static_cast<size_t>(k)];
                o[0] = e.Q[0].rho; o[1] = e.Q[0].mom; o[2] = e.Q[0].ene;
                o[3] = e.Q[1].rho; o[4] = e.Q[1].mom; o[5] = e.Q[1].ene;
            }
        }
    });
}

// ---- post-processing (inc/perf.hpp, inc/csv.hpp) --------------------------
struct ref_record {
    int equation, method, scheme, mode;
    unsigned long long grid_size, block_width;
    int work_factor, ranks;
    long long steps;
    double avg_us_per_step, setup_us;
    unsigned long long messages_sent, bytes_sent, exchange_rounds;
    double virtual_comm_us;
};

static TimingRecord to_rec(const ref_record& r) {
    TimingRecord t;
    t.equation = r.equation ? Equation::Euler : Equation::Heat;
    t.method = r.method ? Method::Flattening : Method::Lengthening;
    t.scheme = r.scheme ? Scheme::Swept : Scheme::Classic;
    t.mode = r.mode ? Mode::VirtualTime : Mode::WallClock;
    t.grid_size = r.grid_size;
    t.block_width = r.block_width;
    t.work_factor = r.work_factor;
    t.ranks = r.ranks;
    t.steps = static_cast<long>(r.steps);
    t.avg_us_per_step = r.avg_us_per_step;
    t.setup_us = r.setup_us;
    t.stats.messages_sent = r.messages_sent;
    t.stats.bytes_sent = r.bytes_sent;
    t.stats.exchange_rounds = r.exchange_rounds;
    t.stats.virtual_comm_time = r.virtual_comm_us / 1e6;
    return t;
}

int ref_csv_row(const ref_record* r, char* buf, size_t len) {
    const std::string s = csv_row(to_rec(*r));
    if (s.size() + 1 > len) return -1;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int>(s.size());
}

int ref_emit_csv(const ref_record* r, size_t n, const char* path, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<TimingRecord> v;
        for (size_t i = 0; i < n; ++i) v.push_back(to_rec(r[i]));
        emit_csv(v, std::string(path));
    });
}

int ref_power_law_fit(const double* x, const double* y, size_t n, double* A, double* b, double* r2, char* err,
                      size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<std::pair<double, double>> pts;
        for (size_t i = 0; i < n; ++i) pts.emplace_back(x[i], y[i]);
        const FitResult f = power_law_fit(pts);
        *A = f.A;
        *b = f.b;
        *r2 = f.r_squared;
    });
}

long ref_best_config(const ref_record* r, size_t n) {
    std::vector<TimingRecord> v;
    for (size_t i = 0; i < n; ++i) v.push_back(to_rec(r[i]));
    if (v.empty()) return -1;
    const TimingRecord* b = &best_config(v);
    return static_cast<long>(b - v.data());
}

}  // extern "C"
