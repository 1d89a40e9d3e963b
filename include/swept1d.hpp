// swept1d.hpp — header-only C++ host interface over the C ABI (swept1d.h).
//
// Mirrors the reference C++ API names so a sweep1d host ports by changing the
// namespace: LaunchConfig (inc/config.hpp:12-41), run -> RunResult
// (inc/engine.hpp:12-28), measure -> TimingRecord (inc/perf.hpp:16-40),
// emit_csv / read_csv (inc/csv.hpp), power_law_fit / best_config, and the
// exception types of inc/errors.hpp. Everything computes on the B200 through
// libswept1d.so; nothing here runs a CPU solver.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "swept1d.h"

namespace swept1d {

enum class Equation { Heat = S1D_HEAT, Euler = S1D_EULER };
enum class Method { Lengthening = S1D_LENGTHENING, Flattening = S1D_FLATTENING };
enum class Scheme { Classic = S1D_CLASSIC, Swept = S1D_SWEPT };
enum class Mode { WallClock = S1D_WALL, VirtualTime = S1D_VIRTUAL };

struct Sweep1dError : std::runtime_error {
    int status;
    Sweep1dError(int st, const std::string& w) : std::runtime_error(w), status(st) {}
};
#define SWEPT1D_ERR(Name, code) \
    struct Name : Sweep1dError { explicit Name(const std::string& w) : Sweep1dError(code, w) {} };
SWEPT1D_ERR(InvalidConfig, S1D_INVALID_CONFIG)
SWEPT1D_ERR(UnknownInitialCondition, S1D_UNKNOWN_IC)
SWEPT1D_ERR(NonPhysicalState, S1D_NONPHYSICAL)
SWEPT1D_ERR(InvalidWidth, S1D_INVALID_WIDTH)
SWEPT1D_ERR(DegenerateFit, S1D_DEGENERATE_FIT)
SWEPT1D_ERR(TransportAborted, S1D_TRANSPORT_ABORTED)
SWEPT1D_ERR(CudaError, S1D_CUDA_ERROR)
SWEPT1D_ERR(PeerUnavailable, S1D_PEER_UNAVAILABLE)
SWEPT1D_ERR(NoDevice, S1D_NO_DEVICE)
#undef SWEPT1D_ERR

inline void check(int st, const char* msg) {
    switch (st) {
    case S1D_OK: return;
    case S1D_INVALID_CONFIG: throw InvalidConfig(msg);
    case S1D_UNKNOWN_IC: throw UnknownInitialCondition(msg);
    case S1D_NONPHYSICAL: throw NonPhysicalState(msg);
    case S1D_INVALID_WIDTH: throw InvalidWidth(msg);
    case S1D_DEGENERATE_FIT: throw DegenerateFit(msg);
    case S1D_TRANSPORT_ABORTED: throw TransportAborted(msg);
    case S1D_CUDA_ERROR: throw CudaError(msg);
    case S1D_PEER_UNAVAILABLE: throw PeerUnavailable(msg);
    case S1D_NO_DEVICE: throw NoDevice(msg);
    default: throw Sweep1dError(st, msg);
    }
}

struct PhysParams {
    double fourier = 0.4, gamma = 1.4, dt_dx = 0.0, cfl = 0.4;
};
struct TransportParams {
    double alpha = 0.0, beta = 0.0, compute_cost = 1e-8;
};

struct LaunchConfig {
    Equation equation = Equation::Heat;
    Method method = Method::Lengthening;
    Scheme scheme = Scheme::Swept;
    std::size_t grid_size = 1024;
    std::size_t block_width = 32;
    int ranks = 2;
    int work_factor = 0;
    long steps = 50;
    std::string initial;
    Mode mode = Mode::VirtualTime;
    PhysParams phys;
    TransportParams transport;
    int num_devices = 0;

    s1d_config to_c() const {
        s1d_config c;
        s1d_config_defaults(&c);
        c.equation = static_cast<int>(equation);
        c.method = static_cast<int>(method);
        c.scheme = static_cast<int>(scheme);
        c.mode = static_cast<int>(mode);
        c.grid_size = grid_size;
        c.block_width = block_width;
        c.ranks = ranks;
        c.work_factor = work_factor;
        c.steps = steps;
        c.fourier = phys.fourier;
        c.gamma = phys.gamma;
        c.dt_dx = phys.dt_dx;
        c.cfl = phys.cfl;
        c.alpha = transport.alpha;
        c.beta = transport.beta;
        c.compute_cost = transport.compute_cost;
        if (initial.size() >= sizeof(c.initial)) throw InvalidConfig("initial condition id too long");
        std::memcpy(c.initial, initial.c_str(), initial.size() + 1);
        c.num_devices = num_devices;
        return c;
    }
    void validate(bool partitioned = true) const {
        char err[512];
        const s1d_config c = to_c();
        check(s1d_validate(&c, partitioned ? 1 : 0, err, sizeof err), err);
    }
    void finalize(bool partitioned = true) {
        char err[512];
        s1d_config c = to_c();
        check(s1d_finalize(&c, partitioned ? 1 : 0, err, sizeof err), err);
        phys.dt_dx = c.dt_dx;
    }
    int values_per_point() const {
        int vpp = 1;
        s1d_spec(static_cast<int>(equation), static_cast<int>(method), nullptr, nullptr, nullptr, &vpp);
        return vpp;
    }
};

inline void apply_config_entry(LaunchConfig& cfg, const std::string& key, const std::string& value) {
    s1d_config c = cfg.to_c();
    char err[512];
    check(s1d_apply_config_entry(&c, key.c_str(), value.c_str(), err, sizeof err), err);
    cfg.equation = static_cast<Equation>(c.equation);
    cfg.method = static_cast<Method>(c.method);
    cfg.scheme = static_cast<Scheme>(c.scheme);
    cfg.mode = static_cast<Mode>(c.mode);
    cfg.grid_size = c.grid_size;
    cfg.block_width = c.block_width;
    cfg.ranks = c.ranks;
    cfg.work_factor = c.work_factor;
    cfg.steps = static_cast<long>(c.steps);
    cfg.initial = std::string(c.initial, strnlen(c.initial, sizeof c.initial));
    cfg.phys = PhysParams{c.fourier, c.gamma, c.dt_dx, c.cfl};
    cfg.transport = TransportParams{c.alpha, c.beta, c.compute_cost};
    cfg.num_devices = c.num_devices;
}

struct CommStats {
    std::uint64_t messages_sent = 0, bytes_sent = 0, exchange_rounds = 0, kernel_launches = 0;
};
struct EngineTiming {
    double setup_seconds = 0, loop_seconds = 0, virtual_seconds = 0;
};
struct RunResult {
    std::vector<double> state;
    CommStats stats;
    EngineTiming timing;
};

inline RunResult run(const LaunchConfig& cfg) {
    const s1d_config c = cfg.to_c();
    RunResult r;
    r.state.resize(cfg.grid_size * static_cast<std::size_t>(cfg.values_per_point()));
    s1d_stats st;
    s1d_timing tm;
    char err[512];
    check(s1d_run(&c, r.state.data(), r.state.size(), &st, &tm, err, sizeof err), err);
    r.stats = CommStats{st.messages_sent, st.bytes_sent, st.exchange_rounds, st.kernel_launches};
    r.timing = EngineTiming{tm.setup_seconds, tm.loop_seconds, tm.virtual_seconds};
    return r;
}

/// Run instrumentation hooks (the subset of sweep1d::RunOptions,
/// inc/debug.hpp:17-24, that the B200 path implements). Any hook set routes the
/// run through the instrumented kernels (s1d_run_debug: same geometry and
/// arithmetic, slower).
struct RunOptions {
    bool coverage = false;    // count every (point, substep) computation
    bool perturb_ulp = false; // nudge the first kernel write by 1 ulp (mutation hook)
};

/// sweep1d::run(cfg, opts) (inc/engine.hpp:28). With coverage on, `coverage`
/// receives [steps*S][n] counts (index (substep-1)*n + point) when non-null.
inline RunResult run(const LaunchConfig& cfg, const RunOptions& opts, std::vector<std::uint32_t>* coverage = nullptr) {
    if (!opts.coverage && !opts.perturb_ulp) return run(cfg);
    const s1d_config c = cfg.to_c();
    RunResult r;
    r.state.resize(cfg.grid_size * static_cast<std::size_t>(cfg.values_per_point()));
    std::vector<std::uint32_t> cov;
    s1d_debug d{};
    d.coverage = opts.coverage ? 1 : 0;
    d.perturb_ulp = opts.perturb_ulp ? 1 : 0;
    if (opts.coverage) {
        int S = 1;
        s1d_spec(c.equation, c.method, &S, nullptr, nullptr, nullptr);
        cov.assign(static_cast<std::size_t>(cfg.steps) * static_cast<std::size_t>(S) * cfg.grid_size, 0u);
        d.coverage_out = cov.data();
        d.coverage_len = cov.size();
    }
    s1d_stats st;
    s1d_timing tm;
    char err[512];
    check(s1d_run_debug(&c, &d, r.state.data(), r.state.size(), &st, &tm, err, sizeof err), err);
    r.stats = CommStats{st.messages_sent, st.bytes_sent, st.exchange_rounds, st.kernel_launches};
    r.timing = EngineTiming{tm.setup_seconds, tm.loop_seconds, tm.virtual_seconds};
    if (coverage) *coverage = std::move(cov);
    return r;
}

using TimingRecord = s1d_record;

inline TimingRecord measure(const LaunchConfig& cfg) {
    const s1d_config c = cfg.to_c();
    TimingRecord rec;
    char err[512];
    check(s1d_measure(&c, &rec, err, sizeof err), err);
    return rec;
}

inline double speedup(double time_classic, double time_swept) { return time_classic / time_swept; }

inline std::string csv_row(const TimingRecord& r) {
    char buf[1024];
    if (s1d_csv_row(&r, buf, sizeof buf) < 0) throw std::runtime_error("csv row too long");
    return buf;
}
inline void emit_csv(const std::vector<TimingRecord>& recs, const std::string& path) {
    char err[512];
    check(s1d_emit_csv(recs.data(), recs.size(), path.c_str(), err, sizeof err), err);
}
inline std::vector<TimingRecord> read_csv(const std::string& path) {
    std::size_t n = 0;
    char err[512];
    check(s1d_read_csv(path.c_str(), nullptr, 0, &n, err, sizeof err), err);
    std::vector<TimingRecord> out(n);
    check(s1d_read_csv(path.c_str(), out.data(), out.size(), &n, err, sizeof err), err);
    return out;
}

struct FitResult {
    double A = 0, b = 0, r_squared = 0;
};
inline FitResult power_law_fit(const std::vector<std::pair<double, double>>& pts) {
    std::vector<double> x, y;
    for (const auto& p : pts) {
        x.push_back(p.first);
        y.push_back(p.second);
    }
    FitResult f;
    char err[512];
    check(s1d_power_law_fit(x.data(), y.data(), x.size(), &f.A, &f.b, &f.r_squared, err, sizeof err), err);
    return f;
}
inline const TimingRecord& best_config(const std::vector<TimingRecord>& recs) {
    const std::int64_t i = s1d_best_config(recs.data(), recs.size());
    if (i < 0) throw InvalidConfig("best_config over an empty record set");
    return recs[static_cast<std::size_t>(i)];
}

} // namespace swept1d
