// Host-side configuration, geometry and initial conditions of the swept
// solver (no CUDA). Restated from the reference's semantics:
//   LaunchConfig::validate/finalize   src/config.cpp:45-103
//   make_partition / extents / IC     src/partition.cpp:10-113
//   cycle_advance / schedules         src/swept.cpp:11-64
// Errors are thrown as s1d::Error{status, message} and converted to status
// codes at the C ABI (engine.cu, extern "C" section).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "swept1d.h"

namespace s1d {

struct Error : std::runtime_error {
    int status;
    Error(int st, const std::string& what) : std::runtime_error(what), status(st) {}
};

struct Spec {
    int S = 1;     // substeps per time step
    int h = 1;     // stencil half width
    int slots = 2; // doubles per reference record
    int vpp = 1;   // values per point in the output
    int rec = 1;   // doubles per B200 edge record (full live snapshot)
};

Spec make_spec(int equation, int method);

std::string initial_or_default(const s1d_config& cfg);
void validate(const s1d_config& cfg, bool partitioned);
void finalize(s1d_config& cfg, bool partitioned);
void apply_config_entry(s1d_config& cfg, const std::string& key, const std::string& value);

std::vector<double> initial_condition(const std::string& id, std::uint64_t n, int equation, double gamma);
// Points [j0, j0+count) of the same initial condition (vpp doubles each):
// per-point identical to initial_condition(), without materialising all n.
std::vector<double> initial_condition_range(const std::string& id, std::uint64_t n, int equation, double gamma,
                                            std::uint64_t j0, std::uint64_t count);
double max_signal_speed(const double* prim, std::size_t len, double gamma);
// max_signal_speed over the whole initial condition, streamed in chunks.
double max_signal_speed_of(const std::string& id, std::uint64_t n, double gamma);

struct Partition {
    std::vector<std::uint64_t> blocks, start;
    std::vector<int> left, right;
};
Partition make_partition(const s1d_config& cfg);

std::uint64_t cycle_advance(std::uint64_t w, std::uint64_t h);

struct Level {
    std::int64_t substep, lo, hi;
};
std::vector<Level> schedule(int kind, std::uint64_t w, std::uint64_t h);

// The reference's alpha-beta virtual clock for a finalized config (host_model.cpp):
// returns the final max rank clock; *comm_seconds = per-rank sum of round costs.
double virtual_clock(const s1d_config& cfg, double* comm_seconds);

// The reference transport's sorted message log and per-rank counters for a
// config (host_model.cpp).
std::vector<s1d_message> message_log(const s1d_config& cfg);
// Wavefront solve issue order (host_wave.cpp).
enum { kWaveChunk = 0, kWaveSignal = 1, kWaveMiddle = 2 };
struct WaveStep {
    int kind;       // kWaveChunk: chunk c of phase p; kWaveSignal: round of phase p; kWaveMiddle
    std::int64_t p; // phase (0: Up, cycles: Down)
    int c;          // chunk
};
std::vector<WaveStep> wave_schedule(int K, int head, int tail, std::int64_t cycles, bool xs);
std::vector<s1d_rank_stats> rank_stats(const s1d_config& cfg);

} // namespace s1d
