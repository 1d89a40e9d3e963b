// The reference's alpha-beta virtual clock, replayed on the host (no GPU).
//
// In VirtualTime mode the reference advances each rank's clock by
// compute_units * compute_cost after it computes (RingTransport::advance_clock,
// transport.cpp:173-178) and, at every exchange round, sets all clocks to the
// round maximum plus alpha + beta * per_message_bytes (transport.cpp:73-90).
// The per-rank sum of round costs is CommStats::virtual_comm_time (reported
// in both modes). The engine calls advance_clock at fixed points:
//   classic:  apply N  -> advance -> exchange round       (engines_impl.hpp:201-213)
//   swept:    Up -> advance; per cycle: shift round -> phase -> advance;
//             pad: exchange round -> apply N -> advance    (engines_impl.hpp:249-321)
// and reports the final max clock (engines_impl.hpp:413). The work per rank is
// a pure function of the partition and the phase schedules, so the clock is
// replayed here in the reference's floating-point order (bit-identical
// virtual_seconds / virtual_comm_time; checked against the compiled reference
// in tests/test_virtual_time.py). The GPU computes the state for real; this
// model is what the reference's virtual mode reports for the same run.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "host_config.hpp"
#include "swept1d.h"

namespace s1d {

namespace {

std::uint64_t schedule_units(int kind, std::uint64_t w, std::uint64_t h) {
    std::uint64_t u = 0;
    for (const Level& l : schedule(kind, w, h)) u += static_cast<std::uint64_t>(l.hi - l.lo);
    return u;
}

} // namespace

double virtual_clock(const s1d_config& cfg, double* comm_seconds) {
    const Spec sp = make_spec(cfg.equation, cfg.method);
    const Partition part = make_partition(cfg);
    const int R = cfg.ranks;
    const std::uint64_t w = cfg.block_width;
    const std::uint64_t h = static_cast<std::uint64_t>(sp.h);
    const std::uint64_t cell = sizeof(double) * static_cast<std::uint64_t>(sp.slots); // reference Cell size
    const std::int64_t total = cfg.steps * sp.S;

    std::vector<double> clk(static_cast<std::size_t>(R), 0.0);
    double comm = 0.0;
    auto advance = [&](int r, std::uint64_t units) {
        clk[static_cast<std::size_t>(r)] += static_cast<double>(units) * cfg.compute_cost;
    };
    auto round = [&](std::uint64_t per_message) {
        const double cost = cfg.alpha + cfg.beta * static_cast<double>(per_message);
        const double peak = *std::max_element(clk.begin(), clk.end());
        std::fill(clk.begin(), clk.end(), peak + cost);
        comm += cost;
    };
    auto owned = [&](int r) { return part.blocks[static_cast<std::size_t>(r)] * w; };

    if (cfg.scheme == S1D_CLASSIC) {
        for (std::int64_t c = 1; c <= total; ++c) {
            for (int r = 0; r < R; ++r) advance(r, owned(r));
            round(h * cell);
        }
    } else {
        const std::uint64_t m = cycle_advance(w, h);
        const std::int64_t cycles = total / static_cast<std::int64_t>(m);
        if (cycles >= 1) {
            const std::uint64_t up = schedule_units(0, w, h);
            const std::uint64_t dia = schedule_units(1, w, h);
            const std::uint64_t down = schedule_units(2, w, h);
            const std::uint64_t buf = w / 2 + h; // swept_buffer_cells (partition.cpp:46-48)
            for (int r = 0; r < R; ++r) advance(r, part.blocks[static_cast<std::size_t>(r)] * up);
            for (std::int64_t j = 1; j <= cycles; ++j) {
                round(buf * cell);
                const std::uint64_t u = j == cycles ? down : dia;
                for (int r = 0; r < R; ++r) advance(r, part.blocks[static_cast<std::size_t>(r)] * u);
            }
        }
        for (std::int64_t c = cycles * static_cast<std::int64_t>(m) + 1; c <= total; ++c) {
            round(h * cell);
            for (int r = 0; r < R; ++r) advance(r, owned(r));
        }
    }
    if (comm_seconds) *comm_seconds = comm;
    return *std::max_element(clk.begin(), clk.end());
}

// The reference transport's message log and per-rank counters for `cfg`
// (RingTransport::complete_round_locked, transport.cpp:66-110; sorted_log
// :197-206), replayed on the host. The round sequence and every payload size
// are pure functions of the configuration: classic runs one exchange round of
// h cells each way per substep (tag (c << 3) | 1, engines_impl.hpp:211);
// swept runs one shift round per cycle of w/2 + h cells, leftward on odd
// cycles (tags (j << 3) | 2 / 3, :295), then one exchange round per pad
// substep (tag (c << 3) | 5, :317). Payloads are the reference's Cell bytes
// (8 * state slots), the B200 path's own traffic is in s1d_stats.
std::vector<s1d_message> message_log(const s1d_config& cfg) {
    const Spec sp = make_spec(cfg.equation, cfg.method);
    const int R = cfg.ranks;
    const std::uint64_t w = cfg.block_width;
    const std::uint64_t h = static_cast<std::uint64_t>(sp.h);
    const std::uint64_t cell = sizeof(double) * static_cast<std::uint64_t>(sp.slots);
    const std::int64_t total = cfg.steps * sp.S;
    std::vector<s1d_message> log;
    std::uint64_t round = 0;
    auto msg = [&](int src, int dst, std::uint64_t tag, std::uint64_t bytes) {
        s1d_message e{};
        e.round = round;
        e.source = src;
        e.dest = dst;
        e.tag = tag;
        e.bytes = bytes;
        log.push_back(e);
    };
    auto exchange = [&](std::uint64_t tag) {
        for (int r = 0; r < R; ++r) {
            msg(r, (r + R - 1) % R, tag, h * cell);
            msg(r, (r + 1) % R, tag, h * cell);
        }
        ++round;
    };
    auto tag_of = [](std::int64_t counter, std::uint64_t phase) {
        return (static_cast<std::uint64_t>(counter) << 3) | phase;
    };
    if (cfg.scheme == S1D_CLASSIC) {
        for (std::int64_t c = 1; c <= total; ++c) exchange(tag_of(c, 1));
    } else {
        const std::uint64_t m = cycle_advance(w, h);
        const std::int64_t cycles = total / static_cast<std::int64_t>(m);
        for (std::int64_t j = 1; j <= cycles; ++j) {
            const bool left = (j & 1) != 0;
            for (int r = 0; r < R; ++r)
                msg(r, left ? (r + R - 1) % R : (r + 1) % R, tag_of(j, left ? 2 : 3), (w / 2 + h) * cell);
            ++round;
        }
        for (std::int64_t c = cycles * static_cast<std::int64_t>(m) + 1; c <= total; ++c) exchange(tag_of(c, 5));
    }
    std::stable_sort(log.begin(), log.end(), [](const s1d_message& a, const s1d_message& b) {
        if (a.round != b.round) return a.round < b.round;
        if (a.source != b.source) return a.source < b.source;
        return a.dest < b.dest;
    });
    return log;
}

// RankCommStats per rank (transport.hpp:17-25): every rank takes part in
// every round, so the counters are the same for all ranks.
std::vector<s1d_rank_stats> rank_stats(const s1d_config& cfg) {
    const Spec sp = make_spec(cfg.equation, cfg.method);
    const std::uint64_t w = cfg.block_width;
    const std::uint64_t h = static_cast<std::uint64_t>(sp.h);
    const std::uint64_t cell = sizeof(double) * static_cast<std::uint64_t>(sp.slots);
    const std::int64_t total = cfg.steps * sp.S;
    s1d_rank_stats one{};
    auto round = [&](int msgs, std::uint64_t per_message) {
        one.messages_sent += static_cast<std::uint64_t>(msgs);
        one.bytes_sent += static_cast<std::uint64_t>(msgs) * per_message;
        one.exchange_rounds += 1;
        one.virtual_comm_seconds += cfg.alpha + cfg.beta * static_cast<double>(per_message);
    };
    if (cfg.scheme == S1D_CLASSIC) {
        for (std::int64_t c = 1; c <= total; ++c) round(2, h * cell);
    } else {
        const std::uint64_t m = cycle_advance(w, h);
        const std::int64_t cycles = total / static_cast<std::int64_t>(m);
        for (std::int64_t j = 1; j <= cycles; ++j) round(1, (w / 2 + h) * cell);
        for (std::int64_t c = cycles * static_cast<std::int64_t>(m) + 1; c <= total; ++c) round(2, h * cell);
    }
    return std::vector<s1d_rank_stats>(static_cast<std::size_t>(cfg.ranks), one);
}

} // namespace s1d
