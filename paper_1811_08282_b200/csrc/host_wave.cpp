// Issue order of the wavefront solve (engine.cu Solver::wavefront_phases),
// kept free of CUDA so its invariants can be checked on the host
// (s1d_debug_wave_schedule, tests/test_wave_schedule.py).
//
// Phases p = 0 (UpTriangle) .. cycles (DownTriangle); the first `head`
// Diamonds after the Up and the last `tail` before the Down run per chunk of
// tiles (K chunks on a ring), the Diamonds between them whole ("middle").
//   * a chunk (p, c), p >= 1, follows chunks c-1, c, c+1 of phase p-1 (the
//     first tail phase follows the middle);
//   * multi-process (xs): the end chunks 0 and K-1 of a phase follow the
//     whole previous phase and its round signal, and each pipelined phase's
//     signal follows its last chunk;
//   * head: Up chunks in copy order 0..K-1, each after every head Diamond
//     chunk that has become ready (so the Diamonds run while the next copy
//     lands);
//   * tail: Down chunks one at a time, each after the depth-first cone of
//     tail chunks it needs (xs: the chunks whose cones avoid end chunks
//     first).
#include <functional>

#include "host_config.hpp"

namespace s1d {

std::vector<WaveStep> wave_schedule(int K, int head, int tail, std::int64_t cycles, bool xs) {
    if (K < 3 || head < 0 || tail < 0 || cycles < head + tail + 2)
        throw Error(S1D_INVALID_CONFIG, "wavefront schedule: needs K >= 3 and cycles >= head + tail + 2");
    const std::int64_t tail0 = cycles - tail;
    auto slot = [&](std::int64_t p) { return p <= head ? static_cast<int>(p) : head + 1 + static_cast<int>(p - tail0); };
    auto wrap = [&](int c) { return ((c % K) + K) % K; };
    auto end_chunk = [&](int c) { return xs && (c == 0 || c == K - 1); };
    std::vector<char> done(static_cast<std::size_t>((head + tail + 2) * K), 0);
    auto is_done = [&](std::int64_t p, int c) -> char& { return done[static_cast<std::size_t>(slot(p) * K + wrap(c))]; };
    auto phase_done = [&](std::int64_t p) {
        for (int c = 0; c < K; ++c)
            if (!is_done(p, c)) return false;
        return true;
    };
    std::vector<WaveStep> steps;
    std::int64_t next_sig = 0;
    auto signal_ready = [&] {
        while (next_sig <= cycles && (next_sig <= head || next_sig >= tail0) && phase_done(next_sig)) {
            if (xs) steps.push_back({kWaveSignal, next_sig, 0});
            ++next_sig;
        }
    };
    auto issue = [&](std::int64_t p, int c) {
        steps.push_back({kWaveChunk, p, wrap(c)});
        is_done(p, c) = 1;
        signal_ready();
    };
    auto ready = [&](std::int64_t p, int c) {
        if (is_done(p, c)) return false;
        if (end_chunk(c)) return phase_done(p - 1);
        return is_done(p - 1, c - 1) && is_done(p - 1, c) && is_done(p - 1, c + 1);
    };
    auto drain = [&] {
        for (bool progress = true; progress;) {
            progress = false;
            for (std::int64_t p = 1; p <= head; ++p)
                for (int c = 0; c < K; ++c)
                    if (ready(p, c)) {
                        issue(p, c);
                        progress = true;
                    }
        }
    };
    for (int a = 0; a < K; ++a) {
        drain();
        issue(0, a);
    }
    drain();
    steps.push_back({kWaveMiddle, head + 1, 0}); // Diamonds head+1 .. tail0-1, whole
    next_sig = tail0;                            // the middle phases signal their own rounds
    std::function<void(std::int64_t, int)> need = [&](std::int64_t p, int c) {
        c = wrap(c);
        if (p < tail0 || is_done(p, c)) return;
        if (end_chunk(c) && p > tail0)
            for (int q = 0; q < K; ++q) need(p - 1, q);
        for (int d = -1; d <= 1; ++d) need(p - 1, c + d);
        issue(p, c);
    };
    std::vector<int> order;
    if (xs) {
        for (int c = tail; c <= K - 1 - tail; ++c) order.push_back(c);
        for (int c = 0; c < K; ++c)
            if (c < tail || c > K - 1 - tail) order.push_back(c);
    } else {
        for (int c = 0; c < K; ++c) order.push_back(c);
    }
    for (int c : order) need(cycles, c);
    return steps;
}

} // namespace s1d
