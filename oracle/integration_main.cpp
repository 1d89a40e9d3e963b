// TEST INFRASTRUCTURE ONLY. Drop-in check: the C++ shim of INTEGRATION.md
// (included verbatim) runs the reference's own sweep1d::LaunchConfig through
// the B200 library. Each RunResult must match the reference's (compiled from
// source, oracle/_ref): state == sweep1d::run_serial bit for bit; stats
// (totals and per_rank) and, in virtual mode, timing.virtual_seconds ==
// sweep1d::run's. Exit code = mismatches.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "sweep1d/engine.hpp"
#include "integration_shim.inc"

int main() {
    using namespace sweep1d;
    struct Case {
        Equation eq;
        Method me;
        Scheme sc;
        std::size_t n, w;
        int ranks;
        long steps;
        Mode mode;
    };
    const Case cases[] = {
        {Equation::Heat, Method::Lengthening, Scheme::Swept, 16384, 64, 2, 1000, Mode::WallClock},
        {Equation::Heat, Method::Lengthening, Scheme::Classic, 3072, 32, 3, 77, Mode::VirtualTime},
        {Equation::Heat, Method::Lengthening, Scheme::Swept, 6144, 1024, 2, 333, Mode::VirtualTime},
        {Equation::Euler, Method::Lengthening, Scheme::Swept, 4096, 64, 2, 250, Mode::WallClock},
        {Equation::Euler, Method::Flattening, Scheme::Swept, 4096, 128, 4, 111, Mode::VirtualTime},
        {Equation::Euler, Method::Lengthening, Scheme::Classic, 2048, 64, 2, 40, Mode::WallClock},
    };
    int bad = 0;
    for (const Case& k : cases) {
        LaunchConfig c;
        c.equation = k.eq;
        c.method = k.me;
        c.scheme = k.sc;
        c.grid_size = k.n;
        c.block_width = k.w;
        c.ranks = k.ranks;
        c.steps = k.steps;
        c.mode = k.mode;
        c.transport.alpha = 3e-6;
        c.transport.beta = 2e-10;
        const RunResult got = run_on_b200(c);
        const std::vector<double> want = run_serial(c);
        const RunResult ref = run(c);
        bool ok = got.state.size() == want.size() &&
                  std::memcmp(got.state.data(), want.data(), want.size() * sizeof(double)) == 0;
        ok = ok && got.stats.messages_sent == ref.stats.messages_sent &&
             got.stats.bytes_sent == ref.stats.bytes_sent && got.stats.exchange_rounds == ref.stats.exchange_rounds &&
             got.stats.virtual_comm_time == ref.stats.virtual_comm_time &&
             got.stats.per_rank.size() == ref.stats.per_rank.size();
        for (std::size_t r = 0; ok && r < ref.stats.per_rank.size(); ++r) {
            const auto& a = got.stats.per_rank[r];
            const auto& b = ref.stats.per_rank[r];
            ok = a.messages_sent == b.messages_sent && a.bytes_sent == b.bytes_sent &&
                 a.exchange_rounds == b.exchange_rounds && a.virtual_comm_time == b.virtual_comm_time;
        }
        if (k.mode == Mode::VirtualTime) ok = ok && got.timing.virtual_seconds == ref.timing.virtual_seconds;
        bad += !ok;
        std::printf("%s %s %s %s n=%zu w=%zu ranks=%d T=%ld\n", ok ? "ok " : "BAD", to_string(k.eq).c_str(),
                    to_string(k.me).c_str(), to_string(k.sc).c_str(), k.n, k.w, k.ranks, k.steps);
    }
    return bad;
}
