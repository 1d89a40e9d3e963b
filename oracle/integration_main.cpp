// TEST INFRASTRUCTURE ONLY. Drop-in check: the C++ shim of INTEGRATION.md
// (included verbatim) runs the reference's own sweep1d::LaunchConfig through
// the B200 library; each result must equal the reference's sweep1d::run_serial
// (compiled from source, oracle/_ref) bit for bit. Exit code = mismatches.
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
    };
    const Case cases[] = {
        {Equation::Heat, Method::Lengthening, Scheme::Swept, 16384, 64, 2, 1000},
        {Equation::Heat, Method::Lengthening, Scheme::Classic, 3072, 32, 3, 77},
        {Equation::Heat, Method::Lengthening, Scheme::Swept, 6144, 1024, 2, 333},
        {Equation::Euler, Method::Lengthening, Scheme::Swept, 4096, 64, 2, 250},
        {Equation::Euler, Method::Flattening, Scheme::Swept, 4096, 128, 4, 111},
        {Equation::Euler, Method::Lengthening, Scheme::Classic, 2048, 64, 2, 40},
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
        const std::vector<double> got = run_on_b200(c);
        const std::vector<double> want = run_serial(c);
        const bool ok = got.size() == want.size() &&
                        std::memcmp(got.data(), want.data(), got.size() * sizeof(double)) == 0;
        bad += !ok;
        std::printf("%s %s %s %s n=%zu w=%zu ranks=%d T=%ld\n", ok ? "ok " : "BAD", to_string(k.eq).c_str(),
                    to_string(k.me).c_str(), to_string(k.sc).c_str(), k.n, k.w, k.ranks, k.steps);
    }
    return bad;
}
