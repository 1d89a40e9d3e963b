// s1d — command-line driver for the B200 swept solver (the reference's CLI is
// a stub, R/tools/main.cpp:1; this implements the subcommands SPEC.md
// "bench-cli" describes) on the C++ host interface include/swept1d.hpp.
//
//   s1d solve  [--config F] [key=value ...] [--dump F]  one run: CSV row + fingerprint
//   s1d verify [--config F] [--against DUMP] [--perturb-ulp] [key=value ...]
//                                                       swept vs classic vs serial oracle, bitwise
//   s1d sweep  --n N1,N2.. --w W1,W2.. [--wf A,B..] [--schemes swept,classic]
//              [key=value ...] --out F.csv              measure a grid, emit CSV
//   s1d fit    F.csv [--scheme swept|classic]            Table-1 power law over best configs
//   s1d report F.csv                                     best config per n + swept/classic speedup
//
// key=value keys are the reference's config-file keys (config.cpp:105-124):
// equation, method, scheme, n|grid_size, w|block_width, ranks, wf|work_factor,
// steps, initial, mode, fourier, gamma, cfl, alpha, beta, compute_cost
// (+ num_devices). Precedence: key=value arguments > --config file > defaults.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "swept1d.hpp"

using namespace swept1d;

namespace {

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    std::string cur;
    std::istringstream is(s);
    while (std::getline(is, cur, sep))
        if (!cur.empty()) out.push_back(cur);
    return out;
}

std::uint64_t parse_size(const std::string& v) {
    if (v.rfind("2^", 0) == 0) return 1ull << std::stoi(v.substr(2));
    return std::stoull(v);
}

void apply_file(LaunchConfig& cfg, const std::string& path) {
    std::ifstream in(path);
    if (!in) throw InvalidConfig("cannot open config file '" + path + "'");
    std::string line;
    int lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        const auto hash = line.find('#');
        if (hash != std::string::npos) line.erase(hash);
        std::string t;
        for (char ch : line)
            if (!std::isspace(static_cast<unsigned char>(ch))) t.push_back(ch);
        if (t.empty()) continue;
        const auto eq = t.find('=');
        if (eq == std::string::npos) throw InvalidConfig(path + ":" + std::to_string(lineno) + ": expected key=value");
        apply_config_entry(cfg, t.substr(0, eq), t.substr(eq + 1));
    }
}

struct Args {
    LaunchConfig cfg;
    std::map<std::string, std::string> flags;
    std::vector<std::string> positional;
};

Args parse(int argc, char** argv, int first) {
    Args a;
    a.cfg.ranks = 1;
    a.cfg.mode = Mode::WallClock;
    std::vector<std::pair<std::string, std::string>> kv;
    for (int i = first; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) == 0) {
            const std::string key = s.substr(2);
            const bool boolean = key == "perturb-ulp"; // takes no value
            if (!boolean && i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) a.flags[key] = argv[++i];
            else a.flags[key] = "1";
        } else if (s.find('=') != std::string::npos) {
            const auto eq = s.find('=');
            kv.emplace_back(s.substr(0, eq), s.substr(eq + 1));
        } else {
            a.positional.push_back(s);
        }
    }
    if (a.flags.count("config")) apply_file(a.cfg, a.flags["config"]);
    for (auto& [k, v] : kv) {
        if (k == "n" || k == "grid_size") v = std::to_string(parse_size(v));
        apply_config_entry(a.cfg, k, v);
    }
    return a;
}

std::uint64_t fnv1a64(const std::vector<double>& v) {
    std::uint64_t h = 1469598103934665603ull;
    const unsigned char* b = reinterpret_cast<const unsigned char*>(v.data());
    for (std::size_t i = 0; i < v.size() * sizeof(double); ++i) {
        h ^= b[i];
        h *= 1099511628211ull;
    }
    return h;
}

TimingRecord record_of(const LaunchConfig& cfg, const RunResult& r) {
    TimingRecord rec{};
    rec.equation = static_cast<int>(cfg.equation);
    rec.method = static_cast<int>(cfg.method);
    rec.scheme = static_cast<int>(cfg.scheme);
    rec.mode = static_cast<int>(cfg.mode);
    rec.grid_size = cfg.grid_size;
    rec.block_width = cfg.block_width;
    rec.work_factor = cfg.work_factor;
    rec.ranks = cfg.ranks;
    rec.steps = cfg.steps;
    rec.avg_us_per_step = cfg.steps > 0 ? r.timing.loop_seconds * 1e6 / static_cast<double>(cfg.steps) : 0.0;
    rec.setup_us = r.timing.setup_seconds * 1e6;
    rec.messages_sent = r.stats.messages_sent;
    rec.bytes_sent = r.stats.bytes_sent;
    rec.exchange_rounds = r.stats.exchange_rounds;
    return rec;
}

int cmd_solve(const Args& a) {
    const RunResult r = run(a.cfg);
    std::printf("%s\n%s\n", s1d_csv_header(), csv_row(record_of(a.cfg, r)).c_str());
    std::printf("fnv1a64: %016llx\n", static_cast<unsigned long long>(fnv1a64(r.state)));
    if (a.flags.count("dump")) {
        std::ofstream out(a.flags.at("dump"), std::ios::binary);
        out.write(reinterpret_cast<const char*>(r.state.data()),
                  static_cast<std::streamsize>(r.state.size() * sizeof(double)));
        if (!out) throw std::runtime_error("cannot write '" + a.flags.at("dump") + "'");
    }
    return 0;
}

// Bitwise comparison of two states: mismatch count and max |diff|, where a
// mismatch involving a NaN counts as an infinite difference.
struct Diff {
    std::size_t mismatches = 0;
    double max_abs = 0.0;
};

Diff compare(const std::vector<double>& a, const std::vector<double>& b) {
    Diff d;
    for (std::size_t i = 0; i < a.size(); ++i) {
        if (std::memcmp(&a[i], &b[i], sizeof(double)) == 0) continue;
        ++d.mismatches;
        const double x = std::isnan(a[i]) || std::isnan(b[i]) ? INFINITY : std::fabs(a[i] - b[i]);
        if (x > d.max_abs) d.max_abs = x;
    }
    return d;
}

bool report_pair(const char* what, const Diff& d, std::size_t n) {
    std::printf("%s: bitwise: %s, max|diff| = %.17g (%zu of %zu values differ)\n", what,
                d.mismatches == 0 ? "true" : "false", d.max_abs, d.mismatches, n);
    return d.mismatches == 0;
}

std::vector<double> read_dump(const std::string& path, std::size_t want) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw std::runtime_error("cannot open '" + path + "'");
    const auto bytes = static_cast<std::size_t>(in.tellg());
    if (bytes != want * sizeof(double))
        throw InvalidConfig("'" + path + "' holds " + std::to_string(bytes) + " bytes, " +
                            std::to_string(want * sizeof(double)) + " expected (n*vpp doubles)");
    std::vector<double> v(want);
    in.seekg(0);
    in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(bytes));
    if (!in) throw std::runtime_error("cannot read '" + path + "'");
    return v;
}

// SPEC.md bench-cli verify: swept vs classic vs the serial oracle, max |diff|
// and a bitwise flag per pair; non-zero exit on any difference, in
// particular on an injected 1-ulp kernel perturbation (--perturb-ulp, the
// reference's RunOptions::perturb_ulp, applied to the swept run). The serial
// leg is a dump of the reference's run_serial (--against FILE, written by
// oracle/dump_serial.py): the oracle is test infrastructure and is never
// linked into the product.
int cmd_verify(const Args& a) {
    LaunchConfig sw = a.cfg, cl = a.cfg;
    sw.scheme = Scheme::Swept;
    cl.scheme = Scheme::Classic;
    RunOptions opts;
    opts.perturb_ulp = a.flags.count("perturb-ulp") != 0;
    const RunResult rs = run(sw, opts), rc = run(cl);
    const std::size_t n = rs.state.size();
    if (opts.perturb_ulp) std::printf("swept run perturbed by 1 ulp (mutation hook)\n");
    bool ok = report_pair("swept vs classic", compare(rs.state, rc.state), n);
    if (a.flags.count("against")) {
        const auto ref = read_dump(a.flags.at("against"), n);
        const std::string p = a.flags.at("against");
        ok = report_pair(("swept vs serial oracle " + p).c_str(), compare(rs.state, ref), n) && ok;
        ok = report_pair(("classic vs serial oracle " + p).c_str(), compare(rc.state, ref), n) && ok;
    } else {
        std::printf("serial oracle: not given (--against DUMP, from oracle/dump_serial.py)\n");
    }
    std::printf("verify: %s\n", ok ? "PASS" : "FAIL");
    return ok ? 0 : 1;
}

int cmd_sweep(const Args& a) {
    if (!a.flags.count("out")) throw InvalidConfig("sweep: --out FILE.csv required");
    std::vector<std::uint64_t> ns, ws;
    std::vector<int> wfs{0};
    for (const auto& s : split(a.flags.count("n") ? a.flags.at("n") : std::to_string(a.cfg.grid_size), ','))
        ns.push_back(parse_size(s));
    for (const auto& s : split(a.flags.count("w") ? a.flags.at("w") : std::to_string(a.cfg.block_width), ','))
        ws.push_back(parse_size(s));
    if (a.flags.count("wf")) {
        wfs.clear();
        for (const auto& s : split(a.flags.at("wf"), ',')) wfs.push_back(std::stoi(s));
    }
    const auto schemes = split(a.flags.count("schemes") ? a.flags.at("schemes") : "swept,classic", ',');
    std::vector<TimingRecord> recs;
    for (auto n : ns)
        for (auto w : ws)
            for (int wf : wfs)
                for (const auto& sc : schemes) {
                    LaunchConfig c = a.cfg;
                    c.grid_size = n;
                    c.block_width = w;
                    c.work_factor = wf;
                    c.scheme = sc == "classic" ? Scheme::Classic : Scheme::Swept;
                    try {
                        run(c); // warm-up (module load, allocation paths)
                        recs.push_back(measure(c));
                        std::fprintf(stderr, "%s\n", csv_row(recs.back()).c_str());
                    } catch (const InvalidConfig& e) {
                        std::fprintf(stderr, "skip n=%llu w=%llu wf=%d %s: %s\n", (unsigned long long)n,
                                     (unsigned long long)w, wf, sc.c_str(), e.what());
                    }
                }
    emit_csv(recs, a.flags.at("out"));
    std::printf("wrote %zu records to %s\n", recs.size(), a.flags.at("out").c_str());
    return 0;
}

// best config per (equation, method, scheme, n)
std::map<std::string, std::vector<TimingRecord>> best_by_n(const std::vector<TimingRecord>& recs) {
    std::map<std::string, std::vector<TimingRecord>> groups;
    for (const auto& r : recs) {
        char key[128];
        std::snprintf(key, sizeof key, "%d/%d/%d/%020llu", r.equation, r.method, r.scheme,
                      (unsigned long long)r.grid_size);
        groups[key].push_back(r);
    }
    std::map<std::string, std::vector<TimingRecord>> best;
    for (auto& [k, v] : groups) {
        const TimingRecord& b = best_config(v);
        best[k.substr(0, k.rfind('/'))].push_back(b);
    }
    return best;
}

int cmd_fit(const Args& a) {
    if (a.positional.empty()) throw InvalidConfig("fit: CSV path required");
    const auto recs = read_csv(a.positional[0]);
    const std::string want = a.flags.count("scheme") ? a.flags.at("scheme") : "";
    for (const auto& [k, v] : best_by_n(recs)) {
        const int scheme = v.front().scheme;
        if (!want.empty() && (want == "swept") != (scheme == S1D_SWEPT)) continue;
        std::vector<std::pair<double, double>> pts;
        for (const auto& r : v) pts.emplace_back(static_cast<double>(r.grid_size), r.avg_us_per_step);
        if (pts.size() < 3) {
            std::printf("%s: %zu grid sizes (need 3 for a fit)\n", k.c_str(), pts.size());
            continue;
        }
        const FitResult f = power_law_fit(pts);
        std::printf("%s %s %s: us/step = %.6g * n^%.6g  (R^2 = %.6f, %zu sizes)\n",
                    v.front().equation == S1D_HEAT ? "heat" : "euler",
                    v.front().method == S1D_LENGTHENING ? "lengthening" : "flattening",
                    scheme == S1D_SWEPT ? "swept" : "classic", f.A, f.b, f.r_squared, pts.size());
    }
    return 0;
}

int cmd_report(const Args& a) {
    if (a.positional.empty()) throw InvalidConfig("report: CSV path required");
    const auto recs = read_csv(a.positional[0]);
    std::map<std::uint64_t, std::pair<const TimingRecord*, const TimingRecord*>> by_n; // classic, swept
    std::vector<TimingRecord> store;
    for (const auto& [k, v] : best_by_n(recs)) store.insert(store.end(), v.begin(), v.end());
    std::printf("%-8s %-12s %-8s %12s %6s %14s %14s\n", "equation", "method", "scheme", "n", "w", "us/step",
                "Mpt-upd/s");
    for (const auto& r : store) {
        std::printf("%-8s %-12s %-8s %12llu %6llu %14.3f %14.1f\n", r.equation == S1D_HEAT ? "heat" : "euler",
                    r.method == S1D_LENGTHENING ? "lengthening" : "flattening",
                    r.scheme == S1D_SWEPT ? "swept" : "classic", (unsigned long long)r.grid_size,
                    (unsigned long long)r.block_width, r.avg_us_per_step,
                    static_cast<double>(r.grid_size) / r.avg_us_per_step);
        auto& slot = by_n[r.grid_size * 4 + static_cast<std::uint64_t>(r.equation * 2 + r.method)];
        (r.scheme == S1D_SWEPT ? slot.second : slot.first) = &r;
    }
    for (const auto& [k, p] : by_n)
        if (p.first && p.second)
            std::printf("speedup swept/classic n=%llu: %.3f\n", (unsigned long long)p.first->grid_size,
                        speedup(p.first->avg_us_per_step, p.second->avg_us_per_step));
    return 0;
}

int usage() {
    std::fprintf(stderr,
                 "usage: s1d solve|verify|sweep|fit|report [options] [key=value ...]\n"
                 "  solve  [--config F] [--dump F] key=value...\n"
                 "  verify [--config F] [--against DUMP] [--perturb-ulp] key=value...\n"
                 "  sweep  --n 2^20,2^22 --w 64,1024 [--wf 0,2] [--schemes swept,classic] --out F.csv key=value...\n"
                 "  fit    F.csv [--scheme swept|classic]\n"
                 "  report F.csv\n"
                 "keys: equation method scheme n w ranks wf steps initial mode fourier gamma cfl alpha beta "
                 "compute_cost num_devices\n");
    return 2;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    if (cmd == "-h" || cmd == "--help" || cmd == "help") {
        usage();
        return 0;
    }
    try {
        const Args a = parse(argc, argv, 2);
        if (cmd == "solve") return cmd_solve(a);
        if (cmd == "verify") return cmd_verify(a);
        if (cmd == "sweep") return cmd_sweep(a);
        if (cmd == "fit") return cmd_fit(a);
        if (cmd == "report") return cmd_report(a);
        return usage();
    } catch (const Sweep1dError& e) {
        std::fprintf(stderr, "s1d %s: error (status %d): %s\n", cmd.c_str(), e.status, e.what());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "s1d %s: error: %s\n", cmd.c_str(), e.what());
        return 1;
    }
}
