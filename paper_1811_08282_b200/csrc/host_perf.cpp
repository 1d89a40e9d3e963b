// Host-side measurement records, CSV and fits (no CUDA).
//
// Restates the reference's post-processing so B200 sweeps are reported in the
// same artefacts:
//   TimingRecord / make_record   inc/perf.hpp:16-29, src/perf.cpp:10-27
//   power_law_fit / best_config  src/perf.cpp:42-97 (log-log OLS, tie-breaks)
//   CSV header/row/emit/read     inc/csv.hpp:11-13, src/csv.cpp:14-136
//                                (%.12g, RFC-4180 quoting, config-lexicographic order)
//
// These are deliberate RESTATEMENTS of the reference's formatter and fit: the
// CSV must be byte-identical to emit_csv and the fit bit-identical to
// power_law_fit (tests/test_perf_csv.py), which pins the statement order. They
// sit off the hot path; the rest of the library is written in its own idiom.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "host_config.hpp"
#include "swept1d.h"

namespace s1d {
namespace {

const char* kHeader =
    "equation,method,scheme,n,w,wf,ranks,steps,mode,avg_us_per_step,msgs,bytes,rounds,virtual_comm_us,setup_us";

std::string eq_s(int e) { return e == S1D_HEAT ? "heat" : "euler"; }
std::string me_s(int m) { return m == S1D_LENGTHENING ? "lengthening" : "flattening"; }
std::string sc_s(int s) { return s == S1D_CLASSIC ? "classic" : "swept"; }
std::string mo_s(int m) { return m == S1D_WALL ? "wall" : "virtual"; }

std::string fmt_double(double v) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.12g", v);
    return buf;
}

std::string quoted(const std::string& f) {
    if (f.find_first_of(",\"\n") == std::string::npos) return f;
    std::string out = "\"";
    for (char c : f) {
        if (c == '"') out += '"';
        out += c;
    }
    return out + '"';
}

auto sort_key(const s1d_record& r) {
    return std::make_tuple(eq_s(r.equation), me_s(r.method), sc_s(r.scheme), r.grid_size, r.block_width,
                           r.work_factor, r.ranks, r.steps, mo_s(r.mode));
}

std::vector<std::string> split_row(const std::string& line) {
    std::vector<std::string> fields;
    std::string cur;
    bool inq = false;
    for (std::size_t i = 0; i < line.size(); ++i) {
        const char c = line[i];
        if (inq) {
            if (c == '"' && i + 1 < line.size() && line[i + 1] == '"') {
                cur += '"';
                ++i;
            } else if (c == '"') {
                inq = false;
            } else {
                cur += c;
            }
        } else if (c == '"') {
            inq = true;
        } else if (c == ',') {
            fields.push_back(cur);
            cur.clear();
        } else {
            cur += c;
        }
    }
    fields.push_back(cur);
    return fields;
}

int parse_enum(const std::string& v, const char* a, const char* b, const char* what) {
    if (v == a) return 0;
    if (v == b) return 1;
    throw Error(S1D_INVALID_CONFIG, std::string("unknown ") + what + " '" + v + "' in CSV");
}

} // namespace

std::string csv_row(const s1d_record& r) {
    std::ostringstream os;
    os << quoted(eq_s(r.equation)) << ',' << quoted(me_s(r.method)) << ',' << quoted(sc_s(r.scheme)) << ','
       << r.grid_size << ',' << r.block_width << ',' << r.work_factor << ',' << r.ranks << ',' << r.steps << ','
       << quoted(mo_s(r.mode)) << ',' << fmt_double(r.avg_us_per_step) << ',' << r.messages_sent << ','
       << r.bytes_sent << ',' << r.exchange_rounds << ',' << fmt_double(r.virtual_comm_us) << ','
       << fmt_double(r.setup_us);
    return os.str();
}

std::string emit_csv(std::vector<s1d_record> recs) {
    std::stable_sort(recs.begin(), recs.end(),
                     [](const s1d_record& a, const s1d_record& b) { return sort_key(a) < sort_key(b); });
    std::string out = std::string(kHeader) + "\n";
    for (const auto& r : recs) out += csv_row(r) + "\n";
    return out;
}

std::vector<s1d_record> read_csv(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Error(S1D_INVALID_CONFIG, "cannot open '" + path + "' for reading");
    std::string line;
    if (!std::getline(in, line)) throw Error(S1D_INVALID_CONFIG, "empty CSV '" + path + "'");
    std::vector<s1d_record> out;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        const auto f = split_row(line);
        if (f.size() != 15) throw Error(S1D_INVALID_CONFIG, "malformed CSV row in '" + path + "': " + line);
        s1d_record r{};
        r.equation = parse_enum(f[0], "heat", "euler", "equation");
        r.method = parse_enum(f[1], "lengthening", "flattening", "method");
        r.scheme = parse_enum(f[2], "classic", "swept", "scheme");
        r.grid_size = std::stoull(f[3]);
        r.block_width = std::stoull(f[4]);
        r.work_factor = std::stoi(f[5]);
        r.ranks = std::stoi(f[6]);
        r.steps = std::stoll(f[7]);
        r.mode = parse_enum(f[8], "wall", "virtual", "mode");
        r.avg_us_per_step = std::stod(f[9]);
        r.messages_sent = std::stoull(f[10]);
        r.bytes_sent = std::stoull(f[11]);
        r.exchange_rounds = std::stoull(f[12]);
        r.virtual_comm_us = std::stod(f[13]);
        r.setup_us = std::stod(f[14]);
        out.push_back(r);
    }
    return out;
}

void power_law_fit(const double* x, const double* y, std::size_t n, double* A, double* b, double* r2) {
    if (n < 3) throw Error(S1D_INVALID_CONFIG, "power_law_fit requires at least 3 points");
    double sx = 0.0, sy = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        if (!(x[i] > 0.0) || !(y[i] > 0.0)) throw Error(S1D_INVALID_CONFIG, "power_law_fit requires positive samples");
        sx += std::log(x[i]);
        sy += std::log(y[i]);
    }
    const double mx = sx / static_cast<double>(n), my = sy / static_cast<double>(n);
    double sxx = 0.0, sxy = 0.0, syy = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        const double dx = std::log(x[i]) - mx, dy = std::log(y[i]) - my;
        sxx += dx * dx;
        sxy += dx * dy;
        syy += dy * dy;
    }
    if (sxx == 0.0) throw Error(S1D_DEGENERATE_FIT, "power_law_fit: all grid sizes equal");
    *b = sxy / sxx;
    *A = std::exp(my - *b * mx);
    if (syy == 0.0) {
        *r2 = 1.0;
    } else {
        double ss = 0.0;
        for (std::size_t i = 0; i < n; ++i) {
            const double res = std::log(y[i]) - ((my - *b * mx) + *b * std::log(x[i]));
            ss += res * res;
        }
        *r2 = 1.0 - ss / syy;
    }
}

std::size_t best_config(const s1d_record* r, std::size_t n) {
    if (n == 0) throw Error(S1D_INVALID_CONFIG, "best_config over an empty record set");
    std::size_t best = 0;
    for (std::size_t i = 1; i < n; ++i) {
        const auto& a = r[i];
        const auto& c = r[best];
        const bool better = a.avg_us_per_step < c.avg_us_per_step ||
                            (a.avg_us_per_step == c.avg_us_per_step &&
                             (a.block_width < c.block_width ||
                              (a.block_width == c.block_width && a.work_factor < c.work_factor)));
        if (better) best = i;
    }
    return best;
}

} // namespace s1d

// ---------------------------------------------------------------------------
// C ABI (host-only entry points)
// ---------------------------------------------------------------------------
namespace {
void put(char* err, size_t errlen, const std::string& m) {
    if (!err || !errlen) return;
    const size_t n = std::min(errlen - 1, m.size());
    std::memcpy(err, m.data(), n);
    err[n] = 0;
}
template <class Fn>
int guard(char* err, size_t errlen, Fn&& fn) {
    try {
        fn();
        put(err, errlen, "");
        return S1D_OK;
    } catch (const s1d::Error& e) {
        put(err, errlen, e.what());
        return e.status;
    } catch (const std::exception& e) {
        put(err, errlen, e.what());
        return S1D_INTERNAL;
    }
}
} // namespace

extern "C" {

const char* s1d_csv_header(void) { return s1d::kHeader; }

// Returns the row length, -1 if buf is too small, or -status on an error
// (null arguments, an exception inside the formatter): nothing throws across
// the C boundary.
int64_t s1d_csv_row(const s1d_record* r, char* buf, size_t len) {
    int64_t n = -1;
    const int st = guard(nullptr, 0, [&] {
        if (!r || !buf) throw s1d::Error(S1D_INVALID_CONFIG, "null argument");
        const std::string row = s1d::csv_row(*r);
        if (row.size() + 1 > len) return;
        std::memcpy(buf, row.c_str(), row.size() + 1);
        n = static_cast<int64_t>(row.size());
    });
    return st == S1D_OK ? n : -static_cast<int64_t>(st);
}

int s1d_emit_csv(const s1d_record* recs, size_t n, const char* path, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        if ((!recs && n) || !path) throw s1d::Error(S1D_INVALID_CONFIG, "null argument");
        const std::string text = s1d::emit_csv(std::vector<s1d_record>(recs, recs + n));
        std::ofstream out(path, std::ios::trunc);
        if (!out) throw s1d::Error(S1D_INVALID_CONFIG, std::string("cannot open '") + path + "' for writing");
        out << text;
        out.flush();
        if (!out) throw s1d::Error(S1D_INVALID_CONFIG, std::string("write failed for '") + path + "'");
    });
}

int s1d_read_csv(const char* path, s1d_record* out, size_t cap, size_t* count, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        if (!path || !count || (!out && cap)) throw s1d::Error(S1D_INVALID_CONFIG, "null argument");
        const auto v = s1d::read_csv(path);
        *count = v.size();
        for (size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
    });
}

int s1d_power_law_fit(const double* n, const double* t, size_t count, double* A, double* b, double* r2, char* err,
                      size_t errlen) {
    return guard(err, errlen, [&] {
        if (!n || !t || !A || !b || !r2) throw s1d::Error(S1D_INVALID_CONFIG, "null argument");
        s1d::power_law_fit(n, t, count, A, b, r2);
    });
}

int64_t s1d_best_config(const s1d_record* recs, size_t n) {
    size_t idx = 0;
    const int st = guard(nullptr, 0, [&] {
        if (!recs && n) throw s1d::Error(S1D_INVALID_CONFIG, "null argument");
        idx = s1d::best_config(recs, n);
    });
    return st == S1D_OK ? static_cast<int64_t>(idx) : -st;
}

} // extern "C"
