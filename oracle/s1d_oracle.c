/* TEST INFRASTRUCTURE ONLY — see s1d_oracle.h. A CPU restatement of the
 * reference serial solver, written independently in C over SoA arrays. Every
 * expression keeps the reference's evaluation order (compiled with
 * -ffp-contract=off) so results are bitwise comparable.
 */
#include "s1d_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* heat_step, inc/kernels.hpp:14-16: c + fo*((l - 2c) + r) */
double s1o_heat_step(double l, double c, double r, double fo) { return c + fo * ((l - 2.0 * c) + r); }

/* minmod, inc/kernels.hpp:20-25 (NaN operand falls through to 0). */
double s1o_minmod(double a, double b) {
    if (a * b > 0.0) return fabs(a) < fabs(b) ? a : b;
    return 0.0;
}

/* pressure_ratio_value, inc/kernels.hpp:33-40 (std::max(a,b) == a<b ? b : a). */
double s1o_pressure_ratio_value(double pl, double pc, double pr) {
    const double den = pr - pc;
    const double apc = fabs(pc), apr = fabs(pr);
    const double scale = apc < apr ? apr : apc;
    if (fabs(den) <= 1e-14 * scale) return NAN;
    return (pc - pl) / den;
}

/* pressure, src/kernels.cpp:27-36: (g-1)*(E - ((0.5*m)*m)/rho). */
static int pressure3(double rho, double mom, double ene, double gamma, double* out) {
    if (!(rho > 0.0)) return S1O_NONPHYSICAL;
    const double p = (gamma - 1.0) * (ene - 0.5 * mom * mom / rho);
    if (!(p > 0.0)) return S1O_NONPHYSICAL;
    *out = p;
    return S1O_OK;
}

int s1o_pressure(const double q[3], double gamma, double* out) { return pressure3(q[0], q[1], q[2], gamma, out); }

/* roe_signal_speed, src/kernels.cpp:43-54. */
static int roe_speed(const double* ql, const double* qr, double gamma, double* out) {
    const double srl = sqrt(ql[0]);
    const double srr = sqrt(qr[0]);
    const double inv = 1.0 / (srl + srr);
    const double u = (srl * (ql[1] / ql[0]) + srr * (qr[1] / qr[0])) * inv;
    const double e = (srl * (ql[2] / ql[0]) + srr * (qr[2] / qr[0])) * inv;
    const double por = (gamma - 1.0) * (e - 0.5 * u * u);
    if (!(por > 0.0)) return S1O_NONPHYSICAL;
    *out = fabs(u) + sqrt(gamma * por);
    return S1O_OK;
}

/* interface_flux, src/kernels.cpp:56-67 with physical_flux :38-41 and
 * limited_slope inc/kernels.hpp:48-52. */
int s1o_interface_flux(const double ql[3], const double qr[3], double pr_l, double pr_r, double gamma,
                       double out[3]) {
    double d[3], rl[3], rr[3], fl[3], fr[3];
    const double inv_r = 1.0 / pr_r;
    for (int k = 0; k < 3; ++k) {
        d[k] = qr[k] - ql[k];
        const double sl = s1o_minmod(d[k], pr_l * d[k]);
        const double sr = s1o_minmod(d[k], inv_r * d[k]);
        rl[k] = ql[k] + 0.5 * sl;
        rr[k] = qr[k] - 0.5 * sr;
    }
    double pl, pr, lam;
    int st = pressure3(rl[0], rl[1], rl[2], gamma, &pl);
    if (st) return st;
    st = pressure3(rr[0], rr[1], rr[2], gamma, &pr);
    if (st) return st;
    st = roe_speed(rl, rr, gamma, &lam);
    if (st) return st;
    const double ul = rl[1] / rl[0], ur = rr[1] / rr[0];
    fl[0] = rl[1];
    fl[1] = rl[1] * ul + pl;
    fl[2] = (rl[2] + pl) * ul;
    fr[0] = rr[1];
    fr[1] = rr[1] * ur + pr;
    fr[2] = (rr[2] + pr) * ur;
    for (int k = 0; k < 3; ++k) out[k] = 0.5 * (fl[k] + fr[k]) - 0.5 * (lam * (rr[k] - rl[k]));
    return S1O_OK;
}

/* ---- initial conditions, src/partition.cpp:54-113 ------------------------ */

static double sine_sample(size_t j, size_t n) {
    size_t k = j % n;
    double sign = 1.0;
    if (2 * k >= n) {
        sign = -1.0;
        k -= n / 2;
    }
    const size_t folded = (4 * k > n) ? (n / 2 - k) : k;
    return sign * sin(2.0 * M_PI * (double)folded / (double)n);
}

int s1o_initial_condition(const char* id, size_t n, int equation, double gamma, double* out) {
    if (equation == 0) {
        if (strcmp(id, "heat-sine") == 0) {
            for (size_t j = 0; j < n; ++j) out[j] = sine_sample(j, n);
        } else if (strcmp(id, "uniform") == 0) {
            for (size_t j = 0; j < n; ++j) out[j] = 1.0;
        } else {
            return S1O_UNKNOWN_IC;
        }
        return S1O_OK;
    }
    int sod = strcmp(id, "euler-sod-periodic") == 0;
    if (!sod && strcmp(id, "uniform") != 0) return S1O_UNKNOWN_IC;
    for (size_t j = 0; j < n; ++j) {
        double rho = 1.0, u = 0.0, p = 1.0;
        if (sod && !(2 * j < n)) {
            rho = 0.125;
            p = 0.1;
        }
        out[3 * j] = rho;
        out[3 * j + 1] = rho * u;
        out[3 * j + 2] = p / (gamma - 1.0) + 0.5 * rho * u * u;
    }
    return S1O_OK;
}

int s1o_max_signal_speed(const double* prim, size_t len, double gamma, double* out) {
    double best = 0.0;
    for (size_t j = 0; j + 2 < len; j += 3) {
        double p;
        const int st = pressure3(prim[j], prim[j + 1], prim[j + 2], gamma, &p);
        if (st) return st;
        const double u = prim[j + 1] / prim[j];
        const double s = fabs(u) + sqrt(gamma * p / prim[j]);
        best = best < s ? s : best;
    }
    *out = best;
    return S1O_OK;
}

/* ---- serial solver, engines_impl.hpp:85-128 ------------------------------ */

/* SoA working arrays of length n + 2h (h ghosts each side, periodic). */
typedef struct {
    double* f[7]; /* heat: T0,T1. euler: rho0,mom0,ene0,rho1,mom1,ene1,Pr */
    int nf;
    size_t len;
} soa_t;

static void refresh_halo(soa_t* a, size_t n, size_t h) {
    for (int f = 0; f < a->nf; ++f) {
        double* v = a->f[f];
        for (size_t k = 0; k < h; ++k) {
            v[k] = v[n + k];         /* left ghosts <- last h owned */
            v[h + n + k] = v[h + k]; /* right ghosts <- first h owned */
        }
    }
}

static void q_at(const soa_t* a, int slot, size_t i, double q[3]) {
    q[0] = a->f[3 * slot][i];
    q[1] = a->f[3 * slot + 1][i];
    q[2] = a->f[3 * slot + 2][i];
}

/* euler_flux_update, src/kernels.cpp:69-73 */
static int flux_update(const double* qm1, const double* q0, const double* qp1, double pm1, double p0, double pp1,
                       double gamma, double factor, const double* base, double out[3]) {
    double fl[3], fr[3];
    int st = s1o_interface_flux(qm1, q0, pm1, p0, gamma, fl);
    if (st) return st;
    st = s1o_interface_flux(q0, qp1, p0, pp1, gamma, fr);
    if (st) return st;
    for (int k = 0; k < 3; ++k) out[k] = base[k] - factor * (fr[k] - fl[k]);
    return S1O_OK;
}

static int len_apply(soa_t* a, size_t i, long c, double gamma, double dt_dx) {
    if (c & 1) { /* pressure_ratio_substep, src/kernels.cpp:90-95 */
        const int slot = (c & 3) == 1 ? 0 : 1;
        double q[3], pl, pc, pr;
        int st;
        q_at(a, slot, i - 1, q);
        if ((st = pressure3(q[0], q[1], q[2], gamma, &pl))) return st;
        q_at(a, slot, i, q);
        if ((st = pressure3(q[0], q[1], q[2], gamma, &pc))) return st;
        q_at(a, slot, i + 1, q);
        if ((st = pressure3(q[0], q[1], q[2], gamma, &pr))) return st;
        a->f[6][i] = s1o_pressure_ratio_value(pl, pc, pr);
        return S1O_OK;
    }
    /* euler_flux_substep, src/kernels.cpp:97-105 */
    const int final_stage = (c & 3) == 0;
    const int rs = final_stage ? 1 : 0, ws = final_stage ? 0 : 1;
    const double factor = final_stage ? dt_dx : 0.5 * dt_dx;
    double qm1[3], q0[3], qp1[3], base[3], out[3];
    q_at(a, rs, i - 1, qm1);
    q_at(a, rs, i, q0);
    q_at(a, rs, i + 1, qp1);
    q_at(a, 0, i, base);
    const int st = flux_update(qm1, q0, qp1, a->f[6][i - 1], a->f[6][i], a->f[6][i + 1], gamma, factor, base, out);
    if (st) return st;
    for (int k = 0; k < 3; ++k) a->f[3 * ws + k][i] = out[k];
    return S1O_OK;
}

/* flattened_euler_step / _substep, src/kernels.cpp:107-125 */
static int flat_apply(soa_t* a, size_t i, long c, double gamma, double dt_dx) {
    const int final_stage = (c & 1) == 0;
    const int slot = final_stage ? 1 : 0;
    double p[5], q[3];
    for (int k = 0; k < 5; ++k) {
        q_at(a, slot, i - 2 + (size_t)k, q);
        const int st = pressure3(q[0], q[1], q[2], gamma, &p[k]);
        if (st) return st;
    }
    double qm1[3], q0[3], qp1[3], base[3], out[3];
    q_at(a, slot, i - 1, qm1);
    q_at(a, slot, i, q0);
    q_at(a, slot, i + 1, qp1);
    q_at(a, 0, i, base);
    const double factor = final_stage ? dt_dx : 0.5 * dt_dx;
    const int st = flux_update(qm1, q0, qp1, s1o_pressure_ratio_value(p[0], p[1], p[2]),
                               s1o_pressure_ratio_value(p[1], p[2], p[3]),
                               s1o_pressure_ratio_value(p[2], p[3], p[4]), gamma, factor, base, out);
    if (st) return st;
    const int ws = final_stage ? 0 : 1;
    for (int k = 0; k < 3; ++k) a->f[3 * ws + k][i] = out[k];
    return S1O_OK;
}

int s1o_run_serial(int equation, int method, size_t n, long steps, double fourier, double gamma, double dt_dx,
                   double cfl, const char* initial, double* out) {
    const int heat = equation == 0;
    const int flat = !heat && method == 1;
    const size_t h = flat ? 2 : 1;
    const int vpp = heat ? 1 : 3;
    /* LaunchConfig::validate(partitioned=false), src/config.cpp:45-62 */
    if (n < 2 * h + 1 || steps < 0 || !(fourier > 0.0) || fourier > 0.5 || !(gamma > 1.0)) return S1O_INVALID_CONFIG;
    const char* id = (initial && initial[0]) ? initial : (heat ? "heat-sine" : "euler-sod-periodic");

    double* ic = (double*)malloc(sizeof(double) * n * (size_t)vpp);
    int st = s1o_initial_condition(id, n, equation, gamma, ic);
    if (st) {
        free(ic);
        return st;
    }
    if (!heat && dt_dx == 0.0) { /* LaunchConfig::finalize, src/config.cpp:97-103 */
        double smax;
        st = s1o_max_signal_speed(ic, n * 3, gamma, &smax);
        if (st) {
            free(ic);
            return st;
        }
        dt_dx = cfl / smax;
    }
    st = s1o_run_state(equation, method, n, steps, fourier, gamma, dt_dx, ic, out);
    free(ic);
    return st;
}

/* serial_advance (engines_impl.hpp:85-128) from a given state. */
int s1o_run_state(int equation, int method, size_t n, long steps, double fourier, double gamma, double dt_dx,
                  const double* ic, double* out) {
    const int heat = equation == 0;
    const int flat = !heat && method == 1;
    const size_t h = flat ? 2 : 1;
    const long S = heat ? 1 : (flat ? 2 : 4);
    if (n < 2 * h + 1 || steps < 0) return S1O_INVALID_CONFIG;

    soa_t a;
    a.nf = heat ? 2 : (flat ? 6 : 7);
    a.len = n + 2 * h;
    for (int f = 0; f < a.nf; ++f) a.f[f] = (double*)calloc(a.len, sizeof(double));
    for (size_t j = 0; j < n; ++j) {
        if (heat) {
            a.f[0][h + j] = a.f[1][h + j] = ic[j]; /* HeatModel::make_cell */
        } else {
            for (int k = 0; k < 3; ++k) a.f[k][h + j] = a.f[3 + k][h + j] = ic[3 * j + (size_t)k];
        }
    }

    const long total = steps * S;
    int st = S1O_OK;
    for (long c = 1; c <= total && !st; ++c) {
        refresh_halo(&a, n, h);
        if (heat) {
            const int ws = (int)(c & 1), rs = ws ^ 1;
            const double* r = a.f[rs];
            double* w = a.f[ws];
            for (size_t i = h; i < h + n; ++i) w[i] = s1o_heat_step(r[i - 1], r[i], r[i + 1], fourier);
        } else {
            for (size_t i = h; i < h + n && !st; ++i)
                st = flat ? flat_apply(&a, i, c, gamma, dt_dx) : len_apply(&a, i, c, gamma, dt_dx);
        }
    }
    if (!st) {
        for (size_t j = 0; j < n; ++j) {
            if (heat) {
                out[j] = a.f[total & 1][h + j]; /* HeatModel::extract */
            } else {
                for (int k = 0; k < 3; ++k) out[3 * j + (size_t)k] = a.f[k][h + j];
            }
        }
    }
    for (int f = 0; f < a.nf; ++f) free(a.f[f]);
    return st;
}

unsigned long long s1o_fnv1a64(const double* v, size_t count) {
    const unsigned char* b = (const unsigned char*)v;
    uint64_t hsh = 1469598103934665603ULL;
    for (size_t i = 0; i < count * sizeof(double); ++i) {
        hsh ^= b[i];
        hsh *= 1099511628211ULL;
    }
    return (unsigned long long)hsh;
}
