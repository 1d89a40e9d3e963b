/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into, loaded by, or
 * called from the product path (paper_1811_08282_b200/). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may use it, and only as the checker.
 *
 * Plain-C restatement of the reference's serial solver
 * (/root/reference/proj/core/include/sweep1d/detail/engines_impl.hpp:85-128)
 * and the per-point kernels it applies (src/kernels.cpp, inc/kernels.hpp),
 * plus the initial conditions (src/partition.cpp:54-113).
 *
 * Parity pinned: tests/test_oracle.py checks this restatement bitwise against
 * (a) the reference compiled from source (oracle/_ref/libsweep1d_ref.so) and
 * (b) the committed golden fixtures in tests/golden/ (reference KATs and the
 * survey's FNV-1a fingerprints).
 */
#ifndef S1D_ORACLE_H
#define S1D_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: identical numbering to include/swept1d.h (S1D_*). */
enum {
    S1O_OK = 0,
    S1O_INVALID_CONFIG = 1,
    S1O_UNKNOWN_IC = 2,
    S1O_NONPHYSICAL = 3,
};

double s1o_heat_step(double l, double c, double r, double fo);
double s1o_minmod(double a, double b);
double s1o_pressure_ratio_value(double pl, double pc, double pr);
int s1o_pressure(const double q[3], double gamma, double* out);
int s1o_interface_flux(const double ql[3], const double qr[3], double pr_l, double pr_r, double gamma,
                       double out[3]);

/* Initial condition: vpp doubles per point (1 heat, 3 euler). equation 0/1. */
int s1o_initial_condition(const char* id, size_t n, int equation, double gamma, double* out);
int s1o_max_signal_speed(const double* prim, size_t len, double gamma, double* out);

/* Serial periodic solver. equation 0 heat / 1 euler; method 0 len / 1 flat.
 * dt_dx == 0 for Euler derives cfl / max_signal_speed(IC) (config.cpp:97-103).
 * `initial` NULL or "" selects the per-equation default. out: n*vpp doubles. */
int s1o_run_serial(int equation, int method, size_t n, long steps, double fourier, double gamma,
                   double dt_dx, double cfl, const char* initial, double* out);

/* The same periodic solver from a caller-given state (n*vpp doubles) with an
 * explicit dt_dx (no finalize): the windowed full-size parity tests run it on
 * a point's dependency cone. */
int s1o_run_state(int equation, int method, size_t n, long steps, double fourier, double gamma, double dt_dx,
                  const double* ic, double* out);

/* FNV-1a 64 over the little-endian bytes of `count` doubles. */
unsigned long long s1o_fnv1a64(const double* v, size_t count);

#ifdef __cplusplus
}
#endif
#endif
