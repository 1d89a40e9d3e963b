// Device restatement of the reference Euler arithmetic (FP64), bit for bit.
//
// Every operation is an explicit round-to-nearest intrinsic in the
// reference's evaluation order, so no FMA contraction or reassociation can
// change a result (the reference builds with -ffp-contract=off). Division and
// square root are the IEEE correctly rounded __ddiv_rn / __dsqrt_rn, equal to
// x86-64 divsd/sqrtsd.
//
//   pressure            src/kernels.cpp:27-36
//   physical_flux       src/kernels.cpp:38-41
//   roe_signal_speed    src/kernels.cpp:43-54
//   interface_flux      src/kernels.cpp:56-67
//   minmod              inc/kernels.hpp:20-25
//   pressure_ratio_value inc/kernels.hpp:33-40
//   limited_slope       inc/kernels.hpp:48-52
//   euler_flux_update   src/kernels.cpp:69-73 (the base - f*(F_R - F_L) step)
//
// Non-physical states (the reference throws NonPhysicalState) set `bad`; the
// kernels OR it into a device flag that the host turns into S1D_NONPHYSICAL.
#pragma once

namespace s1d {
namespace em {

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
// IEEE division with the two special cases the Sod problem hits constantly
// resolved inline: 0/x (zero momentum on the plateaus) and NaN operands (the
// degenerate-ratio sentinel, 1/Pr). __ddiv_rn sends both to its out-of-line
// slow path (a third of all executed instructions before this). Results are
// bit-identical: 0/x (x finite, nonzero) is a zero whose sign is the XOR of
// the operand signs, and any NaN operand yields a NaN (payloads never reach a
// non-NaN value: a NaN ratio only feeds minmod, which returns 0).
__device__ __forceinline__ double dvd(double a, double b) {
    const long long ab = __double_as_longlong(a), bb = __double_as_longlong(b);
    const long long bm = bb & 0x7fffffffffffffffLL;
    if ((ab & 0x7fffffffffffffffLL) == 0 && bm != 0 && bm < 0x7ff0000000000000LL)
        return __longlong_as_double((ab ^ bb) & (long long)0x8000000000000000ULL);
    if (a != a) return a;
    if (b != b) return b;
    return __ddiv_rn(a, b);
}
// Call-site specialisations (same results as dvd): zero dividend with a
// positive finite divisor (momentum / density on the plateaus; density is
// checked positive by the caller's physicality test or is a sqrt sum), and
// a possibly-NaN divisor with dividend 1 (1/Pr).
__device__ __forceinline__ double dvd_z(double a, double b) {
    if (a == 0.0 && b > 0.0 && b < __longlong_as_double(0x7ff0000000000000LL))
        return __longlong_as_double(__double_as_longlong(a) & (long long)0x8000000000000000ULL);
    return __ddiv_rn(a, b);
}
__device__ __forceinline__ double rcp_n(double b) {
    if (b != b) return b;
    return __ddiv_rn(1.0, b);
}

// (g-1)*(E - ((0.5*m)*m)/rho); non-physical when !(rho > 0) or !(p > 0).
__device__ __forceinline__ double pressure(double rho, double mom, double ene, double gamma, bool& bad) {
    const double p = mul(sub(gamma, 1.0), sub(ene, dvd_z(mul(mul(0.5, mom), mom), rho)));
    bad |= !(rho > 0.0) || !(p > 0.0);
    return p;
}

__device__ __forceinline__ double minmod(double a, double b) {
    if (mul(a, b) > 0.0) return fabs(a) < fabs(b) ? a : b;
    return 0.0;
}

// std::max(a, b) == (a < b) ? b : a
__device__ __forceinline__ double ratio(double pl, double pc, double pr) {
    const double den = sub(pr, pc);
    const double apc = fabs(pc), apr = fabs(pr);
    const double scale = apc < apr ? apr : apc;
    if (fabs(den) <= mul(1e-14, scale)) return __longlong_as_double(0x7ff8000000000000LL); // quiet NaN
    return dvd(sub(pc, pl), den); // 0/den on one-sided plateaus
}

// Reconstructed Rusanov flux between cells L and R with stored ratios.
__device__ __forceinline__ void iflux(double lr, double lm, double le, double rr, double rm, double re, double pr_l,
                                      double pr_r, double gamma, double& f0, double& f1, double& f2, bool& bad) {
    const double inv_r = rcp_n(pr_r);
    const double d0 = sub(rr, lr), d1 = sub(rm, lm), d2 = sub(re, le);
    // recon_l = ql + 0.5*minmod(d, pr_l*d); recon_r = qr - 0.5*minmod(d, (1/pr_r)*d)
    const double al = add(lr, mul(0.5, minmod(d0, mul(pr_l, d0))));
    const double am = add(lm, mul(0.5, minmod(d1, mul(pr_l, d1))));
    const double ae = add(le, mul(0.5, minmod(d2, mul(pr_l, d2))));
    const double br = sub(rr, mul(0.5, minmod(d0, mul(inv_r, d0))));
    const double bm = sub(rm, mul(0.5, minmod(d1, mul(inv_r, d1))));
    const double be = sub(re, mul(0.5, minmod(d2, mul(inv_r, d2))));
    const double pl = pressure(al, am, ae, gamma, bad);
    const double pr = pressure(br, bm, be, gamma, bad);
    // Roe-averaged |u| + c
    const double srl = __dsqrt_rn(al), srr = __dsqrt_rn(br);
    const double ul = dvd_z(am, al), ur = dvd_z(bm, br); // also the physical fluxes' u
    const double inv = __ddiv_rn(1.0, add(srl, srr));
    const double u = mul(add(mul(srl, ul), mul(srr, ur)), inv);
    const double e = mul(add(mul(srl, __ddiv_rn(ae, al)), mul(srr, __ddiv_rn(be, br))), inv);
    const double por = mul(sub(gamma, 1.0), sub(e, mul(mul(0.5, u), u)));
    bad |= !(por > 0.0);
    const double lam = add(fabs(u), __dsqrt_rn(mul(gamma, por)));
    // physical fluxes
    const double fl0 = am, fl1 = add(mul(am, ul), pl), fl2 = mul(add(ae, pl), ul);
    const double fr0 = bm, fr1 = add(mul(bm, ur), pr), fr2 = mul(add(be, pr), ur);
    // 0.5*(fl + fr) - 0.5*(lam*(recon_r - recon_l))
    f0 = sub(mul(0.5, add(fl0, fr0)), mul(0.5, mul(lam, sub(br, al))));
    f1 = sub(mul(0.5, add(fl1, fr1)), mul(0.5, mul(lam, sub(bm, am))));
    f2 = sub(mul(0.5, add(fl2, fr2)), mul(0.5, mul(lam, sub(be, ae))));
}

// base - factor*(F_right - F_left)
__device__ __forceinline__ double update(double base, double factor, double fr, double fl) {
    return sub(base, mul(factor, sub(fr, fl)));
}

} // namespace em
} // namespace s1d
