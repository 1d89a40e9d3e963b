// Heat-equation (FTCS, 3-point) kernels for sm_100a, FP64.
//
//   heat_classic_kernel   one substep per launch, the naive comparison and the
//                         swept pad (reference classic_worker,
//                         engines_impl.hpp:201-213)
//   heat_tile_kernel<Q,K> one swept phase: K = Up (UpTriangle,
//                         engines_impl.hpp:280-291), Diamond (:293-307) or
//                         Down (DownTriangle, last cycle). Boundary tiles read
//                         their neighbour shard's edge directly (SplitDiamond).
//
// The point update is heat_step (inc/kernels.hpp:14-16),
//   T' = c + Fo*((l - 2c) + r),
// evaluated with explicit round-to-nearest intrinsics so no FMA contraction
// can change a bit (the reference builds with -ffp-contract=off).
//
// Production tiles (heat_tile_kernel<Q,K>) use
// the folded slot-major layout described above the kernel: each thread holds
// Q = P/2 point pairs symmetric about the tile centre, so the busy threads of
// every level are a prefix of warps. Per level: publish first/last pair to
// shared memory, one barrier, 5P FP64 ops from registers.
//
// Edges: the left producer's R edges and the right producer's L edges (2
// values per level each) go through a shared-memory ring per tile. Short
// tiles (m <= 32) load the whole edge at once with cp.async and stage their
// exports for one coalesced write-back; longer tiles stream the ring
// (cp.async, kRing-2 levels ahead). Inserts reload the two entering distances
// per side, exports store the two leaving ones.
//
// The instrumented debug kernel (heat_tile_debug_kernel) keeps an
// independent contiguous layout (thread lt owns x = 1 + lt*P + k) with plain
// level loops, so debug runs cross-check the production geometry.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "device_util.cuh"
#include "kernels.hpp"

namespace s1d {
namespace {

__device__ __forceinline__ double heat_f(double l, double c, double r, double fo) {
    return __dadd_rn(c, __dmul_rn(fo, __dadd_rn(__dsub_rn(l, __dmul_rn(2.0, c)), r)));
}

// The tile kernels' fast form: 4 FP64 instructions instead of 5, bit for bit
// the same result whenever 2c does not overflow. 2c is exact (a power-of-two
// scaling; subnormals included), so l - 2c rounded once (the reference's
// separately rounded sub of an exact product) equals fma(-2, c, l) rounded
// once; signed zeros agree (checked case by case), and infinities/NaNs
// propagate alike. The only difference is |c| >= 2^1023, where 2c overflows
// to inf in the reference but not inside the fma. The tile kernels therefore
// use this form only when no value of the launch can reach 2^1023: with
// 0 <= Fo <= 0.5 each FTCS step is a convex combination, so
// |T'| <= max(|l|,|c|,|r|) * (1 + 7*2^-53) after rounding, and a launch of at
// most 2m <= 16384 levels whose inputs (state or producer edges) all satisfy
// |v| < 2^1022 keeps every value below 2^1022 * (1 + 2^-35) < 2^1023
// (intermediates: |l - 2c| <= 3M, |(l - 2c) + r| <= 4M < 2^1024). Any other
// launch (a NaN/inf or |v| >= 2^1022 input, or Fo outside [0, 0.5]) runs
// heat_f. The check reads every input once (tile_inputs_fit).
template <bool FU>
__device__ __forceinline__ double heat_step(double l, double c, double r, double fo) {
    if (FU) return __dadd_rn(c, __dmul_rn(fo, __dadd_rn(__fma_rn(-2.0, c, l), r)));
    return heat_f(l, c, r, fo);
}

// |v| >= 2^1022, inf or NaN (biased exponent >= 0x7fd)
__device__ __forceinline__ bool too_big(double v) { return (__double2hiint(v) & 0x7fffffff) >= 0x7fd00000; }
__device__ __forceinline__ int ld_flag(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

__global__ void __launch_bounds__(256) heat_classic_kernel(const ClassicArgs a) {
    // Two points per thread (N is a multiple of the even block width). Only the
    // threads owning points 0 and N-1 touch the neighbours: they wait for the
    // neighbour's previous round (one process per GPU), read the halo, and
    // signal this round once their boundary value is stored.
    const std::uint64_t pairs = a.N >> 1;
    const double fo = a.fourier;
    for (std::uint64_t p = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; p < pairs;
         p += (std::uint64_t)gridDim.x * blockDim.x) {
        const std::uint64_t i = p << 1;
        const double2 c = __ldg(reinterpret_cast<const double2*>(a.in) + p);
        double l, r;
        if (i > 0) {
            l = __ldg(a.in + i - 1);
        } else {
            if (a.nb_flags) flag_wait(a.nb_flags, *a.seq_base + a.round, a.error_flag, a.timeout_ns);
            l = *a.halo_l;
        }
        if (i + 2 < a.N) {
            r = __ldg(a.in + i + 2);
        } else {
            if (a.nb_flags) flag_wait(a.nb_flags + 1, *a.seq_base + a.round, a.error_flag, a.timeout_ns);
            r = *a.halo_r;
        }
        double2 o;
        o.x = heat_f(l, c.x, c.y, fo);
        o.y = heat_f(c.x, c.y, r, fo);
        if (a.dbg.perturb && a.counter == 1 && i == 0) o.x = next_up(o.x); // debug runs only
        if (a.dbg.cov) {
            unsigned* row = a.dbg.cov + (std::uint64_t)(a.counter - 1) * a.dbg.cov_n;
            atomicAdd(row + (a.dbg.gstart + i) % a.dbg.cov_n, 1u);
            atomicAdd(row + (a.dbg.gstart + i + 1) % a.dbg.cov_n, 1u);
        }
        reinterpret_cast<double2*>(a.out)[p] = o;
        if (a.nb_flags) {
            if (i == 0) flag_signal(a.sig_left, *a.seq_base + a.round + 1);
            if (i + 2 >= a.N) flag_signal(a.sig_right, *a.seq_base + a.round + 1);
        }
    }
}

// Incoming edges stream through a per-tile ring of at most kRing levels (2
// values per level per side) filled with cp.async kRing-2 levels ahead of
// use, so shared memory per tile is O(1) in w (S1D_HEAT_RING: build knob).
#ifndef S1D_HEAT_RING
#define S1D_HEAT_RING 16
#endif
constexpr int kRing = S1D_HEAT_RING; // levels held per side (power of two)
constexpr int kRingMask = 2 * kRing - 1;

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Diagnostic builds (-DS1D_NO_LEVEL_BARRIER) replace the level barrier with
// __syncwarp() to time the level loop without it (results are then wrong);
// see level_sync.

// ---------------------------------------------------------------------------
// Production tile kernel: folded, slot-major layout.
//
// A tile's core x in [1, w] is folded about its centre (between x = w/2 and
// w/2+1): distance d pairs the left point x = w/2-d with the right point
// x = w/2+1+d. Every level's span is a distance prefix — [0, r) expanding,
// [0, m-d) contracting — so slot s (distances [sQ, sQ+Q), Q = P/2, both
// sides in registers vl[], vr[]) is busy exactly while sQ lies inside it.
// Thread t = s*G + g (g = tile in the CTA): a warp holds one slot of 32 tiles
// (G >= 32) or a few consecutive slots, so the busy threads are a prefix of
// warps and whole warps drop out as the span shrinks; no warp straddles a
// span edge on each side as in a contiguous x layout.
//
// Inserts (expanding level r: left R[r-1] = (x=lo-1, lo) = left distances
// (r, r-1); right L[r-1] = (x=hi-1, hi) = right distances (r-1, r)) and
// exports (contracting d: L[d] = left (m-1-d, m-2-d), R[d] = right
// (m-2-d, m-1-d), where "distance -1" is the other side's distance 0) fall in
// one slot row. Per level a thread publishes its first and last pair
// (double2) to shared memory, one barrier, then 5P FP64 ops from registers.
// Edge rings are tile-minor ([level*2+j][G], XOR-swizzled) so a slot row's
// insert reads hit distinct banks.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}

#ifndef S1D_HEAT_XPORT_LEVELS
#define S1D_HEAT_XPORT_LEVELS 32
#endif
constexpr int kXportLevels = S1D_HEAT_XPORT_LEVELS; // short tiles (XS builds): m <= this (w <= 64)

// Production rings hold pow2ceil(m) levels for short tiles (the whole edge,
// loaded at once; their shared-memory region is sized by the staged exports
// anyway) and kRing levels, streamed, for longer ones.
__host__ __device__ inline int ring_levels(int m) {
    if (m > kXportLevels) return kRing;
    int l = 1;
    while (l < m) l *= 2;
    return l;
}

// Ring element i (edge value index 2*level+j, wrapped by mask = 2*levels-1) of
// tile g; G is a power of two.
__device__ __forceinline__ int ridx(int i, int mask, int g, int G) {
    i &= mask;
    return i * G + (g ^ (i & (G - 1)));
}

template <int Q>
struct Fold {
    int m, G, s, g;      // levels, tiles per CTA, slot, tile in CTA
    int sa, sb;          // slot range of my warp (warp-uniform)
    double2* F;          // [2][(tt+2)G]: (vl[0], vr[0]) of slot s at (s+1)G+g
    double2* Lst;        // [2][(tt+2)G]: (vl[Q-1], vr[Q-1]) of slot s at (s+1)G+g
    int xs;              // parity stride (double2 elements)
    int rmask;           // ring index mask
    int* err;            // launch error flag (checked builds: bounds violations)
    const double* ringR; // left producer's R edges
    const double* ringL; // right producer's L edges
};

// One CTA barrier per level. (Neighbour-only synchronisation — hardware named
// barriers per pair of neighbour warps — was measured 23% slower, DESIGN.md
// section 8.) Diagnostic builds (-DS1D_NO_LEVEL_BARRIER) drop it.
__device__ __forceinline__ void level_sync() {
#ifdef S1D_NO_LEVEL_BARRIER
    __syncwarp();
#else
    __syncthreads();
#endif
}

template <int Q>
__device__ __forceinline__ void fpublish(const Fold<Q>& c, const double (&vl)[Q], const double (&vr)[Q], int r) {
    const int i = (r & 1) * c.xs + (c.s + 1) * c.G + c.g;
    S1D_CHECK(i >= 0 && i < 2 * c.xs, c.err);
    c.F[i] = make_double2(vl[0], vr[0]);
    c.Lst[i] = make_double2(vl[Q - 1], vr[Q - 1]);
}

template <int Q, bool FU>
__device__ __forceinline__ void fcompute(const Fold<Q>& c, double (&vl)[Q], double (&vr)[Q], int r, double fo) {
    const int par = (r & 1) * c.xs;
    const double2 in = c.Lst[par + c.s * c.G + c.g];      // slot s-1: distance sQ-1
    const double2 out = c.F[par + (c.s + 2) * c.G + c.g]; // slot s+1: distance sQ+Q
    S1D_CHECK(par + (c.s + 2) * c.G + c.g < 2 * c.xs, c.err);
    const double inL = c.s == 0 ? vr[0] : in.x;           // x+1 of left distance sQ
    const double inR = c.s == 0 ? vl[0] : in.y;           // x-1 of right distance sQ
    double nl[Q], nr[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        // right x = w/2+1+d: (x-1, x, x+1) = distances (d-1, d, d+1)
        nr[k] = heat_step<FU>(k == 0 ? inR : vr[k - 1], vr[k], k == Q - 1 ? out.y : vr[k + 1], fo);
        // left x = w/2-d: (x-1, x, x+1) = distances (d+1, d, d-1)
        nl[k] = heat_step<FU>(k == Q - 1 ? out.x : vl[k + 1], vl[k], k == 0 ? inL : vl[k - 1], fo);
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        vl[k] = nl[k];
        vr[k] = nr[k];
    }
}

// Expanding level r: distances r-1 and r from the rings (left value of
// distance e at ring index 2(r-1) + r - e, right at 2(r-1) + e - (r-1)).
// Distances beyond r are outside the dependency cone and take any value, so a
// one-sided predicate suffices.
template <int Q>
__device__ __forceinline__ void finsert(const Fold<Q>& c, double (&vl)[Q], double (&vr)[Q], int r) {
    const int d0 = c.s * Q;
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        if (d0 + k >= r - 1) {
            S1D_CHECK(ridx(3 * r - 2 - d0 - k, c.rmask, c.g, c.G) < (c.rmask + 1) * c.G &&
                          ridx(r - 1 + d0 + k, c.rmask, c.g, c.G) < (c.rmask + 1) * c.G,
                      c.err);
            vl[k] = c.ringR[ridx(3 * r - 2 - d0 - k, c.rmask, c.g, c.G)];
            vr[k] = c.ringL[ridx(r - 1 + d0 + k, c.rmask, c.g, c.G)];
        }
    }
}

// Contracting exports of level m+d (edge layout [level][2]).
template <int Q>
__device__ __forceinline__ void fexport(const Fold<Q>& c, const double (&vl)[Q], const double (&vr)[Q], int d,
                                        double* oL, double* oR, bool live) {
    const int d0 = c.s * Q, e1 = c.m - 1 - d, e2 = c.m - 2 - d;
    S1D_CHECK(d >= 0 && d < c.m, c.err); // edge slots 2d, 2d+1 of the tile's w = 2m
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        if (live && d0 + k == e1) {
            oL[2 * d] = vl[k];
            oR[2 * d + 1] = vr[k];
        }
        if (live && d0 + k == e2) {
            oL[2 * d + 1] = vl[k];
            oR[2 * d] = vr[k];
        }
    }
    if (live && e2 < 0 && c.s == 0) { // last level: (x=m, m+1) = (left 0, right 0)
        oL[2 * d + 1] = vr[0];
        oR[2 * d] = vl[0];
    }
}

// Level loops in segments with compile-time roles (control flow warp-uniform:
// the loops contain barriers; `live` only predicates stores).
// U: unroll of the long compute-only segments (lets the compiler rename the
// loop-carried registers instead of copying them; measured per width).
template <int Q, int U, bool FU, bool INS, bool CP, class Feed>
__device__ __forceinline__ void fexpand_seg(const Fold<Q>& c, double (&vl)[Q], double (&vr)[Q], int r0, int r1,
                                            double fo, Feed& feed) {
    constexpr int UN = (!INS && CP) ? U : 1;
#pragma unroll UN
    for (int r = r0; r < r1; ++r) {
        if (INS) finsert(c, vl, vr, r);
        if (INS || CP) fpublish(c, vl, vr, r);
        feed(r);
        level_sync();
        if (CP) fcompute<Q, FU>(c, vl, vr, r, fo);
    }
}

// Expanding levels [r0, r1), span distances [0, r): idle below sa*Q, insert
// while r in [sa*Q, (sb+1)*Q], compute from sa*Q + 1.
template <int Q, int U, bool FU, class Feed>
__device__ __forceinline__ void fexpand(const Fold<Q>& c, double (&vl)[Q], double (&vr)[Q], int r0, int r1,
                                        double fo, Feed& feed) {
    const int a = c.sa * Q, bi = (c.sb + 1) * Q + 1;
    const int e0 = min(max(a, r0), r1), e1 = min(max(a + 1, r0), r1), e2 = min(max(bi, r0), r1);
    fexpand_seg<Q, U, FU, false, false>(c, vl, vr, r0, e0, fo, feed);
    fexpand_seg<Q, U, FU, true, false>(c, vl, vr, e0, e1, fo, feed);
    fexpand_seg<Q, U, FU, true, true>(c, vl, vr, e1, e2, fo, feed);
    fexpand_seg<Q, U, FU, false, true>(c, vl, vr, e2, r1, fo, feed);
}

// Expanding levels when a warp holds exactly one slot s (G >= 32 tiles per
// CTA, Q divides m: the fixed-width builds). Slot s inserts at levels
// r = sQ + j, j = 0..Q: only distances r-1 and r are new inside the
// dependency cone (larger ones are out of it and may hold anything, finsert),
// and with the level loop unrolled over j their registers (j-1, j) are
// compile-time: four ring loads from two indices instead of finsert's
// 2·Q predicated loads, each with its own swizzled index.
template <int Q, int U, bool FU, class Feed>
__device__ __forceinline__ void fexpand_slot(const Fold<Q>& c, double (&vl)[Q], double (&vr)[Q], int r0, int r1,
                                             double fo, Feed& feed) {
    const int a = c.s * Q;
    const int e0 = min(max(a, r0), r1), e2 = min(max(a + Q + 1, r0), r1);
    fexpand_seg<Q, U, FU, false, false>(c, vl, vr, r0, e0, fo, feed);
#pragma unroll
    for (int j = 0; j <= Q; ++j) {
        const int r = a + j;
        if (r >= e0 && r < e2) { // warp-uniform
            const int i0 = ridx(2 * r - 2, c.rmask, c.g, c.G), i1 = ridx(2 * r - 1, c.rmask, c.g, c.G);
            S1D_CHECK(i0 < (c.rmask + 1) * c.G && i1 < (c.rmask + 1) * c.G, c.err);
            if (j >= 1) { // distance r-1: left at ring index 2r-1, right at 2r-2
                vl[j >= 1 ? j - 1 : 0] = c.ringR[i1];
                vr[j >= 1 ? j - 1 : 0] = c.ringL[i0];
            }
            if (j < Q) { // distance r: left at 2r-2, right at 2r-1
                vl[j < Q ? j : 0] = c.ringR[i0];
                vr[j < Q ? j : 0] = c.ringL[i1];
            }
            fpublish(c, vl, vr, r);
            feed(r);
            level_sync();
            if (j >= 1) fcompute<Q, FU>(c, vl, vr, r, fo); // compute from sQ+1
        }
    }
    fexpand_seg<Q, U, FU, false, true>(c, vl, vr, e2, r1, fo, feed);
}

// The same when a warp holds NS > 1 consecutive slots (G = 32/NS tiles per
// CTA): the warp's insert levels are r = saQ + jw, jw = 0..NS·Q, and a lane
// of slot sa+q fills registers jw-qQ-1 and jw-qQ, compile-time for each q,
// chosen by the lane's q at run time (one predicated move per candidate).
template <int Q, int U, bool FU, int NS, class Feed>
__device__ __forceinline__ void fexpand_slots(const Fold<Q>& c, double (&vl)[Q], double (&vr)[Q], int r0, int r1,
                                              double fo, Feed& feed) {
    const int a = c.sa * Q, q = c.s - c.sa;
    const int e0 = min(max(a, r0), r1), e1 = min(max(a + 1, r0), r1), e2 = min(max(a + NS * Q + 1, r0), r1);
    fexpand_seg<Q, U, FU, false, false>(c, vl, vr, r0, e0, fo, feed);
#pragma unroll
    for (int jw = 0; jw <= NS * Q; ++jw) {
        const int r = a + jw;
        if (r >= e0 && r < e2) { // warp-uniform
            const int i0 = ridx(2 * r - 2, c.rmask, c.g, c.G), i1 = ridx(2 * r - 1, c.rmask, c.g, c.G);
            const double l1 = c.ringR[i1], r0v = c.ringL[i0], l0 = c.ringR[i0], r1v = c.ringL[i1];
#pragma unroll
            for (int qq = 0; qq < NS; ++qq) {
                constexpr int kQ = Q;
                const int j = jw - qq * kQ;
                if (q == qq) {
                    if (j >= 1 && j <= kQ) { // distance r-1
                        vl[(j >= 1 && j <= kQ) ? j - 1 : 0] = l1;
                        vr[(j >= 1 && j <= kQ) ? j - 1 : 0] = r0v;
                    }
                    if (j >= 0 && j < kQ) { // distance r
                        vl[(j >= 0 && j < kQ) ? j : 0] = l0;
                        vr[(j >= 0 && j < kQ) ? j : 0] = r1v;
                    }
                }
            }
            fpublish(c, vl, vr, r);
            feed(r);
            level_sync();
            if (r >= e1) fcompute<Q, FU>(c, vl, vr, r, fo);
        }
    }
    fexpand_seg<Q, U, FU, false, true>(c, vl, vr, e2, r1, fo, feed);
}

template <int Q, int U, bool FU, bool PB, bool CP, bool EX>
__device__ __forceinline__ void fcontract_seg(const Fold<Q>& c, double (&vl)[Q], double (&vr)[Q], int r0, int r1,
                                              double fo, double* oL, double* oR, bool live) {
    constexpr int UN = (PB && CP && !EX) ? U : 1;
#pragma unroll UN
    for (int r = r0; r < r1; ++r) {
        if (PB) fpublish(c, vl, vr, r);
        level_sync();
        if (CP) fcompute<Q, FU>(c, vl, vr, r, fo);
        if (EX) fexport(c, vl, vr, r - c.m, oL, oR, live);
    }
}

// Contracting levels [r0, r1), r = m+d, span distances [0, m-d): compute
// while r <= 2m-1-sa*Q, export from 2m-1-(sb+1)*Q on, publish one level longer.
template <int Q, int U, bool FU>
__device__ __forceinline__ void fcontract(const Fold<Q>& c, double (&vl)[Q], double (&vr)[Q], int r0, int r1,
                                          double fo, double* oL, double* oR, bool live) {
    const int rce = 2 * c.m - 1 - c.sa * Q, ae = 2 * c.m - 1 - (c.sb + 1) * Q;
    const int e0 = min(max(ae, r0), r1), e1 = min(max(rce + 1, r0), r1), e2 = min(max(rce + 2, r0), r1);
    fcontract_seg<Q, U, FU, true, true, false>(c, vl, vr, r0, e0, fo, oL, oR, live);
    fcontract_seg<Q, U, FU, true, true, true>(c, vl, vr, e0, e1, fo, oL, oR, live);
    fcontract_seg<Q, U, FU, true, false, false>(c, vl, vr, e1, e2, fo, oL, oR, live);
    fcontract_seg<Q, U, FU, false, false, false>(c, vl, vr, e2, r1, fo, oL, oR, live);
}

// Shared memory (doubles): exchange 8*(tt+2)*G, then one region reused in turn:
// ring 4*levels*G (Diamond/Down), state staging G*(w+1) (Up/Down) and, for
// short tiles, export staging 2*G*(w+1) (Up/Diamond, after the last ring read).
// Slots of a folded tile: ceil(m / Q) with m = w/2 distances per side and
// Q = P/2 per slot. When Q does not divide m, the last slot's top distances
// (>= m) are padding: outside every level's span (no export reads them) and
// filled by the inserts' one-sided predicate; distance m itself, the halo of
// level m, then lives in a register instead of slot tt's exchange entry.
__host__ __device__ inline int fold_slots(int w, int P) { return (w / 2 + P / 2 - 1) / (P / 2); }

__host__ __device__ inline std::size_t fold_smem_doubles(int kind, int w, int P, int G) {
    const std::size_t tt = (std::size_t)fold_slots(w, P);
    const std::size_t ring = kind != kUp ? 4 * (std::size_t)ring_levels(w / 2) * G : 0;
    const std::size_t stage = kind != kDiamond ? (std::size_t)G * (w + 1) : 0;
    // short tiles stage their exports ([2][G][w+1]) in the same region
    const std::size_t xport = kind != kDown && w / 2 <= kXportLevels ? 2 * (std::size_t)G * (w + 1) : 0; // XS builds
    std::size_t region = ring > stage ? ring : stage;
    if (xport > region) region = xport;
    return 8 * (tt + 2) * G + region;
}

// MINB > 1 caps registers for occupancy (P = 8: 64 registers, 4 CTAs/SM, no
// spills; measured +4-10% over the uncapped build).
// XS: short-tile build (m <= kXportLevels): cp.async ring init and staged
// exports; wide tiles instantiate XS = false (code identical to before).
// One swept phase of the CTA's G tiles. FU: the fast build (heat_step<true>),
// followed in the same stream by the exact build gated on the shard's
// sticky flag *a.big_self ("a value >= 2^1022 may be here"):
//  * Up (inputs: the state): a CTA whose loaded state holds such a value
//    sets the flag and stops before writing anything;
//  * every CTA of a fast launch first reads its shard's and both ring
//    neighbours' flags and, if any is set, sets its own and stops.
// The exact build then recomputes the whole launch when the flag is set (the
// CTAs the fast build completed had small inputs, so their exact results are
// the same bits). Why this is enough: with 0 < Fo <= 0.5 every value of a
// solve is a convex combination of values one launch earlier (heat_step), so
// a launch's inputs can exceed 2^1022 only if an Up input did, and a launch
// reads edges only from its own shard and its ring neighbours, whose flags
// were final when their previous launch completed (the launch waits for it).
// Without a.big_self the exact build runs ungated.
// WT > 0: the tile width as a compile-time constant (then tiles per CTA and
// every index stride fold into immediates).
template <int Q, int KIND, int MAXT, int MINB, int U, bool XS, bool FU, int WT = 0>
__global__ void __launch_bounds__(MAXT, MINB) heat_tile_kernel(const TileArgs a, int G) {
    extern __shared__ __align__(16) double sm[];
    if (!FU && a.big_self && ld_flag(a.big_self) == 0) return; // the fast build computed every CTA
    const int w = WT ? WT : a.w, m = WT ? WT / 2 : a.m;
    if (WT) G = MAXT / ((WT / 2 + Q - 1) / Q);
    const int tt = (m + Q - 1) / Q; // slots per tile (fold_slots)
    const int nt = tt * G;
    const int t = threadIdx.x;
    const int s = t / G, g = t - s * G;
    const int bfirst = a.b0 + blockIdx.x * G; // first tile of this CTA
    const int bend = a.b1 < 0 ? a.nb : a.b1;
    const int ntiles = min(G, bend - bfirst);
    const int b = bfirst + g;
    const bool live = g < ntiles;
    const double fo = a.fourier;

    Fold<Q> c;
    c.m = m;
    c.G = G;
    c.s = s;
    c.g = g;
    c.xs = (tt + 2) * G;
    c.F = reinterpret_cast<double2*>(sm);
    c.Lst = c.F + 2 * c.xs;
    const int rl = ring_levels(m);
    const int rmask = 2 * rl - 1;
    c.rmask = rmask;
    c.err = a.error_flag;
    double* const region = sm + 8 * c.xs;
    double* const ringR = region; // [2*rl][G]
    double* const ringL = ringR + 2 * rl * G;
    double* const stage = region;        // Up/Down [G][w+1]
    c.ringR = ringR;
    c.ringL = ringL;
    {
        const unsigned full = __activemask();
        c.sa = (int)__reduce_min_sync(full, (unsigned)s);
        c.sb = (int)__reduce_max_sync(full, (unsigned)s);
    }
    const int ws = w + 1;
    double vl[Q], vr[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) vl[k] = vr[k] = 0.0;

    // FU: this shard or a ring neighbour may hold a value >= 2^1022 (flags,
    // monotone) or an Up input is one; made uniform at the CTA's first
    // barrier, before anything is written
    bool big = FU && (ld_flag(a.big_self) | ld_flag(a.big_left) | ld_flag(a.big_right)) != 0;
    if (KIND == kUp) { // coalesced staging of the CTA's ntiles*w contiguous points
        const double* src = a.state_in + (std::size_t)bfirst * w;
        for (int j = t; j < ntiles * w; j += nt) {
            const int gg = j / w;
            const double v = src[j];
            if (FU) big |= too_big(v);
            stage[gg * ws + (j - gg * w)] = v;
        }
        if (FU) {
            if (__syncthreads_or(big)) { // nothing written yet
                if (t == 0) atomicOr(a.big_self, 1); // sticky; propagates one shard per launch
                return;
            }
        } else {
            __syncthreads();
        }
        const double* my = stage + g * ws; // core x-1: left d at m-1-d, right d at m+d
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            if (s * Q + k < m) { // padding distances stay 0
                vl[k] = my[m - 1 - (s * Q + k)];
                vr[k] = my[m + s * Q + k];
            }
        }
    }

    // Edge sources: left producer's R edges and right producer's L edges.
    auto srcR = [&](int bb) -> const double* {
        if (a.seam) return a.in_R + (std::size_t)bb * w;
        return bb > 0 ? a.in_R + (std::size_t)(bb - 1) * w : a.peer_R;
    };
    auto srcL = [&](int bb) -> const double* {
        if (a.seam) return bb + 1 < a.nb ? a.in_L + (std::size_t)(bb + 1) * w : a.peer_L;
        return a.in_L + (std::size_t)bb * w;
    };
    const double* pR = nullptr;
    const double* pL = nullptr;
    const bool feeder = live && s == 0 && KIND != kUp && m > rl;
    if (KIND != kUp) {
        if (live) {
            pR = srcR(b);
            pL = srcL(b);
        }
        // Levels 1..min(m, rl), whole CTA, coalesced per tile. Short tiles
        // (the whole edge fits the ring) use cp.async so all of a thread's
        // loads are in flight at once (measured: +10% at w = 32, -2.6% at
        // w = 1024, where plain loads win).
        const int n0 = 2 * (m < rl ? m : rl);
        if (XS) {
            for (int j = t; j < ntiles * n0; j += nt) {
                const int gg = j / n0, i = j - gg * n0;
                S1D_CHECK(i < 2 * m && ridx(i, rmask, gg, G) < 2 * rl * G, a.error_flag);
                cp_async8(ringR + ridx(i, rmask, gg, G), srcR(bfirst + gg) + i);
                cp_async8(ringL + ridx(i, rmask, gg, G), srcL(bfirst + gg) + i);
            }
            cp_async_commit();
            cp_async_wait<0>();
        } else {
            for (int j = t; j < ntiles * n0; j += nt) {
                const int gg = j / n0, i = j - gg * n0;
                ringR[ridx(i, rmask, gg, G)] = srcR(bfirst + gg)[i];
                ringL[ridx(i, rmask, gg, G)] = srcL(bfirst + gg)[i];
            }
        }
        if (FU) {
            if (__syncthreads_or(big)) { // nothing written yet (XS: its copies have landed)
                if (t == 0) atomicOr(a.big_self, 1);
                return;
            }
        } else {
            __syncthreads();
        }
    }
    // Longer tiles: slot-0 threads queue level r+kRing-1 into the ring entries
    // freed by level r-1 (cp.async, one group per level) and wait so that
    // level r+1 has landed before barrier r.
    auto feed = [&](int r) {
        if (feeder) {
            const int q = r + kRing - 2; // 0-based index of level r+kRing-1
            if (q < m) {
                S1D_CHECK(2 * q + 1 < w && ridx(2 * q + 1, rmask, g, G) < 2 * rl * G, a.error_flag);
                cp_async8(ringR + ridx(2 * q, rmask, g, G), pR + 2 * q);
                cp_async8(ringR + ridx(2 * q + 1, rmask, g, G), pR + 2 * q + 1);
                cp_async8(ringL + ridx(2 * q, rmask, g, G), pL + 2 * q);
                cp_async8(ringL + ridx(2 * q + 1, rmask, g, G), pL + 2 * q + 1);
            }
            cp_async_commit();
            cp_async_wait<kRing - 2>();
        }
    };

    double* oL = a.out_L + (std::size_t)b * w;
    double* oR = a.out_R + (std::size_t)b * w;

    if (KIND != kUp) {
        // Fixed-width builds: one slot per warp (G >= 32 tiles per CTA) or 2 /
        // 4 slots per warp (G = 16 / 8) insert through the unrolled loops;
        // the generic builds (and -DS1D_HEAT_NO_SLOTS, a diagnostic) use finsert.
        constexpr int kG = WT > 0 && (WT / 2) % Q == 0 ? MAXT / ((WT / 2) / Q) : 0; // tiles per CTA
        if constexpr (kG >= 32) fexpand_slot<Q, U, FU>(c, vl, vr, 1, m, fo, feed);
#ifndef S1D_HEAT_NO_SLOTS
        else if constexpr (kG == 16 || kG == 8 || kG == 4) fexpand_slots<Q, U, FU, 32 / kG>(c, vl, vr, 1, m, fo, feed);
#endif
        else fexpand<Q, U, FU>(c, vl, vr, 1, m, fo, feed);
        { // level m: full span; the halo pair (x = 0, w+1) is distance m
            const int r = m;
            finsert(c, vl, vr, r);
            fpublish(c, vl, vr, r);
            if (s == tt - 1 && m % Q == 0) // else distance m is a register of slot tt-1 (finsert)
                c.F[(r & 1) * c.xs + (tt + 1) * G + g] =
                    make_double2(ringR[ridx(2 * (m - 1), rmask, g, G)], ringL[ridx(2 * (m - 1) + 1, rmask, g, G)]);
            level_sync();
            fcompute<Q, FU>(c, vl, vr, r, fo);
        }
    }
    if (KIND != kDown) {
        // Short tiles (m <= kXportLevels) stage their exports in the freed ring /
        // staging region and write the CTA's contiguous edge block coalesced at
        // the end (lanes hold different tiles, so direct stores would be 8-byte
        // scatters at stride w; measured +25% at w = 32, +10% at w = 64).
        const bool sx = XS; // launcher guarantees m <= kXportLevels
        double* const xL = ringR; // [G][w+1]
        double* const xR = ringR + (std::size_t)G * ws;
        if (KIND == kUp && sx) __syncthreads(); // state staging reads done
        double* eL = sx ? xL + g * ws : oL;
        double* eR = sx ? xR + g * ws : oR;
        fexport(c, vl, vr, 0, eL, eR, live);
        fcontract<Q, U, FU>(c, vl, vr, m + 1, 2 * m, fo, eL, eR, live);
        if (sx) {
            __syncthreads();
            double* gL = a.out_L + (std::size_t)bfirst * w;
            double* gR = a.out_R + (std::size_t)bfirst * w;
            for (int j = t; j < ntiles * w; j += nt) {
                const int gg = j / w, i = j - gg * w;
                gL[j] = xL[gg * ws + i];
                gR[j] = xR[gg * ws + i];
            }
        }
    } else {
        __syncthreads(); // ring reads done before the staging reuses it
        double* my = stage + g * ws;
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            if (s * Q + k < m) {
                my[m - 1 - (s * Q + k)] = vl[k];
                my[m + s * Q + k] = vr[k];
            }
        }
        __syncthreads();
        const std::int64_t centre0 = a.seam ? (std::int64_t)(bfirst + 1) * w : (std::int64_t)bfirst * w + w / 2;
        const std::int64_t p0 = centre0 - w / 2; // shard position of the CTA's first core point
        for (int j = t; j < ntiles * w; j += nt) {
            const int gg = j / w;
            const double val = stage[gg * ws + (j - gg * w)];
            const std::uint64_t gp = (std::uint64_t)(p0 + j);
            S1D_CHECK(gp < a.N + (std::uint64_t)w, a.error_flag); // spill into the right shard <= w/2
            if (gp < a.N) a.state_out[gp] = val;
            else a.state_right[gp - a.N] = val;
        }
    }
}

// ---------------------------------------------------------------------------
// Debug-kernel helpers: the contiguous layout (tile thread lt owns x = 1 +
// lt*P + k), an independent restatement of the tile geometry.
// ---------------------------------------------------------------------------
__host__ __device__ inline int tile_edge_stride(int) { return 4 * kRing; }

template <int P>
struct TileCtx {
    int w, m, tt, lt;     // width, levels, threads per tile, thread-in-tile
    int my_lo;            // x of v[0]
    int wlo, whi;         // x range of my warp (superset if it spans tiles)
    double* XL;           // exchange: last values, [2][G*(tt+2)]
    double* XF;           // exchange: first values
    int xs;               // parity stride of XL/XF
    int slot;             // my slot (tile base + lt + 1)
    const double* einR;   // my tile's ring of left-producer R edges [kRing][2]
    const double* einL;   // ring of right-producer L edges
};

template <int P>
__device__ __forceinline__ void publish(const TileCtx<P>& c, const double (&v)[P], int r) {
    const int par = (r & 1) * c.xs;
    c.XF[par + c.slot] = v[0];
    c.XL[par + c.slot] = v[P - 1];
}

template <int P>
__device__ __forceinline__ void compute_level(const TileCtx<P>& c, double (&v)[P], int r, int lo, int hi,
                                              double fo) {
    if (c.whi >= lo && c.wlo < hi) {
        const int par = (r & 1) * c.xs;
        const double lft = c.XL[par + c.slot - 1];
        const double rgt = c.XF[par + c.slot + 1];
        double nv[P];
        if (P == 1) {
            nv[0] = heat_f(lft, v[0], rgt, fo);
        } else {
            nv[0] = heat_f(lft, v[0], v[1], fo);
#pragma unroll
            for (int k = 1; k < P - 1; ++k) nv[k] = heat_f(v[k - 1], v[k], v[k + 1], fo);
            nv[P - 1] = heat_f(v[P - 2], v[P - 1], rgt, fo);
        }
#pragma unroll
        for (int k = 0; k < P; ++k) v[k] = nv[k];
    }
}

// Exports of level r (contracting half, d = r - m): L[d] = x in {lo, lo+1},
// R[d] = x in {hi-2, hi-1}; edge layout [level][2].
template <int P>
__device__ __forceinline__ void export_level(const TileCtx<P>& c, const double (&v)[P], int d, int lo, int hi,
                                             double* oL, double* oR) {
    if (c.wlo <= lo + 1 && c.whi >= lo) {
        double* dst = oL + 2 * d - lo + c.my_lo; // address of x = my_lo + k is dst + k
#pragma unroll
        for (int k = 0; k < P; ++k)
            if ((unsigned)(c.my_lo + k - lo) < 2u) dst[k] = v[k];
    }
    if (c.wlo <= hi - 1 && c.whi >= hi - 2) {
        double* dst = oR + 2 * d - (hi - 2) + c.my_lo;
#pragma unroll
        for (int k = 0; k < P; ++k)
            if ((unsigned)(c.my_lo + k - (hi - 2)) < 2u) dst[k] = v[k];
    }
}

// Inserts of level r (expanding half): left producer's R[r-1] at x = lo-1, lo
// and right producer's L[r-1] at x = hi-1, hi. Points beyond (x < lo-1,
// x > hi) are outside the dependency cone and may take any value, so one-sided
// predicates suffice and the smem address stays affine in x.
template <int P>
__device__ __forceinline__ void insert_level(const TileCtx<P>& c, double (&v)[P], int r, int lo, int hi) {
    if (c.wlo <= lo && c.whi >= lo - 1) {
        // ring index of x at level r: 2(r-1) + x - (lo-1)
        const int base = 2 * (r - 1) - (lo - 1) + c.my_lo;
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (c.my_lo + k <= lo) v[k] = c.einR[(base + k) & kRingMask];
    }
    if (c.whi >= hi - 1 && c.wlo <= hi) {
        const int base = 2 * (r - 1) - (hi - 1) + c.my_lo;
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (c.my_lo + k >= hi - 1) v[k] = c.einL[(base + k) & kRingMask];
    }
}

// ---------------------------------------------------------------------------
// Instrumented tile kernel (debug runs only): the same tile geometry, insert /
// export rules and arithmetic, run as plain level loops, counting every
// (point, counter) it computes inside the level's span and optionally nudging
// the run's first computed value (reference perturb_ulp: the up-triangle's
// first level, global point h, shard 0).
// ---------------------------------------------------------------------------
template <int P, int KIND>
__global__ void __launch_bounds__(256) heat_tile_debug_kernel(const TileArgs a, int G) {
    extern __shared__ double sm[];
    const int w = a.w, m = a.m;
    const int tt = w / P;
    const int t = threadIdx.x;
    const int g = t / tt;
    const int b = a.b0 + blockIdx.x * G + g;
    const bool live = b < (a.b1 < 0 ? a.nb : a.b1);
    const double fo = a.fourier;
    TileCtx<P> c;
    c.w = w;
    c.m = m;
    c.tt = tt;
    c.lt = t - g * tt;
    c.my_lo = 1 + c.lt * P;
    c.xs = G * (tt + 2);
    c.XL = sm;
    c.XF = sm + 2 * c.xs;
    c.slot = g * (tt + 2) + c.lt + 1;
    double* einR = sm + 4 * c.xs + (std::size_t)g * tile_edge_stride(w);
    double* einL = einR + 2 * kRing;
    c.einR = einR;
    c.einL = einL;
    {
        const unsigned full = __activemask();
        c.wlo = __reduce_min_sync(full, c.my_lo);
        c.whi = __reduce_max_sync(full, c.my_lo + P - 1);
    }
    const std::int64_t centre = a.seam ? (std::int64_t)(b + 1) * w : (std::int64_t)b * w + w / 2;
    const std::int64_t g0 = centre - w / 2 - 1; // shard position of local x = 0
    auto count = [&](int r, int lo, int hi) {
        if (!live || !a.dbg.cov) return;
        unsigned* row = a.dbg.cov + (std::uint64_t)(a.base + r - 1) * a.dbg.cov_n;
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const int x = c.my_lo + k;
            if (x >= lo && x < hi) atomicAdd(row + (a.dbg.gstart + (std::uint64_t)(g0 + x)) % a.dbg.cov_n, 1u);
        }
    };
    double v[P];
#pragma unroll
    for (int k = 0; k < P; ++k) v[k] = 0.0;
    if (KIND == kUp && live) {
        const double* src = a.state_in + (std::size_t)b * w + (std::size_t)c.lt * P;
#pragma unroll
        for (int k = 0; k < P; ++k) v[k] = src[k];
    }
    if (KIND != kUp) { // whole edges staged (debug sizes are small)
        const double* pR = nullptr;
        const double* pL = nullptr;
        if (live) {
            if (a.seam) {
                pR = a.in_R + (std::size_t)b * w;
                pL = (b + 1 < a.nb) ? a.in_L + (std::size_t)(b + 1) * w : a.peer_L;
            } else {
                pR = (b > 0) ? a.in_R + (std::size_t)(b - 1) * w : a.peer_R;
                pL = a.in_L + (std::size_t)b * w;
            }
        }
        for (int r = 1; r <= m; ++r) {
            const int lo = w / 2 + 1 - r, hi = w / 2 + 1 + r;
            __syncthreads(); // previous level's ring reads done
            if (live) // stage level r's 2+2 values into the ring slot
                for (int i = c.lt; i < 4; i += tt) {
                    const int q = r - 1, j = i & 1;
                    double* ring = (i < 2 ? einR : einL);
                    ring[(2 * q + j) & kRingMask] = (i < 2 ? pR : pL)[2 * q + j];
                }
            __syncthreads();
            insert_level(c, v, r, lo, hi);
            publish(c, v, r);
            if (r == m) {
                const int par = (r & 1) * c.xs, base = g * (tt + 2);
                if (c.lt == 0) c.XL[par + base] = einR[(2 * (m - 1)) & kRingMask];
                if (c.lt == tt - 1) c.XF[par + base + tt + 1] = einL[(2 * (m - 1) + 1) & kRingMask];
            }
            __syncthreads();
            compute_level(c, v, r, lo, hi, fo);
            count(r, lo, hi);
        }
    }
    double* oL = a.out_L + (std::size_t)b * w;
    double* oR = a.out_R + (std::size_t)b * w;
    if (KIND != kDown) {
        if (live) export_level(c, v, 0, 1, w + 1, oL, oR);
        for (int r = m + 1; r <= 2 * m - 1; ++r) {
            const int d = r - m, lo = 1 + d, hi = 1 + w - d;
            publish(c, v, r);
            __syncthreads();
            compute_level(c, v, r, lo, hi, fo);
            count(r, lo, hi);
            if (KIND == kUp && r == m + 1 && a.dbg.perturb && b == 0) {
                const int x = 2; // global point h = 1 of shard 0 (g0 = -1)
#pragma unroll
                for (int k = 0; k < P; ++k)
                    if (c.my_lo + k == x) v[k] = next_up(v[k]);
            }
            if (live) export_level(c, v, d, lo, hi, oL, oR);
        }
    } else if (live) {
        const std::int64_t gp0 = centre - w / 2 + (std::int64_t)c.lt * P;
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const std::uint64_t gp = (std::uint64_t)(gp0 + k);
            if (gp < a.N) a.state_out[gp] = v[k];
            else a.state_right[gp - a.N] = v[k];
        }
    }
}

} // namespace

bool heat_fast_form(const TileArgs& a) { return a.big_self != nullptr && a.m >= 64; }

namespace {

constexpr int kWideCta = 512; // threads per CTA of the P = 16 tiles from w = 256

int tiles_per_cta(int w, int p, int maxt = 256) {
    const int tt = fold_slots(w, p);
    int G = 1;
    if (tt > maxt) return 1;
    while ((G * 2) * tt <= maxt && G * 2 <= 64) G *= 2;
    return G;
}

template <int P, int MAXT = 256, int MINB = 1, int U = 1, bool XS = false, int WT = 0>
cudaError_t launch_tile_p(int kind, const TileArgs& a, cudaStream_t st) {
    static_assert(P % 2 == 0, "the folded layout holds P/2 distance pairs per thread");
    if (XS != (a.m <= kXportLevels)) return cudaErrorInvalidValue;
    const int tt = fold_slots(a.w, P);
    if (tt > MAXT) return cudaErrorInvalidValue;
    const int G = tiles_per_cta(a.w, P, MAXT);
    if (WT && (a.w != WT || G * tt != MAXT)) return cudaErrorInvalidValue; // the compile-time shape must match
    const int nt = G * tt;
    const size_t smem = sizeof(double) * fold_smem_doubles(kind, a.w, P, G);
    const int count = (a.b1 < 0 ? a.nb : a.b1) - a.b0;
    if (count <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((count + G - 1) / G);
    // The fast build + its gated exact build for tiles of at least 64 levels
    // (the extra launch is then noise); shorter tiles, or no flag, run the
    // exact build alone. With a.gated == 0 (single process) the engine reads
    // the flags after the run instead and reruns it exactly if one is set. (0 < Fo <= 0.5, heat_step's precondition,
    // is guaranteed by validation.)
    const bool fast = heat_fast_form(a);
    for (int pass = fast ? 0 : 1; pass < (fast && !a.gated ? 1 : 2); ++pass) {
        const bool fu = pass == 0;
        void (*k)(const TileArgs, int) =
            kind == kUp ? (fu ? heat_tile_kernel<P / 2, kUp, MAXT, MINB, U, XS, true, WT>
                              : heat_tile_kernel<P / 2, kUp, MAXT, MINB, U, XS, false, WT>)
            : kind == kDiamond ? (fu ? heat_tile_kernel<P / 2, kDiamond, MAXT, MINB, U, XS, true, WT>
                                     : heat_tile_kernel<P / 2, kDiamond, MAXT, MINB, U, XS, false, WT>)
                               : (fu ? heat_tile_kernel<P / 2, kDown, MAXT, MINB, U, XS, true, WT>
                                     : heat_tile_kernel<P / 2, kDown, MAXT, MINB, U, XS, false, WT>);
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
        TileArgs ka = a;
        if (!fast) ka.big_self = nullptr; // ungated exact build
        k<<<grid, nt, smem, st>>>(ka, G);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

} // namespace

int heat_points_per_thread(int w, long long tiles) {
    if (const char* e = std::getenv("S1D_HEAT_P")) {
        const int p = std::atoi(e);
        if ((p == 2 || p == 4 || p == 8 || p == 16) && fold_slots(w, p) <= 256) return p;
    }
    // Folded layout: P even (P/2 distance pairs per thread), ceil(m / (P/2))
    // slots (fold_slots: a ragged last slot pads). Measured on B200 (n = 2^27,
    // each with its register cap / unroll): P = 16 from w = 128 (twice the
    // work per level barrier of P = 8: +9% at w = 1024; w = 1000, padded:
    // 1.75 T vs 1.60 T with P = 8), except 128 < w < 256 when 16 does not
    // divide w (w = 200: P = 8 1.46 T, padded P = 16 1.37 T); P = 8 at
    // w = 32..127; narrower tiles P = 4 (w = 0 mod 4) or 2. Tiles wider than
    // 256 slots run P = 16 in CTAs of up to 1024 threads (w <= 16384).
    int p = 2;
    if (w >= 256 || (w >= 128 && w % 16 == 0)) p = 16;
    else if (w >= 32) p = 8;
    else if (w % 4 == 0) p = 4;
    if (fold_slots(w, p) > 1024) return -1; // no valid decomposition (caller reports it)
    // Small grids: P = 16 packs twice the tiles per CTA of P = 8; below one
    // full wave (4 CTAs per SM) P = 8 fills the GPU better (measured n = 2^20:
    // 1.29-1.32 T with P = 8 vs 1.01-1.04 T with P = 16 at w = 256..1024) —
    // except for the fixed-width P = 16 builds (w = 256 / 512 / 1024), which
    // win there too (n = 2^20: 1.70-1.73 T vs 1.47-1.52 T with P = 8).
    const bool fixed16 = w == 256 || w == 512 || w == 1024;
    if (p == 16 && !fixed16 && tiles >= 0 && fold_slots(w, 8) <= 256) {
        static int sms = 0;
        if (sms == 0) {
            int dev = 0;
            cudaGetDevice(&dev);
            if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
                cudaGetLastError();
                sms = 148;
            }
        }
        // P = 16 runs 2 CTAs of kWideCta threads per SM from w = 256, 3 CTAs
        // of 256 below (launch_heat_tile)
        const long long g = w >= 256 ? tiles_per_cta(w, 16, kWideCta) : tiles_per_cta(w, 16);
        if ((tiles + g - 1) / g < (w >= 256 ? 2LL : 4LL) * sms) p = 8;
    }
    return p;
}

cudaError_t launch_heat_classic(const ClassicArgs& a, cudaStream_t st) {
    const std::uint64_t pairs = a.N >> 1;
    std::uint64_t blocks = (pairs + 255) / 256;
    const std::uint64_t cap = (std::uint64_t)a.sms * 8 * 4;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    heat_classic_kernel<<<(unsigned)blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

template <int P>
cudaError_t launch_tile_debug(int kind, const TileArgs& a, cudaStream_t st) {
    const int tt = a.w / P;
    const int G = tiles_per_cta(a.w, P);
    const size_t smem = sizeof(double) * (4 * (size_t)G * (tt + 2) + (size_t)G * tile_edge_stride(a.w));
    void (*k)(const TileArgs, int) = kind == kUp ? heat_tile_debug_kernel<P, kUp>
                                     : kind == kDiamond ? heat_tile_debug_kernel<P, kDiamond>
                                                        : heat_tile_debug_kernel<P, kDown>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int count = (a.b1 < 0 ? a.nb : a.b1) - a.b0;
    if (count <= 0) return cudaSuccess;
    k<<<(unsigned)((count + G - 1) / G), G * tt, smem, st>>>(a, G);
    return cudaGetLastError();
}

cudaError_t launch_heat_tile(int kind, const TileArgs& a, cudaStream_t st, bool debug) {
    if (debug) {
        // the instrumented kernel's contiguous layout needs P | w, w/P <= 256
        for (int p : {16, 8, 4, 2}) {
            if (a.w % p || a.w / p > 256) continue;
            switch (p) {
            case 2: return launch_tile_debug<2>(kind, a, st);
            case 4: return launch_tile_debug<4>(kind, a, st);
            case 8: return launch_tile_debug<8>(kind, a, st);
            default: return launch_tile_debug<16>(kind, a, st);
            }
        }
        return cudaErrorInvalidValue;
    }
    const int slots = fold_slots(a.w, a.p);
    if (slots > 1024) return cudaErrorInvalidValue;
    if (slots > 256) // very wide tiles: one tile per CTA of up to 1024 threads
        return a.p == 16 ? launch_tile_p<16, 1024>(kind, a, st) : cudaErrorInvalidValue;
    const bool xs = a.m <= kXportLevels; // short tiles: staged exports (XS build)
    switch (a.p) {
    case 2: return xs ? launch_tile_p<2, 256, 1, 1, true>(kind, a, st) : launch_tile_p<2>(kind, a, st);
    case 4: // (w = 32: register caps / unroll measured slower)
        return xs ? launch_tile_p<4, 256, 1, 1, true>(kind, a, st) : launch_tile_p<4>(kind, a, st);
    case 8: // measured (w = 64 and widths 16 does not divide): 64-register cap (4 CTAs/SM) + unroll 2
        if (a.w == 32 && tiles_per_cta(32, 8, 256) * fold_slots(32, 8) == 256)
            return launch_tile_p<8, 256, 4, 2, true, 32>(kind, a, st); // fixed width (64 registers: +16-18%)
        if (a.w < 64) return launch_tile_p<8, 256, 1, 2, true>(kind, a, st); // w = 32: unroll only
        if (a.w == 64 && xs && tiles_per_cta(64, 8, 256) * fold_slots(64, 8) == 256)
            return launch_tile_p<8, 256, 4, 2, true, 64>(kind, a, st); // fixed width
        return xs ? launch_tile_p<8, 256, 4, 2, true>(kind, a, st) : launch_tile_p<8, 256, 4, 2>(kind, a, st);
    case 16: // measured (n = 2^27): 4 CTAs/SM + unroll 2 from w = 256 (1.95-1.97 T), 3 CTAs/SM at w = 128
        if (xs) return launch_tile_p<16, 256, 1, 1, true>(kind, a, st);
        if (a.w == 128 && tiles_per_cta(128, 16, 256) * fold_slots(128, 16) == 256)
            return launch_tile_p<16, 256, 3, 2, false, 128>(kind, a, st); // fixed width (unroll 2: +2%)
        if (a.w < 256) return launch_tile_p<16, 256, 3, 1>(kind, a, st);
        // 512-thread CTAs (2 per SM, 64 registers): twice the tiles per CTA, so
        // a warp spans half the distances and the busy/idle boundary of each
        // level wastes half as many lanes. Measured (n = 2^27) against 256-thread
        // CTAs at 4 per SM: w = 256 / 1024 / 2048: 2.27 / 2.17 / 2.14 T vs
        // 2.13 / 2.10 / 2.09 T; 1024-thread CTAs: 1.99 / 2.09 T.
        // The common widths with the width as a compile-time constant.
        if (tiles_per_cta(a.w, 16, kWideCta) * fold_slots(a.w, 16) == kWideCta) {
            if (a.w == 256) return launch_tile_p<16, kWideCta, 2, 2, false, 256>(kind, a, st);
            if (a.w == 512) return launch_tile_p<16, kWideCta, 2, 2, false, 512>(kind, a, st);
            if (a.w == 1024) return launch_tile_p<16, kWideCta, 2, 2, false, 1024>(kind, a, st);
            if (a.w == 2048) return launch_tile_p<16, kWideCta, 2, 2, false, 2048>(kind, a, st);
        }
        return launch_tile_p<16, kWideCta, 2, 2>(kind, a, st);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace s1d
