// Heat-equation (FTCS, 3-point) kernels for sm_100a, FP64.
//
//   heat_classic_kernel   one substep per launch, the naive comparison and the
//                         swept pad (reference classic_worker,
//                         engines_impl.hpp:201-213)
//   heat_tile_kernel<P,K> one swept phase: K = Up (UpTriangle,
//                         engines_impl.hpp:280-291), Diamond (:293-307) or
//                         Down (DownTriangle, last cycle). Boundary tiles read
//                         their neighbour shard's edge directly (SplitDiamond).
//
// The point update is heat_step (inc/kernels.hpp:14-16),
//   T' = c + Fo*((l - 2c) + r),
// evaluated with explicit round-to-nearest intrinsics so no FMA contraction
// can change a bit (the reference builds with -ffp-contract=off).
//
// Tile layout: a CTA runs G tiles side by side;
// tile thread lt owns P consecutive points of the w-point core in registers
// (local x = 1 + lt*P + k, x in [1, w]). Per level a thread publishes its
// first/last value to shared memory, one barrier, and computes its P points
// from registers plus the two neighbour values. Warps whose points lie
// outside the level's span skip the arithmetic (the diamond grows/shrinks by
// one point per side per level).
//
// Edges: the left producer's R edges and the right producer's L edges (2
// values per level each) stream into a small shared-memory ring per tile
// (cp.async, kRing-2 levels ahead). The insert of level r lands at x = lo-1, lo (left) and hi-1, hi (right); its
// shared-memory address is affine in x, so the warp that holds those points
// reloads them with predicated loads (points further out are don't-care:
// they are outside the dependency cone). Exports L[d], R[d] are written by
// the owning threads with exactly-predicated stores.
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

__global__ void __launch_bounds__(256) heat_classic_kernel(const ClassicArgs a) {
    // Two points per thread (N is a multiple of the even block width).
    const std::uint64_t pairs = a.N >> 1;
    const double fo = a.fourier;
    const double hl = *a.halo_l;
    const double hr = *a.halo_r;
    for (std::uint64_t p = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; p < pairs;
         p += (std::uint64_t)gridDim.x * blockDim.x) {
        const std::uint64_t i = p << 1;
        const double2 c = __ldg(reinterpret_cast<const double2*>(a.in) + p);
        const double l = i > 0 ? __ldg(a.in + i - 1) : hl;
        const double r = i + 2 < a.N ? __ldg(a.in + i + 2) : hr;
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
    }
}

// Incoming edges stream through a per-tile ring of kRing levels (2 values per
// level per side) filled with cp.async kRing-2 levels ahead of use, so shared
// memory per tile is O(1) in w. Ring index of (level r, x) is affine in x and
// wrapped with a mask, so predicated insert loads stay contiguous.
constexpr int kRing = 32;             // levels held per side (power of two)
constexpr int kRingMask = 2 * kRing - 1;
__host__ __device__ inline int tile_edge_stride(int) { return 4 * kRing; }

__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

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

// Diagnostic builds (-DS1D_NO_LEVEL_BARRIER) replace the level barrier with
// __syncwarp() to time the level loop without it (results are then wrong).
#ifdef S1D_NO_LEVEL_BARRIER
#define S1D_LEVEL_BARRIER() __syncwarp()
#else
#define S1D_LEVEL_BARRIER() __syncthreads()
#endif

// ---------------------------------------------------------------------------
// Level loops in segments. Over a phase each warp's role changes only at a
// handful of levels (the span edges sweep across it once), so the levels are
// run in segments with compile-time role flags: an idle warp costs a barrier
// per level, a computing warp publish + barrier + 5P FP64 ops.
// ---------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void compute_span(const TileCtx<P>& c, double (&v)[P], int r, double fo) {
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

template <int P>
__device__ __forceinline__ void insert_left(const TileCtx<P>& c, double (&v)[P], int r, int lo) {
    const int base = 2 * (r - 1) - (lo - 1) + c.my_lo;
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (c.my_lo + k <= lo) v[k] = c.einR[(base + k) & kRingMask];
}
template <int P>
__device__ __forceinline__ void insert_right(const TileCtx<P>& c, double (&v)[P], int r, int hi) {
    const int base = 2 * (r - 1) - (hi - 1) + c.my_lo;
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (c.my_lo + k >= hi - 1) v[k] = c.einL[(base + k) & kRingMask];
}
// (`live` only predicates the stores: control flow must stay warp-uniform
// because the segment loops contain barriers.)
template <int P>
__device__ __forceinline__ void export_left(const TileCtx<P>& c, const double (&v)[P], int d, int lo, double* oL,
                                            bool live) {
    double* dst = oL + 2 * d - lo + c.my_lo;
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (live && (unsigned)(c.my_lo + k - lo) < 2u) dst[k] = v[k];
}
template <int P>
__device__ __forceinline__ void export_right(const TileCtx<P>& c, const double (&v)[P], int d, int hi, double* oR,
                                             bool live) {
    double* dst = oR + 2 * d - (hi - 2) + c.my_lo;
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (live && (unsigned)(c.my_lo + k - (hi - 2)) < 2u) dst[k] = v[k];
}

// Expanding levels [r0, r1): span [w/2+1-r, w/2+1+r).
template <int P, bool IL, bool IR, bool CP, class Feed>
__device__ __forceinline__ void expand_seg(const TileCtx<P>& c, double (&v)[P], int r0, int r1, double fo,
                                           Feed& feed) {
    for (int r = r0; r < r1; ++r) {
        const int lo = c.w / 2 + 1 - r, hi = c.w / 2 + 1 + r;
        if (IL) insert_left(c, v, r, lo);
        if (IR) insert_right(c, v, r, hi);
        if (IL || IR || CP) publish(c, v, r);
        feed(r);
        S1D_LEVEL_BARRIER();
        if (CP) compute_span(c, v, r, fo);
    }
}

template <int P, class Feed>
__device__ __forceinline__ void expand_levels(const TileCtx<P>& c, double (&v)[P], int r0, int r1, double fo,
                                              Feed& feed) {
    const int h2 = c.w / 2;
    // role ranges (inclusive) for this warp's x in [wlo, whi]
    const int rc = max(h2 + 1 - c.whi, c.wlo - h2);  // computes from rc on
    const int aL = h2 - c.whi, bL = h2 + 1 - c.wlo;  // left inserts
    const int aR = c.wlo - h2 - 1, bR = c.whi - h2;  // right inserts
    int bnd[6] = {rc, aL, bL + 1, aR, bR + 1, r1};
#pragma unroll
    for (int i = 1; i < 6; ++i) // insertion sort (6 warp-uniform ints)
        for (int j = i; j > 0 && bnd[j - 1] > bnd[j]; --j) {
            const int tmp = bnd[j];
            bnd[j] = bnd[j - 1];
            bnd[j - 1] = tmp;
        }
    int r = r0;
#pragma unroll 1
    for (int i = 0; i < 6 && r < r1; ++i) {
        const int e = min(max(bnd[i], r), r1);
        if (e <= r) continue;
        const int f = ((r >= aL && r <= bL) ? 4 : 0) | ((r >= aR && r <= bR) ? 2 : 0) | (r >= rc ? 1 : 0);
        switch (f) {
        case 0: expand_seg<P, false, false, false>(c, v, r, e, fo, feed); break;
        case 1: expand_seg<P, false, false, true>(c, v, r, e, fo, feed); break;
        case 2: expand_seg<P, false, true, false>(c, v, r, e, fo, feed); break;
        case 3: expand_seg<P, false, true, true>(c, v, r, e, fo, feed); break;
        case 4: expand_seg<P, true, false, false>(c, v, r, e, fo, feed); break;
        case 5: expand_seg<P, true, false, true>(c, v, r, e, fo, feed); break;
        case 6: expand_seg<P, true, true, false>(c, v, r, e, fo, feed); break;
        default: expand_seg<P, true, true, true>(c, v, r, e, fo, feed); break;
        }
        r = e;
    }
}

// Contracting levels [r0, r1): d = r-m, span [1+d, 1+w-d).
template <int P, bool PB, bool CP, bool EL, bool ER>
__device__ __forceinline__ void contract_seg(const TileCtx<P>& c, double (&v)[P], int r0, int r1, double fo,
                                             double* oL, double* oR, bool live) {
    for (int r = r0; r < r1; ++r) {
        const int d = r - c.m, lo = 1 + d, hi = 1 + c.w - d;
        if (PB) publish(c, v, r);
        S1D_LEVEL_BARRIER();
        if (CP) compute_span(c, v, r, fo);
        if (EL) export_left(c, v, d, lo, oL, live);
        if (ER) export_right(c, v, d, hi, oR, live);
    }
}

template <int P>
__device__ __forceinline__ void contract_levels(const TileCtx<P>& c, double (&v)[P], int r0, int r1, double fo,
                                                double* oL, double* oR, bool live) {
    const int m = c.m, w = c.w;
    const int rce = m + min(c.whi - 1, w - c.wlo);      // computes while r <= rce
    const int rpe = m + min(c.whi, w + 1 - c.wlo);      // publishes while r <= rpe
    const int aL = m + c.wlo - 2, bL = m + c.whi - 1;   // left exports
    const int aR = m + w - 1 - c.whi, bR = m + w - c.wlo; // right exports
    int bnd[7] = {rce + 1, rpe + 1, aL, bL + 1, aR, bR + 1, r1};
#pragma unroll
    for (int i = 1; i < 7; ++i)
        for (int j = i; j > 0 && bnd[j - 1] > bnd[j]; --j) {
            const int tmp = bnd[j];
            bnd[j] = bnd[j - 1];
            bnd[j - 1] = tmp;
        }
    int r = r0;
#pragma unroll 1
    for (int i = 0; i < 7 && r < r1; ++i) {
        const int e = min(max(bnd[i], r), r1);
        if (e <= r) continue;
        const bool pb = r <= rpe, cp = r <= rce;
        const bool el = r >= aL && r <= bL, er = r >= aR && r <= bR; // warp-uniform
        if (!pb) contract_seg<P, false, false, false, false>(c, v, r, e, fo, oL, oR, live);
        else if (!cp) contract_seg<P, true, false, false, false>(c, v, r, e, fo, oL, oR, live);
        else if (el && er) contract_seg<P, true, true, true, true>(c, v, r, e, fo, oL, oR, live);
        else if (el) contract_seg<P, true, true, true, false>(c, v, r, e, fo, oL, oR, live);
        else if (er) contract_seg<P, true, true, false, true>(c, v, r, e, fo, oL, oR, live);
        else contract_seg<P, true, true, false, false>(c, v, r, e, fo, oL, oR, live);
        r = e;
    }
}

template <int P, int KIND, int MAXT>
__global__ void __launch_bounds__(MAXT) heat_tile_kernel(const TileArgs a, int G) {
    extern __shared__ double sm[];
    const int w = a.w, m = a.m;
    const int tt = w / P;                 // threads per tile
    const int t = threadIdx.x;
    const int g = t / tt;                 // tile within the CTA
    const int b = a.b0 + blockIdx.x * G + g; // tile index in the shard
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
        // Warp x-range (superset when a warp spans several tiles).
        const unsigned full = __activemask();
        c.wlo = __reduce_min_sync(full, c.my_lo);
        c.whi = __reduce_max_sync(full, c.my_lo + P - 1);
    }

    const std::int64_t centre = a.seam ? (std::int64_t)(b + 1) * w : (std::int64_t)b * w + w / 2;
    double v[P];
#pragma unroll
    for (int k = 0; k < P; ++k) v[k] = 0.0;

    if (KIND == kUp) {
        if (live) {
            const double* src = a.state_in + (std::size_t)b * w + (std::size_t)c.lt * P;
#pragma unroll
            for (int k = 0; k < P; ++k) v[k] = src[k];
        }
    }
    // Edge streaming (Diamond/Down). The tile's threads load levels
    // 1..min(m, kRing) cooperatively; for longer tiles thread lt == 0 then
    // queues level r+kRing-1 into the slot freed by level r-1 (cp.async, one
    // group per level) and waits so that level r+1 has landed before barrier r.
    const double* pR = nullptr;
    const double* pL = nullptr;
    const bool feeder = live && c.lt == 0 && KIND != kUp && m > kRing;
    if (KIND != kUp) {
        if (live) {
            if (a.seam) {
                pR = a.in_R + (std::size_t)b * w;
                pL = (b + 1 < a.nb) ? a.in_L + (std::size_t)(b + 1) * w : a.peer_L;
            } else {
                pR = (b > 0) ? a.in_R + (std::size_t)(b - 1) * w : a.peer_R;
                pL = a.in_L + (std::size_t)b * w;
            }
            const int n0 = 2 * (m < kRing ? m : kRing);
            for (int i = c.lt; i < n0; i += tt) {
                einR[i] = pR[i];
                einL[i] = pL[i];
            }
        }
        __syncthreads();
    }
    auto feed = [&](int r) {
        if (feeder) {
            const int q = r + kRing - 2; // 0-based index of level r+kRing-1
            if (q < m) {
                cp_async16(einR + ((2 * q) & kRingMask), pR + 2 * q);
                cp_async16(einL + ((2 * q) & kRingMask), pL + 2 * q);
            }
            cp_async_commit();
            cp_async_wait<kRing - 2>();
        }
    };

    double* oL = a.out_L + (std::size_t)b * w;
    double* oR = a.out_R + (std::size_t)b * w;

    if (KIND != kUp) {
        // Expanding half, levels 1..m-1 (span [w/2+1-r, w/2+1+r)), then m.
        expand_levels(c, v, 1, m, fo, feed);
        {
            const int r = m, lo = 1, hi = w + 1;
            insert_level(c, v, r, lo, hi);
            publish(c, v, r);
            const int par = (r & 1) * c.xs;
            const int base = g * (tt + 2);
            if (c.lt == 0) c.XL[par + base] = einR[(2 * (m - 1)) & kRingMask];               // x = 0
            if (c.lt == tt - 1) c.XF[par + base + tt + 1] = einL[(2 * (m - 1) + 1) & kRingMask]; // x = w+1
            __syncthreads();
            compute_level(c, v, r, lo, hi, fo);
        }
    }
    if (KIND != kDown) {
        // Contracting half, levels m..2m-1: span [1+d, 1+w-d), d = r-m.
        if (live) export_level(c, v, 0, 1, w + 1, oL, oR);
        contract_levels(c, v, m + 1, 2 * m, fo, oL, oR, live);
    } else if (live) {
        const std::int64_t g0 = centre - w / 2 + (std::int64_t)c.lt * P;
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const std::uint64_t gp = (std::uint64_t)(g0 + k);
            if (gp < a.N) a.state_out[gp] = v[k];
            else a.state_right[gp - a.N] = v[k];
        }
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

int tiles_per_cta(int w, int p) {
    const int tt = w / p;
    int G = 1;
    if (tt > 256) return 1;
    while ((G * 2) * tt <= 256 && G * 2 <= 64) G *= 2;
    return G;
}

template <int P, int MAXT = 256>
cudaError_t launch_tile_p(int kind, const TileArgs& a, cudaStream_t st) {
    const int tt = a.w / P;
    const int G = tiles_per_cta(a.w, P);
    const int nt = G * tt;
    const size_t smem = sizeof(double) * (4 * (size_t)G * (tt + 2) + (size_t)G * tile_edge_stride(a.w));
    void (*k)(const TileArgs, int) = kind == kUp ? heat_tile_kernel<P, kUp, MAXT>
                                     : kind == kDiamond ? heat_tile_kernel<P, kDiamond, MAXT>
                                                        : heat_tile_kernel<P, kDown, MAXT>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int count = (a.b1 < 0 ? a.nb : a.b1) - a.b0;
    if (count <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((count + G - 1) / G);
    k<<<grid, nt, smem, st>>>(a, G);
    return cudaGetLastError();
}

} // namespace

int heat_points_per_thread(int w) {
    if (const char* e = std::getenv("S1D_HEAT_P")) {
        const int p = std::atoi(e);
        if ((p == 1 || p == 2 || p == 4 || p == 8 || p == 16) && w % p == 0 && w / p <= 256) return p;
    }
    // 256 threads per tile for wide tiles (P = w/256); P = 4 for narrow ones
    // (several tiles per CTA); always P | w, 2 <= P <= 16, w/P <= 256.
    int p = 2;
    if (w % 4 == 0) p = 4;
    while (w / p > 256 && w % (2 * p) == 0 && p < 16) p *= 2;
    if (w / p > 1024) return -1; // no valid decomposition (caller reports it)
    return p;                    // w/p in (256, 1024] only for w = 2 mod 4 (P = 2, wide CTA)
}

cudaError_t launch_heat_classic(const ClassicArgs& a, cudaStream_t st) {
    const std::uint64_t pairs = a.N >> 1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    std::uint64_t blocks = (pairs + 255) / 256;
    const std::uint64_t cap = (std::uint64_t)sms * 8 * 4;
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
    if (a.w % a.p || a.w / a.p > 1024) return cudaErrorInvalidValue;
    if (debug) {
        if (a.w / a.p > 256) return cudaErrorInvalidValue;
        switch (a.p) {
        case 2: return launch_tile_debug<2>(kind, a, st);
        case 4: return launch_tile_debug<4>(kind, a, st);
        case 8: return launch_tile_debug<8>(kind, a, st);
        case 16: return launch_tile_debug<16>(kind, a, st);
        default: return cudaErrorInvalidValue;
        }
    }
    if (a.w / a.p > 256) return a.p == 2 ? launch_tile_p<2, 1024>(kind, a, st) : cudaErrorInvalidValue;
    switch (a.p) {
    case 1: return launch_tile_p<1>(kind, a, st);
    case 2: return launch_tile_p<2>(kind, a, st);
    case 4: return launch_tile_p<4>(kind, a, st);
    case 8: return launch_tile_p<8>(kind, a, st);
    case 16: return launch_tile_p<16>(kind, a, st);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace s1d
