// Euler (Sod) kernels for sm_100a, FP64: second-order MUSCL/minmod
// predictor-corrector with a Rusanov flux and Roe-averaged signal speed.
//
// Two data-structure strategies of the reference (inc/kernels.hpp:128-185):
//   lengthening (EulerLenModel, S=4, h=1, record Q0,Q1,Pr = 7 doubles):
//     c%4==1 Pr <- ratio(p(Q0));  c%4==2 Q1 <- Q0 - dt/2dx (F+ - F-)[Q0,Pr]
//     c%4==3 Pr <- ratio(p(Q1));  c%4==0 Q0 <- Q0 - dt/dx  (F+ - F-)[Q1,Pr]
//   flattening (EulerFlatModel, S=2, h=2, record Q0,Q1 = 6 doubles): the
//     ratios are recomputed inline from a 5-point pressure window.
//
// State in HBM is SoA by field: field f of point i at st[f*fstride + i]
// (f: 0..2 Q0, 3..5 Q1, 6 Pr).
//
// Every interface flux and every pressure is computed ONCE and shared by the
// cells that read it (the reference evaluates each flux twice and each
// pressure 3-5 times); the arguments are identical, so results are too.
//
//   euler_len_classic<K>, euler_flat_classic<F>: one substep per launch
//     (reference classic_worker, engines_impl.hpp:201-213), in place.
//   euler_tile<FLAT,KIND>: one swept phase (Up / Diamond / Down), the tile's
//     records resident in shared memory; each phase maps the CTA's threads
//     onto exactly the points of the level's span (no wasted or speculative
//     arithmetic, so the non-physical-state flag is exact).
#include <cstdint>
#include <cstdlib>

#include "euler_math.cuh"
#include "device_util.cuh"
#include "kernels.hpp"

namespace s1d {
namespace {

constexpr int kClassicB = 256; // points per CTA in the classic kernels
// 4 resident CTAs of 256 threads per SM (<= 64 registers): the FP64
// div/sqrt chains of the flux are latency-bound, so occupancy beats the
// few bytes of spill this costs (measured: +8% swept, +20% classic).
#ifndef S1D_EULER_MINB
#define S1D_EULER_MINB 4
#endif
#ifndef S1D_EULER_CLASSIC_MINB
#define S1D_EULER_CLASSIC_MINB 4
#endif

struct Fields {
    double* st;
    std::uint64_t N, fs;
    const double* hl;
    std::uint64_t hlfs;
    const double* hr;
    std::uint64_t hrfs;
    int h;
    __device__ __forceinline__ double ld(int f, std::int64_t x) const {
        if (x < 0) return hl[(std::uint64_t)(x + h) + f * hlfs];
        if ((std::uint64_t)x >= N) return hr[((std::uint64_t)x - N) + f * hrfs];
        return st[(std::uint64_t)x + f * fs];
    }
};

__device__ __forceinline__ Fields fields_of(const ClassicArgs& a) {
    return Fields{a.out, a.N, a.fstride, a.halo_l, a.halo_l_fstride, a.halo_r, a.halo_r_fstride, a.h};
}

__device__ __forceinline__ void classic_count(const ClassicArgs& a, std::uint64_t x) {
    atomicAdd(a.dbg.cov + (std::uint64_t)(a.counter - 1) * a.dbg.cov_n + (a.dbg.gstart + x) % a.dbg.cov_n, 1u);
}

// One process per GPU: the first / last block of the shard waits for the
// neighbour's previous round before its first halo read, and signals this
// round after the block's final barrier (its boundary records are stored;
// other blocks neither read nor write what the neighbours touch).
__device__ __forceinline__ void classic_round_wait(const ClassicArgs& a, bool lb, bool rb) {
    if (!a.nb_flags || !(lb || rb)) return;
    if (threadIdx.x == 0) {
        const unsigned seq = *a.seq_base + a.round;
        if (lb) flag_wait(a.nb_flags, seq, a.error_flag, a.timeout_ns);
        if (rb) flag_wait(a.nb_flags + 1, seq, a.error_flag, a.timeout_ns);
    }
    __syncthreads();
}
__device__ __forceinline__ void classic_round_signal(const ClassicArgs& a, bool lb, bool rb) {
    if (!a.nb_flags || threadIdx.x != 0) return;
    const unsigned seq = *a.seq_base + a.round + 1;
    if (lb) flag_signal(a.sig_left, seq);
    if (rb) flag_signal(a.sig_right, seq);
}

__device__ __forceinline__ void raise_flag(int* flag, bool bad) {
    if (__any_sync(__activemask(), bad) && bad) atomicOr(flag, 1);
}

// ---------------------------------------------------------------------------
// classic, lengthening. KIND = counter % 4 (1 PR on Q0, 2 predictor, 3 PR on
// Q1, 0 corrector).
// ---------------------------------------------------------------------------
// Points per CTA pass: the pass's pressures (ratio substeps: B + 2, two per
// thread) or interface fluxes (B + 1, one per thread) exactly. (A 256-point
// pass left one thread computing a 257th flux alone while the CTA waited at
// the barrier: a second full div/sqrt latency chain per pass.)
__host__ __device__ constexpr int len_classic_points(int kind) {
    return (kind & 1) ? 2 * kClassicB - 2 : kClassicB - 1;
}
constexpr int kFlatClassicPoints = kClassicB - 4; // B + 4 pressures per pass

template <int KIND>
__global__ void __launch_bounds__(kClassicB, S1D_EULER_CLASSIC_MINB) euler_len_classic(const ClassicArgs a) {
    constexpr int B = len_classic_points(KIND);
    __shared__ double sh[3][kClassicB + 2];
    const Fields F = fields_of(a);
    const double gamma = a.gamma;
    bool bad = false;
    for (std::uint64_t i0 = (std::uint64_t)blockIdx.x * B; i0 < a.N; i0 += (std::uint64_t)gridDim.x * B) {
        const int nb = (int)min((std::uint64_t)B, a.N - i0);
        const bool lb = i0 == 0, rb = i0 + nb == a.N; // boundary blocks read / feed the neighbours
        classic_round_wait(a, lb, rb);
        if (KIND & 1) {
            // B + 2 = two pressures per thread, all six loads issued before
            // the math: the ratio substep is memory-latency-bound (ncu: long
            // scoreboard), so twice the loads in flight per thread
            double* P = &sh[0][0];
            const int s = (KIND == 1) ? 0 : 3;
            const int t0 = threadIdx.x, t1 = threadIdx.x + blockDim.x;
            const bool v0 = t0 < nb + 2, v1 = t1 < nb + 2;
            const std::int64_t x0 = (std::int64_t)i0 + t0 - 1, x1 = (std::int64_t)i0 + t1 - 1;
            double q0[3] = {1.0, 0.0, 1.0}, q1[3] = {1.0, 0.0, 1.0};
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                if (v0) q0[f] = F.ld(s + f, x0);
                if (v1) q1[f] = F.ld(s + f, x1);
            }
            if (v0) P[t0] = em::pressure(q0[0], q0[1], q0[2], gamma, bad);
            if (v1) P[t1] = em::pressure(q1[0], q1[1], q1[2], gamma, bad);
            __syncthreads();
            for (int t = threadIdx.x; t < nb; t += blockDim.x) {
                double pr = em::ratio(P[t], P[t + 1], P[t + 2]);
                if (a.dbg.perturb && a.counter == 1 && i0 + t == 0) pr = next_up(pr); // debug runs only
                if (a.dbg.cov) classic_count(a, i0 + t);
                a.out[i0 + t + 6 * a.fstride] = pr;
            }
        } else {
            const bool fin = (KIND == 0);
            const int rs = fin ? 3 : 0, ws = fin ? 0 : 3;
            const double factor = fin ? a.dt_dx : em::mul(0.5, a.dt_dx);
            // interface t sits between points i0+t-1 and i0+t
            for (int t = threadIdx.x; t < nb + 1; t += blockDim.x) {
                const std::int64_t x = (std::int64_t)i0 + t;
                double f0, f1, f2;
                em::iflux(F.ld(rs, x - 1), F.ld(rs + 1, x - 1), F.ld(rs + 2, x - 1), F.ld(rs, x), F.ld(rs + 1, x),
                          F.ld(rs + 2, x), F.ld(6, x - 1), F.ld(6, x), gamma, f0, f1, f2, bad);
                sh[0][t] = f0;
                sh[1][t] = f1;
                sh[2][t] = f2;
            }
            __syncthreads();
            for (int t = threadIdx.x; t < nb; t += blockDim.x) {
                const std::uint64_t x = i0 + t;
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    a.out[x + (ws + k) * a.fstride] =
                        em::update(a.out[x + k * a.fstride], factor, sh[k][t + 1], sh[k][t]);
                if (a.dbg.cov) classic_count(a, x);
            }
        }
        __syncthreads();
        classic_round_signal(a, lb, rb);
    }
    raise_flag(a.error_flag, bad);
}

// classic, flattening. FIN = 0 predictor (Q1 <- from Q0), 1 corrector.
template <int FIN>
__global__ void __launch_bounds__(kClassicB, S1D_EULER_CLASSIC_MINB) euler_flat_classic(const ClassicArgs a) {
    constexpr int B = kFlatClassicPoints;
    __shared__ double sp[kClassicB + 4];
    __shared__ double sf[3][kClassicB + 1];
    const Fields F = fields_of(a);
    const double gamma = a.gamma;
    const int s = FIN ? 3 : 0, ws = FIN ? 0 : 3;
    const double factor = FIN ? a.dt_dx : em::mul(0.5, a.dt_dx);
    bool bad = false;
    for (std::uint64_t i0 = (std::uint64_t)blockIdx.x * B; i0 < a.N; i0 += (std::uint64_t)gridDim.x * B) {
        const int nb = (int)min((std::uint64_t)B, a.N - i0);
        const bool lb = i0 == 0, rb = i0 + nb == a.N;
        classic_round_wait(a, lb, rb);
        for (int t = threadIdx.x; t < nb + 4; t += blockDim.x) { // sp[t] = p(i0 + t - 2)
            const std::int64_t x = (std::int64_t)i0 + t - 2;
            sp[t] = em::pressure(F.ld(s, x), F.ld(s + 1, x), F.ld(s + 2, x), gamma, bad);
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nb + 1; t += blockDim.x) { // interface between i0+t-1 and i0+t
            const std::int64_t x = (std::int64_t)i0 + t;
            const double rl = em::ratio(sp[t], sp[t + 1], sp[t + 2]);     // ratio at x-1
            const double rr = em::ratio(sp[t + 1], sp[t + 2], sp[t + 3]); // ratio at x
            double f0, f1, f2;
            em::iflux(F.ld(s, x - 1), F.ld(s + 1, x - 1), F.ld(s + 2, x - 1), F.ld(s, x), F.ld(s + 1, x),
                      F.ld(s + 2, x), rl, rr, gamma, f0, f1, f2, bad);
            sf[0][t] = f0;
            sf[1][t] = f1;
            sf[2][t] = f2;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nb; t += blockDim.x) {
            const std::uint64_t x = i0 + t;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                a.out[x + (ws + k) * a.fstride] = em::update(a.out[x + k * a.fstride], factor, sf[k][t + 1], sf[k][t]);
            if (a.dbg.perturb && a.counter == 1 && x == 0) a.out[ws * a.fstride] = next_up(a.out[ws * a.fstride]);
            if (a.dbg.cov) classic_count(a, x);
        }
        __syncthreads();
        classic_round_signal(a, lb, rb);
    }
    raise_flag(a.error_flag, bad);
}

// ---------------------------------------------------------------------------
// swept tile (one CTA per tile)
// ---------------------------------------------------------------------------
constexpr int kERing = 16; // ring levels per side
constexpr int kELook = 8;  // cp.async lookahead (levels)

__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int FLAT>
struct TileGeom {
    static constexpr int H = FLAT ? 2 : 1;
    static constexpr int REC = FLAT ? 6 : 7;
    static constexpr int LVL = 2 * H * REC;   // doubles per level per side in an edge
    static constexpr int CHUNKS = LVL / 2;    // 16-byte chunks per level per side
};

// Shared memory of one tile (doubles): records, pressures, fluxes, ring.
inline std::size_t euler_tile_doubles(int flat, int w) {
    const int H = flat ? 2 : 1, REC = flat ? 6 : 7;
    const std::size_t W2 = (std::size_t)w + 2 * H;
    return REC * W2 + (W2 + 1) + 3 * (W2 + 1) + 2 * (std::size_t)kERing * 2 * H * REC;
}
inline std::size_t euler_tile_smem(int flat, int w) { return euler_tile_doubles(flat, w) * sizeof(double); }

// Narrow tiles share a CTA (GT tiles side by side) so each phase has enough
// points for the CTA's threads.
inline int euler_tiles_per_cta(int flat, int w) {
    const int H = flat ? 2 : 1, chunks = flat ? 12 : 7; // 16-byte edge chunks per level and side
    // measured (B200, n=2^22): lengthening best at GT*w ~ 512 for w <= 128;
    // flattening at GT = 8, 4, 4 for w = 32, 64, 128; wide tiles alone.
    int gt = 1;
    const int want = w > 128 ? 1 : flat ? (w <= 32 ? 8 : 4) : 512 / w;
    while (gt < want && gt < 16 && (std::size_t)(2 * gt) * euler_tile_smem(flat, w) <= 100 * 1024 &&
           2 * chunks * (2 * gt) <= 256)
        gt *= 2;
    (void)H;
    if (const char* e = std::getenv("S1D_EULER_GT")) {
        const int v = std::atoi(e);
        if (v >= 1 && v <= 64 && 2 * chunks * v <= 256) gt = v;
    }
    return gt;
}

// MAXT = 1024: one thread per point of the widest span (latency-bound small
// grids, where the CTA count is below one wave).
// GMEM: tiles whose records exceed a CTA's shared memory (lengthening
// w > ~2600, flattening w > ~2800; the reference's check_width has no upper
// bound, R/core/src/swept.cpp:10-19) keep records, pressures and fluxes in a
// per-CTA global scratch block (L1/L2-resident) and only the edge ring in
// shared memory; same code, same barriers, same arithmetic.
// Resident CTAs the register budget is sized for: 64 registers per thread
// (2048 / MAXT CTAs, at most 4 of 256), except the w = 128 build (4 tiles per
// CTA), which measured 4-6% faster at 85 registers and 3 CTAs/SM (w = 64..512
// were 5-12% slower that way).
constexpr int euler_min_blocks(int maxt, int wt) {
    return maxt > 512 ? 1 : maxt > 256 ? 2 : maxt > 128 ? (wt == 128 ? 3 : S1D_EULER_MINB) : 2 * S1D_EULER_MINB;
}

// WT > 0: the tile width (and then the CTA size, MAXT) as compile-time
// constants, so tile offsets fold into immediates (the common widths).
// ONE: one tile per CTA (every width above 128) as a compile-time fact, so
// the multi-tile paths (a division per visited point, per-tile liveness)
// fold away: measured +9-10% at w = 512. GTC > 0: the tiles per CTA of a
// narrow fixed-width build as a compile-time constant.
template <int FLAT, int KIND, bool DBG, int MAXT, bool GMEM = false, int WT = 0, bool ONE = false, int GTC = 0>
__global__ void __launch_bounds__(MAXT, euler_min_blocks(MAXT, WT)) euler_tile(const TileArgs a, int GT) {
    if (ONE) GT = 1;
    else if (GTC) GT = GTC;
    using G = TileGeom<FLAT>;
    constexpr int H = G::H, REC = G::REC, LVL = G::LVL;
    extern __shared__ double sm[];
    const int w = WT ? WT : a.w, m = WT ? WT / (2 * H) : a.m, t = threadIdx.x;
    const int NT = WT ? MAXT : (int)blockDim.x;
    const int W2 = w + 2 * H;
    const std::size_t TR = (std::size_t)REC * W2 + 4 * (std::size_t)(W2 + 1); // records + pressures + fluxes
    const std::size_t TRING = 2 * (std::size_t)kERing * LVL;
    const std::size_t TS = TR + TRING;
    // per-tile views: S [REC][W2] records (local x in [0, W2)), P [W2+1]
    // pressures, Fx [3][W2+1] interface fluxes (interface x between x-1 and
    // x), ring [2 sides][kERing][LVL]
    double* const tbase = GMEM ? a.scratch + (std::size_t)blockIdx.x * GT * TR : sm;
    const std::size_t tstep = GMEM ? TR : TS;
    auto S = [&](int gi) { return tbase + gi * tstep; };
    auto Pp = [&](int gi) { return tbase + gi * tstep + REC * W2; };
    auto Fx = [&](int gi) { return tbase + gi * tstep + REC * W2 + (W2 + 1); };
    auto ring = [&](int gi) { return GMEM ? sm + gi * TRING : sm + gi * TS + TR; };
    const double gamma = a.gamma;
    const double dt_dx = a.dt_dx;
    const std::size_t tstride = (std::size_t)w * REC; // edge doubles per tile per side
    bool bad = false;

    auto tile_of = [&](int gi) { return a.b0 + (int)blockIdx.x * GT + gi; };
    // one tile per CTA: the launcher's grid is exactly the tile count
    auto live = [&](int gi) { return ONE || tile_of(gi) < (a.b1 < 0 ? a.nb : a.b1); };
    auto origin = [&](int gi) { // shard position of local x = 0
        const int b = tile_of(gi);
        const std::int64_t centre = a.seam ? (std::int64_t)(b + 1) * w : (std::int64_t)b * w + w / 2;
        return centre - w / 2 - H;
    };
    // debug: count (point, counter) computations; nudge the run's first value
    auto count = [&](int gi, int x, std::int64_t c) {
        if (DBG && a.dbg.cov) {
            unsigned* row = a.dbg.cov + (std::uint64_t)(c - 1) * a.dbg.cov_n;
            atomicAdd(row + (a.dbg.gstart + (std::uint64_t)(origin(gi) + x)) % a.dbg.cov_n, 1u);
        }
    };
    auto perturb = [&](int gi, int x, std::int64_t c, int field) {
        // reference perturb_one_ulp: the up-triangle's first level at global
        // point h of shard 0 (tile 0: local x = 2H)
        if (DBG && KIND == kUp && a.dbg.perturb && c == 1 && tile_of(gi) == 0 && x == 2 * H)
            S(gi)[field * W2 + x] = next_up(S(gi)[field * W2 + x]);
    };
    // Visit (tile, x) for x in [x0, x1) of every live tile, threads spread
    // over the concatenation of the tiles' ranges.
    auto for_all = [&](int x0, int x1, auto&& f) {
        const int cnt = x1 - x0;
        if (cnt <= 0) return;
        S1D_CHECK(x0 >= 0 && x1 <= W2, a.error_flag); // phase ranges stay inside the tile's records
        if (GT == 1) {
            if (live(0))
                for (int x = x0 + t; x < x1; x += NT) f(0, x);
            return;
        }
        // i / cnt through a float reciprocal: (i + 1/2) / cnt sits at least
        // 1/(2 cnt) >= 4.5e-4 from an integer, and the float error is below
        // GT · 2^-23 <= 2e-6 (GT <= 16), so the truncation is exact
        const float inv = __frcp_rn((float)cnt);
        for (int i = t; i < GT * cnt; i += NT) {
            const int gi = __float2int_rz(__fmul_rn((float)i + 0.5f, inv));
            S1D_CHECK(gi == i / cnt, a.error_flag);
            if (live(gi)) f(gi, x0 + (i - gi * cnt));
        }
    };

    // producers' edges (Diamond/Down); feeders: per tile, CHUNKS threads per side
    auto producers = [&](int gi, const double*& pR, const double*& pL) {
        const int b = tile_of(gi);
        if (a.seam) {
            pR = a.in_R + (std::size_t)b * tstride;
            pL = (b + 1 < a.nb) ? a.in_L + (std::size_t)(b + 1) * tstride : a.peer_L;
        } else {
            pR = (b > 0) ? a.in_R + (std::size_t)(b - 1) * tstride : a.peer_R;
            pL = a.in_L + (std::size_t)b * tstride;
        }
    };
    const int fg = t / (2 * G::CHUNKS);
    const bool feeder = KIND != kUp && fg < GT && live(fg);
    const int fside = (t % (2 * G::CHUNKS)) < G::CHUNKS ? 0 : 1, fchunk = t % G::CHUNKS;
    const double* fsrc = nullptr;
    double* fring = nullptr;
    if (feeder) {
        const double* pR;
        const double* pL;
        producers(fg, pR, pL);
        fsrc = (fside == 0 ? pR : pL) + 2 * fchunk;
        fring = ring(fg) + (std::size_t)fside * kERing * LVL + 2 * fchunk;
    }
    auto issue = [&](int q) { // level q (1-based) into its ring slot
        if (feeder && q <= m) cp_async16(fring + (std::size_t)((q - 1) % kERing) * LVL, fsrc + (std::size_t)(q - 1) * LVL);
    };
    // copy level q's ring slot into S: left records at x in [lo-H, lo+H),
    // right at [hi-H, hi+H) with lo/hi the span of level q.
    auto insert = [&](int q) {
        const int lo = w / 2 + H - q * H, hi = w / 2 + H + q * H;
        for (int i = t; i < GT * 2 * LVL; i += NT) {
            const int gi = i / (2 * LVL), k = i % (2 * LVL);
            if (!live(gi)) continue;
            const int side = k / LVL, j = k % LVL, rec = j / REC, f = j % REC;
            const int x = side == 0 ? lo - H + rec : hi - H + rec;
            S1D_CHECK(x >= 0 && x < W2, a.error_flag);
            S(gi)[f * W2 + x] = ring(gi)[((std::size_t)side * kERing + (q - 1) % kERing) * LVL + j];
        }
    };

    if (KIND == kUp) {
        for (int gi = 0; gi < GT; ++gi) {
            if (!live(gi)) continue;
            const std::int64_t g0 = origin(gi);
            for (int f = 0; f < REC; ++f)
                for (int x = H + t; x < w + H; x += NT)
                    S(gi)[f * W2 + x] = a.state_in[(std::size_t)f * a.fstride + (std::size_t)(g0 + x)];
        }
    } else {
        for (int q = 1; q <= kELook; ++q) {
            issue(q);
            if (feeder) cp_async_commit();
        }
        if (feeder) cp_async_wait<kELook - 1>();
        __syncthreads();
        insert(1);
    }
    __syncthreads();

    // One level: counter c, span [lo, hi). `between` runs after the level's
    // last reads of S outside the span and before its final barrier (inserts
    // of the next level, ring refill).
    auto level = [&](std::int64_t c, int lo, int hi, auto&& between) {
        if (!FLAT) {
            if (c & 1) {
                const int s = ((c & 3) == 1) ? 0 : 3;
                for_all(lo - 1, hi + 1, [&](int gi, int x) {
                    const double* St = S(gi);
                    Pp(gi)[x] = em::pressure(St[s * W2 + x], St[(s + 1) * W2 + x], St[(s + 2) * W2 + x], gamma, bad);
                });
                between(0);
                __syncthreads();
                for_all(lo, hi, [&](int gi, int x) {
                    const double* P = Pp(gi);
                    S(gi)[6 * W2 + x] = em::ratio(P[x - 1], P[x], P[x + 1]);
                    count(gi, x, c);
                    perturb(gi, x, c, 6);
                });
                between(1);
            } else {
                const bool fin = (c & 3) == 0;
                const int rs = fin ? 3 : 0, ws = fin ? 0 : 3;
                const double factor = fin ? dt_dx : em::mul(0.5, dt_dx);
                for_all(lo, hi + 1, [&](int gi, int x) {
                    const double* St = S(gi);
                    double* F = Fx(gi);
                    double f0, f1, f2;
                    em::iflux(St[rs * W2 + x - 1], St[(rs + 1) * W2 + x - 1], St[(rs + 2) * W2 + x - 1], St[rs * W2 + x],
                              St[(rs + 1) * W2 + x], St[(rs + 2) * W2 + x], St[6 * W2 + x - 1], St[6 * W2 + x], gamma,
                              f0, f1, f2, bad);
                    F[x] = f0;
                    F[(W2 + 1) + x] = f1;
                    F[2 * (W2 + 1) + x] = f2;
                });
                between(0);
                __syncthreads();
                for_all(lo, hi, [&](int gi, int x) {
                    double* St = S(gi);
                    const double* F = Fx(gi);
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        St[(ws + k) * W2 + x] =
                            em::update(St[k * W2 + x], factor, F[k * (W2 + 1) + x + 1], F[k * (W2 + 1) + x]);
                    count(gi, x, c);
                });
                between(1);
            }
        } else {
            const bool fin = (c & 1) == 0;
            const int s = fin ? 3 : 0, ws = fin ? 0 : 3;
            const double factor = fin ? dt_dx : em::mul(0.5, dt_dx);
            for_all(lo - 2, hi + 2, [&](int gi, int x) {
                const double* St = S(gi);
                Pp(gi)[x] = em::pressure(St[s * W2 + x], St[(s + 1) * W2 + x], St[(s + 2) * W2 + x], gamma, bad);
            });
            __syncthreads();
            for_all(lo, hi + 1, [&](int gi, int x) {
                const double* St = S(gi);
                const double* P = Pp(gi);
                double* F = Fx(gi);
                const double rl = em::ratio(P[x - 2], P[x - 1], P[x]);
                const double rr = em::ratio(P[x - 1], P[x], P[x + 1]);
                double f0, f1, f2;
                em::iflux(St[s * W2 + x - 1], St[(s + 1) * W2 + x - 1], St[(s + 2) * W2 + x - 1], St[s * W2 + x],
                          St[(s + 1) * W2 + x], St[(s + 2) * W2 + x], rl, rr, gamma, f0, f1, f2, bad);
                F[x] = f0;
                F[(W2 + 1) + x] = f1;
                F[2 * (W2 + 1) + x] = f2;
            });
            between(0);
            __syncthreads();
            for_all(lo, hi, [&](int gi, int x) {
                double* St = S(gi);
                const double* F = Fx(gi);
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    St[(ws + k) * W2 + x] =
                        em::update(St[k * W2 + x], factor, F[k * (W2 + 1) + x + 1], F[k * (W2 + 1) + x]);
                count(gi, x, c);
                perturb(gi, x, c, ws);
            });
            between(1);
        }
        __syncthreads();
    };

    auto export_level = [&](int d, int lo, int hi) {
        for (int i = t; i < GT * 2 * LVL; i += NT) {
            const int gi = i / (2 * LVL), k = i % (2 * LVL);
            if (!live(gi)) continue;
            const int b = tile_of(gi);
            const int side = k / LVL, j = k % LVL, rec = j / REC, f = j % REC;
            const int x = side == 0 ? lo + rec : hi - 2 * H + rec;
            S1D_CHECK(x >= 0 && x < W2 && d >= 0 && d < m, a.error_flag);
            double* o = (side == 0 ? a.out_L : a.out_R) + (std::size_t)b * tstride + (std::size_t)d * LVL;
            o[j] = S(gi)[f * W2 + x];
        }
    };

    const std::int64_t base = a.base;
    if (KIND != kUp) {
        for (int r = 1; r <= m; ++r) {
            const int lo = w / 2 + H - r * H, hi = w / 2 + H + r * H;
            if (feeder) { // queue level r+kELook; level r+1 must land before the phase barrier
                issue(r + kELook);
                cp_async_commit();
            }
            level(base + r, lo, hi, [&](int phase) {
                if (phase == 0) {
                    if (feeder) cp_async_wait<kELook - 1>();
                } else if (r < m) {
                    insert(r + 1);
                }
            });
        }
    }
    if (KIND != kDown) {
        export_level(0, H, w + H);
        for (int r = m + 1; r <= 2 * m - 1; ++r) {
            const int d = r - m, lo = H + d * H, hi = w + H - d * H;
            level(base + r, lo, hi, [](int) {});
            export_level(d, lo, hi);
        }
    } else {
        for (int gi = 0; gi < GT; ++gi) {
            if (!live(gi)) continue;
            const std::int64_t g0 = origin(gi);
            for (int f = 0; f < REC; ++f)
                for (int x = H + t; x < w + H; x += NT) {
                    const std::uint64_t gp = (std::uint64_t)(g0 + x);
                    if (gp < a.N) a.state_out[(std::size_t)f * a.fstride + gp] = S(gi)[f * W2 + x];
                    else a.state_right[(std::size_t)f * a.right_fstride + (gp - a.N)] = S(gi)[f * W2 + x];
                }
        }
    }
    raise_flag(a.error_flag, bad);
}

// Largest dynamic shared memory a CTA may opt into (read once per process).
std::size_t smem_optin() {
    static const std::size_t v = [] {
        int dev = 0, b = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&b, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || b <= 0) {
            cudaGetLastError();
            b = 227 * 1024;
        }
        return (std::size_t)b;
    }();
    return v;
}

template <int FLAT, bool DBG = false, int MAXT = 256, bool GMEM = false, int WT = 0, int GTC = 0>
cudaError_t launch_tile_f(int kind, const TileArgs& a_in, cudaStream_t st, int cap_threads = 0) {
    TileArgs a = a_in;
    const int GT = GMEM ? 1 : GTC ? GTC : euler_tiles_per_cta(FLAT, a.w);
    const std::size_t ring_doubles = 2 * (std::size_t)kERing * TileGeom<FLAT>::LVL;
    const size_t smem = GMEM ? GT * ring_doubles * sizeof(double) : (size_t)GT * euler_tile_smem(FLAT, a.w);
    void (*k)(const TileArgs, int) = nullptr;
    if constexpr (GTC > 1) {
        k = kind == kUp ? euler_tile<FLAT, kUp, DBG, MAXT, false, WT, false, GTC>
            : kind == kDiamond ? euler_tile<FLAT, kDiamond, DBG, MAXT, false, WT, false, GTC>
                               : euler_tile<FLAT, kDown, DBG, MAXT, false, WT, false, GTC>;
    } else {
        if (GT == 1 || WT || GMEM) {
            k = kind == kUp ? euler_tile<FLAT, kUp, DBG, MAXT, GMEM, WT, true>
                : kind == kDiamond ? euler_tile<FLAT, kDiamond, DBG, MAXT, GMEM, WT, true>
                                   : euler_tile<FLAT, kDown, DBG, MAXT, GMEM, WT, true>;
        } else if constexpr (!WT && !GMEM) {
            k = kind == kUp ? euler_tile<FLAT, kUp, DBG, MAXT, false, 0, false>
                : kind == kDiamond ? euler_tile<FLAT, kDiamond, DBG, MAXT, false, 0, false>
                                   : euler_tile<FLAT, kDown, DBG, MAXT, false, 0, false>;
        }
    }
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    // narrow tiles: 128-thread CTAs (more tiles in flight per SM)
    int cap = cap_threads > 0 ? cap_threads : MAXT > 256 ? MAXT : a.w <= 256 && GT == 1 ? 128 : 256;
    if (const char* e = std::getenv("S1D_EULER_NT")) cap = std::atoi(e);
    if (cap < 32 || cap > MAXT) cap = MAXT;
    int nt = ((GT * (a.w + 2 * TileGeom<FLAT>::H) + 31) / 32) * 32;
    if (nt > cap) nt = cap;
    const int need = 32 * ((2 * TileGeom<FLAT>::CHUNKS * GT + 31) / 32); // feeder threads
    if (nt < need) nt = need;
    if (WT && (a.w != WT || nt != MAXT)) return cudaErrorInvalidValue; // compile-time shape must match
    const int count = (a.b1 < 0 ? a.nb : a.b1) - a.b0;
    if (count <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((count + GT - 1) / GT);
    if (GMEM) { // stream-ordered scratch for this launch (graph-capturable)
        const std::size_t bytes = sizeof(double) * grid * GT * (euler_tile_doubles(FLAT, a.w) - ring_doubles);
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&a.scratch), bytes, st);
        if (e != cudaSuccess) return e;
    }
    k<<<grid, nt, smem, st>>>(a, GT);
    cudaError_t e = cudaGetLastError();
    if (GMEM) {
        const cudaError_t f = cudaFreeAsync(a.scratch, st);
        if (e == cudaSuccess) e = f;
    }
    return e;
}

__global__ void unpack_kernel(const double* __restrict__ aos, double* __restrict__ st, std::uint64_t N,
                              std::uint64_t fs, int rec) {
    for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < N;
         i += (std::uint64_t)gridDim.x * blockDim.x) {
        const double q0 = aos[3 * i], q1 = aos[3 * i + 1], q2 = aos[3 * i + 2];
        st[i] = q0;
        st[i + fs] = q1;
        st[i + 2 * fs] = q2;
        st[i + 3 * fs] = q0;
        st[i + 4 * fs] = q1;
        st[i + 5 * fs] = q2;
        if (rec == 7) st[i + 6 * fs] = 0.0; // make_cell: Pr = 0 (inc/kernels.hpp:144-149)
    }
}

__global__ void pack_kernel(const double* __restrict__ st, double* __restrict__ aos, std::uint64_t N,
                            std::uint64_t fs) {
    for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < N;
         i += (std::uint64_t)gridDim.x * blockDim.x) {
        aos[3 * i] = st[i];
        aos[3 * i + 1] = st[i + fs];
        aos[3 * i + 2] = st[i + 2 * fs];
    }
}

unsigned grid_for(std::uint64_t n, int per_block, int sms) {
    std::uint64_t blocks = (n + per_block - 1) / per_block;
    const std::uint64_t cap = (std::uint64_t)sms * 16;
    if (blocks > cap) blocks = cap;
    return (unsigned)(blocks ? blocks : 1);
}

} // namespace

cudaError_t launch_euler_classic(int flat, const ClassicArgs& a, cudaStream_t st) {
    const unsigned grid = grid_for(a.N, flat ? kFlatClassicPoints : len_classic_points((int)(a.counter & 3)), a.sms);
    if (flat) {
        if (a.counter & 1) euler_flat_classic<0><<<grid, kClassicB, 0, st>>>(a);
        else euler_flat_classic<1><<<grid, kClassicB, 0, st>>>(a);
    } else {
        switch (a.counter & 3) {
        case 1: euler_len_classic<1><<<grid, kClassicB, 0, st>>>(a); break;
        case 2: euler_len_classic<2><<<grid, kClassicB, 0, st>>>(a); break;
        case 3: euler_len_classic<3><<<grid, kClassicB, 0, st>>>(a); break;
        default: euler_len_classic<0><<<grid, kClassicB, 0, st>>>(a); break;
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_euler_tile(int flat, int kind, const TileArgs& a, cudaStream_t st, bool debug) {
    if (euler_tile_smem(flat, a.w) > smem_optin()) { // records in global scratch
        if (debug) return flat ? launch_tile_f<1, true, 256, true>(kind, a, st)
                               : launch_tile_f<0, true, 256, true>(kind, a, st);
        return flat ? launch_tile_f<1, false, 1024, true>(kind, a, st, 512)
                    : launch_tile_f<0, false, 1024, true>(kind, a, st, 512);
    }
    if (debug) return flat ? launch_tile_f<1, true>(kind, a, st) : launch_tile_f<0, true>(kind, a, st);
    // Latency-bound launches (at most one CTA per SM, e.g. 2^16 points per GPU)
    // run one thread per span point (1024-thread CTAs): measured +15-20% at
    // 2^16; with more CTAs than SMs the 256-thread build's occupancy wins (2x).
    const int sms = a.sms;
    const int count = (a.b1 < 0 ? a.nb : a.b1) - a.b0;
    const int GT = euler_tiles_per_cta(flat, a.w);
    bool wide = (count + GT - 1) / GT <= sms;
    // Tiles whose shared memory already limits the SM to two CTAs (w >= 1024)
    // run 512 threads per CTA: measured +11-14% at w = 1024 (slower at w <= 512).
    const int cap = !wide && (size_t)GT * euler_tile_smem(flat, a.w) > 76 * 1024 ? 512 : 0;
    if (const char* e = std::getenv("S1D_EULER_NT")) wide = std::atoi(e) > 256;
    // The common widths run builds with the tile width and CTA size as
    // compile-time constants (w = 256: 128 threads; 512: 256; 1024: 512).
    const bool fixed = GT == 1 && !std::getenv("S1D_EULER_NT");
    if (!wide && cap == 512 && fixed && a.w == 1024)
        return flat ? launch_tile_f<1, false, 512, false, 1024>(kind, a, st)
                    : launch_tile_f<0, false, 512, false, 1024>(kind, a, st);
    if (!wide && cap == 512 && fixed && a.w == 2048)
        return flat ? launch_tile_f<1, false, 512, false, 2048>(kind, a, st)
                    : launch_tile_f<0, false, 512, false, 2048>(kind, a, st);
    // latency-bound grids at w = 512: one thread per span point, 17 warps
    if (wide && fixed && a.w == 512)
        return flat ? launch_tile_f<1, false, 544, false, 512>(kind, a, st)
                    : launch_tile_f<0, false, 544, false, 512>(kind, a, st);
    if (wide || cap)
        return flat ? launch_tile_f<1, false, 1024>(kind, a, st, cap) : launch_tile_f<0, false, 1024>(kind, a, st, cap);
    if (fixed && a.w == 512)
        return flat ? launch_tile_f<1, false, 256, false, 512>(kind, a, st)
                    : launch_tile_f<0, false, 256, false, 512>(kind, a, st);
    if (fixed && a.w == 256)
        return flat ? launch_tile_f<1, false, 128, false, 256>(kind, a, st)
                    : launch_tile_f<0, false, 128, false, 256>(kind, a, st);
    // narrow fixed widths: several tiles per 256-thread CTA (GT as measured
    // by euler_tiles_per_cta, a compile-time constant here)
    if (!std::getenv("S1D_EULER_NT") && !std::getenv("S1D_EULER_GT")) {
        if (flat) {
            if (a.w == 128 && GT == 4) return launch_tile_f<1, false, 256, false, 128, 4>(kind, a, st);
            if (a.w == 64 && GT == 4) return launch_tile_f<1, false, 256, false, 64, 4>(kind, a, st);
            if (a.w == 32 && GT == 8) return launch_tile_f<1, false, 256, false, 32, 8>(kind, a, st);
        } else {
            if (a.w == 128 && GT == 4) return launch_tile_f<0, false, 256, false, 128, 4>(kind, a, st);
            if (a.w == 64 && GT == 8) return launch_tile_f<0, false, 256, false, 64, 8>(kind, a, st);
            if (a.w == 32 && GT == 8) return launch_tile_f<0, false, 256, false, 32, 8>(kind, a, st);
        }
    }
    return flat ? launch_tile_f<1>(kind, a, st) : launch_tile_f<0>(kind, a, st);
}

cudaError_t launch_euler_unpack(const double* aos, double* st_fields, std::uint64_t N, std::uint64_t fs, int rec,
                                cudaStream_t st) {
    unpack_kernel<<<grid_for(N, 256, 148), 256, 0, st>>>(aos, st_fields, N, fs, rec);
    return cudaGetLastError();
}

cudaError_t launch_euler_pack(const double* st_fields, double* aos, std::uint64_t N, std::uint64_t fs,
                              cudaStream_t st) {
    pack_kernel<<<grid_for(N, 256, 148), 256, 0, st>>>(st_fields, aos, N, fs);
    return cudaGetLastError();
}

std::size_t euler_tile_smem_bytes(int flat, int w) { return euler_tile_smem(flat, w); }

} // namespace s1d
