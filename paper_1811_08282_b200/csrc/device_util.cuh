// Small device helpers shared by the kernels.
#pragma once

namespace s1d {

// std::nextafter(x, +inf) for finite x (the reference's perturb_one_ulp,
// inc/kernels.hpp:122-125).
__device__ __forceinline__ double next_up(double x) {
    if (x != x) return x;
    if (x == 0.0) return __longlong_as_double(1LL); // smallest positive subnormal
    const long long b = __double_as_longlong(x);
    return __longlong_as_double(x > 0.0 ? b + 1 : b - 1);
}

// Checked builds (-DS1D_CHECKED): index bounds of the tile kernels' shared
// and global accesses are verified at run time; a violation sets bit 2 (value
// 4) of the launch's error flag (no trap, so the GPU never needs a reset) and
// the host reports S1D_INTERNAL.
#ifdef S1D_CHECKED
#define S1D_CHECK(cond, flag)                                                                                      \
    do {                                                                                                           \
        if (!(cond)) atomicOr((flag), 4);                                                                          \
    } while (0)
#else
#define S1D_CHECK(cond, flag)                                                                                      \
    do {                                                                                                           \
    } while (0)
#endif

// Round hand-off between shards of different processes (one process per GPU):
// a shard's flag word holds the rounds completed by one ring neighbour, stored
// by that neighbour over NVLink (system-scope release) and polled here
// (system-scope acquire). The spin is bounded: after timeout_ns it sets bit 1
// of *err and returns, so a dead peer cannot wedge the GPU. The abort is
// sticky: once bit 1 is set (by any wait of the run), every later wait
// returns at once, so a run of R rounds after a peer died costs one timeout,
// not R (the host then reports S1D_TRANSPORT_ABORTED).
__device__ __forceinline__ unsigned flag_ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void flag_st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ bool transport_aborted(const int* err) {
    return (*reinterpret_cast<const volatile int*>(err) & 2) != 0;
}
__device__ __forceinline__ void flag_wait(const unsigned* f, unsigned seq, int* err, unsigned long long timeout_ns) {
    if ((int)(flag_ld_acquire(f) - seq) >= 0) return;
    if (transport_aborted(err)) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while ((int)(flag_ld_acquire(f) - seq) < 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns || transport_aborted(err)) {
            atomicOr(err, 2);
            return;
        }
    }
}
__device__ __forceinline__ void flag_signal(unsigned* f, unsigned seq) {
    __threadfence_system();
    flag_st_release(f, seq);
}

} // namespace s1d
