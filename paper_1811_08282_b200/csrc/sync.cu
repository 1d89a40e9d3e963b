// Cross-process round ordering for one-process-per-GPU shards.
//
// Each shard owns `flags[2]` in its device memory: flags[0] = rounds completed
// by its LEFT ring neighbour, flags[1] = by its RIGHT neighbour. After a round
// a shard's stream runs signal_kernel, which publishes its round count into
// both neighbours' flags (peer stores over NVLink, system-scope release).
// Before the next round, wait_kernel spins (system-scope acquire) until both
// of its own flags have caught up. The spin is bounded: after `timeout_ns` it
// sets bit 1 of the shard's error flag and returns, so a dead peer can never
// wedge the GPU (the host reports S1D_TRANSPORT_ABORTED). The abort is sticky
// (bit 1 already set: return at once), so only the first round pays it.
//
// This replaces RingTransport's mutex/condvar round barrier
// (src/transport.cpp:112-171) with device-side ordering: no host round trip
// per round, and the payload itself never moves (consumers read the
// producer's edge buffer in place).
#include <cstdint>

#include "device_util.cuh"
#include "kernels.hpp"

namespace s1d {
namespace {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ std::uint64_t globaltimer() {
    std::uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void wait_kernel(const unsigned* flags, unsigned seq, int* err, std::uint64_t timeout_ns) {
    if (threadIdx.x != 0) return;
    const std::uint64_t t0 = globaltimer();
    while (true) {
        const unsigned a = ld_acquire_sys(flags), b = ld_acquire_sys(flags + 1);
        if ((int)(a - seq) >= 0 && (int)(b - seq) >= 0) break;
        if (transport_aborted(err)) break;
        if (globaltimer() - t0 > timeout_ns) {
            atomicOr(err, 2);
            break;
        }
        __nanosleep(256);
    }
    __threadfence_system();
}

__global__ void signal_kernel(unsigned* left_flags_slot, unsigned* right_flags_slot, unsigned seq) {
    if (threadIdx.x != 0) return;
    __threadfence_system();
    st_release_sys(left_flags_slot, seq);
    st_release_sys(right_flags_slot, seq);
}

// Transport calibration (s1d_calibrate_transport): `iters` flag hand-offs
// between two devices. The starter stores i into the peer's flag and spins
// until i comes back; the echo spins for i, then stores it back. One-way
// latency = elapsed / (2 iters). Bounded by `timeout_ns` like wait_kernel.
__global__ void pingpong_kernel(const unsigned* mine, unsigned* peer, int iters, int starter, int* err,
                                std::uint64_t timeout_ns) {
    if (threadIdx.x != 0) return;
    const std::uint64_t t0 = globaltimer();
    for (unsigned i = 1; i <= (unsigned)iters; ++i) {
        if (starter) st_release_sys(peer, i);
        while ((int)(ld_acquire_sys(mine) - i) < 0) {
            if (globaltimer() - t0 > timeout_ns) {
                atomicOr(err, 2);
                return;
            }
        }
        if (!starter) st_release_sys(peer, i);
    }
}

__global__ void set_u32_kernel(unsigned* p, unsigned v) { *p = v; }

} // namespace

cudaError_t launch_set_u32(unsigned* p, unsigned v, cudaStream_t st) {
    set_u32_kernel<<<1, 1, 0, st>>>(p, v);
    return cudaGetLastError();
}

cudaError_t launch_pingpong(const unsigned* mine, unsigned* peer, int iters, int starter, int* err,
                            std::uint64_t timeout_ns, cudaStream_t st) {
    pingpong_kernel<<<1, 32, 0, st>>>(mine, peer, iters, starter, err, timeout_ns);
    return cudaGetLastError();
}

cudaError_t launch_wait_flags(const unsigned* flags, unsigned seq, int* err, std::uint64_t timeout_ns,
                              cudaStream_t st) {
    wait_kernel<<<1, 32, 0, st>>>(flags, seq, err, timeout_ns);
    return cudaGetLastError();
}

cudaError_t launch_signal_flags(unsigned* left_slot, unsigned* right_slot, unsigned seq, cudaStream_t st) {
    signal_kernel<<<1, 32, 0, st>>>(left_slot, right_slot, seq);
    return cudaGetLastError();
}

} // namespace s1d
