// FP64 pipe peak microbenchmark (roofline denominator for the swept kernels).
// Eight independent DADD/DMUL chains per thread; -fmad=false keeps them as
// separate DADD and DMUL instructions, exactly the op mix of heat_step.
#include <cuda_runtime.h>

#include <string>

#include "host_config.hpp"
#include "swept1d.h"

namespace {

__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            x[i] = __dadd_rn(x[i], a);
            x[i] = __dmul_rn(x[i], b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s = __dadd_rn(s, x[i]);
    if (s == 12345.678) out[0] = s; // keep the chains live
}

} // namespace

extern "C" int s1d_measure_fp64_peak(int device, double* ops_per_second, char* err, size_t errlen) {
    auto fail = [&](const char* what, cudaError_t e) {
        if (err && errlen) {
            std::string m = std::string(what) + ": " + cudaGetErrorString(e);
            size_t n = m.size() < errlen - 1 ? m.size() : errlen - 1;
            m.copy(err, n);
            err[n] = 0;
        }
        return (int)S1D_CUDA_ERROR;
    };
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        if (err && errlen) {
            const std::string m = "no CUDA device visible";
            const size_t n = m.size() < errlen - 1 ? m.size() : errlen - 1;
            m.copy(err, n);
            err[n] = 0;
        }
        return (int)S1D_NO_DEVICE;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail("cudaSetDevice", e);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* out = nullptr;
    if ((e = cudaMalloc(&out, sizeof(double))) != cudaSuccess) return fail("cudaMalloc", e);
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    const int iters = 4096, blocks = sms * 8, threads = 256;
    fp64_peak_kernel<<<blocks, threads>>>(out, 256, 1.0000001, 0.9999999); // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(t0);
        fp64_peak_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 0.9999999);
        cudaEventRecord(t1);
        cudaEventSynchronize(t1);
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        if (ms < best) best = ms;
    }
    e = cudaGetLastError();
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaFree(out);
    if (e != cudaSuccess) return fail("fp64_peak_kernel", e);
    const double ops = 16.0 * iters * (double)blocks * threads;
    *ops_per_second = ops / (best * 1e-3);
    if (err && errlen) err[0] = 0;
    return S1D_OK;
}
