// misc_kernels.cu — device KAT hooks for the RNG and the FP64 roofline
// microbenchmark.
#include <cuda_runtime.h>

#include "kernels.h"
#include "fastmath.cuh"
#include "smc_device.cuh"

namespace smc {
namespace {

__global__ void philox_kernel(int64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const u32x4 r = philox4x32_10(u32x4{ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]}, key[2 * i],
                                  key[2 * i + 1]);
    out[4 * i] = r.x;
    out[4 * i + 1] = r.y;
    out[4 * i + 2] = r.z;
    out[4 * i + 3] = r.w;
}

// Box-Muller pairs exactly as the fast particle kernel draws them.
__global__ void normal_pairs_kernel(uint64_t seed, uint32_t obs, uint32_t particle, int64_t n, double* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Uniform2 u = uniform_block(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), obs, particle,
                                     static_cast<uint64_t>(i));
    const double r = fm::sqrt_pos(-2.0 * fm::log_tab(u.u0));
    double sn, cs;
    fm::sincospi(2.0 * u.u1, &sn, &cs);
    out[2 * i] = r * cs;
    out[2 * i + 1] = r * sn;
}

// 8 independent DFMA chains per thread; 2 flops per DFMA.
__global__ void __launch_bounds__(256) dfma_peak_kernel(int iters, double* sink) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = 1.0 + 1e-9 * (threadIdx.x + q);
    const double b = 0.999999999, c = 1e-12;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = fma(a[q], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += a[q];
    if (s == 12345.0) sink[blockIdx.x] = s;  // never true; keeps the chains live
}

// The FP32 counterpart: 8 independent FFMA chains per thread.
__global__ void __launch_bounds__(256) ffma_peak_kernel(int iters, double* sink) {
    float a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = 1.0f + 1e-6f * float(threadIdx.x + q);
    const float b = 0.9999999f, c = 1e-9f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = fmaf(a[q], b, c);
    }
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += a[q];
    if (s == 12345.0f) sink[blockIdx.x] = s;  // never true; keeps the chains live
}

}  // namespace

cudaError_t launch_philox(int64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out, cudaStream_t s) {
    philox_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(n, ctr, key, out);
    return cudaGetLastError();
}

cudaError_t launch_normal_pairs(uint64_t seed, uint32_t obs, uint32_t particle, int64_t n, double* out,
                                cudaStream_t s) {
    normal_pairs_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(seed, obs, particle, n, out);
    return cudaGetLastError();
}

cudaError_t launch_dfma_peak(int n_blocks, int iters, double* sink, cudaStream_t s) {
    dfma_peak_kernel<<<n_blocks, 256, 0, s>>>(iters, sink);
    return cudaGetLastError();
}

cudaError_t launch_ffma_peak(int n_blocks, int iters, double* sink, cudaStream_t s) {
    ffma_peak_kernel<<<n_blocks, 256, 0, s>>>(iters, sink);
    return cudaGetLastError();
}

}  // namespace smc
