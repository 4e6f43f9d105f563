// galerkin_kernels.cu — spectral Galerkin reference solver on the device
// (src/galerkin.cpp).
//
// The explicit Euler step Theta <- Theta + dt A Theta is a dense complex
// GEMV: A (nb^2 x 16 B, 19 MB at box cutoff 16) stays in L2 / HBM and each
// step streams it once, so the step is bandwidth-bound (4 DFMA per 16 B).
// One warp per row: the lanes read the row with coalesced 16-byte loads and
// the axpy is fused into the row's epilogue (ping-pong Theta buffers, since
// every row reads the whole previous Theta).
#include <cuda_runtime.h>

#include "kernels.h"
#include "scalar_eval.cuh"

namespace smc {
namespace {

constexpr int kRowsPerBlock = 8;  // 8 warps

__global__ void __launch_bounds__(32 * kRowsPerBlock) gemv_step_kernel(const double2* __restrict__ A,
                                                                       const double2* __restrict__ th,
                                                                       double2* __restrict__ out, int64_t nb,
                                                                       double dt) {
    const int lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock + (threadIdx.x >> 5);
    if (row >= nb) return;
    const double2* a = A + row * nb;
    double re = 0.0, im = 0.0, re2 = 0.0, im2 = 0.0;
    int64_t m = lane;
    for (; m + 32 < nb; m += 64) {  // two independent accumulators per lane
        const double2 x = __ldg(a + m), y = __ldg(th + m);
        const double2 x2 = __ldg(a + m + 32), y2 = __ldg(th + m + 32);
        re = fma(x.x, y.x, fma(-x.y, y.y, re));
        im = fma(x.x, y.y, fma(x.y, y.x, im));
        re2 = fma(x2.x, y2.x, fma(-x2.y, y2.y, re2));
        im2 = fma(x2.x, y2.y, fma(x2.y, y2.x, im2));
    }
    if (m < nb) {
        const double2 x = __ldg(a + m), y = __ldg(th + m);
        re = fma(x.x, y.x, fma(-x.y, y.y, re));
        im = fma(x.x, y.y, fma(x.y, y.x, im));
    }
    re += re2;
    im += im2;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, off);
        im += __shfl_xor_sync(0xffffffffu, im, off);
    }
    if (lane == 0) {
        const double2 t = th[row];
        out[row] = make_double2(t.x + dt * re, t.y + dt * im);  // theta += dt * scratch (galerkin.cpp:208-209)
    }
}

// Theta_l = (1/n^2) sum_jk theta_0(j/n, k/n) e^{-2 pi i (l1 j + l2 k)/n}
// (galerkin.cpp:83-101): one block per mode.
__global__ void quadrature_kernel(ScalarImg f, const int* __restrict__ k1s, const int* __restrict__ k2s, int n,
                                  double2* __restrict__ theta) {
    __shared__ double sr[256], si[256];
    const int l = blockIdx.x;
    const double l1 = k1s[l], l2 = k2s[l];
    double re = 0.0, im = 0.0;
    const int64_t total = static_cast<int64_t>(n) * n;
    for (int64_t q = threadIdx.x; q < total; q += blockDim.x) {
        const int j = static_cast<int>(q / n), k = static_cast<int>(q - static_cast<int64_t>(j) * n);
        const double v = scalar_eval(f, double(j) / n, double(k) / n);
        double s, c;
        sincospi(-2.0 * (l1 * j / n + l2 * k / n), &s, &c);
        re += v * c;
        im += v * s;
    }
    sr[threadIdx.x] = re;
    si[threadIdx.x] = im;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            sr[threadIdx.x] += sr[threadIdx.x + w];
            si[threadIdx.x] += si[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) theta[l] = make_double2(sr[0] / double(n) / double(n), si[0] / double(n) / double(n));
}

// Re sum_l Theta_l e^{2 pi i l.x} (galerkin.cpp:213-219) for one point.
__global__ void observe_kernel(const double2* __restrict__ th, const int* __restrict__ k1s,
                               const int* __restrict__ k2s, int64_t nb, double x1, double x2, double* out) {
    __shared__ double sr[256];
    double re = 0.0;
    for (int64_t l = threadIdx.x; l < nb; l += blockDim.x) {
        double s, c;
        sincospi(2.0 * (double(k1s[l]) * x1 + double(k2s[l]) * x2), &s, &c);
        const double2 t = th[l];
        re += t.x * c - t.y * s;
    }
    sr[threadIdx.x] = re;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sr[threadIdx.x] += sr[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sr[0];
}

// galerkin_field_grid (galerkin.cpp:233-250): one thread per grid point.
__global__ void field_grid_kernel(const double2* __restrict__ c, const int* __restrict__ k1s,
                                  const int* __restrict__ k2s, int64_t nb, int n, double* __restrict__ grid) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= static_cast<int64_t>(n) * n) return;
    const int i = static_cast<int>(q / n), j = static_cast<int>(q - static_cast<int64_t>(i) * n);
    double v = 0.0;
    for (int64_t l = 0; l < nb; ++l) {
        double s, co;
        sincospi(2.0 * (double(k1s[l]) * i / n + double(k2s[l]) * j / n), &s, &co);
        const double2 t = c[l];
        v += t.x * co - t.y * s;
    }
    grid[q] = v;
}

}  // namespace

cudaError_t launch_galerkin_step(const double* A, const double* th, double* out, int64_t nb, double dt,
                                 cudaStream_t s) {
    const unsigned blocks = static_cast<unsigned>((nb + kRowsPerBlock - 1) / kRowsPerBlock);
    gemv_step_kernel<<<blocks, 32 * kRowsPerBlock, 0, s>>>(reinterpret_cast<const double2*>(A),
                                                           reinterpret_cast<const double2*>(th),
                                                           reinterpret_cast<double2*>(out), nb, dt);
    return cudaGetLastError();
}

cudaError_t launch_galerkin_quadrature(const ScalarImg& f, const int* k1, const int* k2, int64_t nb, int n,
                                       double* theta, cudaStream_t s) {
    quadrature_kernel<<<static_cast<unsigned>(nb), 256, 0, s>>>(f, k1, k2, n, reinterpret_cast<double2*>(theta));
    return cudaGetLastError();
}

cudaError_t launch_galerkin_observe(const double* th, const int* k1, const int* k2, int64_t nb, double x1, double x2,
                                    double* out, cudaStream_t s) {
    observe_kernel<<<1, 256, 0, s>>>(reinterpret_cast<const double2*>(th), k1, k2, nb, x1, x2, out);
    return cudaGetLastError();
}

cudaError_t launch_galerkin_field_grid(const double* c, const int* k1, const int* k2, int64_t nb, int n, double* grid,
                                       cudaStream_t s) {
    const int64_t total = static_cast<int64_t>(n) * n;
    field_grid_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const double2*>(c), k1, k2, nb, n, grid);
    return cudaGetLastError();
}

}  // namespace smc
