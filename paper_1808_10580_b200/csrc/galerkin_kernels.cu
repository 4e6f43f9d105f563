// galerkin_kernels.cu — spectral Galerkin reference solver on the device
// (src/galerkin.cpp).
//
// The explicit Euler step Theta <- Theta + dt A Theta is a dense complex
// GEMV: A (nb^2 x 16 B, 19 MB at box cutoff 16) stays in L2 / HBM and each
// step streams it once, so the step is bandwidth-bound (4 DFMA per 16 B).
// The threads of a block read their row with coalesced 16-byte loads and
// the axpy is fused into the row's epilogue (ping-pong Theta buffers, since
// every row reads the whole previous Theta).  One block per row.
#include <cuda_runtime.h>

#include "kernels.h"
#include "scalar_eval.cuh"

namespace smc {
namespace {

constexpr int kStepThreads = 128;

// One block per row: every thread streams a strided slice of the row (all its
// loads independent, so a whole row is one L2/HBM round trip instead of a
// warp-serial walk), then a shuffle + shared-memory reduction.
__global__ void __launch_bounds__(kStepThreads) gemv_step_kernel(const double2* __restrict__ A,
                                                                 const double2* __restrict__ th,
                                                                 double2* __restrict__ out, int64_t nb, double dt) {
    const int64_t row = blockIdx.x;
    const double2* a = A + row * nb;
    double re = 0.0, im = 0.0, re2 = 0.0, im2 = 0.0;
    int64_t m = threadIdx.x;
    for (; m + kStepThreads < nb; m += 2 * kStepThreads) {
        const double2 x = __ldg(a + m), y = __ldg(th + m);
        const double2 x2 = __ldg(a + m + kStepThreads), y2 = __ldg(th + m + kStepThreads);
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
    __shared__ double2 part[kStepThreads / 32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = make_double2(re, im);
    __syncthreads();
    if (threadIdx.x == 0) {
        double sr = 0.0, si = 0.0;
#pragma unroll
        for (int w = 0; w < kStepThreads / 32; ++w) {
            sr += part[w].x;
            si += part[w].y;
        }
        const double2 t = th[row];
        out[row] = make_double2(t.x + dt * sr, t.y + dt * si);  // theta += dt * scratch (galerkin.cpp:208-209)
    }
}

// A_lm (galerkin.cpp:108-142) with the reference's std::complex operation
// sequence, uncontracted (explicit _rn intrinsics), so A is bit-identical to
// the host assembly: vhat from a dense (2K+1)^2 grid of vector coefficients
// [c1re, c1im, c2re, c2im], present[] marks the stored wavenumbers.
__global__ void assemble_kernel(const double4* __restrict__ vhat, const unsigned char* __restrict__ present, int K,
                                const int* __restrict__ k1s, const int* __restrict__ k2s, int64_t nb, double kappa,
                                int constant, double v1, double v2, double2* __restrict__ A) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t l = blockIdx.y;
    if (j >= nb) return;
    const double two_pi = 6.283185307179586;
    const int l1 = k1s[l], l2 = k2s[l], m1 = k1s[j], m2 = k2s[j];
    double re = 0.0, im = 0.0;
    if (constant) {
        if (l == j) {  // A_ll -= i2pi * (v . l): complex * double = (0 x, 2 pi x)
            const double x = __dadd_rn(__dmul_rn(v1, double(l1)), __dmul_rn(v2, double(l2)));
            re = __dsub_rn(re, __dmul_rn(0.0, x));
            im = __dsub_rn(im, __dmul_rn(two_pi, x));
        }
    } else {
        const int d1 = l1 - m1, d2 = l2 - m2;
        if (d1 >= -K && d1 <= K && d2 >= -K && d2 <= K) {
            const int64_t g = static_cast<int64_t>(d1 + K) * (2 * K + 1) + (d2 + K);
            if (present[g]) {
                const double4 c = vhat[g];
                // (c1 m1 + c2 m2) * (0 + 2 pi i): (a 0 - b 2pi, a 2pi + b 0)
                const double a = __dadd_rn(__dmul_rn(c.x, double(m1)), __dmul_rn(c.z, double(m2)));
                const double b = __dadd_rn(__dmul_rn(c.y, double(m1)), __dmul_rn(c.w, double(m2)));
                const double tr = __dsub_rn(__dmul_rn(a, 0.0), __dmul_rn(b, two_pi));
                const double ti = __dadd_rn(__dmul_rn(a, two_pi), __dmul_rn(b, 0.0));
                re = __dsub_rn(re, tr);
                im = __dsub_rn(im, ti);
            }
        }
    }
    if (l == j) {
        const double ksq = __dmul_rn(__dmul_rn(two_pi, two_pi),
                                     __dadd_rn(__dmul_rn(double(l1), double(l1)), __dmul_rn(double(l2), double(l2))));
        re = __dsub_rn(re, __dmul_rn(kappa, ksq));
    }
    A[l * nb + j] = make_double2(re, im);
}

// Gershgorin bound max_l sum_m |A_lm| (galerkin.cpp:153-156, :170-171):
// one block per row, the maximum through the bit pattern of a non-negative
// double (monotone as an unsigned integer).
__global__ void radius_kernel(const double2* __restrict__ A, int64_t nb, unsigned long long* out) {
    __shared__ double part[8];
    double s = 0.0;
    const double2* a = A + static_cast<int64_t>(blockIdx.x) * nb;
    for (int64_t m = threadIdx.x; m < nb; m += blockDim.x) s += hypot(a[m].x, a[m].y);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
        atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(t)));
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
    gemv_step_kernel<<<static_cast<unsigned>(nb), kStepThreads, 0, s>>>(reinterpret_cast<const double2*>(A),
                                                           reinterpret_cast<const double2*>(th),
                                                           reinterpret_cast<double2*>(out), nb, dt);
    return cudaGetLastError();
}

cudaError_t launch_galerkin_assemble(const double* vhat, const unsigned char* present, int K, const int* k1,
                                     const int* k2, int64_t nb, double kappa, int constant, double v1, double v2,
                                     double* A, unsigned long long* radius_bits, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((nb + 255) / 256), static_cast<unsigned>(nb));
    assemble_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const double4*>(vhat), present, K, k1, k2, nb, kappa,
                                         constant, v1, v2, reinterpret_cast<double2*>(A));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(radius_bits, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    radius_kernel<<<static_cast<unsigned>(nb), 256, 0, s>>>(reinterpret_cast<const double2*>(A), nb, radius_bits);
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
