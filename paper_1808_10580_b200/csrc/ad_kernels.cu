// ad_kernels.cu — K1: fused advection-diffusion particle kernel (sm_100a).
//
// One thread owns one particle for its whole path (Algorithm 1,
// PAPER.md:130-143): Philox block -> Box-Muller -> Fourier velocity ->
// Euler-Maruyama step -> torus wrap, repeated n_j times in registers, then
// theta_0 at the terminal point.  Replaces simulate_to_time
// (src/sde.cpp:37-50), FourierVelocityField::operator() (src/fields.cpp:71-89)
// and the per-particle work lambda of estimate_observation
// (src/forward_ad.cpp:41-47).  Only the terminal value touches HBM.
//
// FP64 is the parity path; FP32 is the optional fast mode (3-SE gate): same
// streams, single-precision state and series, theta_0 in FP64.
#include <cuda_runtime.h>

#include "kernels.h"
#include "scalar_eval.cuh"
#include "smc_device.cuh"
#include "velocity.cuh"

namespace smc {
namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ double log_t(double x) { return log(x); }
__device__ __forceinline__ float log_t(float x) { return __logf(x); }

template <class T>
__global__ void __launch_bounds__(kBlock) ad_particles(const AdLaunch L) {
    const int obs = blockIdx.y;
    const int sample = blockIdx.z;
    const int64_t local = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const int64_t span = L.p_end - L.p_begin;
    if (local >= span) return;
    const int64_t particle = L.p_begin + local;

    const AdObsImg o = L.obs[obs];
    const uint64_t seed = L.seeds ? __ldg(L.seeds + sample) : L.seed;
    const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
    const uint32_t slot = L.obs_slot0 + obs;

    const LatticeImg& lat = L.vel.lat;
    const int64_t soff = static_cast<int64_t>(sample) * lat.sample_stride;
    const double* coef = lat.coef + soff;
    const double* row0 = lat.row0 + soff;
    const double* g0 = lat.g0 + soff;

    T x1 = T(o.x1 - floor(o.x1)), x2 = T(o.x2 - floor(o.x2));
    const T dt = T(o.dt), dt_last = T(o.dt_last), sr = T(o.sr), sr_last = T(o.sr_last);
    const int64_t n = o.n_steps;
    for (int64_t step = 0; step < n; ++step) {
        const Uniform2 u = uniform_block(k0, k1, slot, static_cast<uint32_t>(particle), static_cast<uint64_t>(step));
        const T rad = sqrt(T(-2) * log_t(T(u.u0)));
        T sn, cs;
        sincospi_t(T(2) * T(u.u1), &sn, &cs);
        const T xi1 = rad * cs, xi2 = rad * sn;
        T v1, v2;
        if (L.vel.is_constant) {
            v1 = T(L.vel.c1);
            v2 = T(L.vel.c2);
        } else {
            velocity_lattice<T>(lat, coef, row0, g0, x1, x2, v1, v2);
        }
        const bool last = step + 1 == n;
        const T h = last ? dt_last : dt;
        const T s = last ? sr_last : sr;
        x1 = fma(s, xi1, fma(-v1, h, x1));
        x2 = fma(s, xi2, fma(-v2, h, x2));
        x1 -= floor(x1);
        x2 -= floor(x2);
    }
    const double val = scalar_eval(L.theta0, double(x1), double(x2));
    L.values[(static_cast<int64_t>(sample) * L.n_obs + obs) * span + local] = val;
}

template <class T>
cudaError_t launch(const AdLaunch& L, cudaStream_t s) {
    const int64_t span = L.p_end - L.p_begin;
    if (span <= 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>((span + kBlock - 1) / kBlock), static_cast<unsigned>(L.n_obs),
                    static_cast<unsigned>(L.n_samples));
    ad_particles<T><<<grid, kBlock, 0, s>>>(L);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_ad_particles(const AdLaunch& L, cudaStream_t s) { return launch<double>(L, s); }
cudaError_t launch_ad_particles_fp32(const AdLaunch& L, cudaStream_t s) { return launch<float>(L, s); }

}  // namespace smc
