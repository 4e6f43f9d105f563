// ad_kernels.cu — K1 with the generic lattice velocity (any K, any mode set,
// per-sample coefficients for batched evaluation).  See ad_body.cuh for the
// particle loop and velocity.cuh for the lattice series.  FP64 is the parity
// path; FP32 is the optional fast mode (3-SE gate).
#include <cuda_runtime.h>

#include "ad_body.cuh"

namespace smc {

namespace {

constexpr int kBlock = 256;

template <class T>
__global__ void __launch_bounds__(kBlock) ad_particles(const AdLaunch L) {
    const int obs = blockIdx.y;
    const int sample = blockIdx.z;
    const int64_t local = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const int64_t span = L.p_end - L.p_begin;
    if (local >= span) return;
    const LatticeImg& lat = L.vel.lat;
    const int64_t soff = static_cast<int64_t>(sample) * lat.sample_stride;
    const double* coef = lat.coef + soff;
    const double* row0 = lat.row0 + soff;
    const double* g0 = lat.g0 + soff;
    const bool is_const = L.vel.is_constant;
    const T c1 = T(L.vel.c1), c2 = T(L.vel.c2);
    ad_particle<T>(L, obs, sample, local, span, [&](T x1, T x2, T& v1, T& v2) {
        if (is_const) {
            v1 = c1;
            v2 = c2;
        } else {
            velocity_lattice<T>(lat, coef, row0, g0, x1, x2, v1, v2);
        }
    });
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
