// ad_strict.cu — K1 "strict" FP64 diagnostic build (compiled with
// -fmad=false).
//
// Same particle loop as ad_kernels.cu, but every floating-point operation is
// the reference's, in the reference's order and association, with no FMA
// contraction: fill_powers' complex recurrence (src/fields.cpp:23-31), the
// (k1,k2)-sorted mode loop with w = 2(re e.re - im e.im) (fields.cpp:78-87),
// em_step's (x - v dt) + (sigma sqrt(dt)) xi (src/sde.cpp:13-15), Box-Muller
// with a = (2 pi) u1 (src/rng.cpp:67-72).  The only remaining source of
// difference from the reference is libm: CUDA's log/sin/cos vs glibc's.  The
// parity tests use this kernel to show the per-particle values are bitwise
// equal to the reference except where libm rounds differently.
#define SMC_STRICT_TU 1
#include <cuda_runtime.h>

#include "ad_unit.cuh"
#include "kernels.h"
#include "scalar_eval.cuh"
#include "smc_device.cuh"
#include "velocity.cuh"

namespace smc {
namespace {

constexpr int kBlock = 128;

template <int KCAP>
__global__ void __launch_bounds__(kBlock) ad_particles_strict(const AdLaunch L) {
    int obs = blockIdx.y;
    int64_t local = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
    int64_t span = L.p_end - L.p_begin;
    if (local >= span) return;
    if (L.unit_cpo > 0) {  // sharded launch (kernels.h unit mode)
        if (!unit_coords(L, local, obs, local)) return;
        span = L.n_particles;
    }
    const int64_t particle = L.p_begin + local;
    const AdObsImg o = L.obs[obs];
    const uint64_t seed = L.seed;
    const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
    const uint32_t slot = L.obs_slot0 + obs;
    cd p1[KCAP + 1], p2[KCAP + 1];

    double x1 = o.x1 - floor(o.x1), x2 = o.x2 - floor(o.x2);
    const int64_t n = o.n_steps;
    for (int64_t step = 0; step < n; ++step) {
        const Uniform2 u = uniform_block(k0, k1, slot, static_cast<uint32_t>(particle), static_cast<uint64_t>(step));
        const double r = sqrt(-2.0 * log(u.u0));
        const double a = 2.0 * kPi * u.u1;
        const double xi1 = r * cos(a), xi2 = r * sin(a);
        double v1, v2;
        velocity_strict<KCAP>(L.vel, p1, p2, x1, x2, v1, v2);
        const bool last = step + 1 == n;
        const double h = last ? o.dt_last : o.dt;
        const double root_dt = last ? o.rdt_last : o.rdt;
        x1 = x1 - v1 * h + L.sigma * root_dt * xi1;
        x2 = x2 - v2 * h + L.sigma * root_dt * xi2;
        x1 = x1 - floor(x1);
        x2 = x2 - floor(x2);
    }
    ad_out_row(L, 0, obs, span)[local] = scalar_eval(L.theta0, x1, x2);
}

}  // namespace

cudaError_t launch_ad_particles_strict(const AdLaunch& L, cudaStream_t s) {
    const int64_t span = L.p_end - L.p_begin;
    if (span <= 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>((span + kBlock - 1) / kBlock),
                    static_cast<unsigned>(L.unit_cpo > 0 ? 1 : L.n_obs), 1);
    const int K = L.vel.is_constant ? 0 : L.vel.K;
    if (K <= 8) ad_particles_strict<8><<<grid, kBlock, 0, s>>>(L);
    else if (K <= 32) ad_particles_strict<32><<<grid, kBlock, 0, s>>>(L);
    else if (K <= 128) ad_particles_strict<128><<<grid, kBlock, 0, s>>>(L);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace smc
