// ad_body.cuh — the per-particle loop of K1, shared by the generic-lattice
// kernel (ad_kernels.cu) and the compile-time disk kernels (ad_disk.cu).
//
// Each thread owns P particles of one observation for their whole paths
// (Algorithm 1): Philox block -> Box-Muller -> velocity ->
// Euler-Maruyama step -> torus wrap, n_j times in registers, then theta_0 at
// the terminal point (simulate_to_time, src/sde.cpp:37-50; work lambda,
// src/forward_ad.cpp:41-47).  Only the terminal values touch HBM.  With P > 1
// the velocity evaluator loads each coefficient once for all P particles.
#pragma once

#include "ad_unit.cuh"
#include "kernels.h"
#include "scalar_eval.cuh"
#include "smc_device.cuh"
#include "velocity.cuh"

namespace smc {

__device__ __forceinline__ double log_t(double x) { return fm::log_tab(x); }  // x = uniform in (0,1)
__device__ __forceinline__ float log_t(float x) { return __logf(x); }

// Particles local[p] (p < P) of observation `obs`; entries >= span are
// computed on a clamped index and not stored.  RK: the launch carries the
// Philox round keys of L.seed (L.rk; single-sample launches without per-sample
// seeds).
template <class T, int P, class Vel, bool RK = false, bool UNIT = true>
__device__ __forceinline__ void ad_particles_p(const AdLaunch& L, int obs, int sample, const int64_t (&local)[P],
                                               int64_t span, Vel&& velocity) {
    const AdObsImg o = L.obs[obs];
    const uint64_t seed = L.seeds ? __ldg(L.seeds + sample) : L.seed;
    const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
    const uint32_t slot = L.obs_slot0 + obs;
    uint32_t particle[P];
    T x1[P], x2[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        particle[p] = static_cast<uint32_t>(L.p_begin + (local[p] < span ? local[p] : span - 1));
        x1[p] = T(o.x1 - floor(o.x1));
        x2[p] = T(o.x2 - floor(o.x2));
    }
    const T dt = T(o.dt), dt_last = T(o.dt_last), sr = T(o.sr), sr_last = T(o.sr_last);
    const int64_t n = o.n_steps;
    // The noise of step s+1 does not depend on the path, so it is drawn one
    // step ahead: its Philox/Box-Muller chain and step s's velocity series are
    // independent instruction streams the scheduler interleaves (ILP that
    // hides DFMA latency at modest occupancy).
    T nx1[P], nx2[P];
    auto draw = [&](int64_t step, T (&z1)[P], T (&z2)[P]) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const Uniform2 u = RK ? uniform_block(L.rk, slot, particle[p], static_cast<uint64_t>(step))
                                  : uniform_block(k0, k1, slot, particle[p], static_cast<uint64_t>(step));
            const T rad = sqrt(T(-2) * log_t(T(u.u0)));
            T sn, cs;
            sincospi_t(T(2) * T(u.u1), &sn, &cs);
            z1[p] = rad * cs;
            z2[p] = rad * sn;
        }
    };
    draw(0, nx1, nx2);
    for (int64_t step = 0; step < n; ++step) {
        T xi1[P], xi2[P], v1[P], v2[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            xi1[p] = nx1[p];
            xi2[p] = nx2[p];
        }
        draw(step + 1, nx1, nx2);  // one block past the last step is drawn and discarded
        // `zero` is 0 for every reachable step but depends on the (uniform)
        // step counter, so constant-bank coefficient reads indexed by it
        // cannot be hoisted out of the loop (see ad_disk.cu ConstCoef)
        const int zero = static_cast<int>(static_cast<uint64_t>(step) >> 62);
        velocity(x1, x2, v1, v2, zero);
        const bool last = step + 1 == n;
        const T h = last ? dt_last : dt;
        const T s = last ? sr_last : sr;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            x1[p] = fma(s, xi1[p], fma(-v1[p], h, x1[p]));
            x2[p] = fma(s, xi2[p], fma(-v2[p], h, x2[p]));
            x1[p] -= floor(x1[p]);
            x2[p] -= floor(x2[p]);
        }
    }
    // UNIT = false: a launch that is never in unit mode (its output row
    // needs no runtime mode check)
    double* out = UNIT ? ad_out_row(L, sample, obs, span)
                       : L.values + (static_cast<int64_t>(sample) * L.n_obs + obs) * span;
#pragma unroll
    for (int p = 0; p < P; ++p)
        if (local[p] < span) out[local[p]] = scalar_eval(L.theta0, double(x1[p]), double(x2[p]));
}

// Single-particle convenience wrapper.
template <class T, bool UNIT = true, class Vel>
__device__ __forceinline__ void ad_particle(const AdLaunch& L, int obs, int sample, int64_t local, int64_t span,
                                            Vel&& velocity) {
    const int64_t loc[1] = {local};
    auto vel = [&](const T (&x1)[1], const T (&x2)[1], T (&v1)[1], T (&v2)[1], int) {
        velocity(x1[0], x2[0], v1[0], v2[0]);
    };
    ad_particles_p<T, 1, decltype(vel)&, false, UNIT>(L, obs, sample, loc, span, vel);
}

}  // namespace smc
