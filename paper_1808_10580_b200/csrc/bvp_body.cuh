// bvp_body.cuh — K2 exit-time walker kernel body (Algorithm 2).
//
// Per walker (forward_bvp.cpp:39-46 -> simulate_to_exit, sde.cpp:52-77):
//   loop step < max_steps:
//     next = x - v(x) dt + sigma sqrt(dt) xi            (em_step, sde.cpp:8-16)
//     if next leaves D: exit point by segment crossing (geometry.cpp:56-114),
//        f_int += f(x) frac dt, tau = step dt + frac dt, value = bc(exit) - f_int
//     else f_int += f(x) dt, x = next
//   failed (value 0, excluded) after max_steps.
//
// Exit times are heavy-tailed, so walkers are not pinned to threads: each warp
// is persistent and refills lanes whose walker finished from a global queue
// (ballot -> one atomicAdd per refill -> rank by popc), keeping all 32 lanes
// busy until the queue drains.  Every walker's randomness is addressed by
// (seed, obs, particle, step), so refill order never changes results.
//
// Included by bvp_kernels.cu (FMA contraction on; FP64 + FP32) and
// bvp_strict.cu (-fmad=false; the reference's operation order).
#pragma once

#include <type_traits>

#include "kernels.h"
#include "scalar_eval.cuh"
#include "smc_device.cuh"
#include "velocity.cuh"
#include "disk_velocity.cuh"

namespace smc {

constexpr int kBvpBlock = 128;
// Walker steps per run between queue refills (see the run loop below;
// C3: 4 -> 226.2, 8 -> 222.4, 16 -> 219.7, 32 -> 219.1 ms, same box).
#ifndef SMC_BVP_RUN
#define SMC_BVP_RUN 16
#endif
constexpr int kBvpRun = SMC_BVP_RUN;
// Minimum resident walker blocks per SM the register allocation must allow,
// for the constant-velocity walkers (the paper's Dirichlet problem, C3).
// Before the run loop and the table exponential, 7 (72 registers) was best
// (C3 263.9 -> 254.9 ms on one box; 8 blocks at 64 registers spilled in the
// step: 267.9 ms).  With the shorter step, 8 blocks at 64 registers (a few
// spill loads per step) beat 7 blocks at 72: 219.7 -> 218.0 ms
// (profiles/r02_ab_k2_expbump_runloop.log).  The Fourier-velocity walkers
// need their registers (they spill at 72) and stay unconstrained.
#ifndef SMC_BVP_MINB
#define SMC_BVP_MINB 8
#endif

// uniform in (0,1); FP64 from the log table staged in shared memory
__device__ __forceinline__ double log_u(double x, const double* tab) { return fm::log_tab(x, tab); }
__device__ __forceinline__ float log_u(float x, const double*) { return __logf(x); }
__device__ __forceinline__ double sqrt_u(double v) { return fm::sqrt_pos(v); }
__device__ __forceinline__ float sqrt_u(float v) { return sqrtf(v); }

// Forcing f(x) evaluated every step.  NB > 0: a Gaussian-bump sum of exactly
// NB terms held in registers for the whole walk (no per-step loads or
// dispatch); NB == 0: the generic ScalarField evaluator.  FAST (FP64 value
// walkers): the bump exponentials by fm::exp_bump from the 2 KB table `tab`
// staged in shared memory — valid only for arguments in [-708, 0], which
// launch_bvp_walkers proves for the domain before it selects NB > 0.
template <int NB, bool FAST = false>
struct Forcing {
    double c1[NB > 0 ? NB : 1], c2[NB > 0 ? NB : 1], amp[NB > 0 ? NB : 1];
    double neg_a = 0.0;
    const double* tab = nullptr;
    __device__ __forceinline__ explicit Forcing(const ScalarImg& f, const double* exp_tab = nullptr) : tab(exp_tab) {
        if constexpr (NB > 0) {
            neg_a = f.neg_sharpness;
#pragma unroll
            // volatile loads: ptxas may not re-issue them inside the walker
            // loop (it rematerialises plain read-only loads there instead of
            // keeping the values in registers: 11 loads per walker-step, C3
            // 296 -> 283 ms without them)
            const volatile double* center = f.center;
            const volatile double* amps = f.amp;
            for (int i = 0; i < NB; ++i) {
                c1[i] = center[2 * i];
                c2[i] = center[2 * i + 1];
                amp[i] = amps[i];
            }
        }
    }
    // the unit-amplitude bumps phi_j(x) = exp(-a |x - c_j|^2) (forcing basis)
    __device__ __forceinline__ void basis(double x1, double x2, double (&phi)[NB > 0 ? NB : 1]) const {
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const double d1 = x1 - c1[i], d2 = x2 - c2[i];
            phi[i] = SMC_SCALAR_EXP(neg_a * (d1 * d1 + d2 * d2));
        }
    }
    // FP32 variant (3-SE gate): the bump sum in float with the SFU exponential
    __device__ __forceinline__ float operator()(const ScalarImg& f, float x1, float x2) const {
        if constexpr (NB == 0) {
            return float(scalar_eval(f, double(x1), double(x2)));
        } else {
            float s = 0.0f;
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const float d1 = x1 - float(c1[i]), d2 = x2 - float(c2[i]);
                s = fmaf(float(amp[i]), __expf(float(neg_a) * fmaf(d1, d1, d2 * d2)), s);
            }
            return s;
        }
    }
    __device__ __forceinline__ double operator()(const ScalarImg& f, double x1, double x2) const {
        if constexpr (NB == 0) {
            return scalar_eval(f, x1, x2);
        } else {
            double s = 0.0;  // same order as ScalarField::operator() (fields.cpp:244-248)
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const double d1 = x1 - c1[i], d2 = x2 - c2[i];
                if constexpr (FAST) s += amp[i] * fm::exp_bump(neg_a * (d1 * d1 + d2 * d2), tab);
                else s += amp[i] * SMC_SCALAR_EXP(neg_a * (d1 * d1 + d2 * d2));
            }
            return s;
        }
    }
};

// VEL: 0 = runtime dispatch (constant or Fourier), 1 = constant velocity
// only (the lattice series is compiled out, which frees registers).
// BASIS (NB > 0, FP64): instead of one forcing integral, accumulate the NB
// unit-bump integrals I_j = int phi_j(X_t) dt and store value = bc(X_tau), so
// G(F) = E[bc] - sum_j F_j E[I_j] for every amplitude vector F from one pass
// (common random numbers: the paths do not depend on F).
// DISK_K > 0 (FP64, Fourier velocity filling the disk |k| <= DISK_K): the
// compile-time disk series of K1 (disk_velocity.cuh) from a coefficient block
// staged in shared memory, instead of the runtime-tiled lattice loop.
// DOM: 1 = box domain compiled in (domain_contains<T, 1>), 0 = any kind.
template <class T, bool STRICT, int KCAP, int NB = 0, int VEL = 0, bool BASIS = false, int DISK_K = 0, int DOM = 0>
__global__ void __launch_bounds__(kBvpBlock, (VEL == 1 && DISK_K == 0 && !STRICT) ? SMC_BVP_MINB : 1)
    bvp_walkers(const BvpLaunch L) {
    constexpr unsigned FULL = 0xffffffffu;
    __shared__ __align__(16) T disk_coef[DISK_K > 0 ? DiskShape<DISK_K>::n_coef : 2];
    if constexpr (DISK_K > 0) {
        for (int i = threadIdx.x; i < DiskShape<DISK_K>::n_coef; i += blockDim.x) disk_coef[i] = T(L.disk_coef[i]);
        __syncthreads();
    }
    // shared-memory copies of the log table (FP64 Box-Muller: 32-bit LDS
    // addressing instead of 64-bit global) and of exp_bump's table
    constexpr bool kLogTab = !STRICT && std::is_same<T, double>::value;
    __shared__ __align__(16) double log_tab[kLogTab ? 512 : 2];
    if constexpr (kLogTab) {
        for (int i = threadIdx.x; i < 512; i += blockDim.x) log_tab[i] = fm::g_logtab[i];
        __syncthreads();
    }
    constexpr bool kFastBump = NB > 0 && !STRICT && !BASIS && std::is_same<T, double>::value;
    __shared__ __align__(16) double exp_tab[kFastBump ? 256 : 1];
    if constexpr (kFastBump) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) exp_tab[i] = fm::g_exptab[i];
        __syncthreads();
    }
    const disk::SmemCoef<T> dc{static_cast<uint32_t>(__cvta_generic_to_shared(disk_coef))};
    const int lane = threadIdx.x & 31;
    const unsigned long long total = static_cast<unsigned long long>(L.n_obs) * L.n_particles;
    const LatticeImg& lat = L.vel.lat;
    const T dt = T(L.dt), sr = T(L.sr);

    bool active = false, exhausted = false;
    unsigned long long w = 0;
    uint32_t obs = 0, particle = 0;
    int64_t step = 0;
    T x1 = T(0), x2 = T(0), f_int = T(0);
    double I[NB > 0 ? NB : 1];
    unsigned long long my_steps = 0;
    cd p1[STRICT ? KCAP + 1 : 1], p2[STRICT ? KCAP + 1 : 1];
    const Forcing<NB, kFastBump> forcing(L.forcing, exp_tab);

    for (;;) {
        if (!exhausted) {
            const unsigned need = __ballot_sync(FULL, !active);
            if (need) {
                const int leader = __ffs(need) - 1;
                unsigned long long base = 0;
                if (lane == leader) base = atomicAdd(L.counter, static_cast<unsigned long long>(__popc(need)));
                base = __shfl_sync(FULL, base, leader);
                if (base + __popc(need) >= total) exhausted = true;
                if (!active) {
                    const unsigned long long idx = base + __popc(need & ((1u << lane) - 1u));
                    if (idx < total) {
                        w = idx;
                        obs = static_cast<uint32_t>(idx / static_cast<unsigned long long>(L.n_particles));
                        particle = static_cast<uint32_t>(L.p_begin + static_cast<int64_t>(
                                       idx - static_cast<unsigned long long>(obs) * L.n_particles));
                        x1 = T(__ldg(L.obs_x + 2 * obs));
                        x2 = T(__ldg(L.obs_x + 2 * obs + 1));
                        f_int = T(0);
                        if constexpr (BASIS) {
#pragma unroll
                            for (int q = 0; q < NB; ++q) I[q] = 0.0;
                        }
                        step = 0;
                        active = true;
                    }
                }
            }
        }
        if (!__any_sync(FULL, active)) break;
        if (!active) continue;
        // up to kBvpRun steps between refills: the refill vote, the loop-carried
        // moves and the max_steps test are paid once per run, not per step (a
        // lane whose walker exits idles for the rest of the run: (kBvpRun - 1)/2
        // steps per walker against ~800 on C3).  max_steps is hit exactly.
        {
            const int64_t left = L.max_steps - step;
            const int n_run = left < kBvpRun ? static_cast<int>(left) : kBvpRun;
            int run = 0;
            // (not unrolled: two steps per iteration lose the uniform-register
            // constants to per-thread LDC and spill)
#pragma unroll 1
            for (; run < n_run; ++run) {
                const Uniform2 u = uniform_block(L.rk, L.obs_slot0 + obs, particle, static_cast<uint64_t>(step));
                T xi1, xi2, v1, v2;
                if constexpr (STRICT) {
                    const double r = sqrt(-2.0 * log(u.u0));
                    const double a = 2.0 * kPi * u.u1;
                    xi1 = r * cos(a);
                    xi2 = r * sin(a);
                    velocity_strict<KCAP>(L.vel, p1, p2, x1, x2, v1, v2);
                } else {
                    const T rad = sqrt_u(T(-2) * log_u(T(u.u0), log_tab));
                    T sn, cs;
                    sincospi_shift(T(2) * T(u.u1), &sn, &cs);
                    xi1 = rad * cs;
                    xi2 = rad * sn;
                    if (VEL == 1 || L.vel.is_constant) {
                        v1 = T(L.vel.c1);
                        v2 = T(L.vel.c2);
                    } else if constexpr (VEL == 0 && DISK_K > 0) {
                        const T xa[1] = {x1}, xb[1] = {x2};
                        T va[1], vb[1];
                        disk::velocity_disk<DISK_K, T, 1>(dc, xa, xb, va, vb);
                        v1 = va[0];
                        v2 = vb[0];
                    } else if constexpr (VEL == 0) {
                        velocity_lattice<T, double>(lat, lat.coef, x1, x2, v1, v2);
                    }
                }
                T n1, n2;
                if constexpr (STRICT) {
                    n1 = x1 - v1 * L.dt + L.sigma * L.root_dt * xi1;
                    n2 = x2 - v2 * L.dt + L.sigma * L.root_dt * xi2;
                } else {
                    n1 = fma(sr, xi1, fma(-v1, dt, x1));
                    n2 = fma(sr, xi2, fma(-v2, dt, x2));
                }
                T f = T(0);
                double phi[NB > 0 ? NB : 1];
                if constexpr (BASIS) forcing.basis(double(x1), double(x2), phi);
                else f = forcing(L.forcing, x1, x2);  // FP64, or the float variant for T = float
                if (!domain_contains<T, DOM>(L.domain, n1, n2)) {
                    T h1, h2;
                    const T frac = boundary_exit<T>(L.domain, x1, x2, n1, n2, h1, h2);
                    const T tau = T(double(step)) * dt + frac * dt;
                    if constexpr (BASIS) {
                        const unsigned long long nw = total;
#pragma unroll
                        for (int q = 0; q < NB; ++q) L.basis[q * nw + w] = I[q] + phi[q] * double(frac) * double(dt);
                        L.values[w] = scalar_eval(L.boundary, double(h1), double(h2));
                    } else {
                        f_int += f * frac * dt;
                        L.values[w] = scalar_eval(L.boundary, double(h1), double(h2)) - double(f_int);
                    }
                    L.aux[w] = double(tau);
                    L.failed[w] = 0;
                    active = false;
                    ++run;
                    break;
                }
                if constexpr (BASIS) {
#pragma unroll
                    for (int q = 0; q < NB; ++q) I[q] += phi[q] * double(dt);
                } else {
                    f_int += f * dt;
                }
                x1 = n1;
                x2 = n2;
                ++step;
            }
            my_steps += static_cast<unsigned>(run);
        }
        if (active && step >= L.max_steps) {
            L.values[w] = 0.0;
            L.aux[w] = 0.0;
            L.failed[w] = 1;
            if constexpr (BASIS) {
#pragma unroll
                for (int q = 0; q < NB; ++q) L.basis[q * total + w] = 0.0;
            }
            active = false;
        }
    }
    // one atomic per warp for the walker-step count
    unsigned long long s = my_steps;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(FULL, s, off);
    if (lane == 0 && s) atomicAdd(L.step_total, s);
}

}  // namespace smc
