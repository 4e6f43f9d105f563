// kernels.h — launch interface between the host runtime (capi.cu) and the
// sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "geometry.cuh"
#include "images.h"
#include "smc_device.cuh"

namespace smc {

constexpr int kChunk = 1024;  // == SMC_CHUNK: reduction tree leaf block

// K1: advection-diffusion particles to a fixed time (Algorithm 1;
// sde.cpp:37-50 + fields.cpp:71-89 + forward_ad.cpp:41-47), one particle per
// thread.  Grid: x over particle blocks of this shard, y over observations,
// z over parameter samples.
struct AdLaunch {
    VelImg vel;
    ScalarImg theta0;
    const AdObsImg* obs;       // [n_obs]
    int32_t n_obs;
    uint32_t obs_slot0;        // stream-key obs slot of obs[0] (spec slot, forward_ad.cpp:43)
    uint64_t seed;             // CRN seed
    const uint64_t* seeds;     // [n_samples] per-sample seeds, or nullptr (CRN)
    int64_t n_particles;       // particles per observation
    int64_t p_begin, p_end;    // this launch's particle range [p_begin, p_end)
    int32_t n_samples;
    int32_t precision;         // smc_precision
    double sigma;              // sqrt(2 kappa)
    double* values;            // [n_samples][n_obs][p_end - p_begin]
    const double* host_disk;   // host copy of the single-sample disk coefficient block (or null)
    const int32_t* obs_order;  // [n_obs] observations by decreasing step count
    int32_t obs_major;         // batched grid order: 1 = (blocks, samples, obs longest first), 0 = (blocks, obs, samples)
    int32_t unit_cpo;          // > 0: unit mode (sharded single-sample launch), = chunks per observation
    int64_t unit0;             // unit mode: first (observation, chunk) unit, unit = obs * unit_cpo + chunk
    RoundKeys rk;              // Philox round keys of `seed` (filled by the launcher that uses them)
};

// Unit mode (multi-GPU sharding of one evaluation): a launch
// covers the (observation, chunk) units [unit0, unit0 + n_units) of the
// image's observations, with p_begin = 0 and p_end = n_units * kChunk.  The
// flat thread index f maps to unit unit0 + f / kChunk and particle
// (unit % unit_cpo) * kChunk + f % kChunk of observation unit / unit_cpo, and
// its terminal value lands at values[f] (chunk-contiguous), so a chunk tree
// over values[u * kChunk ...] is that unit's exact aligned partial.  Threads
// past their observation's last particle do nothing (the partial kernel masks
// them).  Grid y = 1.

cudaError_t launch_ad_particles(const AdLaunch& L, cudaStream_t s);
// Batched grid order (AdLaunch::obs_major) for a launch of this shape.
int batched_obs_major(const AdLaunch& L, int64_t blocks_per_obs);
cudaError_t launch_ad_particles_fp32(const AdLaunch& L, cudaStream_t s);
cudaError_t launch_ad_particles_strict(const AdLaunch& L, cudaStream_t s);

// K1 specialised for the full disk |k| <= K (K <= kDiskMaxK, disk_shape.h):
// coef = device blocks of disk_n_coef(K) doubles, one per sample.  Returns
// cudaErrorNotSupported when K has no specialisation.
cudaError_t launch_ad_disk(const AdLaunch& L, int K, const double* coef, cudaStream_t s);

// K2: Dirichlet exit-time walkers (Algorithm 2, PAPER.md:162-178;
// sde.cpp:52-77 + forward_bvp.cpp:39-46).  Persistent warps: a lane whose
// walker exits (or fails at max_steps) writes its result and is refilled with
// the next walker index from a global counter (one atomic per warp refill).
struct BvpLaunch {
    VelImg vel;
    ScalarImg forcing, boundary;
    DomainImg domain;
    const double* obs_x;       // [n_obs][2]
    int32_t n_obs;
    uint32_t obs_slot0;
    uint64_t seed;
    int64_t n_particles;       // walkers per observation launched: particles [p_begin, p_begin + n)
    int64_t max_steps;
    double dt, root_dt, sigma, sr;  // sr = sigma * sqrt(dt)
    int32_t precision;
    int32_t bump_exp_ok;       // every bump exponent provably in [-708, 0] (fm::exp_bump valid; prepare_bvp)
    unsigned long long* counter;     // walker queue head (zeroed before launch)
    unsigned long long* step_total;  // total walker-steps executed (atomicAdd)
    double* values;            // [n_obs][n_particles]
    double* aux;               // exit time
    uint8_t* failed;
    double* basis;             // forcing-basis mode: [n_bumps][n_obs][n_particles] unit-bump integrals
    const double* disk_coef;   // disk_shape.h coefficient block when disk_K > 0
    int32_t disk_K;            // > 0: dense Fourier velocity on |k| <= disk_K (FP64 walkers use bvp_disk.cu)
    int32_t pad2_;
    int64_t p_begin;           // first walker index of this launch (walker sharding; 0 otherwise)
    RoundKeys rk;              // Philox round keys of `seed` (with_round_keys, set by every K2 launcher)
};

inline BvpLaunch with_round_keys(const BvpLaunch& L) {
    BvpLaunch K = L;
    K.rk = make_round_keys(L.seed);
    return K;
}

cudaError_t launch_bvp_walkers(const BvpLaunch& L, int n_sms, cudaStream_t s);
cudaError_t launch_bvp_walkers_strict(const BvpLaunch& L, int n_sms, cudaStream_t s);
// FP64 walkers with the compile-time disk velocity (L.disk_K in 1..kDiskMaxK).
cudaError_t launch_bvp_disk(const BvpLaunch& L, unsigned blocks, cudaStream_t s);
// Forcing-basis mode (Gaussian-bump forcing with 1..4 terms, FP64).
cudaError_t launch_bvp_basis(const BvpLaunch& L, int n_sms, cudaStream_t s);

// Stable compaction of valid walkers per segment (reduce_observation's
// valid/valid_aux vectors, executor.cpp:93-101).  chunk_tmp: 2 * n_seg *
// ceil(n/1024) int64.  Writes counts[seg] (valid walkers).
cudaError_t compact_valid(const double* values, const double* aux, const uint8_t* failed, int64_t n,
                          int64_t n_seg, double* cvalues, double* caux, int64_t* counts, int64_t* chunk_tmp,
                          cudaStream_t s);

// K3: deterministic pairwise tree (executor.cpp:11-26) over aligned chunks.
// One pass turns each segment's n values into ceil(n / 1024) chunk partials.
//   mode 0: x_i;  mode 1: (x_i - center[seg])^2
// Out-of-range leaves are -0.0, the exact additive identity.
cudaError_t launch_tree_pass(const double* in, int64_t in_stride, const int64_t* counts,
                             int64_t n_uniform, int64_t n_seg, double* out, int64_t out_stride,
                             const double* center, int mode, cudaStream_t s);

// Sharded AD: the chunk partial of each unit [unit0, unit0 + n_units) from the
// unit-mode K1 values (chunk-contiguous); out[u - unit0].  mode 0: x_i;
// mode 1: (x_i - center[obs])^2.
cudaError_t launch_unit_partials(const double* values, int64_t n_units, int64_t unit0, int64_t cpo,
                                 int64_t n_particles, const double* center, int mode, double* out, cudaStream_t s);

// Sharded Dirichlet reduction (reduce_kernels.cu): this rank's compacted valid
// walkers of every observation -> the tree sums of the aligned dyadic blocks of
// its interval in the global compacted order, kDyadicSlots per (obs, quantity);
// and the receiver's merge of all ranks' blocks into the per-observation sums.
constexpr int kDyadicSlots = 64;
cudaError_t launch_dyadic_blocks(const double* vals, int64_t qstride, int nq, int64_t vstride, const int64_t* gcounts,
                                 int world, int rank, int64_t n_obs, const double* center, int mode, double* rec,
                                 double* scratch, int64_t sstride, cudaStream_t s);
cudaError_t launch_dyadic_finish(const double* rec, const int64_t* gcounts, int world, int64_t n_obs, int nq,
                                 double* sums, int64_t* counts_total, double* means, cudaStream_t s);

// Runs tree passes until one value per segment remains.  scratch must hold
// 2 * n_seg * ceil(n/1024) doubles.  counts may be null (all segments n).
cudaError_t tree_reduce(const double* in, int64_t in_stride, const int64_t* counts, int64_t n,
                        int64_t n_seg, double* sums, const double* center, int mode,
                        double* scratch, cudaStream_t s, int* launches);

// means[seg] = sums[seg] / counts[seg]
cudaError_t launch_divide(const double* sums, const int64_t* counts, int64_t n_uniform, int64_t n_seg,
                          double* means, cudaStream_t s);

// Finish reduce_observation (executor.cpp:104-116) on device.
cudaError_t launch_estimates(const double* means, const double* sumsq, const double* sumaux,
                             const int64_t* counts, int64_t n_uniform, int64_t n_particles,
                             int64_t n_seg, void* out_estimates, cudaStream_t s);

// Device-resident multi-chain pCN (pcn_kernels.cu).
struct PcnStep {
    int64_t n_chains, dim, M, n_obs, n_steps, n_samples;
    const double* stds;      // [M] per-mode prior std (PriorSpec::component_stds, pairwise)
    double contraction, beta;
    const uint64_t* seeds;   // [n_chains] chain seeds
    uint64_t blk0;           // first stream block of this step's prior draw
    uint64_t ublk;           // block of this step's uniform
    int32_t uhalf;           // which of its two uniforms
    int32_t init;            // 1: chain_init (accept the proposal unconditionally)
    int32_t noise_inf;       // noise_std infinite: Phi == 0
    int32_t pad_;
    double noise_std;
    const double* data;      // [n_obs]
    double* U;               // [n_chains][dim] state
    double* Up;              // [n_chains][dim] proposal
    double* norm_prop;       // [n_chains]
    double* norm_cur;
    double* phi;
    double* map_obj;
    int64_t* accepted;
    uint8_t* acc_flag;
    uint8_t* map_flag;
    double* map_u;           // [n_chains][dim]
    double* phi_trace;       // [n_chains][n_steps] or null
    double* samples;         // [n_chains][n_samples][dim] or null
    int64_t step;            // 0-based step index
    int64_t sample_slot;     // >= 0: store the state as sample #slot
    // Graph mode (it_dev != null): the step index lives on the device and the
    // kernels derive blk0 / ublk / uhalf / step / sample_slot from it, so one
    // captured step replays unchanged; pcn_advance bumps it.
    const int64_t* it_dev;
    uint64_t blk_base;       // stream block counter after chain_init
    int64_t burn_in, thin;
};
cudaError_t launch_pcn_advance(int64_t* it_dev, cudaStream_t s);
cudaError_t launch_pcn_propose(const PcnStep& S, cudaStream_t s);
// u -> coefficient blocks on the device (host_problem.h PackMap, uploaded).
// grid.y = n_samples <= 65535 per launch.
struct PackDev {
    int64_t stride;
    const int32_t* ip;
    const int32_t* im;
    const double* kp;
    const double* km;
    const int8_t* ms;
};
cudaError_t launch_pack(const PackDev& M, const double* Up, int64_t dim, int64_t n_samples, double* blocks, int* bad,
                        cudaStream_t s);
cudaError_t launch_pcn_accept(const PcnStep& S, const void* est, cudaStream_t s);
cudaError_t launch_pcn_commit(const PcnStep& S, cudaStream_t s);

// Spectral Galerkin reference solver (galerkin_kernels.cu).
cudaError_t launch_galerkin_step(const double* A, const double* th, double* out, int64_t nb, double dt,
                                 cudaStream_t s);
cudaError_t launch_galerkin_assemble(const double* vhat, const unsigned char* present, int K, const int* k1,
                                     const int* k2, int64_t nb, double kappa, int constant, double v1, double v2,
                                     double* A, unsigned long long* radius_bits, cudaStream_t s);
cudaError_t launch_galerkin_quadrature(const ScalarImg& f, const int* k1, const int* k2, int64_t nb, int n,
                                       double* theta, cudaStream_t s);
cudaError_t launch_galerkin_observe(const double* th, const int* k1, const int* k2, int64_t nb, double x1, double x2,
                                    double* out, cudaStream_t s);
cudaError_t launch_galerkin_field_grid(const double* c, const int* k1, const int* k2, int64_t nb, int n, double* grid,
                                       cudaStream_t s);

// Diagnostics / microbenchmarks.
cudaError_t launch_philox(int64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out,
                          cudaStream_t s);
cudaError_t launch_normal_pairs(uint64_t seed, uint32_t obs, uint32_t particle, int64_t n,
                                double* out, cudaStream_t s);
cudaError_t launch_dfma_peak(int n_blocks, int iters, double* sink, cudaStream_t s);
cudaError_t launch_ffma_peak(int n_blocks, int iters, double* sink, cudaStream_t s);

}  // namespace smc
