/*
 * scalarmc_b200.h — C ABI of the B200-native particle forward map G(u).
 *
 * This is the drop-in boundary for the reference library `scalarmc`
 * (/root/reference/proj, arXiv 1808.10580).  Every entry point below replaces
 * one reference C++ function on the hot path; the reference symbol it stands
 * in for is cited next to it (paths relative to /root/reference/proj).  The C++
 * shim in paper_1808_10580_b200/host/scalarmc_forward_gpu.cpp re-implements the
 * unchanged C++ signatures (`observe_ad`, `observe_ad_single`, `observe_bvp`)
 * on top of these calls, and the Python mirror (paper_1808_10580_b200/api.py)
 * binds them with ctypes.
 *
 * Conventions
 *   - Plain C types only: caller-owned POD inputs, caller-owned output arrays.
 *   - Every function returns an smc_status; on failure smc_last_error() returns
 *     a thread-local message.  The status maps 1:1 onto the exception type the
 *     reference throws for the same condition (invalid_argument, out_of_range,
 *     runtime_error), and the message text matches the reference's.
 *   - Calls are synchronous: they return once host outputs are written.
 *   - There is no CPU fallback: without a CUDA device smc_create fails.
 */
#ifndef SCALARMC_B200_H
#define SCALARMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Every declaration below is exported even when the library is built with
 * -fvisibility=hidden. */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define SMC_ABI_VERSION 1

/* Status codes; the comment names the reference exception type. */
typedef enum smc_status {
    SMC_OK = 0,
    SMC_EINVAL = 1,   /* std::invalid_argument */
    SMC_ERANGE = 2,   /* std::out_of_range */
    SMC_ERUNTIME = 3, /* std::runtime_error (all particles failed, ...) */
    SMC_ECUDA = 4     /* CUDA / device failure (no reference analogue) */
} smc_status;

/* ParticleEstimate (include/scalarmc/executor.hpp:13-19), same field order. */
typedef struct smc_estimate {
    double mean;
    double std_error;
    int64_t n_particles;
    int64_t n_failed;
    double aux_mean;
} smc_estimate;

/* ScalarField (include/scalarmc/fields.hpp:121-164; eval src/fields.cpp:235-253).
 * kind: 0 constant, 1 cosine series, 2 Gaussian bumps, 3 linear (affine).
 * Arrays are SoA with n_terms entries; unused pointers may be NULL. */
typedef enum smc_scalar_kind {
    SMC_SCALAR_CONSTANT = 0,
    SMC_SCALAR_COSINE = 1,
    SMC_SCALAR_BUMPS = 2,
    SMC_SCALAR_LINEAR = 3
} smc_scalar_kind;

typedef struct smc_scalar_field {
    int32_t kind;
    int32_t n_terms;
    double constant;        /* constant value, or affine offset */
    double gradient[2];     /* linear: gradient */
    double sharpness;       /* bumps: a in exp(-a |x-c|^2) */
    const double* amplitude;/* cosine/bumps: [n_terms] */
    const double* freq;     /* cosine: [n_terms][2] angular frequency (2 pi k for torus modes) */
    const double* phase;    /* cosine: [n_terms] */
    const double* center;   /* bumps: [n_terms][2] */
} smc_scalar_field;

/* VelocityField (include/scalarmc/fields.hpp:67-86): constant vector or a
 * FourierVelocityField (fields.hpp:24-64).  Modes are given as the caller holds
 * them (any sign convention); the library canonicalises and sorts exactly like
 * the reference constructor (src/fields.cpp:35-69). */
typedef struct smc_velocity {
    int32_t is_constant;
    int32_t max_wavenumber; /* K, > 0 for Fourier fields */
    double constant[2];
    int64_t n_modes;
    const int32_t* k;       /* [n_modes][2] (k1, k2) */
    const double* coeff;    /* [n_modes][2] (re, im) */
} smc_velocity;

typedef enum smc_scheme { SMC_EULER_MARUYAMA = 0, SMC_MILSTEIN = 1 } smc_scheme;

/* Precision of the particle kernels.  FP64 is the parity path (1e-10 relative
 * gate); FP32 is the optional fast mode (3 Monte Carlo SE gate). STRICT is the
 * FP64 diagnostic build that keeps the reference's operation order and does no
 * FMA contraction. */
typedef enum smc_precision { SMC_FP64 = 0, SMC_FP32 = 1, SMC_FP64_STRICT = 2 } smc_precision;

/* AdProblemSpec (include/scalarmc/forward_ad.hpp:23-34).  The diffusion is the
 * isotropic model sigma = sqrt(2 kappa) (fields.cpp:158-165); diagonal
 * std::function models have no device representation and are rejected by the
 * C++ shim with std::invalid_argument. */
typedef struct smc_ad_problem {
    smc_velocity velocity;
    double kappa;
    smc_scalar_field initial_condition;
    int64_t n_obs;
    const double* obs_t;    /* [n_obs] */
    const double* obs_x;    /* [n_obs][2] */
    double dt;              /* <= 0: min_j t_j / 200 (forward_ad.cpp:10-15) */
    int64_t n_particles;
    int32_t scheme;         /* smc_scheme; Milstein == EM for isotropic sigma (sde.cpp:21) */
    int32_t precision;      /* smc_precision */
} smc_ad_problem;

/* Domain (include/scalarmc/geometry.hpp:36-74). */
typedef enum smc_domain_kind { SMC_DOMAIN_TORUS = 0, SMC_DOMAIN_BOX = 1, SMC_DOMAIN_DISK = 2 } smc_domain_kind;

typedef struct smc_domain {
    int32_t kind;
    int32_t pad_;
    double lower[2], upper[2];  /* box */
    double center[2];           /* disk */
    double radius;              /* disk */
} smc_domain;

/* BvpProblemSpec (include/scalarmc/forward_bvp.hpp:16-30). */
typedef struct smc_bvp_problem {
    smc_velocity velocity;
    double kappa;
    smc_scalar_field forcing;
    smc_scalar_field boundary_data;
    smc_domain domain;
    int64_t n_obs;
    const double* obs_x;    /* [n_obs][2] */
    double dt;              /* <= 0: clipped default rule (forward_bvp.cpp:9-18) */
    int64_t n_particles;
    int32_t scheme;
    int32_t precision;
    int64_t max_steps;
} smc_bvp_problem;

/* PriorSpec (include/scalarmc/inference.hpp:22-38): fixes the u layout
 * [Re, Im] per mode in |k|^2-then-(k1,k2) order (inference.cpp:24-40, :63-73). */
typedef struct smc_prior {
    int32_t cutoff;
    int32_t pad_;
    double s0;
    double alpha;
} smc_prior;

/* ---- context ------------------------------------------------------------ */
typedef struct smc_ctx smc_ctx;

/* One context per process per GPU (torch.distributed launches one process per
 * GPU).  Owns the stream and the persistent device buffers reused across calls
 * (MCMC calls the forward map 1e5+ times). */
smc_status smc_create(int device, smc_ctx** out);
void smc_destroy(smc_ctx* ctx);
const char* smc_last_error(void);
int smc_abi_version(void);

/* ---- multi-device contexts ------------------------------
 * A context over several GPUs of one box.  smc_ad_observe, smc_ad_observe_single,
 * smc_bvp_observe(_range), smc_ad_observe_batched and smc_pcn_chains on it shard
 * their work over the GPUs (particle chunks / walker ranges / parameter samples /
 * chains) and combine ranks with a small deterministic NCCL exchange over
 * NVLink, so the estimates are bit-identical to one GPU for any device count;
 * every other call runs on the first device.  The reference's parallelism knob
 * is `workers` (executor.cpp:45-85); here it is the device list.
 *
 * One process, several GPUs: smc_create_multi(ndev, devs) (ncclCommInitAll).
 * A list that repeats a device is allowed (NCCL is then replaced by peer copies
 * ordered by events — the same arithmetic, used to test sharding on one GPU).
 * One process per GPU (torchrun): rank 0 calls smc_nccl_unique_id, the caller
 * broadcasts the 128 bytes (e.g. torch.distributed), and every rank calls
 * smc_create_rank(device, rank, world, id) — collective, like ncclCommInitRank.
 * Every rank then calls the forward maps with the same arguments and receives
 * the full result. */
#define SMC_UNIQUE_ID_BYTES 128
smc_status smc_nccl_unique_id(uint8_t* out /* [SMC_UNIQUE_ID_BYTES] */);
smc_status smc_create_multi(int ndev, const int* devs, smc_ctx** out);
smc_status smc_create_rank(int device, int rank, int world, const uint8_t* unique_id, smc_ctx** out);
/* Host-staged variant for ranks that cannot share an NCCL communicator (e.g.
 * several ranks on one GPU when testing the plumbing): at every exchange the
 * library writes this rank's contribution to buf[displ[rank], +bytes[rank]) and
 * calls exchange(user, buf, displ, bytes, world), which must fill the other
 * ranks' slices (an all-gather over the caller's transport, e.g.
 * torch.distributed over gloo) and return 0. */
typedef int (*smc_exchange_fn)(void* user, uint8_t* buf, const uint64_t* displ, const uint64_t* bytes, int world);
smc_status smc_create_rank_hosted(int device, int rank, int world, smc_exchange_fn exchange, void* user,
                                  smc_ctx** out);
typedef struct smc_group_desc {
    int32_t world;      /* ranks the forward maps are sharded over */
    int32_t rank;       /* rank of this context's first device */
    int32_t n_local;    /* devices driven by this process */
    int32_t nccl;       /* 1: NCCL exchange, 0: single device or emulated exchange */
    int32_t devices[8]; /* first 8 local devices (-1 unused) */
} smc_group_desc;
smc_status smc_group_query(smc_ctx* ctx, smc_group_desc* out);

/* ---- forward maps (the drop-in boundary) --------------------------------- */

/* observe_ad (include/scalarmc/forward_ad.hpp:39-40, src/forward_ad.cpp:53-60).
 * out: [n_obs]. */
smc_status smc_ad_observe(smc_ctx* ctx, const smc_ad_problem* prob, uint64_t seed,
                          smc_estimate* out);

/* observe_ad_single (forward_ad.hpp:43-44, forward_ad.cpp:62-69). */
smc_status smc_ad_observe_single(smc_ctx* ctx, const smc_ad_problem* prob, uint64_t obs_index,
                                 uint64_t seed, smc_estimate* out);

/* Batched AD forward map: B parameter samples per launch.  u: [B][2M] in the
 * prior's component order — each row is what velocity_from_coefficients
 * (inference.cpp:63-73) turns into a field, so row b reproduces
 * LikelihoodSpec::misfit's observe_ad call (inference.cpp:93-104) for u_b.
 * seeds: [B], or NULL for common random numbers (every sample uses `seed`).
 * The velocity slot of `base` is ignored. out: [B][n_obs].  At most 65535
 * observations per call (one grid dimension; smc_ad_observe has no limit). */
smc_status smc_ad_observe_batched(smc_ctx* ctx, const smc_ad_problem* base, const smc_prior* prior,
                                  int64_t n_samples, const double* u, const uint64_t* seeds,
                                  uint64_t seed, smc_estimate* out);

/* observe_bvp (include/scalarmc/forward_bvp.hpp:35-36, src/forward_bvp.cpp:34-49).
 * out: [n_obs]; aux_mean is the mean exit time. */
smc_status smc_bvp_observe(smc_ctx* ctx, const smc_bvp_problem* prob, uint64_t seed,
                           smc_estimate* out);

/* observe_bvp restricted to observations [obs_begin, obs_begin + obs_count)
 * with their original stream slots (observation sharding across GPUs: the
 * result for slot j never depends on which rank computes it).
 * out: [obs_count]. */
smc_status smc_bvp_observe_range(smc_ctx* ctx, const smc_bvp_problem* prob, uint64_t seed, int64_t obs_begin,
                                 int64_t obs_count, smc_estimate* out);

/* Forcing basis of the Dirichlet map.  With common
 * random numbers the walker paths do not depend on the forcing amplitudes F,
 * so for a Gaussian-bump forcing (1..4 bumps; the amplitudes in `prob` are
 * ignored) one pass yields, per observation j,
 *   mean_bc[j]            = E[theta_bc(X_tau)]
 *   mean_basis[j][k]      = E[int_0^tau phi_k(X_t) dt],  phi_k = exp(-a |x - c_k|^2)
 * and observe_bvp's mean for any F is mean_bc[j] - sum_k F_k mean_basis[j][k]
 * (forward_bvp.cpp:45 by linearity) — what forcing_cost (optimize.cpp:161-173)
 * evaluates at every Nelder-Mead vertex.  mean_tau / n_failed as
 * observe_bvp's aux_mean / n_failed.  Any output may be NULL. */
smc_status smc_bvp_forcing_basis(smc_ctx* ctx, const smc_bvp_problem* prob, uint64_t seed, double* mean_bc,
                                 double* mean_basis, double* mean_tau, int64_t* n_failed);

/* ---- device-resident multi-chain pCN ------------
 * run_chain (include/scalarmc/inference.hpp:95-99, src/inference.cpp:170-194)
 * for n_chains independent chains at once: every step evaluates all chains'
 * proposals with ONE batched forward map (common random numbers:
 * forward_seed, as LikelihoodSpec::misfit), and the proposal draw, the
 * u -> field packing, Phi, the accept/reject and the MAP tracking stay on the
 * device.  Chain c uses the stream NormalStream{chain_seeds[c], 0xFFFFFFFF, 0}
 * exactly as run_chain does with config.seed (inference.cpp:12, :175), so
 * chain c reproduces run_chain(config with seed = chain_seeds[c]).
 * `forward` is the likelihood's AdProblemSpec (its velocity slot is ignored),
 * or NULL for run_chain(..., likelihood = nullptr): Phi == 0, every proposal
 * accepted, no forward map (data / noise_std / forward_seed unused);
 * data: [n_obs] (LikelihoodSpec::data); u0: [n_chains][dim] or NULL (draw from
 * the prior).  Output arrays are caller-owned; any may be NULL except
 * final_u. */
typedef struct smc_chain_config { /* ChainConfig (inference.hpp:87-93) */
    int64_t n_steps;
    double beta;
    int64_t burn_in;
    int64_t thin;
} smc_chain_config;

typedef struct smc_chain_outputs {
    double* final_u;        /* [n_chains][dim] */
    double* final_phi;      /* [n_chains] */
    double* map_u;          /* [n_chains][dim] */
    double* map_objective;  /* [n_chains] */
    int64_t* accepted;      /* [n_chains] */
    double* phi_trace;      /* [n_chains][n_steps] */
    double* samples;        /* [n_chains][smc_pcn_num_samples(cfg)][dim] */
} smc_chain_outputs;

int64_t smc_pcn_num_samples(const smc_chain_config* cfg);
smc_status smc_pcn_chains(smc_ctx* ctx, const smc_ad_problem* forward, const smc_prior* prior, const double* data,
                          double noise_std, uint64_t forward_seed, int64_t n_chains, const uint64_t* chain_seeds,
                          const double* u0, const smc_chain_config* cfg, smc_chain_outputs* out);

/* ---- spectral Galerkin reference solver ---------
 * galerkin_solve_ad (include/scalarmc/galerkin.hpp:36-40,
 * src/galerkin.cpp:159-227): project theta_0 onto the Fourier basis, assemble
 * the dense system A_lm = -vhat_{l-m}.(2 pi i m) - delta_lm kappa (2 pi |l|)^2,
 * integrate Theta_i = (I + dt A) Theta_{i-1} through the sorted observation
 * times (shortened steps land exactly on each t_j) and evaluate
 * Re sum_l Theta_l(t_j) e^{2 pi i l.x_j}.  A lives in HBM/L2; each explicit
 * Euler step is one fused complex GEMV + axpy kernel, replayed from a CUDA
 * graph.  Basis modes: k1 = -L..L outer, k2 = -L..L inner, disk keeps
 * |k|_2 <= L (galerkin.cpp:20-33). */
typedef struct smc_galerkin_basis { /* GalerkinBasis (galerkin.hpp:14-18) */
    int32_t kind;   /* 0 box, 1 disk */
    int32_t cutoff;
} smc_galerkin_basis;

typedef struct smc_galerkin_result { /* GalerkinResult (galerkin.hpp:20-27); caller-owned arrays */
    double* observation_values;            /* [n_obs] (required) */
    double* coefficients_at_observations;  /* [n_obs][n_basis][2] or NULL */
    double* final_coefficients;            /* [n_basis][2] or NULL */
    double dt_used;
    int64_t steps;
} smc_galerkin_result;

/* Number of basis modes and the mode list [n][2] (host only). */
int64_t smc_galerkin_n_basis(const smc_galerkin_basis* basis);
smc_status smc_galerkin_modes(const smc_galerkin_basis* basis, int32_t* modes);
/* galerkin_spectral_radius (galerkin.cpp:151-157): Gershgorin row-sum bound. */
smc_status smc_galerkin_spectral_radius(smc_ctx* ctx, const smc_ad_problem* prob, const smc_galerkin_basis* basis,
                                        double* out);
smc_status smc_galerkin_solve_ad(smc_ctx* ctx, const smc_ad_problem* prob, const smc_galerkin_basis* basis,
                                 double dt_ref, smc_galerkin_result* out);
/* galerkin_field_grid (galerkin.cpp:233-250): Re sum_l c_l e^{2 pi i l.(i/n, j/n)}
 * on an n x n grid (row-major, x2 fastest) from coefficients in basis order. */
smc_status smc_galerkin_field_grid(smc_ctx* ctx, const smc_galerkin_basis* basis, const double* coefficients,
                                   int32_t n, double* grid);

/* ---- resolved step sizes (host only, no device needed) ------------------- */
/* AdProblemSpec::resolved_dt (forward_ad.cpp:10-15). */
smc_status smc_ad_resolved_dt(const smc_ad_problem* prob, double* out);
/* BvpProblemSpec::resolved_dt (forward_bvp.cpp:9-18). */
smc_status smc_bvp_resolved_dt(const smc_bvp_problem* prob, double* out);
/* Validation only (forward_ad.cpp:17-28, forward_bvp.cpp:20-32). */
smc_status smc_ad_validate(const smc_ad_problem* prob);
smc_status smc_bvp_validate(const smc_bvp_problem* prob);
/* FourierVelocityField constructor checks (fields.cpp:35-69). */
smc_status smc_velocity_validate(const smc_velocity* v);
/* sizeof of the ABI structs, in declaration order (estimate, scalar_field,
 * velocity, ad_problem, domain, bvp_problem, prior, stats) — lets bindings
 * check their layout.  Returns the number written. */
int smc_struct_sizes(int64_t* out, int cap);

/* ---- chunking -------------------------------------------------------------
 * The reduction tree's leaf block: sharded forward maps split each
 * observation's particles into chunks of SMC_CHUNK (executor.cpp:11-26 tree
 * aligned at 1024 leaves). */
#define SMC_CHUNK 1024

/* Number of chunks per observation for n_particles. */
int64_t smc_num_chunks(int64_t n_particles);

/* Device stream the context launches on (cudaStream_t as void*).  A caller
 * that already owns a stream (torch, NCCL) can hand it to the context so the
 * forward map and the collectives are ordered on one stream; NULL restores the
 * context's own stream. */
void* smc_stream(smc_ctx* ctx);
smc_status smc_set_stream(smc_ctx* ctx, void* stream);

/* ---- diagnostics ---------------------------------------------------------- */
/* Per-particle terminal values theta_0(X_T) for one observation, particles
 * [0, n) (parity diagnostics). out: [n] host. */
smc_status smc_ad_particle_values(smc_ctx* ctx, const smc_ad_problem* prob, uint64_t obs_index,
                                   uint64_t seed, int64_t n, double* out);

/* Per-walker (value, exit time, failed) for one BVP observation. */
smc_status smc_bvp_particle_values(smc_ctx* ctx, const smc_bvp_problem* prob, uint64_t obs_index,
                                   uint64_t seed, int64_t n, double* values, double* aux,
                                   uint8_t* failed);

/* Philox4x32-10 block and Box-Muller pair evaluated ON THE DEVICE for n
 * (counter, key) inputs (rng.cpp:33-41, :53-72) — the KAT hook. */
smc_status smc_philox_device(smc_ctx* ctx, int64_t n, const uint32_t* ctr, const uint32_t* key,
                             uint32_t* out);
smc_status smc_normal_pairs_device(smc_ctx* ctx, uint64_t seed, uint64_t obs, uint64_t particle,
                                   int64_t n_blocks, double* out);

/* Stats of the last forward-map call on this context: kernel time of the
 * particle kernel (ms, CUDA events on the launching stream), its launch count,
 * and the total particle-steps executed.  After smc_pcn_chains,
 * particle_kernel_ms is the device time of the whole step loop. */
typedef struct smc_stats {
    double particle_kernel_ms;
    double reduce_ms;
    int64_t kernel_launches;   /* this call */
    int64_t particle_steps;
    int64_t total_launches;    /* cumulative over the context's life */
} smc_stats;
smc_status smc_last_stats(smc_ctx* ctx, smc_stats* out);

/* FP64 DFMA peak microbenchmark (roofline denominator): runs a DFMA-only
 * kernel over all SMs for about `ms` milliseconds; returns TFLOP/s. */
smc_status smc_fp64_peak(smc_ctx* ctx, double ms, double* tflops);
/* The FP32 counterpart (FFMA-only kernel): the roofline denominator of the
 * SMC_FP32 variant. */
smc_status smc_fp32_peak(smc_ctx* ctx, double ms, double* tflops);

/* Guard-zone self-test (diagnostic; the GPU pool refuses compute-sanitizer).
 * With SMC_GUARD=1 in the environment every device buffer carries 4 KB guard
 * zones before and after it, checked at the end of every C-ABI call.  This
 * entry writes `nbytes` zero bytes at byte `offset` of a 1024-byte context
 * buffer: an offset range outside [0, 1024) must fail with SMC_ERUNTIME
 * ("device buffer overrun ...").  Returns SMC_EINVAL when guard mode is off
 * (the write would land outside any buffer). */
smc_status smc_guard_selftest(smc_ctx* ctx, int64_t offset, int64_t nbytes);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* SCALARMC_B200_H */
