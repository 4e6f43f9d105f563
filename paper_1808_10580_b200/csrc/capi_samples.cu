// capi_samples.cu — C ABI entry points over many parameter samples:
// batched forward maps (u -> coefficient blocks packed on the device) and the
// device-resident multi-chain pCN driver.
#include <exception>
#include <thread>

#include <deque>

#include "capi_internal.h"

using namespace smc;
using namespace smc::capi;

extern "C" {

}  // extern "C"

namespace smc::capi {

// Enqueue one batched evaluation of samples [0, n_samples) of (u, seeds) on
// ctx's stream: pack -> K1 -> K3; estimates [n_samples][n_obs] stay on the
// device (R.est).  R.d_bad: the FourierVelocityField ctor's non-finite check
// (fields.cpp:46-47), read by the caller after the stream completes.
struct BatchedRun {
    smc_estimate* est = nullptr;
    int* d_bad = nullptr;
    int64_t steps = 0;
};

BatchedRun batched_enqueue(smc_ctx* ctx, const smc_ad_problem& p, const smc_prior& prior, int64_t n_samples,
                           const double* u, const uint64_t* seeds, uint64_t seed) {
    BatchedRun R;
    ctx->stats = smc_stats{};
    const int64_t n = p.n_particles, n_obs = p.n_obs;
    // One FourierVelocityField per sample from u in prior order
    // (velocity_from_coefficients, inference.cpp:63-73), built on the
    // device: the image carries the full prior disk's structure and the
    // pack kernel writes every sample's coefficient block from u.
    const PreparedVelocity structure = prior_structure(prior.cutoff);
    const int64_t dim = 2 * static_cast<int64_t>(structure.modes.size());
    AdPrepared P = prepare_ad(ctx, p, {&structure}, structure, 0, n_obs);
    P.L.host_disk = nullptr;  // the coefficient blocks come from the pack kernel
    const LatticeHost Lh = lattice_structure(structure);
    const PackMap pmap = pack_map(prior.cutoff, P.disk_K > 0, &Lh);
    const PackDev pdev = upload_pack_map(ctx, pmap);
    double* d_u = ctx->pk_u.get<double>(static_cast<size_t>(n_samples * dim));
    CK(cudaMemcpyAsync(d_u, u, sizeof(double) * n_samples * dim, cudaMemcpyHostToDevice, ctx->stream));
    double* blocks = ctx->pk_blocks.get<double>(static_cast<size_t>(n_samples * pmap.stride));
    R.d_bad = ctx->pk_bad.get<int>(1);
    CK(cudaMemsetAsync(R.d_bad, 0, sizeof(int), ctx->stream));
    CK(launch_pack(pdev, d_u, dim, n_samples, blocks, R.d_bad, ctx->stream));
    count_launches(ctx, 1);
    if (P.disk_K > 0) {
        P.disk = blocks;
    } else {
        P.L.vel.lat.coef = blocks;
        P.L.vel.lat.sample_stride = pmap.stride;
    }
    uint64_t* d_seeds = nullptr;
    if (seeds) {
        d_seeds = ctx->tmp_a.get<uint64_t>(static_cast<size_t>(n_samples));
        CK(cudaMemcpyAsync(d_seeds, seeds, sizeof(uint64_t) * n_samples, cudaMemcpyHostToDevice, ctx->stream));
    }
    double* values = ctx->values.get<double>(static_cast<size_t>(std::max<int64_t>(n_samples * n_obs * n, 1)));
    CK(cudaEventRecord(ctx->ev[0], ctx->stream));
    constexpr int64_t kMaxZ = 65535;
    for (int64_t b0 = 0; b0 < n_samples; b0 += kMaxZ) {
        const int64_t nb = std::min(kMaxZ, n_samples - b0);
        AdLaunch L = P.L;
        L.seed = seed;
        L.seeds = d_seeds ? d_seeds + b0 : nullptr;
        L.n_samples = static_cast<int32_t>(nb);
        if (!L.vel.is_constant) L.vel.lat.coef += b0 * L.vel.lat.sample_stride;
        L.values = values + b0 * n_obs * n;
        run_particles(ctx, L, &P, b0);
    }
    CK(cudaEventRecord(ctx->ev[1], ctx->stream));
    R.est = n_samples > 0 ? reduce_ad_device(ctx, values, n, n_samples * n_obs) : nullptr;
    CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    R.steps = P.steps_per_particle_sum * n * n_samples;
    return R;
}

// observe_ad_batched's checks (validate() without the velocity slot).
smc_ad_problem batched_problem(const smc_ad_problem* base, const smc_prior* prior, int64_t n_samples) {
    if (n_samples < 1) raise(SMC_EINVAL, "observe_ad_batched: need at least one sample");
    if (prior->cutoff <= 0) raise(SMC_EINVAL, "FourierVelocityField: max_wavenumber must be positive");
    smc_ad_problem p = *base;
    p.velocity.is_constant = 0;
    p.velocity.max_wavenumber = prior->cutoff;
    check_kappa(p.kappa);
    check_scalar(p.initial_condition);
    ad_validate(p);
    check_particle_range(p.n_particles);
    if (p.precision == SMC_FP64_STRICT) raise(SMC_EINVAL, "strict precision is single-sample only");
    if (p.n_obs > 65535) raise(SMC_ERUNTIME, "observe_ad_batched: at most 65535 observations per batched launch");
    return p;
}

// Sample sharding: rank r evaluates samples [B r / W, B (r+1) / W); the
// estimate rows are all-gathered (n_obs x 40 B per sample) so every rank
// returns the whole [B][n_obs].  No arithmetic crosses ranks: bit-identical.
void group_ad_observe_batched(smc_ctx* ctx, const smc_ad_problem& p, const smc_prior& prior, int64_t B,
                              const double* u, const uint64_t* seeds, uint64_t seed, smc_estimate* out) {
    smc_group* g = ctx->group;
    const int W = g->world, nloc = static_cast<int>(g->members.size());
    const int64_t n_obs = p.n_obs;
    const int64_t dim = 2 * static_cast<int64_t>(prior_modes(prior.cutoff).size());
    const size_t row = sizeof(smc_estimate) * static_cast<size_t>(n_obs);
    std::vector<size_t> displ(W), bytes(W);
    for (int r = 0; r < W; ++r) {
        displ[r] = static_cast<size_t>(B * r / W) * row;
        bytes[r] = static_cast<size_t>(B * (r + 1) / W - B * r / W) * row;
    }
    std::vector<unsigned char*> ex(nloc);
    std::vector<int*> bad(nloc);
    int64_t local_steps = 0;
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        const int r = g->rank0 + m;
        const int64_t sb = B * r / W, nb = B * (r + 1) / W - sb;
        CK(cudaSetDevice(c->device));
        ex[m] = c->gx_d.get<unsigned char>(static_cast<size_t>(B) * row);
        if (nb == 0) {
            c->stats = smc_stats{};
            CK(cudaEventRecord(c->ev[0], c->stream));
            CK(cudaEventRecord(c->ev[1], c->stream));
            CK(cudaEventRecord(c->ev[2], c->stream));
            bad[m] = nullptr;
            continue;
        }
        const BatchedRun R = batched_enqueue(c, p, prior, nb, u + sb * dim, seeds ? seeds + sb : nullptr, seed);
        CK(cudaMemcpyAsync(ex[m] + displ[r], R.est, bytes[r], cudaMemcpyDeviceToDevice, c->stream));
        bad[m] = R.d_bad;
        local_steps += R.steps;
    }
    group_exchange(g, ex, displ, bytes);
    std::vector<int> bad_h(static_cast<size_t>(nloc), 0);
    {
        smc_ctx* c = g->members[0];
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpyAsync(c->est_host.get<unsigned char>(static_cast<size_t>(B) * row), ex[0],
                           static_cast<size_t>(B) * row, cudaMemcpyDeviceToHost, c->stream));
    }
    smc_stats agg{};
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        CK(cudaSetDevice(c->device));
        if (bad[m]) CK(cudaMemcpyAsync(&bad_h[m], bad[m], sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        finish_stats(c);
        agg.particle_kernel_ms = std::max(agg.particle_kernel_ms, c->stats.particle_kernel_ms);
        agg.reduce_ms = std::max(agg.reduce_ms, c->stats.reduce_ms);
        agg.kernel_launches += c->stats.kernel_launches;
    }
    CK(cudaSetDevice(ctx->device));
    agg.particle_steps = local_steps;
    ctx->stats = agg;
    for (int b : bad_h)
        if (b) raise(SMC_EINVAL, "FourierVelocityField: non-finite coefficient");
    std::memcpy(out, ctx->est_host.p, static_cast<size_t>(B) * row);
}

}  // namespace smc::capi

extern "C" {

smc_status smc_ad_observe_batched(smc_ctx* ctx, const smc_ad_problem* base, const smc_prior* prior,
                                  int64_t n_samples, const double* u, const uint64_t* seeds, uint64_t seed,
                                  smc_estimate* out) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        const smc_ad_problem p = batched_problem(base, prior, n_samples);
        if (is_sharded(ctx)) {
            group_ad_observe_batched(ctx, p, *prior, n_samples, u, seeds, seed, out);
            return;
        }
        const BatchedRun R = batched_enqueue(ctx, p, *prior, n_samples, u, seeds, seed);
        const size_t bytes = sizeof(smc_estimate) * static_cast<size_t>(n_samples * p.n_obs);
        smc_estimate* h = ctx->est_host.get<smc_estimate>(static_cast<size_t>(n_samples * p.n_obs));
        CK(cudaMemcpyAsync(h, R.est, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        int bad = 0;
        CK(cudaMemcpyAsync(&bad, R.d_bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        finish_stats(ctx);
        ctx->stats.particle_steps = R.steps;
        // the FourierVelocityField ctor throws before any particle work (fields.cpp:46-47)
        if (bad) raise(SMC_EINVAL, "FourierVelocityField: non-finite coefficient");
        std::memcpy(out, h, bytes);
    });
}

int64_t smc_pcn_num_samples(const smc_chain_config* cfg) {
    // iterations i = 1..n_steps with i > burn_in and (i - burn_in - 1) % thin
    // == 0 (inference.cpp:183-185): from the first such i0 every thin-th one.
    // A negative burn_in moves i0 off 1 (burn_in = -2, thin 4: i0 = 3).
    if (!cfg || cfg->thin < 1 || cfg->n_steps < 1) return 0;
    const int64_t thin = cfg->thin;
    const int64_t lo = cfg->burn_in + 1 > 1 ? cfg->burn_in + 1 : 1;
    const int64_t r = ((lo - cfg->burn_in - 1) % thin + thin) % thin;
    const int64_t i0 = r == 0 ? lo : lo + (thin - r);
    return cfg->n_steps >= i0 ? (cfg->n_steps - i0) / thin + 1 : 0;
}

}  // extern "C"

namespace smc::capi {

// run_chain's checks (inference.cpp:172-173), prior_draw/chain_init's
// (inference.cpp:17-21, :89-91, :125-133), pcn_step's (:138).
void pcn_validate(const smc_ad_problem* forward, const smc_prior* prior, double noise_std, int64_t n_chains,
                  const smc_chain_config* cfg, const smc_chain_outputs* out) {
    if (cfg->n_steps < 0) raise(SMC_EINVAL, "run_chain: n_steps must be >= 0");
    if (cfg->thin < 1) raise(SMC_EINVAL, "run_chain: thin must be >= 1");
    if (prior->cutoff < 1) raise(SMC_EINVAL, "PriorSpec: cutoff must be >= 1");
    if (!(prior->s0 >= 0.0)) raise(SMC_EINVAL, "PriorSpec: s0 must be >= 0");
    if (!std::isfinite(prior->alpha)) raise(SMC_EINVAL, "PriorSpec: alpha must be finite");
    // forward == nullptr: run_chain(..., likelihood = nullptr) — Phi == 0, no forward map
    if (forward != nullptr && !(noise_std > 0.0)) raise(SMC_EINVAL, "LikelihoodSpec: noise_std must be positive");
    if (cfg->n_steps > 0 && !(cfg->beta > 0.0 && cfg->beta <= 1.0)) raise(SMC_EINVAL, "pcn_step: beta must be in (0,1]");
    if (n_chains < 1) raise(SMC_EINVAL, "pcn_chains: need at least one chain");
    if (!out || !out->final_u) raise(SMC_EINVAL, "pcn_chains: final_u output is required");
    if (forward != nullptr) {
        const smc_ad_problem& p = *forward;
        check_kappa(p.kappa);
        check_scalar(p.initial_condition);
        ad_validate(p);
        check_particle_range(p.n_particles);
        if (p.precision == SMC_FP64_STRICT) raise(SMC_EINVAL, "strict precision is single-sample only");
        if (p.n_obs > 65535)
            raise(SMC_ERUNTIME, "smc_pcn_chains: at most 65535 observations in the likelihood's forward map");
    }
}

// The chains [0, n_chains) of one device (one batched forward map per step).
void pcn_chains_impl(smc_ctx* ctx, const smc_ad_problem* forward, const smc_prior* prior, const double* data,
                     double noise_std, uint64_t forward_seed, int64_t n_chains, const uint64_t* chain_seeds,
                     const double* u0, const smc_chain_config* cfg, smc_chain_outputs* out) {
    CK(cudaSetDevice(ctx->device));
    pcn_validate(forward, prior, noise_std, n_chains, cfg, out);
    const bool prior_only = forward == nullptr;
    smc_ad_problem p{};
    if (!prior_only) p = *forward;
    cudaStream_t s = ctx->stream;
    const int64_t n_obs = p.n_obs, n = p.n_particles, B = n_chains;

    // prior modes (|k|^2 then (k1,k2) order) and per-mode stds (inference.cpp:24-53)
    const std::vector<HostMode> pm = prior_modes(prior->cutoff);
    const int64_t M = static_cast<int64_t>(pm.size()), dim = 2 * M;
    std::vector<double> stds(static_cast<size_t>(M));
    for (int64_t i = 0; i < M; ++i) {
        const double kn = std::sqrt(double(pm[i].k1) * pm[i].k1 + double(pm[i].k2) * pm[i].k2);
        stds[static_cast<size_t>(i)] = prior->s0 * std::pow(kn, -prior->alpha);
    }
    // lattice structure of the full prior disk and the u -> block gather map
    // (disk layout for K <= kDiskMaxK, tiled lattice otherwise)
    const PreparedVelocity structure = prior_structure(prior->cutoff);
    const bool use_disk =
        disk_kernel_for(prior->cutoff, p.precision == SMC_FP64) && std::getenv("SMC_DISABLE_DISK") == nullptr;
    const LatticeHost Lh = lattice_structure(structure);
    const PackMap pmap = pack_map(prior->cutoff, use_disk, &Lh);
    const int64_t stride = pmap.stride;
    if (!prior_only && static_cast<int64_t>(p.n_obs) <= 0) raise(SMC_EINVAL, "AdProblemSpec: no observations");
    if (!prior_only && p.n_obs > 65535)
        raise(SMC_ERUNTIME, "smc_pcn_chains: at most 65535 observations in the likelihood's forward map");

    // device buffers (RAII: freed at the end of the call, guard zones under SMC_GUARD)
    std::deque<DevBuf> owned;
    auto dalloc = [&](size_t bytes) -> void* {
        owned.emplace_back();
        return owned.back().get<unsigned char>(bytes);
    };
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    };
    const int64_t n_samples = smc_pcn_num_samples(cfg);
    PcnStep S{};
    S.n_chains = B;
    S.dim = dim;
    S.M = M;
    S.n_obs = n_obs;
    S.n_steps = cfg->n_steps;
    S.n_samples = n_samples;
    S.noise_std = noise_std;
    S.noise_inf = (prior_only || std::isinf(noise_std)) ? 1 : 0;
    auto* d_stds = static_cast<double*>(dalloc(8 * M));
    h2d(d_stds, stds.data(), 8 * M);
    S.stds = d_stds;
    auto* d_seeds = static_cast<uint64_t*>(dalloc(8 * B));
    h2d(d_seeds, chain_seeds, 8 * B);
    S.seeds = d_seeds;
    auto* d_data = static_cast<double*>(dalloc(8 * std::max<int64_t>(n_obs, 1)));
    if (!prior_only) h2d(d_data, data, 8 * n_obs);
    S.data = d_data;
    const PackDev pdev = upload_pack_map(ctx, pmap);
    S.U = static_cast<double*>(dalloc(8 * B * dim));
    S.Up = static_cast<double*>(dalloc(8 * B * dim));
    S.map_u = static_cast<double*>(dalloc(8 * B * dim));
    S.norm_prop = static_cast<double*>(dalloc(8 * B));
    S.norm_cur = static_cast<double*>(dalloc(8 * B));
    S.phi = static_cast<double*>(dalloc(8 * B));
    S.map_obj = static_cast<double*>(dalloc(8 * B));
    S.accepted = static_cast<int64_t*>(dalloc(8 * B));
    S.acc_flag = static_cast<uint8_t*>(dalloc(B));
    S.map_flag = static_cast<uint8_t*>(dalloc(B));
    S.phi_trace = out->phi_trace ? static_cast<double*>(dalloc(8 * B * std::max<int64_t>(1, cfg->n_steps))) : nullptr;
    S.samples = (out->samples && n_samples > 0) ? static_cast<double*>(dalloc(8 * B * n_samples * dim)) : nullptr;
    auto* d_blocks = static_cast<double*>(dalloc(8 * B * stride));
    CK(cudaMemsetAsync(S.U, 0, 8 * B * dim, s));
    CK(cudaMemsetAsync(S.accepted, 0, 8 * B, s));
    CK(cudaMemsetAsync(S.phi, 0, 8 * B, s));

    // forward image (theta_0, observations, lattice tiles); coefficient
    // blocks come from the pack kernel
    AdPrepared P{};
    double* values = nullptr;
    if (!prior_only) {
        p.velocity.is_constant = 0;
        p.velocity.max_wavenumber = prior->cutoff;
        P = prepare_ad(ctx, p, {&structure}, structure, 0, n_obs);
        P.L.host_disk = nullptr;  // the coefficient blocks come from the pack kernel
        P.L.seed = forward_seed;
        P.L.seeds = nullptr;
        if (!use_disk) {
            P.L.vel.lat.coef = d_blocks;
            P.L.vel.lat.sample_stride = stride;
        }
        values = ctx->values.get<double>(static_cast<size_t>(B * n_obs * n));
    }

    auto forward_map = [&]() -> smc_estimate* {
        if (prior_only) return nullptr;  // Phi == 0 (noise_inf), nothing to evaluate
        for (int64_t b0 = 0; b0 < B; b0 += 65535)
            CK(launch_pack(pdev, S.Up + b0 * dim, dim, std::min<int64_t>(65535, B - b0), d_blocks + b0 * stride,
                           nullptr, s));
        constexpr int64_t kMaxZ = 65535;
        for (int64_t b0 = 0; b0 < B; b0 += kMaxZ) {
            AdLaunch L = P.L;
            L.n_samples = static_cast<int32_t>(std::min(kMaxZ, B - b0));
            L.values = values + b0 * n_obs * n;
            if (use_disk) {
                CK(launch_ad_disk(L, prior->cutoff, d_blocks + b0 * stride, s));
            } else {
                L.vel.lat.coef = d_blocks + b0 * stride;
                run_particles(ctx, L);
            }
        }
        count_launches(ctx, 1);
        return reduce_ad_device(ctx, values, n, B * n_obs);
    };

    // chain_init (inference.cpp:125-134): u0 given, or prior_draw from the stream
    uint64_t blk = 0;
    if (u0) {
        h2d(S.U, u0, 8 * B * dim);
        S.contraction = 1.0;  // Up = 1 U + 0 xi = U
        S.beta = 0.0;
    } else {
        S.contraction = 0.0;  // Up = 0 U + 1 xi = xi = prior_draw
        S.beta = 1.0;
        blk = static_cast<uint64_t>(M);
    }
    S.blk0 = 0;
    S.init = 1;
    S.step = 0;
    S.sample_slot = -1;
    CK(launch_pcn_propose(S, s));
    CK(launch_pcn_accept(S, forward_map(), s));
    CK(launch_pcn_commit(S, s));
    count_launches(ctx, 3);

    // the steps (pcn_step, inference.cpp:136-166; run_chain loop :182-189)
    S.init = 0;
    S.contraction = std::sqrt(1.0 - cfg->beta * cfg->beta);
    S.beta = cfg->beta;
    ctx->stats = smc_stats{};
    CK(cudaEventRecord(ctx->ev[0], s));
    const char* ge = std::getenv("SMC_PCN_GRAPH");
    const bool use_graph = cfg->n_steps >= 2 && s != nullptr && !(ge && std::atoi(ge) == 0);
    if (use_graph) {
        // Graph mode: the step index is a device counter, so a captured
        // group of G steps (propose, pack, K1, K3, accept, commit, advance)
        // replays unchanged; the launch cost per step drops to a share of
        // one graph launch.  Same kernels, same arguments: bit-identical.
        auto* d_it = static_cast<int64_t*>(dalloc(8));
        CK(cudaMemsetAsync(d_it, 0, 8, s));
        S.it_dev = d_it;
        S.blk_base = blk;
        S.burn_in = cfg->burn_in;
        S.thin = cfg->thin;
        const int64_t before = ctx->total_launches;
        auto capture = [&](int64_t g) {
            cudaGraph_t graph = nullptr;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            try {
                for (int64_t k = 0; k < g; ++k) {
                    CK(launch_pcn_propose(S, s));
                    CK(launch_pcn_accept(S, forward_map(), s));
                    CK(launch_pcn_commit(S, s));
                    CK(launch_pcn_advance(d_it, s));
                }
            } catch (...) {
                cudaStreamEndCapture(s, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            CK(cudaStreamEndCapture(s, &graph));
            cudaGraphExec_t exec = nullptr;
            const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
            cudaGraphDestroy(graph);
            CK(e);
            return exec;
        };
        const int64_t G = std::min<int64_t>(16, cfg->n_steps);
        cudaGraphExec_t group = capture(G);
        const int64_t per_step = (ctx->total_launches - before) / G + 4;
        const int64_t rest = cfg->n_steps % G;
        cudaGraphExec_t single = rest ? capture(1) : nullptr;
        struct ExecFree {
            cudaGraphExec_t a, b;
            ~ExecFree() {
                if (a) cudaGraphExecDestroy(a);
                if (b) cudaGraphExecDestroy(b);
            }
        } exec_free{group, single};
        for (int64_t q = 0; q < cfg->n_steps / G; ++q) CK(cudaGraphLaunch(group, s));
        for (int64_t r = 0; r < rest; ++r) CK(cudaGraphLaunch(single, s));
        ctx->total_launches = before + per_step * cfg->n_steps;
    }
    bool ucache = false;
    uint64_t ublk = 0;
    for (int64_t it = 0; !use_graph && it < cfg->n_steps; ++it) {
        S.blk0 = blk;
        blk += static_cast<uint64_t>(M);
        if (!ucache) {  // uniform() draws a fresh block and caches its second value
            ublk = blk;
            blk += 1;
            S.uhalf = 0;
            ucache = true;
        } else {
            S.uhalf = 1;
            ucache = false;
        }
        S.ublk = ublk;
        S.step = it;
        const int64_t iteration = it + 1;
        S.sample_slot = (iteration > cfg->burn_in && (iteration - cfg->burn_in - 1) % cfg->thin == 0)
                            ? (iteration - std::max<int64_t>(cfg->burn_in, 0) - 1) / cfg->thin
                            : -1;
        CK(launch_pcn_propose(S, s));
        CK(launch_pcn_accept(S, forward_map(), s));
        CK(launch_pcn_commit(S, s));
        count_launches(ctx, 3);
    }
    CK(cudaEventRecord(ctx->ev[1], s));
    CK(cudaEventRecord(ctx->ev[2], s));
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
        if (dst) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    };
    d2h(out->final_u, S.U, 8 * B * dim);
    d2h(out->final_phi, S.phi, 8 * B);
    d2h(out->map_u, S.map_u, 8 * B * dim);
    d2h(out->map_objective, S.map_obj, 8 * B);
    d2h(out->accepted, S.accepted, 8 * B);
    if (S.phi_trace && cfg->n_steps > 0) d2h(out->phi_trace, S.phi_trace, 8 * B * cfg->n_steps);
    if (S.samples) d2h(out->samples, S.samples, 8 * B * n_samples * dim);
    CK(cudaStreamSynchronize(s));
    finish_stats(ctx);  // particle_kernel_ms = device time of the step loop
}

// Chain sharding: rank r runs chains [B r / W, B (r+1) / W) — chains are
// independent, so nothing crosses ranks but the outputs.  One process with
// several GPUs: one host thread per device writes its rows of `out`.  One
// process per GPU: each rank's rows are packed, all-gathered (group_exchange)
// and unpacked, so every rank returns every chain.
void group_pcn_chains(smc_ctx* ctx, const smc_ad_problem* forward, const smc_prior* prior, const double* data,
                      double noise_std, uint64_t forward_seed, int64_t B, const uint64_t* chain_seeds,
                      const double* u0, const smc_chain_config* cfg, smc_chain_outputs* out) {
    smc_group* g = ctx->group;
    const int W = g->world, nloc = static_cast<int>(g->members.size());
    const int64_t dim = 2 * static_cast<int64_t>(prior_modes(prior->cutoff).size());
    const int64_t T = cfg->n_steps, NS = smc_pcn_num_samples(cfg);
    auto block = [&](int r) { return std::make_pair(B * r / W, B * (r + 1) / W - B * r / W); };
    auto shifted = [&](smc_chain_outputs* o, int64_t cb) {
        smc_chain_outputs s{};
        s.final_u = o->final_u + cb * dim;
        s.final_phi = o->final_phi ? o->final_phi + cb : nullptr;
        s.map_u = o->map_u ? o->map_u + cb * dim : nullptr;
        s.map_objective = o->map_objective ? o->map_objective + cb : nullptr;
        s.accepted = o->accepted ? o->accepted + cb : nullptr;
        s.phi_trace = o->phi_trace ? o->phi_trace + cb * T : nullptr;
        s.samples = o->samples ? o->samples + cb * NS * dim : nullptr;
        return s;
    };
    smc_stats agg{};
    auto collect = [&](smc_ctx* c) {
        agg.particle_kernel_ms = std::max(agg.particle_kernel_ms, c->stats.particle_kernel_ms);
        agg.reduce_ms = std::max(agg.reduce_ms, c->stats.reduce_ms);
        agg.kernel_launches += c->stats.kernel_launches;
        agg.particle_steps += c->stats.particle_steps;
    };
    if (nloc == W) {  // one process: a host thread per device
        std::vector<std::thread> threads;
        std::vector<std::exception_ptr> errs(static_cast<size_t>(nloc));
        for (int m = 0; m < nloc; ++m) {
            const auto [cb, nb] = block(m);
            if (nb == 0) continue;
            threads.emplace_back([&, m, cb = cb, nb = nb] {
                try {
                    smc_ctx* c = g->members[m];
                    CK(cudaSetDevice(c->device));
                    smc_chain_outputs o = shifted(out, cb);
                    pcn_chains_impl(c, forward, prior, data, noise_std, forward_seed, nb, chain_seeds + cb,
                                    u0 ? u0 + cb * dim : nullptr, cfg, &o);
                } catch (...) {
                    errs[static_cast<size_t>(m)] = std::current_exception();
                }
            });
        }
        for (auto& t : threads) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        for (smc_ctx* c : g->members) collect(c);
        CK(cudaSetDevice(ctx->device));
        ctx->stats = agg;
        return;
    }
    // one rank per process: run the own block into a packed row per chain
    //   [final_u dim | final_phi | map_u dim | map_objective | accepted | phi_trace T | samples NS*dim]
    const int64_t R = 2 * dim + 3 + (out->phi_trace ? T : 0) + (out->samples ? NS * dim : 0);
    const int r = g->rank0;
    const auto [cb, nb] = block(r);
    std::vector<double> fu(static_cast<size_t>(nb * dim)), fp(static_cast<size_t>(nb)), mu(static_cast<size_t>(nb * dim)),
        mo(static_cast<size_t>(nb)), pt(out->phi_trace ? static_cast<size_t>(nb * T) : 0),
        sm(out->samples ? static_cast<size_t>(nb * NS * dim) : 0);
    std::vector<int64_t> ac(static_cast<size_t>(nb));
    if (nb > 0) {
        smc_chain_outputs o{fu.data(), fp.data(), mu.data(), mo.data(), ac.data(),
                            out->phi_trace ? pt.data() : nullptr, out->samples ? sm.data() : nullptr};
        pcn_chains_impl(ctx, forward, prior, data, noise_std, forward_seed, nb, chain_seeds + cb,
                        u0 ? u0 + cb * dim : nullptr, cfg, &o);
    } else {
        ctx->stats = smc_stats{};
    }
    collect(ctx);
    std::vector<double> rows(static_cast<size_t>(B * R));
    for (int64_t i = 0; i < nb; ++i) {
        double* w = rows.data() + (cb + i) * R;
        std::copy_n(fu.data() + i * dim, dim, w);
        w[dim] = fp[i];
        std::copy_n(mu.data() + i * dim, dim, w + dim + 1);
        w[2 * dim + 1] = mo[i];
        std::memcpy(&w[2 * dim + 2], &ac[i], sizeof(double));
        int64_t k = 2 * dim + 3;
        if (out->phi_trace) {
            std::copy_n(pt.data() + i * T, T, w + k);
            k += T;
        }
        if (out->samples) std::copy_n(sm.data() + i * NS * dim, NS * dim, w + k);
    }
    std::vector<size_t> displ(W), bytes(W);
    for (int q = 0; q < W; ++q) {
        displ[q] = static_cast<size_t>(block(q).first * R) * sizeof(double);
        bytes[q] = static_cast<size_t>(block(q).second * R) * sizeof(double);
    }
    unsigned char* d = ctx->gx_d.get<unsigned char>(static_cast<size_t>(B * R) * sizeof(double));
    CK(cudaSetDevice(ctx->device));
    if (bytes[r])
        CK(cudaMemcpyAsync(d + displ[r], reinterpret_cast<unsigned char*>(rows.data()) + displ[r], bytes[r],
                           cudaMemcpyHostToDevice, ctx->stream));
    group_exchange(g, {d}, displ, bytes);
    CK(cudaMemcpyAsync(rows.data(), d, static_cast<size_t>(B * R) * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int64_t b = 0; b < B; ++b) {
        const double* w = rows.data() + b * R;
        std::copy_n(w, dim, out->final_u + b * dim);
        if (out->final_phi) out->final_phi[b] = w[dim];
        if (out->map_u) std::copy_n(w + dim + 1, dim, out->map_u + b * dim);
        if (out->map_objective) out->map_objective[b] = w[2 * dim + 1];
        if (out->accepted) std::memcpy(&out->accepted[b], &w[2 * dim + 2], sizeof(int64_t));
        int64_t k = 2 * dim + 3;
        if (out->phi_trace) {
            std::copy_n(w + k, T, out->phi_trace + b * T);
            k += T;
        }
        if (out->samples) std::copy_n(w + k, NS * dim, out->samples + b * NS * dim);
    }
    ctx->stats = agg;
}

}  // namespace smc::capi

extern "C" {

smc_status smc_pcn_chains(smc_ctx* ctx, const smc_ad_problem* forward, const smc_prior* prior, const double* data,
                          double noise_std, uint64_t forward_seed, int64_t n_chains, const uint64_t* chain_seeds,
                          const double* u0, const smc_chain_config* cfg, smc_chain_outputs* out) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        pcn_validate(forward, prior, noise_std, n_chains, cfg, out);
        if (is_sharded(ctx))
            group_pcn_chains(ctx, forward, prior, data, noise_std, forward_seed, n_chains, chain_seeds, u0, cfg, out);
        else
            pcn_chains_impl(ctx, forward, prior, data, noise_std, forward_seed, n_chains, chain_seeds, u0, cfg, out);
    });
}

}  // extern "C"

