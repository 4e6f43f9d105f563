// capi_group.cu — multi-device contexts: one forward map sharded over the
// GPUs of a box, behind the same C-ABI calls.
//
// A group is either the GPUs of one process (smc_create_multi: one thread
// drives every device, NCCL communicators from ncclCommInitAll) or one GPU per
// process (smc_create_rank: torchrun / MPI style, ncclCommInitRank with a
// unique id the caller broadcasts).  smc_ad_observe / smc_bvp_observe /
// smc_ad_observe_batched / smc_pcn_chains on a group context shard their work
// internally; everything else runs on the owning context's device.
//
// The exchange is an all-gather of variable-size contributions done as one
// NCCL group of in-place broadcasts (rank q broadcasts its slice into the
// same offset of every rank's buffer), on each member's stream — no host
// synchronisation between the compute phases.  A single process whose device
// list repeats a GPU (NCCL rejects duplicate devices) exchanges with peer
// copies ordered by events instead ("emulated"); the arithmetic is the same,
// so results are bit-identical either way.
//
// NCCL is loaded at run time (dlopen libnccl.so.2): a process that already
// loaded one (torch) reuses it, and single-device contexts never need it.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "capi_internal.h"

using namespace smc;
using namespace smc::capi;

namespace smc::capi {
namespace {

// ---- NCCL, loaded on first use ---------------------------------------------
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

const NcclApi* nccl(std::string* why) {
    static NcclApi api;
    static std::string err;
    static bool ok = false;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* name = std::getenv("SMC_NCCL_LIB");
        void* h = dlopen(name ? name : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot load NCCL: ") + dlerror();
            return;
        }
        auto sym = [&](const char* s) {
            void* f = dlsym(h, s);
            if (!f && err.empty()) err = std::string("NCCL symbol missing: ") + s;
            return f;
        };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(sym("ncclGetVersion"));
        ok = err.empty();
    });
    if (!ok) {
        if (why) *why = err;
        return nullptr;
    }
    return &api;
}

void NK(const NcclApi* api, ncclResult_t r, const char* what) {
    if (r != ncclSuccess) raise(SMC_ECUDA, std::string("NCCL error: ") + api->GetErrorString(r) + " (" + what + ")");
}

const NcclApi* need_nccl() {
    std::string why;
    const NcclApi* api = nccl(&why);
    if (!api) raise(SMC_ECUDA, why);
    return api;
}

smc_ctx* new_member(int device) {
    smc_ctx* c = nullptr;
    const smc_status st = smc_create(device, &c);
    if (st != SMC_OK) raise(st, smc_last_error());
    return c;
}

}  // namespace

void group_destroy(smc_ctx* ctx) {
    smc_group* g = ctx->group;
    ctx->group = nullptr;
    if (!g) return;
    for (smc_ctx* m : g->members) {
        cudaSetDevice(m->device);
        cudaStreamSynchronize(m->stream);
    }
    if (!g->comms.empty()) {
        if (const NcclApi* api = nccl(nullptr))
            for (void* c : g->comms)
                if (c) api->CommDestroy(static_cast<ncclComm_t>(c));
    }
    for (size_t i = 0; i < g->ready.size(); ++i) {
        cudaSetDevice(g->members[i]->device);
        if (g->ready[i]) cudaEventDestroy(g->ready[i]);
    }
    for (size_t i = 1; i < g->members.size(); ++i) smc_destroy(g->members[i]);
    delete g;
}

// Rank r's contribution occupies bytes [displ[r], displ[r] + bytes[r]) of
// every member's buffer bufs[m] and is already in place on the member that
// owns rank r; afterwards every member holds all of them.  Enqueued on the
// members' streams (no host synchronisation).
void group_exchange(smc_group* g, const std::vector<unsigned char*>& bufs, const std::vector<size_t>& displ,
                    const std::vector<size_t>& bytes) {
    const int nloc = static_cast<int>(g->members.size());
    // a forced one-rank group (SMC_GROUP_FORCE) still runs its NCCL calls
    if (g->world == 1 && g->comms.empty()) return;
    if (g->hook) {  // one member: stage through the host, the caller's all-gather fills the rest
        smc_ctx* c = g->members[0];
        const int r = g->rank0;
        size_t total = 0;
        for (int q = 0; q < g->world; ++q) total = std::max(total, displ[q] + bytes[q]);
        unsigned char* h = g->hook_buf.get<unsigned char>(total);
        CK(cudaSetDevice(c->device));
        if (bytes[r]) CK(cudaMemcpyAsync(h + displ[r], bufs[0] + displ[r], bytes[r], cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        std::vector<uint64_t> d(displ.begin(), displ.end()), b(bytes.begin(), bytes.end());
        if (g->hook(g->hook_user, h, d.data(), b.data(), g->world) != 0)
            raise(SMC_ERUNTIME, "smc group exchange: the host exchange callback failed");
        for (int q = 0; q < g->world; ++q)
            if (q != r && bytes[q])
                CK(cudaMemcpyAsync(bufs[0] + displ[q], h + displ[q], bytes[q], cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));  // h is reused by the next exchange
        return;
    }
    if (!g->comms.empty()) {
        const NcclApi* api = need_nccl();
        NK(api, api->GroupStart(), "ncclGroupStart");
        for (int q = 0; q < g->world; ++q) {
            if (bytes[q] == 0) continue;
            for (int m = 0; m < nloc; ++m) {
                unsigned char* p = bufs[m] + displ[q];
                const ncclResult_t r = api->Broadcast(p, p, bytes[q], ncclUint8, q,
                                                      static_cast<ncclComm_t>(g->comms[m]), g->members[m]->stream);
                if (r != ncclSuccess) {
                    api->GroupEnd();
                    NK(api, r, "ncclBroadcast");
                }
            }
        }
        NK(api, api->GroupEnd(), "ncclGroupEnd");
        return;
    }
    // emulated: every member's stream waits for the others' contributions and
    // copies them in
    for (int m = 0; m < nloc; ++m) {
        CK(cudaSetDevice(g->members[m]->device));
        CK(cudaEventRecord(g->ready[m], g->members[m]->stream));
    }
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* dst = g->members[m];
        CK(cudaSetDevice(dst->device));
        for (int q = 0; q < nloc; ++q) {
            if (q == m || bytes[g->rank0 + q] == 0) continue;
            smc_ctx* src = g->members[q];
            CK(cudaStreamWaitEvent(dst->stream, g->ready[q], 0));
            const size_t off = displ[g->rank0 + q];
            CK(cudaMemcpyPeerAsync(bufs[m] + off, dst->device, bufs[q] + off, src->device, bytes[g->rank0 + q],
                                   dst->stream));
        }
    }
}

// Balanced contiguous split of n_items weighted items over `world` ranks:
// bounds[r] = first item of rank r (bounds[world] = n_items).  cost(i) >= 0.
template <class Cost>
std::vector<int64_t> weighted_split(int64_t n_items, int world, Cost&& cost) {
    std::vector<double> prefix(static_cast<size_t>(n_items) + 1, 0.0);
    for (int64_t i = 0; i < n_items; ++i) prefix[i + 1] = prefix[i] + cost(i);
    const double total = prefix.back();
    std::vector<int64_t> b(static_cast<size_t>(world) + 1, n_items);
    b[0] = 0;
    int64_t i = 0;
    for (int r = 1; r < world; ++r) {
        const double target = total * r / world;
        // first item whose prefix-before is >= target, or the nearer boundary
        while (i < n_items && prefix[i + 1] <= target) ++i;
        int64_t cut = i;
        if (i < n_items && (target - prefix[i]) > (prefix[i + 1] - target)) cut = i + 1;
        b[r] = std::max(b[r - 1], std::min(cut, n_items));
    }
    return b;
}

// ---- sharded observe_ad ------------------------------------------------------
// Units are the (observation, 1024-particle chunk) pairs in observation-major
// order, split into contiguous ranges balanced by particle-steps.  Each rank
// runs the unit-mode K1 over its range and reduces every unit to its exact
// chunk partial (the first K3 pass of reduce_observation's tree,
// executor.cpp:11-26); the exchange assembles [n_obs][chunks] on every rank,
// which finishes the same tree passes, the division (executor.cpp:103), the
// squared-deviation partials of the two-pass variance (:104-112) — exchanged
// the same way — and the estimates.  Bit-identical to one device for any
// split.  Exchange: 2 x n_obs x chunks doubles (C2: 2 x 7 KB).
void group_ad_observe(smc_ctx* ctx, const smc_ad_problem& p, uint64_t seed, int64_t obs_begin, int64_t obs_count,
                      smc_estimate* out) {
    smc_group* g = ctx->group;
    const PreparedVelocity v = prepare_velocity(p.velocity);
    check_kappa(p.kappa);
    check_scalar(p.initial_condition);
    ad_validate(p);
    check_particle_range(p.n_particles);
    const AdImage A = build_ad_image(p, {&v}, v, obs_begin, obs_count);
    const int64_t n = p.n_particles, cpo = smc_num_chunks(n), U = obs_count * cpo;
    const std::vector<int64_t> bounds = weighted_split(U, g->world, [&](int64_t u) {
        const int64_t c = u % cpo;
        return double(A.obs_steps[static_cast<size_t>(u / cpo)]) * double(std::min<int64_t>(kChunk, n - c * kChunk));
    });
    std::vector<size_t> displ(g->world), bytes(g->world);
    for (int r = 0; r < g->world; ++r) {
        displ[r] = static_cast<size_t>(bounds[r]) * sizeof(double);
        bytes[r] = static_cast<size_t>(bounds[r + 1] - bounds[r]) * sizeof(double);
    }
    const int nloc = static_cast<int>(g->members.size());
    std::vector<unsigned char*> ex1(nloc), ex2(nloc);
    std::vector<AdPrepared> prep(nloc);
    std::vector<double*> values(nloc), means(nloc);
    int64_t local_steps = 0;
    // phase 1: particles + chunk partials of the own units
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        const int r = g->rank0 + m;
        const int64_t u0 = bounds[r], nu = bounds[r + 1] - bounds[r];
        CK(cudaSetDevice(c->device));
        c->stats = smc_stats{};
        prep[m] = upload_ad_image(c, A);
        AdLaunch& L = prep[m].L;
        L.seed = seed;
        L.unit_cpo = static_cast<int32_t>(cpo);
        L.unit0 = u0;
        L.p_begin = 0;
        L.p_end = nu * kChunk;
        values[m] = c->values.get<double>(static_cast<size_t>(std::max<int64_t>(nu * kChunk, 1)));
        L.values = values[m];
        ex1[m] = reinterpret_cast<unsigned char*>(c->gx_a.get<double>(static_cast<size_t>(U)));
        ex2[m] = reinterpret_cast<unsigned char*>(c->gx_b.get<double>(static_cast<size_t>(U)));
        CK(cudaEventRecord(c->ev[0], c->stream));
        if (nu > 0) {
            if (cpo > INT32_MAX) raise(SMC_ERUNTIME, "observe_ad: too many particle chunks per observation");
            run_particles(c, L, &prep[m]);
            CK(launch_unit_partials(values[m], nu, u0, cpo, n, nullptr, 0,
                                    reinterpret_cast<double*>(ex1[m]) + u0, c->stream));
            count_launches(c, 1);
        }
        CK(cudaEventRecord(c->ev[1], c->stream));
        for (int64_t u = u0; u < u0 + nu; ++u)
            local_steps += A.obs_steps[static_cast<size_t>(u / cpo)] * std::min<int64_t>(kChunk, n - (u % cpo) * kChunk);
    }
    group_exchange(g, ex1, displ, bytes);
    // phase 2: finish the sums, means, squared-deviation partials
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        const int r = g->rank0 + m;
        const int64_t u0 = bounds[r], nu = bounds[r + 1] - bounds[r];
        CK(cudaSetDevice(c->device));
        double* scratch = c->scratch.get<double>(static_cast<size_t>(2 * obs_count * cpo));
        double* sums = c->sums.get<double>(static_cast<size_t>(obs_count));
        means[m] = c->means.get<double>(static_cast<size_t>(obs_count));
        int launches = 0;
        CK(tree_reduce(reinterpret_cast<double*>(ex1[m]), cpo, nullptr, cpo, obs_count, sums, nullptr, 0, scratch,
                       c->stream, &launches));
        CK(launch_divide(sums, nullptr, n, obs_count, means[m], c->stream));
        if (nu > 0)
            CK(launch_unit_partials(values[m], nu, u0, cpo, n, means[m], 1,
                                    reinterpret_cast<double*>(ex2[m]) + u0, c->stream));
        count_launches(c, launches + 1 + (nu > 0 ? 1 : 0));
    }
    group_exchange(g, ex2, displ, bytes);
    // phase 3: variance, estimates; the owning context copies them out
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        CK(cudaSetDevice(c->device));
        double* scratch = c->scratch.get<double>(static_cast<size_t>(2 * obs_count * cpo));
        double* sumsq = c->sumsq.get<double>(static_cast<size_t>(obs_count));
        smc_estimate* est = c->est.get<smc_estimate>(static_cast<size_t>(obs_count));
        int launches = 0;
        CK(tree_reduce(reinterpret_cast<double*>(ex2[m]), cpo, nullptr, cpo, obs_count, sumsq, nullptr, 0, scratch,
                       c->stream, &launches));
        CK(launch_estimates(means[m], sumsq, nullptr, nullptr, n, n, obs_count, est, c->stream));
        count_launches(c, launches + 1);
        if (m == 0) {
            smc_estimate* h = c->est_host.get<smc_estimate>(static_cast<size_t>(obs_count));
            CK(cudaMemcpyAsync(h, est, sizeof(smc_estimate) * obs_count, cudaMemcpyDeviceToHost, c->stream));
        }
        CK(cudaEventRecord(c->ev[2], c->stream));
    }
    smc_stats agg{};
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->stream));
        finish_stats(c);
        agg.particle_kernel_ms = std::max(agg.particle_kernel_ms, c->stats.particle_kernel_ms);
        agg.reduce_ms = std::max(agg.reduce_ms, c->stats.reduce_ms);
        agg.kernel_launches += c->stats.kernel_launches;
    }
    CK(cudaSetDevice(ctx->device));
    std::memcpy(out, ctx->est_host.p, sizeof(smc_estimate) * obs_count);
    agg.particle_steps = local_steps;
    ctx->stats = agg;
}

// ---- sharded observe_bvp -------------------------------------------------------
// Rank r runs walkers [n r / W, n (r+1) / W) of every observation (their own
// stream keys, so the walkers do not depend on the split) and compacts its
// valid ones.  The reference compacts before its tree (executor.cpp:93-101),
// so a walker's tree position depends on failures on lower ranks: the first
// exchange carries the valid counts (n_obs int64 per rank), after which rank r
// knows its interval [off, off + cnt) of each observation's global compacted
// order and sends the tree sums of that interval's aligned dyadic blocks
// (value and exit time, 64 slots each); every rank merges them into the exact
// roots.  The variance pass sends the blocks of (v - mean)^2.  Exchange:
// n_obs x (8 + 2 x 512 + 512) bytes per rank (C3: 38 KB), bit-identical to
// one device for any split.
void group_bvp_observe(smc_ctx* ctx, const smc_bvp_problem& p, uint64_t seed, int64_t obs_begin, int64_t obs_count,
                       smc_estimate* out) {
    smc_group* g = ctx->group;
    const int W = g->world, nloc = static_cast<int>(g->members.size());
    const int64_t n = p.n_particles, no = obs_count;
    auto range = [&](int r) { return std::make_pair(n * r / W, n * (r + 1) / W); };
    const size_t rec1 = static_cast<size_t>(no) * 2 * kDyadicSlots, rec2 = static_cast<size_t>(no) * kDyadicSlots;
    std::vector<size_t> d0(W), b0(W), d1(W), b1(W), d2(W), b2(W);
    for (int r = 0; r < W; ++r) {
        d0[r] = static_cast<size_t>(r * no) * sizeof(int64_t);
        b0[r] = static_cast<size_t>(no) * sizeof(int64_t);
        d1[r] = r * rec1 * sizeof(double);
        b1[r] = rec1 * sizeof(double);
        d2[r] = r * rec2 * sizeof(double);
        b2[r] = rec2 * sizeof(double);
    }
    std::vector<unsigned char*> ex0(nloc), ex1(nloc), ex2(nloc);
    std::vector<double*> comp(nloc), scr(nloc), sums(nloc), means(nloc);
    std::vector<int64_t*> nvalid(nloc);
    std::vector<unsigned long long*> steps(nloc);
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        const int r = g->rank0 + m;
        const auto [wb, we] = range(r);
        const int64_t span = we - wb;
        CK(cudaSetDevice(c->device));
        c->stats = smc_stats{};
        BvpLaunch L = prepare_bvp(c, p, obs_begin, obs_count);
        L.seed = seed;
        L.n_particles = span;
        L.p_begin = wb;
        ex0[m] = reinterpret_cast<unsigned char*>(c->gx_a.get<int64_t>(static_cast<size_t>(W * no)));
        ex1[m] = reinterpret_cast<unsigned char*>(c->gx_b.get<double>(W * rec1));
        ex2[m] = reinterpret_cast<unsigned char*>(c->gx_c.get<double>(W * rec2));
        int64_t* my_counts = reinterpret_cast<int64_t*>(ex0[m]) + r * no;
        const size_t tot = static_cast<size_t>(std::max<int64_t>(no * span, 1));
        comp[m] = c->tmp_a.get<double>(2 * tot);
        scr[m] = c->tmp_b.get<double>(static_cast<size_t>(no * 2 * (span / kChunk + 1)));
        if (span > 0) {
            run_bvp(c, L, no, span);
            steps[m] = L.step_total;
            int64_t* chunk_tmp = c->chunk_tmp.get<int64_t>(static_cast<size_t>(2 * no * smc_num_chunks(span)));
            CK(compact_valid(L.values, L.aux, L.failed, span, no, comp[m], comp[m] + tot, my_counts, chunk_tmp,
                             c->stream));
            count_launches(c, 3);
        } else {
            steps[m] = nullptr;
            CK(cudaEventRecord(c->ev[0], c->stream));
            CK(cudaEventRecord(c->ev[1], c->stream));
            CK(cudaMemsetAsync(my_counts, 0, sizeof(int64_t) * no, c->stream));
        }
    }
    group_exchange(g, ex0, d0, b0);
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        const int r = g->rank0 + m;
        const auto [wb, we] = range(r);
        const int64_t span = we - wb;
        const size_t tot = static_cast<size_t>(std::max<int64_t>(no * span, 1));
        CK(cudaSetDevice(c->device));
        const int64_t* gcounts = reinterpret_cast<const int64_t*>(ex0[m]);
        CK(launch_dyadic_blocks(comp[m], static_cast<int64_t>(tot), 2, span, gcounts, W, r, no, nullptr, 0,
                                reinterpret_cast<double*>(ex1[m]) + r * rec1, scr[m], span / kChunk + 1, c->stream));
        count_launches(c, 1);
    }
    group_exchange(g, ex1, d1, b1);
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        const int r = g->rank0 + m;
        const auto [wb, we] = range(r);
        const int64_t span = we - wb;
        const size_t tot = static_cast<size_t>(std::max<int64_t>(no * span, 1));
        CK(cudaSetDevice(c->device));
        const int64_t* gcounts = reinterpret_cast<const int64_t*>(ex0[m]);
        sums[m] = c->sums.get<double>(static_cast<size_t>(3 * no));  // value, aux, squared deviation
        means[m] = c->means.get<double>(static_cast<size_t>(no));
        nvalid[m] = c->counts.get<int64_t>(static_cast<size_t>(no));
        CK(launch_dyadic_finish(reinterpret_cast<const double*>(ex1[m]), gcounts, W, no, 2, sums[m], nvalid[m],
                                means[m], c->stream));
        CK(launch_dyadic_blocks(comp[m], static_cast<int64_t>(tot), 1, span, gcounts, W, r, no, means[m], 1,
                                reinterpret_cast<double*>(ex2[m]) + r * rec2, scr[m], span / kChunk + 1, c->stream));
        count_launches(c, 2);
    }
    group_exchange(g, ex2, d2, b2);
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        CK(cudaSetDevice(c->device));
        const int64_t* gcounts = reinterpret_cast<const int64_t*>(ex0[m]);
        CK(launch_dyadic_finish(reinterpret_cast<const double*>(ex2[m]), gcounts, W, no, 1, sums[m] + 2 * no, nullptr,
                                nullptr, c->stream));
        smc_estimate* est = c->est.get<smc_estimate>(static_cast<size_t>(no));
        CK(launch_estimates(means[m], sums[m] + 2 * no, sums[m] + no, nvalid[m], n, n, no, est, c->stream));
        count_launches(c, 2);
        unsigned long long* sh = c->steps_host.get<unsigned long long>(1);
        *sh = 0;
        if (steps[m]) CK(cudaMemcpyAsync(sh, steps[m], sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
        if (m == 0) {
            smc_estimate* h = c->est_host.get<smc_estimate>(static_cast<size_t>(no));
            CK(cudaMemcpyAsync(h, est, sizeof(smc_estimate) * no, cudaMemcpyDeviceToHost, c->stream));
        }
        CK(cudaEventRecord(c->ev[2], c->stream));
    }
    smc_stats agg{};
    for (int m = 0; m < nloc; ++m) {
        smc_ctx* c = g->members[m];
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->stream));
        finish_stats(c);
        agg.particle_kernel_ms = std::max(agg.particle_kernel_ms, c->stats.particle_kernel_ms);
        agg.reduce_ms = std::max(agg.reduce_ms, c->stats.reduce_ms);
        agg.kernel_launches += c->stats.kernel_launches;
        agg.particle_steps += static_cast<int64_t>(*c->steps_host.get<unsigned long long>(1));
    }
    CK(cudaSetDevice(ctx->device));
    ctx->stats = agg;
    const smc_estimate* h = static_cast<const smc_estimate*>(ctx->est_host.p);
    for (int64_t j = 0; j < no; ++j)
        if (h[j].n_failed == n) raise(SMC_ERUNTIME, "map_reduce: every particle of an observation failed");
    std::memcpy(out, h, sizeof(smc_estimate) * no);
}

}  // namespace smc::capi

extern "C" {

smc_status smc_nccl_unique_id(uint8_t* out) {
    return guarded(__func__, [&] {
        const NcclApi* api = need_nccl();
        ncclUniqueId id;
        NK(api, api->GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, &id, sizeof(id));
    });
}

smc_status smc_create_multi(int ndev, const int* devs, smc_ctx** out) {
    return guarded(__func__, [&] {
        *out = nullptr;
        if (ndev < 1 || !devs) raise(SMC_EINVAL, "smc_create_multi: need at least one device");
        smc_ctx* lead = new_member(devs[0]);
        // SMC_GROUP_FORCE=1: a one-device list still becomes a (one-rank NCCL)
        // group, so the sharded path and its NCCL calls run on a single GPU
        const bool force = std::getenv("SMC_GROUP_FORCE") && std::atoi(std::getenv("SMC_GROUP_FORCE")) == 1;
        if (ndev == 1 && !force) {
            *out = lead;
            return;
        }
        auto* g = new smc_group();
        lead->group = g;
        g->world = ndev;
        g->rank0 = 0;
        g->members.push_back(lead);
        try {
            for (int i = 1; i < ndev; ++i) g->members.push_back(new_member(devs[i]));
            bool distinct = true;
            for (int i = 0; i < ndev; ++i)
                for (int j = 0; j < i; ++j) distinct = distinct && devs[i] != devs[j];
            const char* ex = std::getenv("SMC_GROUP_EXCHANGE");
            const bool want_emulated = ex && std::strcmp(ex, "emulated") == 0;
            std::string why;
            const NcclApi* api = (distinct && !want_emulated) ? nccl(&why) : nullptr;
            if (ndev == 1 && !api) raise(SMC_ECUDA, "SMC_GROUP_FORCE: " + why);
            if (api) {
                std::vector<ncclComm_t> comms(static_cast<size_t>(ndev));
                NK(api, api->CommInitAll(comms.data(), ndev, devs), "ncclCommInitAll");
                for (ncclComm_t c : comms) g->comms.push_back(c);
            } else {
                if (distinct && !want_emulated) raise(SMC_ECUDA, why);
                g->ready.resize(static_cast<size_t>(ndev), nullptr);
                for (int i = 0; i < ndev; ++i) {
                    CK(cudaSetDevice(devs[i]));
                    CK(cudaEventCreateWithFlags(&g->ready[i], cudaEventDisableTiming));
                    for (int j = 0; j < ndev; ++j) {
                        int can = 0;
                        if (devs[j] != devs[i] && cudaDeviceCanAccessPeer(&can, devs[i], devs[j]) == cudaSuccess &&
                            can) {
                            const cudaError_t e = cudaDeviceEnablePeerAccess(devs[j], 0);
                            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                            else CK(e);
                        }
                    }
                }
            }
            // Modelling knob (emulated groups on one GPU): SMC_GROUP_SERIAL=1
            // puts every member on the lead's stream, so the members' shards
            // run one after another and each member's particle-kernel time is
            // what one rank of a W-GPU group would see (tools/shard_model.py)
            const char* serial = std::getenv("SMC_GROUP_SERIAL");
            if (!api && serial && std::atoi(serial) == 1)
                for (int i = 1; i < ndev; ++i)
                    if (devs[i] == devs[0]) g->members[i]->stream = lead->stream;
            CK(cudaSetDevice(devs[0]));
        } catch (...) {
            smc_destroy(lead);
            throw;
        }
        *out = lead;
    });
}

smc_status smc_create_rank(int device, int rank, int world, const uint8_t* unique_id, smc_ctx** out) {
    return guarded(__func__, [&] {
        *out = nullptr;
        if (world < 1 || rank < 0 || rank >= world) raise(SMC_EINVAL, "smc_create_rank: rank out of range");
        smc_ctx* c = new_member(device);
        const bool force = std::getenv("SMC_GROUP_FORCE") && std::atoi(std::getenv("SMC_GROUP_FORCE")) == 1;
        if (world == 1 && !(force && unique_id)) {
            *out = c;
            return;
        }
        try {
            if (!unique_id) raise(SMC_EINVAL, "smc_create_rank: unique id required for world > 1");
            const NcclApi* api = need_nccl();
            ncclUniqueId id;
            std::memcpy(&id, unique_id, sizeof(id));
            CK(cudaSetDevice(device));
            ncclComm_t comm = nullptr;
            NK(api, api->CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
            auto* g = new smc_group();
            c->group = g;
            g->world = world;
            g->rank0 = rank;
            g->members.push_back(c);
            g->comms.push_back(comm);
        } catch (...) {
            smc_destroy(c);
            throw;
        }
        *out = c;
    });
}

smc_status smc_create_rank_hosted(int device, int rank, int world, smc_exchange_fn exchange, void* user,
                                  smc_ctx** out) {
    return guarded(__func__, [&] {
        *out = nullptr;
        if (world < 1 || rank < 0 || rank >= world) raise(SMC_EINVAL, "smc_create_rank: rank out of range");
        if (!exchange) raise(SMC_EINVAL, "smc_create_rank_hosted: exchange callback required");
        smc_ctx* c = new_member(device);
        if (world == 1) {
            *out = c;
            return;
        }
        auto* g = new smc_group();
        c->group = g;
        g->world = world;
        g->rank0 = rank;
        g->members.push_back(c);
        g->hook = exchange;
        g->hook_user = user;
        *out = c;
    });
}

smc_status smc_group_query(smc_ctx* ctx, smc_group_desc* out) {
    return guarded(__func__, [&] {
        out->world = ctx->group ? ctx->group->world : 1;
        out->rank = ctx->group ? ctx->group->rank0 : 0;
        out->n_local = ctx->group ? static_cast<int32_t>(ctx->group->members.size()) : 1;
        out->nccl = (ctx->group && !ctx->group->comms.empty()) ? 1 : 0;
        for (int i = 0; i < 8; ++i) out->devices[i] = -1;
        if (ctx->group) {
            for (size_t i = 0; i < ctx->group->members.size() && i < 8; ++i)
                out->devices[i] = ctx->group->members[i]->device;
        } else {
            out->devices[0] = ctx->device;
        }
    });
}

}  // extern "C"
