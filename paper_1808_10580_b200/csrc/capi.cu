// capi.cu — the C ABI (include/scalarmc_b200.h): context, device-image
// upload, kernel orchestration and host result return.
//
// One smc_ctx per process per GPU.  A forward-map call is: validate (host, the
// reference's messages) -> pack one image (velocity lattice, theta_0 terms,
// per-observation step schedules) into pinned staging -> one H2D copy -> K1
// particle kernel -> K3 tree reduction passes -> estimates kernel -> one D2H
// copy of n_obs x 40 B.  All on the context's stream; persistent buffers grow
// and are reused across calls.
#include <mutex>
#include <set>

#include "capi_internal.h"

using namespace smc;
using namespace smc::capi;

namespace smc::capi {

thread_local std::string g_err;

// ---- guard zones (SMC_GUARD=1) ----------------------------------------------
namespace {
std::mutex g_guard_mu;
std::set<DevBuf*>& guard_registry() {
    static std::set<DevBuf*> r;
    return r;
}
}  // namespace

bool guard_mode() {
    static const bool on = [] {
        const char* e = std::getenv("SMC_GUARD");
        return e && *e && std::strcmp(e, "0") != 0;
    }();
    return on;
}

void DevBuf::allocate_guarded(size_t bytes) {
    CK(cudaGetDevice(&device));
    void* b = nullptr;
    CK(cudaMalloc(&b, bytes + 2 * kGuardBytes));
    base = static_cast<unsigned char*>(b);
    p = base + kGuardBytes;
    // the zones must hold the pattern before any stream writes: fill them on a
    // private non-blocking stream and wait for it (not a device-wide sync,
    // which another member thread's CUDA-graph capture would reject)
    cudaStream_t fs = nullptr;
    CK(cudaStreamCreateWithFlags(&fs, cudaStreamNonBlocking));
    const cudaError_t e1 = cudaMemsetAsync(base, kGuardByte, kGuardBytes, fs);
    const cudaError_t e2 = cudaMemsetAsync(base + kGuardBytes + bytes, kGuardByte, kGuardBytes, fs);
    const cudaError_t e3 = cudaStreamSynchronize(fs);
    cudaStreamDestroy(fs);
    CK(e1);
    CK(e2);
    CK(e3);
    std::lock_guard<std::mutex> lk(g_guard_mu);
    guard_registry().insert(this);
}

void DevBuf::release() {
    if (base) {
        {
            std::lock_guard<std::mutex> lk(g_guard_mu);
            guard_registry().erase(this);
        }
        cudaFree(base);
    } else if (p) {
        cudaFree(p);
    }
    p = nullptr;
    base = nullptr;
    cap = 0;
}

void guard_check(const char* entry) {
    std::lock_guard<std::mutex> lk(g_guard_mu);
    int prev = 0;
    CK(cudaGetDevice(&prev));
    std::vector<unsigned char> h(kGuardBytes);
    std::set<int> synced;
    for (DevBuf* b : guard_registry()) {
        if (!synced.count(b->device)) {
            CK(cudaSetDevice(b->device));
            CK(cudaDeviceSynchronize());
            synced.insert(b->device);
        }
        CK(cudaSetDevice(b->device));
        for (int side = 0; side < 2; ++side) {
            const unsigned char* z = side == 0 ? b->base : b->base + kGuardBytes + b->cap;
            CK(cudaMemcpy(h.data(), z, kGuardBytes, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < kGuardBytes; ++i) {
                if (h[i] != kGuardByte) {
                    // re-arm the zone: the violation is reported once, by this call
                    cudaMemset(const_cast<unsigned char*>(z), kGuardByte, kGuardBytes);
                    cudaDeviceSynchronize();
                    cudaSetDevice(prev);
                    std::ostringstream os;
                    os << entry << ": device buffer overrun — guard zone " << (side == 0 ? "before" : "after")
                       << " a " << b->cap << "-byte buffer on device " << b->device << " overwritten at byte "
                       << (side == 0 ? static_cast<long long>(i) - static_cast<long long>(kGuardBytes)
                                     : static_cast<long long>(b->cap + i));
                    raise(SMC_ERUNTIME, os.str());
                }
            }
        }
    }
    CK(cudaSetDevice(prev));
}


void count_launches(smc_ctx* ctx, int64_t n) {
    ctx->stats.kernel_launches += n;
    ctx->total_launches += n;
}



ScalarRef add_scalar(Image& im, const smc_scalar_field& f) {
    check_scalar(f);
    ScalarRef r;
    r.img.kind = f.kind;
    r.img.n = f.n_terms;
    r.img.constant = f.constant;
    r.img.g0 = f.gradient[0];
    r.img.g1 = f.gradient[1];
    r.img.neg_sharpness = -f.sharpness;
    const size_t n = static_cast<size_t>(f.n_terms);
    if (f.kind == SMC_SCALAR_COSINE && n) {
        r.amp = im.add(f.amplitude, n * sizeof(double));
        r.freq = im.add(f.freq, 2 * n * sizeof(double));
        r.phase = im.add(f.phase, n * sizeof(double));
    } else if (f.kind == SMC_SCALAR_BUMPS && n) {
        r.amp = im.add(f.amplitude, n * sizeof(double));
        r.center = im.add(f.center, 2 * n * sizeof(double));
    } else {
        r.img.n = (f.kind == SMC_SCALAR_COSINE || f.kind == SMC_SCALAR_BUMPS) ? 0 : r.img.n;
    }
    return r;
}

ScalarImg patch(const ScalarRef& r, unsigned char* base) {
    ScalarImg s = r.img;
    s.amp = reinterpret_cast<const double*>(base + r.amp);
    s.freq = reinterpret_cast<const double*>(base + r.freq);
    s.phase = reinterpret_cast<const double*>(base + r.phase);
    s.center = reinterpret_cast<const double*>(base + r.center);
    return s;
}



// Velocity image: strict mode list + tiled lattice structure + one
// coefficient block per sample (fills[i] for sample i).
VelRef add_velocity(Image& im, const PreparedVelocity& v, const std::vector<const PreparedVelocity*>& fills) {
    VelRef r;
    r.img.is_constant = v.is_constant ? 1 : 0;
    r.img.c1 = v.c1;
    r.img.c2 = v.c2;
    r.img.K = v.K;
    r.img.n_modes = static_cast<int32_t>(v.modes.size());
    if (v.is_constant) return r;
    std::vector<ModeImg> modes;
    modes.reserve(v.modes.size());
    for (const auto& m : v.modes) {
        const double kn = std::sqrt(double(m.k1) * m.k1 + double(m.k2) * m.k2);  // fields.cpp:66
        modes.push_back(ModeImg{m.k1, m.k2, m.re, m.im, -double(m.k2) / kn, double(m.k1) / kn});
    }
    r.modes = im.add_vec(modes);
    const LatticeHost L = lattice_structure(v);
    r.tiles = im.add_vec(L.tiles);
    r.coefs = im.reserve(static_cast<size_t>(L.stride) * fills.size() * sizeof(double));
    for (size_t b = 0; b < fills.size(); ++b)
        lattice_fill(L, *fills[b], reinterpret_cast<double*>(im.bytes.data() + r.coefs) + b * L.stride);
    LatticeImg& li = r.img.lat;
    li.sample_stride = L.stride;
    li.K = L.K;
    li.R = L.R;
    li.J0 = L.J0;
    li.n_tiles = L.n_tiles;
    li.row0_off = static_cast<int32_t>(L.row0_off);
    li.g0_off = static_cast<int32_t>(L.g0_off);
    return r;
}

VelImg patch(const VelRef& r, unsigned char* base) {
    VelImg v = r.img;
    if (v.is_constant) return v;
    v.modes = reinterpret_cast<const ModeImg*>(base + r.modes);
    v.lat.tiles = reinterpret_cast<const int2*>(base + r.tiles);
    v.lat.coef = reinterpret_cast<const double*>(base + r.coefs);
    return v;
}



void check_particle_range(int64_t n_particles) {
    // Stream keys carry the particle index in 32 bits (rng.cpp:46-47); the
    // reference's work lambda throws and map_reduce reports it.
    if (n_particles > (int64_t(1) << 32)) raise(SMC_ERUNTIME, "map_reduce: a particle work function threw");
}

AdImage build_ad_image(const smc_ad_problem& p, const std::vector<const PreparedVelocity*>& fills,
                       const PreparedVelocity& structure, int64_t obs_begin, int64_t obs_count) {
    const double dt = ad_resolved_dt(p);
    AdImage A;
    A.sigma = std::sqrt(2.0 * p.kappa);
    Image& im = A.im;
    std::vector<AdObsImg> obs;
    for (int64_t j = obs_begin; j < obs_begin + obs_count; ++j) {
        obs.push_back(make_ad_obs(p.obs_t[j], p.obs_x[2 * j], p.obs_x[2 * j + 1], dt, A.sigma));
        A.steps_per_particle_sum += obs.back().n_steps;
        A.obs_steps.push_back(obs.back().n_steps);
    }
    A.obs_off = im.add_vec(obs);
    // batched launches schedule the longest observations first (grid z), so
    // the short ones fill the tail instead of a long one trailing alone
    std::vector<int32_t> order(obs.size());
    for (size_t j = 0; j < order.size(); ++j) order[j] = static_cast<int32_t>(j);
    if (std::getenv("SMC_NO_LPT") == nullptr)
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t a, int32_t b) { return obs[a].n_steps > obs[b].n_steps; });
    A.order_off = im.add_vec(order);
    A.th = add_scalar(im, p.initial_condition);
    A.vr = add_velocity(im, structure, fills);
    // Dense fields with a compile-time disk kernel for their K take it
    // (K <= kDiskMaxK; FP64 also the tiled disk kernels' K).
    const bool disk = !structure.is_constant && p.precision != SMC_FP64_STRICT &&
                      disk_kernel_for(structure.K, p.precision == SMC_FP64) &&
                      2 * structure.modes.size() >= static_cast<size_t>(disk_n_modes(structure.K)) &&
                      std::getenv("SMC_DISABLE_DISK") == nullptr;
    if (disk) {
        const size_t nc = static_cast<size_t>(disk_n_coef(structure.K));
        A.disk_off = im.reserve(nc * fills.size() * sizeof(double));
        for (size_t b = 0; b < fills.size(); ++b)
            disk_fill(structure.K, *fills[b], reinterpret_cast<double*>(im.bytes.data() + A.disk_off) + b * nc);
        if (fills.size() == 1) {
            const double* h = reinterpret_cast<const double*>(im.bytes.data() + A.disk_off);
            A.host_disk.assign(h, h + nc);
        }
        A.disk_K = structure.K;
    }
    A.obs_begin = obs_begin;
    A.obs_count = obs_count;
    A.n_particles = p.n_particles;
    A.precision = p.precision;
    return A;
}

AdPrepared upload_ad_image(smc_ctx* ctx, const AdImage& A) {
    AdPrepared out;
    unsigned char* base = ctx->upload(A.im);
    out.host_disk = A.host_disk;
    if (A.disk_K > 0) {
        out.disk_K = A.disk_K;
        out.disk = reinterpret_cast<const double*>(base + A.disk_off);
    }
    out.steps_per_particle_sum = A.steps_per_particle_sum;
    AdLaunch& L = out.L;
    L.vel = patch(A.vr, base);
    L.theta0 = patch(A.th, base);
    L.obs = reinterpret_cast<const AdObsImg*>(base + A.obs_off);
    L.obs_order = reinterpret_cast<const int32_t*>(base + A.order_off);
    L.n_obs = static_cast<int32_t>(A.obs_count);
    L.obs_slot0 = static_cast<uint32_t>(A.obs_begin);
    L.n_particles = A.n_particles;
    L.p_begin = 0;
    L.p_end = A.n_particles;
    L.n_samples = 1;
    L.precision = A.precision;
    L.sigma = A.sigma;
    L.host_disk = out.host_disk.empty() ? nullptr : out.host_disk.data();
    out.n_obs = A.obs_count;
    return out;
}

AdPrepared prepare_ad(smc_ctx* ctx, const smc_ad_problem& p, const std::vector<const PreparedVelocity*>& fills,
                      const PreparedVelocity& structure, int64_t obs_begin, int64_t obs_count) {
    return upload_ad_image(ctx, build_ad_image(p, fills, structure, obs_begin, obs_count));
}

void run_particles(smc_ctx* ctx, AdLaunch& L, const AdPrepared* P, int64_t sample0) {
    if (P && P->disk_K > 0) {
        CK(launch_ad_disk(L, P->disk_K, P->disk + sample0 * disk_n_coef(P->disk_K), ctx->stream));
    } else if (L.precision == SMC_FP64_STRICT) {
        if (L.n_samples != 1) raise(SMC_EINVAL, "strict precision is single-sample only");
        if (!L.vel.is_constant && L.vel.K > 128) raise(SMC_EINVAL, "strict precision supports max_wavenumber <= 128");
        CK(launch_ad_particles_strict(L, ctx->stream));
    } else if (L.precision == SMC_FP32) {
        CK(launch_ad_particles_fp32(L, ctx->stream));
    } else {
        CK(launch_ad_particles(L, ctx->stream));
    }
    count_launches(ctx, 1);
}

// Reduce [n_seg][n] values (no failures) into estimates on the host.
// Reduce [n_seg][n] values (no failures) into estimates left on the device.
smc_estimate* reduce_ad_device(smc_ctx* ctx, const double* values, int64_t n, int64_t n_seg) {
    cudaStream_t s = ctx->stream;
    const int64_t chunks = (n + kChunk - 1) / kChunk;
    double* scratch = ctx->scratch.get<double>(static_cast<size_t>(2 * n_seg * std::max<int64_t>(chunks, 1)));
    double* sums = ctx->sums.get<double>(static_cast<size_t>(n_seg));
    double* means = ctx->means.get<double>(static_cast<size_t>(n_seg));
    double* sumsq = ctx->sumsq.get<double>(static_cast<size_t>(n_seg));
    smc_estimate* est = ctx->est.get<smc_estimate>(static_cast<size_t>(n_seg));
    int launches = 0;
    CK(tree_reduce(values, n, nullptr, n, n_seg, sums, nullptr, 0, scratch, s, &launches));
    CK(launch_divide(sums, nullptr, n, n_seg, means, s));
    CK(tree_reduce(values, n, nullptr, n, n_seg, sumsq, means, 1, scratch, s, &launches));
    CK(launch_estimates(means, sumsq, nullptr, nullptr, n, n, n_seg, est, s));
    count_launches(ctx, launches + 2);
    return est;
}

void reduce_ad(smc_ctx* ctx, const double* values, int64_t n, int64_t n_seg, smc_estimate* out) {
    cudaStream_t s = ctx->stream;
    const int64_t chunks = (n + kChunk - 1) / kChunk;
    double* scratch = ctx->scratch.get<double>(static_cast<size_t>(2 * n_seg * std::max<int64_t>(chunks, 1)));
    double* sums = ctx->sums.get<double>(static_cast<size_t>(n_seg));
    double* means = ctx->means.get<double>(static_cast<size_t>(n_seg));
    double* sumsq = ctx->sumsq.get<double>(static_cast<size_t>(n_seg));
    smc_estimate* est = ctx->est.get<smc_estimate>(static_cast<size_t>(n_seg));
    int launches = 0;
    CK(tree_reduce(values, n, nullptr, n, n_seg, sums, nullptr, 0, scratch, s, &launches));
    CK(launch_divide(sums, nullptr, n, n_seg, means, s));
    CK(tree_reduce(values, n, nullptr, n, n_seg, sumsq, means, 1, scratch, s, &launches));
    CK(launch_estimates(means, sumsq, nullptr, nullptr, n, n, n_seg, est, s));
    count_launches(ctx, launches + 2);
    smc_estimate* h = ctx->est_host.get<smc_estimate>(static_cast<size_t>(n_seg));
    CK(cudaMemcpyAsync(h, est, sizeof(smc_estimate) * n_seg, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(ctx->ev[2], s));
    CK(cudaStreamSynchronize(s));
    std::memcpy(out, h, sizeof(smc_estimate) * n_seg);
}

void finish_stats(smc_ctx* ctx) {
    float a = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]));
    CK(cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]));
    ctx->stats.particle_kernel_ms = a;
    ctx->stats.reduce_ms = b;
}

void ad_observe_range(smc_ctx* ctx, const smc_ad_problem& p, uint64_t seed, int64_t obs_begin, int64_t obs_count,
                      smc_estimate* out) {
    const PreparedVelocity v = prepare_velocity(p.velocity);
    check_kappa(p.kappa);
    check_scalar(p.initial_condition);
    ad_validate(p);
    check_particle_range(p.n_particles);
    smc_stats total{};
    // observations index a grid dimension (<= 65535 per launch); larger sets
    // run in chunks — each observation's estimate depends only on its own
    // slot, so chunking does not change results
    constexpr int64_t kMaxObsPerLaunch = 65535;
    for (int64_t b = obs_begin; b < obs_begin + obs_count; b += kMaxObsPerLaunch) {
        const int64_t cnt = std::min(kMaxObsPerLaunch, obs_begin + obs_count - b);
        ctx->stats = smc_stats{};
        AdPrepared P = prepare_ad(ctx, p, {&v}, v, b, cnt);
        P.L.seed = seed;
        const int64_t n = p.n_particles;
        P.L.values = ctx->values.get<double>(static_cast<size_t>(cnt * n));
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        run_particles(ctx, P.L, &P);
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        reduce_ad(ctx, P.L.values, n, cnt, out + (b - obs_begin));
        finish_stats(ctx);
        total.particle_kernel_ms += ctx->stats.particle_kernel_ms;
        total.reduce_ms += ctx->stats.reduce_ms;
        total.kernel_launches += ctx->stats.kernel_launches;
        total.particle_steps += P.steps_per_particle_sum * n;
    }
    ctx->stats = total;
}

// True when every Gaussian-bump exponent -a |x - c_j|^2 the walkers can form
// lies in [-700, 0] (fm::exp_bump's domain, with margin): a >= 0 and a times
// the largest squared distance from any bump centre to the bounding box of
// the domain and the launched observation points is at most 700.  Walkers
// only ever sit at their start point or at an accepted step inside the domain.
static bool bump_exp_range_ok(const smc_bvp_problem& p, int64_t obs_begin, int64_t obs_count) {
    const smc_scalar_field& f = p.forcing;
    if (f.kind != SMC_SCALAR_BUMPS || f.n_terms < 1 || f.center == nullptr) return false;
    double lo[2], hi[2];
    if (p.domain.kind == 1) {
        for (int a = 0; a < 2; ++a) lo[a] = p.domain.lower[a], hi[a] = p.domain.upper[a];
    } else if (p.domain.kind == 2) {
        for (int a = 0; a < 2; ++a) lo[a] = p.domain.center[a] - p.domain.radius, hi[a] = p.domain.center[a] + p.domain.radius;
    } else {
        return false;
    }
    for (int64_t o = obs_begin; o < obs_begin + obs_count; ++o)
        for (int a = 0; a < 2; ++a) lo[a] = std::min(lo[a], p.obs_x[2 * o + a]), hi[a] = std::max(hi[a], p.obs_x[2 * o + a]);
    if (!(f.sharpness >= 0.0)) return false;
    for (int j = 0; j < f.n_terms; ++j) {
        double d2 = 0.0;
        for (int a = 0; a < 2; ++a) {
            const double c = f.center[2 * j + a];
            const double m = std::max(std::fabs(lo[a] - c), std::fabs(hi[a] - c));
            d2 += m * m;
        }
        if (!(f.sharpness * d2 <= 700.0)) return false;
    }
    return true;
}

BvpLaunch prepare_bvp(smc_ctx* ctx, const smc_bvp_problem& p, int64_t obs_begin, int64_t obs_count) {
    const PreparedVelocity v = prepare_velocity(p.velocity);
    check_kappa(p.kappa);
    check_scalar(p.forcing);
    check_scalar(p.boundary_data);
    check_domain(p.domain);
    bvp_validate(p);
    check_particle_range(p.n_particles);
    const double dt = bvp_resolved_dt(p, v);
    Image im;
    const size_t obs_off = im.add(p.obs_x + 2 * obs_begin, static_cast<size_t>(2 * obs_count) * sizeof(double));
    const ScalarRef fr = add_scalar(im, p.forcing);
    const ScalarRef br = add_scalar(im, p.boundary_data);
    const VelRef vr = add_velocity(im, v, {&v});
    // dense Fourier fields on |k| <= 12: the compile-time disk series (as K1)
    const bool disk = !v.is_constant && p.precision == SMC_FP64 && v.K <= kDiskMaxK &&
                      2 * v.modes.size() >= static_cast<size_t>(disk_n_modes(v.K)) &&
                      std::getenv("SMC_DISABLE_DISK") == nullptr;
    size_t disk_off = 0;
    if (disk) {
        disk_off = im.reserve(static_cast<size_t>(disk_n_coef(v.K)) * sizeof(double));
        disk_fill(v.K, v, reinterpret_cast<double*>(im.bytes.data() + disk_off));
    }
    unsigned char* base = ctx->upload(im);
    BvpLaunch L{};
    if (disk) {
        L.disk_K = v.K;
        L.disk_coef = reinterpret_cast<const double*>(base + disk_off);
    }
    L.vel = patch(vr, base);
    L.forcing = patch(fr, base);
    L.boundary = patch(br, base);
    DomainImg& d = L.domain;
    d.kind = p.domain.kind;
    d.lo1 = p.domain.lower[0];
    d.lo2 = p.domain.lower[1];
    d.hi1 = p.domain.upper[0];
    d.hi2 = p.domain.upper[1];
    d.c1 = p.domain.center[0];
    d.c2 = p.domain.center[1];
    d.r = p.domain.radius;
    d.r2 = p.domain.radius * p.domain.radius;
    L.obs_x = reinterpret_cast<const double*>(base + obs_off);
    L.n_obs = static_cast<int32_t>(obs_count);
    L.obs_slot0 = static_cast<uint32_t>(obs_begin);
    L.n_particles = p.n_particles;
    L.max_steps = p.max_steps;
    L.dt = dt;
    L.sigma = std::sqrt(2.0 * p.kappa);
    L.root_dt = std::sqrt(dt);
    L.sr = L.sigma * L.root_dt;
    L.precision = p.precision;
    L.bump_exp_ok = bump_exp_range_ok(p, obs_begin, obs_count) ? 1 : 0;
    return L;
}

void run_bvp(smc_ctx* ctx, BvpLaunch& L, int64_t n_obs, int64_t n) {
    cudaStream_t s = ctx->stream;
    const size_t total = static_cast<size_t>(n_obs * n);
    L.values = ctx->values.get<double>(total);
    L.aux = ctx->aux.get<double>(total);
    L.failed = ctx->flags.get<uint8_t>(total);
    // walker-queue head + step total; ctx->counts is reused for the valid
    // counts only after the kernel has finished with these.
    unsigned long long* ctr = ctx->flags2.get<unsigned long long>(2);
    CK(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), s));
    L.counter = ctr;
    L.step_total = ctr + 1;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    CK(cudaEventRecord(ctx->ev[0], s));
    if (L.precision == SMC_FP64_STRICT) {
        if (!L.vel.is_constant && L.vel.K > 128) raise(SMC_EINVAL, "strict precision supports max_wavenumber <= 128");
        CK(launch_bvp_walkers_strict(L, sms, s));
    } else {
        CK(launch_bvp_walkers(L, sms, s));
    }
    count_launches(ctx, 1);
    CK(cudaEventRecord(ctx->ev[1], s));
}


// Upload a PackMap into the context's pack buffers (reused across calls).
PackDev upload_pack_map(smc_ctx* ctx, const PackMap& m) {
    const size_t n = static_cast<size_t>(m.stride);
    auto* ip = ctx->pk_ip.get<int32_t>(n);
    auto* im = ctx->pk_im.get<int32_t>(n);
    auto* kp = ctx->pk_kp.get<double>(n);
    auto* km = ctx->pk_km.get<double>(n);
    auto* ms = ctx->pk_ms.get<int8_t>(n);
    CK(cudaMemcpyAsync(ip, m.ip.data(), 4 * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(im, m.im.data(), 4 * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(kp, m.kp.data(), 8 * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(km, m.km.data(), 8 * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ms, m.ms.data(), n, cudaMemcpyHostToDevice, ctx->stream));
    return PackDev{m.stride, ip, im, kp, km, ms};
}

}  // namespace smc::capi

extern "C" {

int smc_abi_version(void) { return SMC_ABI_VERSION; }

const char* smc_last_error(void) { return g_err.c_str(); }

smc_status smc_create(int device, smc_ctx** out) {
    return guarded(__func__, [&] {
        *out = nullptr;
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) raise(SMC_ECUDA, "smc_create: no such CUDA device");
        CK(cudaSetDevice(device));
        auto* c = new smc_ctx();
        c->device = device;
        CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
        *out = c;
    });
}

void smc_destroy(smc_ctx* ctx) {
    if (!ctx) return;
    if (ctx->group) group_destroy(ctx);  // the other members and the communicators
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;  // every DevBuf / PinnedBuf member frees itself (RAII)
}

void* smc_stream(smc_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

smc_status smc_set_stream(smc_ctx* ctx, void* stream) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    });
}

smc_status smc_ad_resolved_dt(const smc_ad_problem* p, double* out) {
    return guarded(__func__, [&] { *out = ad_resolved_dt(*p); });
}

smc_status smc_bvp_resolved_dt(const smc_bvp_problem* p, double* out) {
    return guarded(__func__, [&] {
        const PreparedVelocity v = prepare_velocity(p->velocity);
        *out = bvp_resolved_dt(*p, v);
    });
}

smc_status smc_velocity_validate(const smc_velocity* v) {
    return guarded(__func__, [&] { (void)prepare_velocity(*v); });
}

smc_status smc_ad_validate(const smc_ad_problem* p) {
    return guarded(__func__, [&] {
        (void)prepare_velocity(p->velocity);
        check_kappa(p->kappa);
        check_scalar(p->initial_condition);
        ad_validate(*p);
    });
}

smc_status smc_bvp_validate(const smc_bvp_problem* p) {
    return guarded(__func__, [&] {
        (void)prepare_velocity(p->velocity);
        check_kappa(p->kappa);
        check_scalar(p->forcing);
        check_scalar(p->boundary_data);
        check_domain(p->domain);
        bvp_validate(*p);
    });
}

int smc_struct_sizes(int64_t* out, int cap) {
    const int64_t s[] = {sizeof(smc_estimate), sizeof(smc_scalar_field), sizeof(smc_velocity),
                         sizeof(smc_ad_problem), sizeof(smc_domain), sizeof(smc_bvp_problem),
                         sizeof(smc_prior), sizeof(smc_stats)};
    const int n = static_cast<int>(sizeof(s) / sizeof(s[0]));
    for (int i = 0; i < n && i < cap; ++i) out[i] = s[i];
    return n;
}

int64_t smc_num_chunks(int64_t n_particles) { return (n_particles + kChunk - 1) / kChunk; }

smc_status smc_ad_observe(smc_ctx* ctx, const smc_ad_problem* p, uint64_t seed, smc_estimate* out) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        if (is_sharded(ctx)) group_ad_observe(ctx, *p, seed, 0, p->n_obs, out);
        else ad_observe_range(ctx, *p, seed, 0, p->n_obs, out);
    });
}

smc_status smc_ad_observe_single(smc_ctx* ctx, const smc_ad_problem* p, uint64_t obs_index, uint64_t seed,
                                 smc_estimate* out) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        // observe_ad_single validates first, then range-checks (forward_ad.cpp:64-67).
        (void)prepare_velocity(p->velocity);
        check_kappa(p->kappa);
        check_scalar(p->initial_condition);
        ad_validate(*p);
        if (obs_index >= static_cast<uint64_t>(p->n_obs))
            raise(SMC_ERANGE, "observe_ad_single: observation index out of range");
        if (is_sharded(ctx)) group_ad_observe(ctx, *p, seed, static_cast<int64_t>(obs_index), 1, out);
        else ad_observe_range(ctx, *p, seed, static_cast<int64_t>(obs_index), 1, out);
    });
}

smc_status smc_ad_particle_values(smc_ctx* ctx, const smc_ad_problem* p, uint64_t obs_index, uint64_t seed,
                                  int64_t n, double* out) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        const PreparedVelocity v = prepare_velocity(p->velocity);
        check_kappa(p->kappa);
        check_scalar(p->initial_condition);
        ad_validate(*p);
        if (obs_index >= static_cast<uint64_t>(p->n_obs)) raise(SMC_ERANGE, "observation index out of range");
        AdPrepared P = prepare_ad(ctx, *p, {&v}, v, static_cast<int64_t>(obs_index), 1);
        P.L.seed = seed;
        P.L.p_end = n;
        P.L.values = ctx->values.get<double>(static_cast<size_t>(n));
        run_particles(ctx, P.L, &P);
        CK(cudaMemcpyAsync(out, P.L.values, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

smc_status smc_philox_device(smc_ctx* ctx, int64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        uint32_t* dc = ctx->tmp_a.get<uint32_t>(static_cast<size_t>(4 * n));
        uint32_t* dk = ctx->tmp_b.get<uint32_t>(static_cast<size_t>(2 * n));
        uint32_t* dout = ctx->tmp_c.get<uint32_t>(static_cast<size_t>(4 * n));
        CK(cudaMemcpyAsync(dc, ctr, 16 * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(dk, key, 8 * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(launch_philox(n, dc, dk, dout, ctx->stream));
        CK(cudaMemcpyAsync(out, dout, 16 * n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

smc_status smc_normal_pairs_device(smc_ctx* ctx, uint64_t seed, uint64_t obs, uint64_t particle, int64_t n_blocks,
                                   double* out) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        if (obs > 0xFFFFFFFFull || particle > 0xFFFFFFFFull)
            raise(SMC_EINVAL, "StreamKey: obs/particle index exceeds 32-bit stream space");
        double* d = ctx->tmp_a.get<double>(static_cast<size_t>(2 * n_blocks));
        CK(launch_normal_pairs(seed, static_cast<uint32_t>(obs), static_cast<uint32_t>(particle), n_blocks, d,
                               ctx->stream));
        CK(cudaMemcpyAsync(out, d, 16 * n_blocks, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

smc_status smc_last_stats(smc_ctx* ctx, smc_stats* out) {
    return guarded(__func__, [&] {
        *out = ctx->stats;
        out->total_launches = ctx->total_launches;
    });
}

namespace {
// Runs the DFMA (fp64) or FFMA peak kernel over all SMs for about `ms`.
double fma_peak(smc_ctx* ctx, double ms, bool fp64) {
    CK(cudaSetDevice(ctx->device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const int blocks = sms * 8;
    double* sink = ctx->tmp_a.get<double>(static_cast<size_t>(blocks));
    int iters = 4096;
    float t = 0.f;
    for (int attempt = 0; attempt < 8; ++attempt) {
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        CK(fp64 ? launch_dfma_peak(blocks, iters, sink, ctx->stream) : launch_ffma_peak(blocks, iters, sink, ctx->stream));
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        CK(cudaEventSynchronize(ctx->ev[1]));
        CK(cudaEventElapsedTime(&t, ctx->ev[0], ctx->ev[1]));
        if (t >= 0.9 * ms) break;
        const double scale = std::min(64.0, std::max(2.0, ms / std::max<double>(t, 1e-3)));
        iters = static_cast<int>(std::min<double>(iters * scale, 1 << 30));
    }
    const double flops = 2.0 * 8.0 * double(iters) * 256.0 * blocks;
    return flops / (double(t) * 1e-3) / 1e12;
}
}  // namespace

smc_status smc_fp32_peak(smc_ctx* ctx, double ms, double* tflops) {
    return guarded(__func__, [&] { *tflops = fma_peak(ctx, ms, false); });
}

smc_status smc_fp64_peak(smc_ctx* ctx, double ms, double* tflops) {
    return guarded(__func__, [&] { *tflops = fma_peak(ctx, ms, true); });
}

smc_status smc_guard_selftest(smc_ctx* ctx, int64_t offset, int64_t nbytes) {
    return guarded(__func__, [&] {
        if (!guard_mode()) raise(SMC_EINVAL, "smc_guard_selftest: guard mode is off (set SMC_GUARD=1)");
        if (nbytes < 0 || offset < -static_cast<int64_t>(kGuardBytes) ||
            offset + nbytes > static_cast<int64_t>(1024 + kGuardBytes))
            raise(SMC_EINVAL, "smc_guard_selftest: the write must stay within the guard zones");
        CK(cudaSetDevice(ctx->device));
        unsigned char* b = ctx->guard_probe.get<unsigned char>(1024);
        CK(cudaMemsetAsync(b + offset, 0, static_cast<size_t>(nbytes), ctx->stream));
    });
}

smc_status smc_bvp_observe(smc_ctx* ctx, const smc_bvp_problem* p, uint64_t seed, smc_estimate* out) {
    return smc_bvp_observe_range(ctx, p, seed, 0, p->n_obs, out);
}

// reduce_observation for every observation of [n_obs][n] walker results on
// the device (executor.cpp:87-117): stable compaction of the valid walkers,
// then the same trees as AD; estimates to the host.  step_total (device,
// optional): the walker-step counter to report in the stats.
static void reduce_bvp(smc_ctx* ctx, const double* values, const double* aux, const uint8_t* failed, int64_t n,
                       int64_t n_obs, const unsigned long long* step_total, smc_estimate* out) {
    cudaStream_t s = ctx->stream;
    const int64_t chunks = smc_num_chunks(n);
    double* cvalues = ctx->tmp_a.get<double>(static_cast<size_t>(n_obs * n));
    double* caux = ctx->tmp_b.get<double>(static_cast<size_t>(n_obs * n));
    int64_t* chunk_tmp = ctx->tmp_c.get<int64_t>(static_cast<size_t>(2 * n_obs * chunks));
    int64_t* counts = ctx->counts.get<int64_t>(static_cast<size_t>(n_obs));
    CK(compact_valid(values, aux, failed, n, n_obs, cvalues, caux, counts, chunk_tmp, s));
    double* scratch = ctx->scratch.get<double>(static_cast<size_t>(2 * n_obs * std::max<int64_t>(chunks, 1)));
    double* sums = ctx->sums.get<double>(static_cast<size_t>(n_obs));
    double* means = ctx->means.get<double>(static_cast<size_t>(n_obs));
    double* sumsq = ctx->sumsq.get<double>(static_cast<size_t>(n_obs));
    double* sumaux = ctx->sumaux.get<double>(static_cast<size_t>(n_obs));
    smc_estimate* est = ctx->est.get<smc_estimate>(static_cast<size_t>(n_obs));
    int launches = 3;
    CK(tree_reduce(cvalues, n, counts, n, n_obs, sums, nullptr, 0, scratch, s, &launches));
    CK(launch_divide(sums, counts, n, n_obs, means, s));
    CK(tree_reduce(cvalues, n, counts, n, n_obs, sumsq, means, 1, scratch, s, &launches));
    CK(tree_reduce(caux, n, counts, n, n_obs, sumaux, nullptr, 0, scratch, s, &launches));
    CK(launch_estimates(means, sumsq, sumaux, counts, n, n, n_obs, est, s));
    count_launches(ctx, launches + 2);
    smc_estimate* h = ctx->est_host.get<smc_estimate>(static_cast<size_t>(n_obs));
    CK(cudaMemcpyAsync(h, est, sizeof(smc_estimate) * n_obs, cudaMemcpyDeviceToHost, s));
    unsigned long long* steps_h = ctx->steps_host.get<unsigned long long>(1);
    *steps_h = 0;
    if (step_total)
        CK(cudaMemcpyAsync(steps_h, step_total, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(ctx->ev[2], s));
    CK(cudaStreamSynchronize(s));
    if (step_total) ctx->stats.particle_steps = static_cast<int64_t>(*steps_h);
    finish_stats(ctx);
    for (int64_t j = 0; j < n_obs; ++j)
        if (h[j].n_failed == n) raise(SMC_ERUNTIME, "map_reduce: every particle of an observation failed");
    std::memcpy(out, h, sizeof(smc_estimate) * n_obs);
}

smc_status smc_bvp_observe_range(smc_ctx* ctx, const smc_bvp_problem* p, uint64_t seed, int64_t obs_begin,
                                 int64_t obs_count, smc_estimate* out) {
    return guarded(__func__, [&] {
        if (obs_begin < 0 || obs_count < 0 || obs_begin + obs_count > p->n_obs)
            raise(SMC_ERANGE, "observe_bvp: observation range out of bounds");
        CK(cudaSetDevice(ctx->device));
        if (is_sharded(ctx)) {
            group_bvp_observe(ctx, *p, seed, obs_begin, obs_count, out);
            return;
        }
        ctx->stats = smc_stats{};
        BvpLaunch L = prepare_bvp(ctx, *p, obs_begin, obs_count);
        L.seed = seed;
        const int64_t n = p->n_particles, n_obs = obs_count;
        run_bvp(ctx, L, n_obs, n);
        reduce_bvp(ctx, L.values, L.aux, L.failed, n, n_obs, L.step_total, out);
    });
}

smc_status smc_bvp_forcing_basis(smc_ctx* ctx, const smc_bvp_problem* p, uint64_t seed, double* mean_bc,
                                 double* mean_basis, double* mean_tau, int64_t* n_failed) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        if (p->forcing.kind != SMC_SCALAR_BUMPS || p->forcing.n_terms < 1 || p->forcing.n_terms > 4)
            raise(SMC_EINVAL, "bvp_forcing_basis: forcing must be a sum of 1..4 Gaussian bumps");
        if (p->precision != SMC_FP64) raise(SMC_EINVAL, "bvp_forcing_basis: FP64 only");
        ctx->stats = smc_stats{};
        BvpLaunch L = prepare_bvp(ctx, *p, 0, p->n_obs);
        L.seed = seed;
        const int64_t n = p->n_particles, n_obs = p->n_obs, nb = p->forcing.n_terms;
        cudaStream_t s = ctx->stream;
        const size_t total = static_cast<size_t>(n_obs * n);
        L.values = ctx->values.get<double>(total);
        L.aux = ctx->aux.get<double>(total);
        L.failed = ctx->flags.get<uint8_t>(total);
        L.basis = ctx->tmp_c.get<double>(total * static_cast<size_t>(nb));
        unsigned long long* ctr = ctx->flags2.get<unsigned long long>(2);
        CK(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), s));
        L.counter = ctr;
        L.step_total = ctr + 1;
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        CK(cudaEventRecord(ctx->ev[0], s));
        CK(launch_bvp_basis(L, sms, s));
        CK(cudaEventRecord(ctx->ev[1], s));
        count_launches(ctx, 1);
        // per quantity: compact valid walkers (executor.cpp:93-101), tree sum, / n_valid
        const int64_t chunks = smc_num_chunks(n);
        double* cvals = ctx->tmp_a.get<double>(total);
        double* caux = ctx->tmp_b.get<double>(total);
        int64_t* chunk_tmp = ctx->chunk_tmp.get<int64_t>(static_cast<size_t>(2 * n_obs * chunks));
        int64_t* counts = ctx->counts.get<int64_t>(static_cast<size_t>(n_obs));
        double* scratch = ctx->scratch.get<double>(static_cast<size_t>(2 * n_obs * std::max<int64_t>(chunks, 1)));
        double* sums = ctx->sums.get<double>(static_cast<size_t>(n_obs * (nb + 2)));
        double* means = ctx->means.get<double>(static_cast<size_t>(n_obs * (nb + 2)));
        int launches = 0;
        // values + exit times
        CK(compact_valid(L.values, L.aux, L.failed, n, n_obs, cvals, caux, counts, chunk_tmp, s));
        CK(tree_reduce(cvals, n, counts, n, n_obs, sums, nullptr, 0, scratch, s, &launches));
        CK(tree_reduce(caux, n, counts, n, n_obs, sums + n_obs, nullptr, 0, scratch, s, &launches));
        for (int64_t q = 0; q < nb; ++q) {
            const double* bq = L.basis + q * static_cast<int64_t>(total);
            CK(compact_valid(bq, bq, L.failed, n, n_obs, cvals, caux, counts, chunk_tmp, s));
            CK(tree_reduce(cvals, n, counts, n, n_obs, sums + (2 + q) * n_obs, nullptr, 0, scratch, s, &launches));
        }
        for (int64_t q = 0; q < nb + 2; ++q)
            CK(launch_divide(sums + q * n_obs, counts, n, n_obs, means + q * n_obs, s));
        count_launches(ctx, launches + 3 * (nb + 1) + nb + 2);
        std::vector<double> h(static_cast<size_t>(n_obs * (nb + 2)));
        std::vector<int64_t> hc(static_cast<size_t>(n_obs));
        CK(cudaMemcpyAsync(h.data(), means, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hc.data(), counts, sizeof(int64_t) * n_obs, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(ctx->ev[2], s));
        CK(cudaStreamSynchronize(s));
        finish_stats(ctx);
        for (int64_t j = 0; j < n_obs; ++j) {
            if (hc[static_cast<size_t>(j)] == 0) raise(SMC_ERUNTIME, "map_reduce: every particle of an observation failed");
            if (mean_bc) mean_bc[j] = h[static_cast<size_t>(j)];
            if (mean_tau) mean_tau[j] = h[static_cast<size_t>(n_obs + j)];
            if (n_failed) n_failed[j] = n - hc[static_cast<size_t>(j)];
            for (int64_t q = 0; q < nb; ++q)
                if (mean_basis) mean_basis[j * nb + q] = h[static_cast<size_t>((2 + q) * n_obs + j)];
        }
    });
}

smc_status smc_bvp_particle_values(smc_ctx* ctx, const smc_bvp_problem* p, uint64_t obs_index, uint64_t seed,
                                   int64_t n, double* values, double* aux, uint8_t* failed) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        if (obs_index >= static_cast<uint64_t>(p->n_obs)) raise(SMC_ERANGE, "observation index out of range");
        BvpLaunch L = prepare_bvp(ctx, *p, static_cast<int64_t>(obs_index), 1);
        L.seed = seed;
        L.n_particles = n;
        run_bvp(ctx, L, 1, n);
        CK(cudaMemcpyAsync(values, L.values, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(aux, L.aux, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(failed, L.failed, n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
