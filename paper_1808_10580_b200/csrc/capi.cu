// capi.cu — the C ABI (include/scalarmc_b200.h): context, device-image
// upload, kernel orchestration and host result return.
//
// One smc_ctx per process per GPU.  A forward-map call is: validate (host, the
// reference's messages) -> pack one image (velocity lattice, theta_0 terms,
// per-observation step schedules) into pinned staging -> one H2D copy -> K1
// particle kernel -> K3 tree reduction passes -> estimates kernel -> one D2H
// copy of n_obs x 40 B.  All on the context's stream; persistent buffers grow
// and are reused across calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <sstream>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/scalarmc_b200.h"
#include "disk_shape.h"
#include "host_problem.h"
#include "kernels.h"

namespace {
constexpr int kLatticeTileHost = 8;  // == kLatticeTile (velocity.cuh) / kTileW (host_problem.cpp)
}

using namespace smc;

namespace {

thread_local std::string g_err;

#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) raise(SMC_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                                    " (" #x ")");                                   \
    } while (0)

template <class F>
smc_status guarded(F&& f) {
    try {
        f();
        return SMC_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return static_cast<smc_status>(e.code);
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return SMC_ERUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SMC_ERUNTIME;
    }
}

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    template <class T>
    T* get(size_t n) {
        const size_t bytes = std::max<size_t>(n * sizeof(T), 16);
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            CK(cudaMalloc(&p, bytes));
            cap = bytes;
        }
        return static_cast<T*>(p);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    template <class T>
    T* get(size_t n) {
        const size_t bytes = std::max<size_t>(n * sizeof(T), 16);
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            CK(cudaMallocHost(&p, bytes));
            cap = bytes;
        }
        return static_cast<T*>(p);
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

// Host-side image under construction: 16-byte aligned blobs in one arena.
struct Image {
    std::vector<unsigned char> bytes;
    size_t add(const void* src, size_t n) {
        const size_t off = (bytes.size() + 15) & ~size_t(15);
        bytes.resize(off + std::max<size_t>(n, 1));
        if (n) std::memcpy(bytes.data() + off, src, n);
        return off;
    }
    template <class T>
    size_t add_vec(const std::vector<T>& v) {
        return add(v.data(), v.size() * sizeof(T));
    }
    size_t reserve(size_t n) {
        const size_t off = (bytes.size() + 15) & ~size_t(15);
        bytes.resize(off + std::max<size_t>(n, 1));
        return off;
    }
};

}  // namespace

struct smc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;      // stream every launch goes to
    cudaStream_t own_stream = nullptr;  // the context's own stream
    int64_t total_launches = 0;
    cudaEvent_t ev[4] = {};
    DevBuf image, values, aux, flags, flags2, scratch, sums, means, sumsq, sumaux, est, counts, tmp_a, tmp_b, tmp_c;
    DevBuf pk_ip, pk_im, pk_kp, pk_km, pk_ms, pk_u, pk_blocks, pk_bad;  // device u -> field packing
    DevBuf gal_A, gal_t0, gal_t1, gal_k1, gal_k2, gal_obs, gal_grid;  // Galerkin reference solver
    PinnedBuf staging, est_host;
    smc_stats stats{};
    // sharded AD state (smc_ad_shard_*)
    int64_t shard_n_obs = 0, shard_span = 0;

    unsigned char* upload(const Image& img) {
        unsigned char* h = staging.get<unsigned char>(img.bytes.size());
        std::memcpy(h, img.bytes.data(), img.bytes.size());
        unsigned char* d = image.get<unsigned char>(img.bytes.size());
        CK(cudaMemcpyAsync(d, h, img.bytes.size(), cudaMemcpyHostToDevice, stream));
        return d;
    }
};

namespace {

void count_launches(smc_ctx* ctx, int64_t n) {
    ctx->stats.kernel_launches += n;
    ctx->total_launches += n;
}

// ScalarField image: term arrays appended to the image; pointers patched
// after upload.
struct ScalarRef {
    ScalarImg img{};
    size_t amp = 0, freq = 0, phase = 0, center = 0;
};

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

struct VelRef {
    VelImg img{};
    size_t modes = 0, tiles = 0, coefs = 0;
};

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

// Everything a K1 launch needs, prepared and uploaded.
struct AdPrepared {
    AdLaunch L{};
    int disk_K = 0;                  // > 0: use the compile-time disk kernel
    const double* disk = nullptr;    // its coefficient blocks (device, one per sample)
    int64_t n_obs = 0;
    int64_t steps_per_particle_sum = 0;  // sum_j n_j
};

void check_particle_range(int64_t n_particles) {
    // Stream keys carry the particle index in 32 bits (rng.cpp:46-47); the
    // reference's work lambda throws and map_reduce reports it.
    if (n_particles > (int64_t(1) << 32)) raise(SMC_ERUNTIME, "map_reduce: a particle work function threw");
}

AdPrepared prepare_ad(smc_ctx* ctx, const smc_ad_problem& p, const std::vector<const PreparedVelocity*>& fills,
                      const PreparedVelocity& structure, int64_t obs_begin, int64_t obs_count) {
    const double dt = ad_resolved_dt(p);
    const double sigma = std::sqrt(2.0 * p.kappa);
    Image im;
    std::vector<AdObsImg> obs;
    AdPrepared out;
    for (int64_t j = obs_begin; j < obs_begin + obs_count; ++j) {
        obs.push_back(make_ad_obs(p.obs_t[j], p.obs_x[2 * j], p.obs_x[2 * j + 1], dt, sigma));
        out.steps_per_particle_sum += obs.back().n_steps;
    }
    const size_t obs_off = im.add_vec(obs);
    const ScalarRef th = add_scalar(im, p.initial_condition);
    const VelRef vr = add_velocity(im, structure, fills);
    // Dense fields with K <= kDiskMaxK take the compile-time disk kernel.
    size_t disk_off = 0;
    const bool disk = !structure.is_constant && p.precision != SMC_FP64_STRICT && structure.K <= kDiskMaxK &&
                      2 * structure.modes.size() >= static_cast<size_t>(disk_n_modes(structure.K)) &&
                      std::getenv("SMC_DISABLE_DISK") == nullptr;
    if (disk) {
        const size_t nc = static_cast<size_t>(disk_n_coef(structure.K));
        disk_off = im.reserve(nc * fills.size() * sizeof(double));
        for (size_t b = 0; b < fills.size(); ++b)
            disk_fill(structure.K, *fills[b], reinterpret_cast<double*>(im.bytes.data() + disk_off) + b * nc);
    }
    unsigned char* base = ctx->upload(im);
    if (disk) {
        out.disk_K = structure.K;
        out.disk = reinterpret_cast<const double*>(base + disk_off);
    }
    AdLaunch& L = out.L;
    L.vel = patch(vr, base);
    L.theta0 = patch(th, base);
    L.obs = reinterpret_cast<const AdObsImg*>(base + obs_off);
    L.n_obs = static_cast<int32_t>(obs_count);
    L.obs_slot0 = static_cast<uint32_t>(obs_begin);
    L.n_particles = p.n_particles;
    L.p_begin = 0;
    L.p_end = p.n_particles;
    L.n_samples = 1;
    L.precision = p.precision;
    L.sigma = sigma;
    out.n_obs = obs_count;
    return out;
}

void run_particles(smc_ctx* ctx, AdLaunch& L, const AdPrepared* P = nullptr, int64_t sample0 = 0) {
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
    ctx->stats = smc_stats{};
    AdPrepared P = prepare_ad(ctx, p, {&v}, v, obs_begin, obs_count);
    P.L.seed = seed;
    const int64_t n = p.n_particles;
    P.L.values = ctx->values.get<double>(static_cast<size_t>(obs_count * n));
    CK(cudaEventRecord(ctx->ev[0], ctx->stream));
    run_particles(ctx, P.L, &P);
    CK(cudaEventRecord(ctx->ev[1], ctx->stream));
    reduce_ad(ctx, P.L.values, n, obs_count, out);
    finish_stats(ctx);
    ctx->stats.particle_steps = P.steps_per_particle_sum * n;
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

}  // namespace

namespace smc {
namespace {
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
}  // namespace
}  // namespace smc

extern "C" {

int smc_abi_version(void) { return SMC_ABI_VERSION; }

const char* smc_last_error(void) { return g_err.c_str(); }

smc_status smc_create(int device, smc_ctx** out) {
    return guarded([&] {
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
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
    for (DevBuf* b : {&ctx->image, &ctx->values, &ctx->aux, &ctx->flags, &ctx->flags2, &ctx->scratch, &ctx->sums, &ctx->means,
                      &ctx->sumsq, &ctx->sumaux, &ctx->est, &ctx->counts, &ctx->tmp_a, &ctx->tmp_b, &ctx->tmp_c})
        b->release();
    ctx->staging.release();
    ctx->est_host.release();
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

void* smc_stream(smc_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

smc_status smc_set_stream(smc_ctx* ctx, void* stream) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    });
}

smc_status smc_ad_resolved_dt(const smc_ad_problem* p, double* out) {
    return guarded([&] { *out = ad_resolved_dt(*p); });
}

smc_status smc_bvp_resolved_dt(const smc_bvp_problem* p, double* out) {
    return guarded([&] {
        const PreparedVelocity v = prepare_velocity(p->velocity);
        *out = bvp_resolved_dt(*p, v);
    });
}

smc_status smc_velocity_validate(const smc_velocity* v) {
    return guarded([&] { (void)prepare_velocity(*v); });
}

smc_status smc_ad_validate(const smc_ad_problem* p) {
    return guarded([&] {
        (void)prepare_velocity(p->velocity);
        check_kappa(p->kappa);
        check_scalar(p->initial_condition);
        ad_validate(*p);
    });
}

smc_status smc_bvp_validate(const smc_bvp_problem* p) {
    return guarded([&] {
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
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        ad_observe_range(ctx, *p, seed, 0, p->n_obs, out);
    });
}

smc_status smc_ad_observe_single(smc_ctx* ctx, const smc_ad_problem* p, uint64_t obs_index, uint64_t seed,
                                 smc_estimate* out) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        // observe_ad_single validates first, then range-checks (forward_ad.cpp:64-67).
        (void)prepare_velocity(p->velocity);
        check_kappa(p->kappa);
        check_scalar(p->initial_condition);
        ad_validate(*p);
        if (obs_index >= static_cast<uint64_t>(p->n_obs))
            raise(SMC_ERANGE, "observe_ad_single: observation index out of range");
        ad_observe_range(ctx, *p, seed, static_cast<int64_t>(obs_index), 1, out);
    });
}

smc_status smc_ad_observe_batched(smc_ctx* ctx, const smc_ad_problem* base, const smc_prior* prior,
                                  int64_t n_samples, const double* u, const uint64_t* seeds, uint64_t seed,
                                  smc_estimate* out) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        if (n_samples < 1) raise(SMC_EINVAL, "observe_ad_batched: need at least one sample");
        if (prior->cutoff <= 0) raise(SMC_EINVAL, "FourierVelocityField: max_wavenumber must be positive");
        smc_ad_problem p = *base;
        p.velocity.is_constant = 0;
        p.velocity.max_wavenumber = prior->cutoff;
        check_kappa(p.kappa);
        check_scalar(p.initial_condition);
        // validate() without the velocity slot
        ad_validate(p);
        check_particle_range(p.n_particles);
        if (p.precision == SMC_FP64_STRICT) raise(SMC_EINVAL, "strict precision is single-sample only");
        ctx->stats = smc_stats{};
        const int64_t n = p.n_particles, n_obs = p.n_obs;
        // One FourierVelocityField per sample from u in prior order
        // (velocity_from_coefficients, inference.cpp:63-73), built on the
        // device: the image carries the full prior disk's structure and the
        // pack kernel writes every sample's coefficient block from u.
        const PreparedVelocity structure = prior_structure(prior->cutoff);
        const int64_t dim = 2 * static_cast<int64_t>(structure.modes.size());
        AdPrepared P = prepare_ad(ctx, p, {&structure}, structure, 0, n_obs);
        const LatticeHost Lh = lattice_structure(structure);
        const PackMap pmap = pack_map(prior->cutoff, P.disk_K > 0, &Lh);
        const PackDev pdev = upload_pack_map(ctx, pmap);
        double* d_u = ctx->pk_u.get<double>(static_cast<size_t>(n_samples * dim));
        CK(cudaMemcpyAsync(d_u, u, sizeof(double) * n_samples * dim, cudaMemcpyHostToDevice, ctx->stream));
        double* blocks = ctx->pk_blocks.get<double>(static_cast<size_t>(n_samples * pmap.stride));
        int* d_bad = ctx->pk_bad.get<int>(1);
        CK(cudaMemsetAsync(d_bad, 0, sizeof(int), ctx->stream));
        for (int64_t b0 = 0; b0 < n_samples; b0 += 65535)
            CK(launch_pack(pdev, d_u + b0 * dim, dim, std::min<int64_t>(65535, n_samples - b0),
                           blocks + b0 * pmap.stride, d_bad, ctx->stream));
        count_launches(ctx, (n_samples + 65534) / 65535);
        // the FourierVelocityField ctor throws before any particle work (fields.cpp:46-47)
        int bad = 0;
        CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (bad) raise(SMC_EINVAL, "FourierVelocityField: non-finite coefficient");
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
        double* values = ctx->values.get<double>(static_cast<size_t>(n_samples * n_obs * n));
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
        reduce_ad(ctx, values, n, n_samples * n_obs, out);
        finish_stats(ctx);
        ctx->stats.particle_steps = P.steps_per_particle_sum * n * n_samples;
    });
}

smc_status smc_ad_shard_partials(smc_ctx* ctx, const smc_ad_problem* p, uint64_t seed, int64_t chunk_begin,
                                 int64_t chunk_end, double* partials_dev) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        const PreparedVelocity v = prepare_velocity(p->velocity);
        check_kappa(p->kappa);
        check_scalar(p->initial_condition);
        ad_validate(*p);
        check_particle_range(p->n_particles);
        const int64_t n_chunks = smc_num_chunks(p->n_particles);
        if (chunk_begin < 0 || chunk_end > n_chunks || chunk_begin > chunk_end)
            raise(SMC_ERANGE, "smc_ad_shard_partials: chunk range out of bounds");
        ctx->stats = smc_stats{};
        AdPrepared P = prepare_ad(ctx, *p, {&v}, v, 0, p->n_obs);
        P.L.seed = seed;
        P.L.p_begin = chunk_begin * kChunk;
        P.L.p_end = std::min(chunk_end * kChunk, p->n_particles);
        const int64_t span = std::max<int64_t>(P.L.p_end - P.L.p_begin, 0);
        P.L.values = ctx->values.get<double>(static_cast<size_t>(std::max<int64_t>(p->n_obs * span, 1)));
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        run_particles(ctx, P.L, &P);
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        const int64_t nloc = chunk_end - chunk_begin;
        if (nloc > 0) {
            CK(launch_tree_pass(P.L.values, span, nullptr, span, p->n_obs, partials_dev, nloc, nullptr, 0, ctx->stream));
            count_launches(ctx, 1);
        }
        CK(cudaEventRecord(ctx->ev[2], ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        finish_stats(ctx);
        ctx->shard_n_obs = p->n_obs;
        ctx->shard_span = span;
        ctx->stats.particle_steps = P.steps_per_particle_sum * span;
    });
}

smc_status smc_tree_finish(smc_ctx* ctx, const double* partials_dev, int64_t n_obs, int64_t n_chunks,
                           double* sums_dev) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        double* scratch = ctx->scratch.get<double>(static_cast<size_t>(2 * n_obs * std::max<int64_t>(1, n_chunks)));
        int launches = 0;
        CK(tree_reduce(partials_dev, n_chunks, nullptr, n_chunks, n_obs, sums_dev, nullptr, 0, scratch, ctx->stream,
                       &launches));
        count_launches(ctx, launches);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

smc_status smc_ad_shard_sq_partials(smc_ctx* ctx, const double* means_dev, int64_t n_obs, int64_t chunk_begin,
                                    int64_t chunk_end, double* partials_dev) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        if (n_obs != ctx->shard_n_obs) raise(SMC_EINVAL, "smc_ad_shard_sq_partials: observation count mismatch");
        const int64_t nloc = chunk_end - chunk_begin;
        const int64_t span = ctx->shard_span;
        if (nloc > 0) {
            CK(launch_tree_pass(static_cast<const double*>(ctx->values.p), span, nullptr, span, n_obs, partials_dev,
                                nloc, means_dev, 1, ctx->stream));
            count_launches(ctx, 1);
        }
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

smc_status smc_ad_particle_values(smc_ctx* ctx, const smc_ad_problem* p, uint64_t obs_index, uint64_t seed,
                                  int64_t n, double* out) {
    return guarded([&] {
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
    return guarded([&] {
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
    return guarded([&] {
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
    return guarded([&] {
        *out = ctx->stats;
        out->total_launches = ctx->total_launches;
    });
}

// ---- spectral Galerkin reference solver (src/galerkin.cpp) ----------------
namespace {
// check_galerkin_inputs (galerkin.cpp:144-149): the spec's own validation
// (isotropic diffusion is the only kind the ABI carries).
PreparedVelocity galerkin_check_inputs(const smc_ad_problem& p) {
    PreparedVelocity v = prepare_velocity(p.velocity);
    check_kappa(p.kappa);
    check_scalar(p.initial_condition);
    ad_validate(p);
    return v;
}
}  // namespace

int64_t smc_galerkin_n_basis(const smc_galerkin_basis* basis) {
    try {
        return galerkin_modes(*basis).size();
    } catch (...) {
        return -1;
    }
}

smc_status smc_galerkin_modes(const smc_galerkin_basis* basis, int32_t* modes) {
    return guarded([&] {
        const GalerkinModes m = galerkin_modes(*basis);
        for (int64_t i = 0; i < m.size(); ++i) {
            modes[2 * i] = m.k1[static_cast<size_t>(i)];
            modes[2 * i + 1] = m.k2[static_cast<size_t>(i)];
        }
    });
}

smc_status smc_galerkin_spectral_radius(smc_ctx*, const smc_ad_problem* prob, const smc_galerkin_basis* basis,
                                        double* out) {
    return guarded([&] {
        const PreparedVelocity v = galerkin_check_inputs(*prob);
        const GalerkinModes m = galerkin_modes(*basis);
        *out = galerkin_radius(galerkin_assemble(prob->kappa, v, m), m.size());
    });
}

smc_status smc_galerkin_solve_ad(smc_ctx* ctx, const smc_ad_problem* prob, const smc_galerkin_basis* basis,
                                 double dt_ref, smc_galerkin_result* out) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        const smc_ad_problem& p = *prob;
        const PreparedVelocity v = galerkin_check_inputs(p);
        if (!(dt_ref > 0.0)) raise(SMC_EINVAL, "galerkin_solve_ad: dt_ref must be positive");
        const GalerkinModes m = galerkin_modes(*basis);
        const int64_t nb = m.size();
        cudaStream_t s = ctx->stream;
        double* dA = ctx->gal_A.get<double>(static_cast<size_t>(2 * nb * nb));
        double* th[2] = {ctx->gal_t0.get<double>(static_cast<size_t>(2 * nb)),
                         ctx->gal_t1.get<double>(static_cast<size_t>(2 * nb))};
        int* dk1 = ctx->gal_k1.get<int>(static_cast<size_t>(nb));
        int* dk2 = ctx->gal_k2.get<int>(static_cast<size_t>(nb));
        double* dobs = ctx->gal_obs.get<double>(static_cast<size_t>(std::max<int64_t>(p.n_obs, 1)));
        CK(cudaMemcpyAsync(dk1, m.k1.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dk2, m.k2.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, s));
        // A assembled on the device (bit-identical to the host restatement of
        // galerkin.cpp:108-142), then the explicit-Euler stability estimate
        // (galerkin.cpp:170-177)
        const VhatGrid vg = galerkin_vhat_grid(v);
        const size_t cells = vg.present.size();
        double* dvh = ctx->gal_grid.get<double>(4 * cells + (cells + 7) / 8 + 1);
        auto* dpres = reinterpret_cast<unsigned char*>(dvh + 4 * cells);
        auto* dradius = ctx->tmp_a.get<unsigned long long>(1);
        CK(cudaMemcpyAsync(dvh, vg.c.data(), sizeof(double) * 4 * cells, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dpres, vg.present.data(), cells, cudaMemcpyHostToDevice, s));
        CK(launch_galerkin_assemble(dvh, dpres, vg.K, dk1, dk2, nb, p.kappa, v.is_constant ? 1 : 0, v.c1, v.c2, dA,
                                    dradius, s));
        count_launches(ctx, 2);
        unsigned long long rbits = 0;
        CK(cudaMemcpyAsync(&rbits, dradius, sizeof(rbits), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double radius;
        std::memcpy(&radius, &rbits, sizeof(radius));
        if (radius * dt_ref >= 2.0) {
            std::ostringstream msg;
            msg << "galerkin_solve_ad: dt_ref " << dt_ref << " violates the stability estimate; suggest dt_ref <= "
                << 1.8 / radius;
            raise(SMC_ERUNTIME, msg.str());
        }
        // projection of theta_0 (galerkin.cpp:43-101)
        std::vector<double> theta0;
        if (galerkin_project_exact(p.initial_condition, m, theta0)) {
            CK(cudaMemcpyAsync(th[0], theta0.data(), sizeof(double) * 2 * nb, cudaMemcpyHostToDevice, s));
        } else {
            Image im;
            const ScalarRef ref = add_scalar(im, p.initial_condition);
            unsigned char* base = ctx->upload(im);
            const int n = std::max(128, 4 * (m.max_abs + 1));
            CK(launch_galerkin_quadrature(patch(ref, base), dk1, dk2, nb, n, th[0], s));
            count_launches(ctx, 1);
        }
        // the step schedule: once through the sorted observation times, shortening
        // the last step of each segment to land on t_j (galerkin.cpp:181-221)
        std::vector<int64_t> order(static_cast<size_t>(p.n_obs));
        for (int64_t i = 0; i < p.n_obs; ++i) order[static_cast<size_t>(i)] = i;
        std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return p.obs_t[a] < p.obs_t[b]; });
        constexpr int kGroup = 16;  // even: a group returns to the buffer it started from
        cudaGraphExec_t group[2] = {nullptr, nullptr};
        struct GraphFree {
            cudaGraphExec_t* g;
            ~GraphFree() {
                for (int i = 0; i < 2; ++i)
                    if (g[i]) cudaGraphExecDestroy(g[i]);
            }
        } graph_free{group};
        auto group_exec = [&](int cur) {
            if (!group[cur]) {
                cudaGraph_t graph = nullptr;
                CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
                cudaError_t e = cudaSuccess;
                for (int k = 0; k < kGroup && e == cudaSuccess; ++k)
                    e = launch_galerkin_step(dA, th[(cur + k) & 1], th[(cur + k + 1) & 1], nb, dt_ref, s);
                const cudaError_t e2 = cudaStreamEndCapture(s, &graph);
                CK(e);
                CK(e2);
                const cudaError_t e3 = cudaGraphInstantiate(&group[cur], graph, 0);
                cudaGraphDestroy(graph);
                CK(e3);
            }
            return group[cur];
        };
        int cur = 0;
        double t = 0.0;
        int64_t steps = 0;
        const bool use_graph = s != nullptr;
        for (const int64_t oi : order) {
            const double target = p.obs_t[oi];
            int64_t run = 0;  // pending full steps of dt_ref
            auto flush = [&] {
                for (; use_graph && run >= kGroup; run -= kGroup) {
                    CK(cudaGraphLaunch(group_exec(cur), s));
                    count_launches(ctx, kGroup);
                }
                for (; run > 0; --run, cur ^= 1) {
                    CK(launch_galerkin_step(dA, th[cur], th[cur ^ 1], nb, dt_ref, s));
                    count_launches(ctx, 1);
                }
            };
            while (t < target - 1e-15) {
                const double dt = std::min(dt_ref, target - t);
                if (dt == dt_ref) {
                    ++run;
                } else {
                    flush();
                    CK(launch_galerkin_step(dA, th[cur], th[cur ^ 1], nb, dt, s));
                    count_launches(ctx, 1);
                    cur ^= 1;
                }
                t += dt;
                ++steps;
            }
            flush();
            CK(launch_galerkin_observe(th[cur], dk1, dk2, nb, p.obs_x[2 * oi], p.obs_x[2 * oi + 1], dobs + oi, s));
            count_launches(ctx, 1);
            if (out->coefficients_at_observations)
                CK(cudaMemcpyAsync(out->coefficients_at_observations + oi * 2 * nb, th[cur], sizeof(double) * 2 * nb,
                                   cudaMemcpyDeviceToHost, s));
        }
        CK(cudaMemcpyAsync(out->observation_values, dobs, sizeof(double) * p.n_obs, cudaMemcpyDeviceToHost, s));
        if (out->final_coefficients)
            CK(cudaMemcpyAsync(out->final_coefficients, th[cur], sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        out->dt_used = dt_ref;
        out->steps = steps;
    });
}

smc_status smc_galerkin_field_grid(smc_ctx* ctx, const smc_galerkin_basis* basis, const double* coefficients,
                                   int32_t n, double* grid) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        if (n < 2) raise(SMC_EINVAL, "galerkin_field_grid: n must be >= 2");
        const GalerkinModes m = galerkin_modes(*basis);
        const int64_t nb = m.size();
        cudaStream_t s = ctx->stream;
        double* dc = ctx->gal_t0.get<double>(static_cast<size_t>(2 * nb));
        int* dk1 = ctx->gal_k1.get<int>(static_cast<size_t>(nb));
        int* dk2 = ctx->gal_k2.get<int>(static_cast<size_t>(nb));
        double* dg = ctx->gal_grid.get<double>(static_cast<size_t>(n) * n);
        CK(cudaMemcpyAsync(dc, coefficients, sizeof(double) * 2 * nb, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dk1, m.k1.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dk2, m.k2.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, s));
        CK(launch_galerkin_field_grid(dc, dk1, dk2, nb, n, dg, s));
        count_launches(ctx, 1);
        CK(cudaMemcpyAsync(grid, dg, sizeof(double) * n * n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

smc_status smc_fp64_peak(smc_ctx* ctx, double ms, double* tflops) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        const int blocks = sms * 8;
        double* sink = ctx->tmp_a.get<double>(static_cast<size_t>(blocks));
        int iters = 4096;
        float t = 0.f;
        for (int attempt = 0; attempt < 8; ++attempt) {
            CK(cudaEventRecord(ctx->ev[0], ctx->stream));
            CK(launch_dfma_peak(blocks, iters, sink, ctx->stream));
            CK(cudaEventRecord(ctx->ev[1], ctx->stream));
            CK(cudaEventSynchronize(ctx->ev[1]));
            CK(cudaEventElapsedTime(&t, ctx->ev[0], ctx->ev[1]));
            if (t >= 0.9 * ms) break;
            const double scale = std::min(64.0, std::max(2.0, ms / std::max<double>(t, 1e-3)));
            iters = static_cast<int>(std::min<double>(iters * scale, 1 << 30));
        }
        const double flops = 2.0 * 8.0 * double(iters) * 256.0 * blocks;
        *tflops = flops / (double(t) * 1e-3) / 1e12;
    });
}

int64_t smc_pcn_num_samples(const smc_chain_config* cfg) {
    // iterations i = 1..n_steps with i > burn_in and (i - burn_in - 1) % thin == 0
    if (!cfg || cfg->thin < 1 || cfg->n_steps <= cfg->burn_in) return 0;
    const int64_t burn = cfg->burn_in < 0 ? 0 : cfg->burn_in;
    return (cfg->n_steps - burn - 1) / cfg->thin + 1;
}

smc_status smc_pcn_chains(smc_ctx* ctx, const smc_ad_problem* forward, const smc_prior* prior, const double* data,
                          double noise_std, uint64_t forward_seed, int64_t n_chains, const uint64_t* chain_seeds,
                          const double* u0, const smc_chain_config* cfg, smc_chain_outputs* out) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        // run_chain's checks (inference.cpp:172-173), prior_draw/chain_init's
        // (inference.cpp:17-21, :89-91, :125-133), pcn_step's (:138).
        if (cfg->n_steps < 0) raise(SMC_EINVAL, "run_chain: n_steps must be >= 0");
        if (cfg->thin < 1) raise(SMC_EINVAL, "run_chain: thin must be >= 1");
        if (prior->cutoff < 1) raise(SMC_EINVAL, "PriorSpec: cutoff must be >= 1");
        if (!(prior->s0 >= 0.0)) raise(SMC_EINVAL, "PriorSpec: s0 must be >= 0");
        if (!std::isfinite(prior->alpha)) raise(SMC_EINVAL, "PriorSpec: alpha must be finite");
        if (!(noise_std > 0.0)) raise(SMC_EINVAL, "LikelihoodSpec: noise_std must be positive");
        if (cfg->n_steps > 0 && !(cfg->beta > 0.0 && cfg->beta <= 1.0))
            raise(SMC_EINVAL, "pcn_step: beta must be in (0,1]");
        if (n_chains < 1) raise(SMC_EINVAL, "pcn_chains: need at least one chain");
        if (!out || !out->final_u) raise(SMC_EINVAL, "pcn_chains: final_u output is required");
        smc_ad_problem p = *forward;
        check_kappa(p.kappa);
        check_scalar(p.initial_condition);
        ad_validate(p);
        check_particle_range(p.n_particles);
        if (p.precision == SMC_FP64_STRICT) raise(SMC_EINVAL, "strict precision is single-sample only");
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
        const bool use_disk = prior->cutoff <= kDiskMaxK && std::getenv("SMC_DISABLE_DISK") == nullptr;
        const LatticeHost Lh = lattice_structure(structure);
        const PackMap pmap = pack_map(prior->cutoff, use_disk, &Lh);
        const int64_t stride = pmap.stride;
        if (static_cast<int64_t>(p.n_obs) <= 0) raise(SMC_EINVAL, "AdProblemSpec: no observations");

        // device buffers (freed at the end of the call)
        std::vector<void*> owned;
        auto dalloc = [&](size_t bytes) {
            void* q = nullptr;
            CK(cudaMalloc(&q, std::max<size_t>(bytes, 16)));
            owned.push_back(q);
            return q;
        };
        struct Freer {
            std::vector<void*>* v;
            ~Freer() {
                for (void* q : *v) cudaFree(q);
            }
        } freer{&owned};
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
        S.noise_inf = std::isinf(noise_std) ? 1 : 0;
        auto* d_stds = static_cast<double*>(dalloc(8 * M));
        h2d(d_stds, stds.data(), 8 * M);
        S.stds = d_stds;
        auto* d_seeds = static_cast<uint64_t*>(dalloc(8 * B));
        h2d(d_seeds, chain_seeds, 8 * B);
        S.seeds = d_seeds;
        auto* d_data = static_cast<double*>(dalloc(8 * n_obs));
        h2d(d_data, data, 8 * n_obs);
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
        p.velocity.is_constant = 0;
        p.velocity.max_wavenumber = prior->cutoff;
        AdPrepared P = prepare_ad(ctx, p, {&structure}, structure, 0, n_obs);
        P.L.seed = forward_seed;
        P.L.seeds = nullptr;
        if (!use_disk) {
            P.L.vel.lat.coef = d_blocks;
            P.L.vel.lat.sample_stride = stride;
        }
        double* values = ctx->values.get<double>(static_cast<size_t>(B * n_obs * n));

        auto forward_map = [&]() -> smc_estimate* {
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
    });
}

smc_status smc_bvp_observe(smc_ctx* ctx, const smc_bvp_problem* p, uint64_t seed, smc_estimate* out) {
    return smc_bvp_observe_range(ctx, p, seed, 0, p->n_obs, out);
}

smc_status smc_bvp_observe_range(smc_ctx* ctx, const smc_bvp_problem* p, uint64_t seed, int64_t obs_begin,
                                 int64_t obs_count, smc_estimate* out) {
    return guarded([&] {
        if (obs_begin < 0 || obs_count < 0 || obs_begin + obs_count > p->n_obs)
            raise(SMC_ERANGE, "observe_bvp: observation range out of bounds");
        CK(cudaSetDevice(ctx->device));
        ctx->stats = smc_stats{};
        BvpLaunch L = prepare_bvp(ctx, *p, obs_begin, obs_count);
        L.seed = seed;
        const int64_t n = p->n_particles, n_obs = obs_count;
        run_bvp(ctx, L, n_obs, n);
        // compaction of valid walkers, then the same tree as AD
        cudaStream_t s = ctx->stream;
        const int64_t chunks = smc_num_chunks(n);
        double* cvalues = ctx->tmp_a.get<double>(static_cast<size_t>(n_obs * n));
        double* caux = ctx->tmp_b.get<double>(static_cast<size_t>(n_obs * n));
        int64_t* chunk_tmp = ctx->tmp_c.get<int64_t>(static_cast<size_t>(2 * n_obs * chunks));
        int64_t* counts = ctx->counts.get<int64_t>(static_cast<size_t>(n_obs));
        CK(compact_valid(L.values, L.aux, L.failed, n, n_obs, cvalues, caux, counts, chunk_tmp, s));
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
        unsigned long long* steps_h = ctx->staging.get<unsigned long long>(1);
        CK(cudaMemcpyAsync(steps_h, L.step_total, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(ctx->ev[2], s));
        CK(cudaStreamSynchronize(s));
        ctx->stats.particle_steps = static_cast<int64_t>(*steps_h);
        finish_stats(ctx);
        for (int64_t j = 0; j < n_obs; ++j)
            if (h[j].n_failed == n) raise(SMC_ERUNTIME, "map_reduce: every particle of an observation failed");
        std::memcpy(out, h, sizeof(smc_estimate) * n_obs);
    });
}

smc_status smc_bvp_forcing_basis(smc_ctx* ctx, const smc_bvp_problem* p, uint64_t seed, double* mean_bc,
                                 double* mean_basis, double* mean_tau, int64_t* n_failed) {
    return guarded([&] {
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
        DevBuf ctmp;
        int64_t* chunk_tmp = ctmp.get<int64_t>(static_cast<size_t>(2 * n_obs * chunks));
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
        ctmp.release();
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
    return guarded([&] {
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
