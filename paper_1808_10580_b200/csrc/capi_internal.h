// capi_internal.h — shared internals of the C ABI translation units
// (capi.cu: context, images, AD/BVP forward maps; capi_samples.cu: batched
// evaluations and multi-chain pCN; capi_galerkin.cu: the spectral reference
// solver).  Not part of the public interface.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

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

namespace smc::capi {

extern thread_local std::string g_err;



#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) ::smc::raise(SMC_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                                    " (" #x ")");                                   \
    } while (0)

// Every C-ABI entry runs inside guarded(__func__, ...): one NVTX range named
// after the entry point (visible in nsys / ncu --nvtx), exceptions mapped to
// the smc_status of the reference's exception type.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Guard zones (SMC_GUARD=1; the pool refuses compute-sanitizer): every device
// buffer is allocated with kGuardBytes of a fixed byte pattern before and
// after it, and every C-ABI entry ends by synchronising and checking every
// live buffer's zones — a kernel or copy that writes past either end of its
// buffer (up to 4 KB) fails that call with SMC_ERUNTIME naming the entry.
bool guard_mode();
void guard_check(const char* entry);

template <class F>
smc_status guarded(const char* name, F&& f) {
    NvtxRange range(name);
    try {
        f();
        if (guard_mode()) guard_check(name);
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

// Device / pinned buffers that grow on demand and are reused across calls.
// RAII and non-copyable: a context's buffers are all released by its
// destructor, so a new buffer cannot be forgotten in smc_destroy.
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    unsigned char* base = nullptr;  // guard mode: the allocation, p = base + kGuardBytes
    int device = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    template <class T>
    T* get(size_t n) {
        const size_t bytes = std::max<size_t>(n * sizeof(T), 16);
        if (bytes > cap) {
            release();
            if (guard_mode()) {
                allocate_guarded(bytes);
            } else {
                CK(cudaMalloc(&p, bytes));
            }
            cap = bytes;
        }
        return static_cast<T*>(p);
    }
    void allocate_guarded(size_t bytes);  // capi.cu
    void release();
};

struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() { release(); }
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


}  // namespace smc::capi

using smc::capi::DevBuf;
using smc::capi::Image;
using smc::capi::PinnedBuf;

// Multi-device group (capi_group.cu): the ranks of one
// sharded forward map.  Single process: members are per-device contexts of
// this process (members[0] is the owning context).  One process per GPU:
// one member, rank0 = this process's rank.  comms: one ncclComm_t per member
// (empty: the emulated exchange of a single process with repeated devices).
struct smc_group {
    int world = 1;
    int rank0 = 0;
    std::vector<smc_ctx*> members;
    std::vector<void*> comms;
    std::vector<cudaEvent_t> ready;  // per member: contribution enqueued (emulated exchange)
    smc_exchange_fn hook = nullptr;  // host-staged exchange (smc_create_rank_hosted)
    void* hook_user = nullptr;
    PinnedBuf hook_buf;
};

struct smc_ctx {
    int device = 0;
    smc_group* group = nullptr;         // non-null: multi-device context (see smc_group)
    cudaStream_t stream = nullptr;      // stream every launch goes to
    cudaStream_t own_stream = nullptr;  // the context's own stream
    int64_t total_launches = 0;
    cudaEvent_t ev[4] = {};
    DevBuf image, values, aux, flags, flags2, scratch, sums, means, sumsq, sumaux, est, counts, tmp_a, tmp_b, tmp_c;
    DevBuf chunk_tmp;  // compaction scan scratch of smc_bvp_forcing_basis
    DevBuf guard_probe;  // smc_guard_selftest
    DevBuf gx_a, gx_b, gx_c, gx_d;  // group exchange buffers (every rank's contribution)
    DevBuf pk_ip, pk_im, pk_kp, pk_km, pk_ms, pk_u, pk_blocks, pk_bad;  // device u -> field packing
    DevBuf gal_A, gal_t0, gal_t1, gal_k1, gal_k2, gal_obs, gal_grid;  // Galerkin reference solver
    // staging: the problem image's H2D source, read by a copy that may still
    // be queued behind earlier work on the stream when the call returns to
    // the host — nothing else may write it before the call's final sync;
    // steps_host: the walker-step count read back at the end of a call
    PinnedBuf staging, est_host, steps_host;
    smc_stats stats{};

    unsigned char* upload(const Image& img) {
        unsigned char* h = staging.get<unsigned char>(img.bytes.size());
        std::memcpy(h, img.bytes.data(), img.bytes.size());
        unsigned char* d = image.get<unsigned char>(img.bytes.size());
        CK(cudaMemcpyAsync(d, h, img.bytes.size(), cudaMemcpyHostToDevice, stream));
        return d;
    }
};

namespace smc::capi {

void count_launches(smc_ctx* ctx, int64_t n);

// ScalarField image: term arrays appended to the image; pointers patched
// after upload.
struct ScalarRef {
    ScalarImg img{};
    size_t amp = 0, freq = 0, phase = 0, center = 0;
};
ScalarRef add_scalar(Image& im, const smc_scalar_field& f);
ScalarImg patch(const ScalarRef& r, unsigned char* base);

struct VelRef {
    VelImg img{};
    size_t modes = 0, tiles = 0, coefs = 0;
};
// Velocity image: strict mode list + tiled lattice structure + one
// coefficient block per sample (fills[i] for sample i).
VelRef add_velocity(Image& im, const PreparedVelocity& v, const std::vector<const PreparedVelocity*>& fills);
VelImg patch(const VelRef& r, unsigned char* base);

// Everything a K1 launch needs, prepared and uploaded.
struct AdPrepared {
    AdLaunch L{};
    int disk_K = 0;                  // > 0: use the compile-time disk kernel
    const double* disk = nullptr;    // its coefficient blocks (device, one per sample)
    std::vector<double> host_disk;   // host copy of a single-sample block (kernel-parameter path)
    int64_t n_obs = 0;
    int64_t steps_per_particle_sum = 0;  // sum_j n_j
};
// The device-independent part of an AD launch: the host image and the offsets
// to patch after upload (multi-device groups build it once and upload it to
// every member).
struct AdImage {
    Image im;
    size_t obs_off = 0, order_off = 0, disk_off = 0;
    ScalarRef th;
    VelRef vr;
    int disk_K = 0;
    std::vector<double> host_disk;
    std::vector<int64_t> obs_steps;  // n_j per image observation
    int64_t steps_per_particle_sum = 0;
    int64_t obs_begin = 0, obs_count = 0, n_particles = 0;
    int32_t precision = 0;
    double sigma = 0.0;
};
AdImage build_ad_image(const smc_ad_problem& p, const std::vector<const PreparedVelocity*>& fills,
                       const PreparedVelocity& structure, int64_t obs_begin, int64_t obs_count);
AdPrepared upload_ad_image(smc_ctx* ctx, const AdImage& A);
void check_particle_range(int64_t n_particles);
AdPrepared prepare_ad(smc_ctx* ctx, const smc_ad_problem& p, const std::vector<const PreparedVelocity*>& fills,
                      const PreparedVelocity& structure, int64_t obs_begin, int64_t obs_count);
void run_particles(smc_ctx* ctx, AdLaunch& L, const AdPrepared* P = nullptr, int64_t sample0 = 0);
// Reduce [n_seg][n] values (no failures) into estimates left on the device.
smc_estimate* reduce_ad_device(smc_ctx* ctx, const double* values, int64_t n, int64_t n_seg);
// ... and copied to the host.
void reduce_ad(smc_ctx* ctx, const double* values, int64_t n, int64_t n_seg, smc_estimate* out);
void finish_stats(smc_ctx* ctx);
void ad_observe_range(smc_ctx* ctx, const smc_ad_problem& p, uint64_t seed, int64_t obs_begin, int64_t obs_count,
                      smc_estimate* out);
BvpLaunch prepare_bvp(smc_ctx* ctx, const smc_bvp_problem& p, int64_t obs_begin, int64_t obs_count);
void run_bvp(smc_ctx* ctx, BvpLaunch& L, int64_t n_obs, int64_t n);
// Multi-device groups (capi_group.cu).  is_sharded: the context is a group of
// more than one rank, so the forward maps run sharded.
inline bool is_sharded(const smc_ctx* ctx) { return ctx->group != nullptr; }
void group_destroy(smc_ctx* ctx);
// All-gather of variable-size byte slices: rank r's slice [displ[r], +bytes[r])
// of bufs[m] (member m's device buffer) is in place on its owner; afterwards
// every member holds every slice.  Enqueued on the members' streams.
void group_exchange(smc_group* g, const std::vector<unsigned char*>& bufs, const std::vector<size_t>& displ,
                    const std::vector<size_t>& bytes);
void group_ad_observe(smc_ctx* ctx, const smc_ad_problem& p, uint64_t seed, int64_t obs_begin, int64_t obs_count,
                      smc_estimate* out);
void group_bvp_observe(smc_ctx* ctx, const smc_bvp_problem& p, uint64_t seed, int64_t obs_begin, int64_t obs_count,
                       smc_estimate* out);
// Upload a PackMap into the context's pack buffers (reused across calls).
PackDev upload_pack_map(smc_ctx* ctx, const PackMap& m);

}  // namespace smc::capi
