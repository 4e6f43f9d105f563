// ad_kernels.cu — K1 with the generic tiled lattice velocity (any K, any mode
// set, per-sample coefficient blocks for batched evaluation).  See
// ad_body.cuh for the particle loop and velocity.cuh for the series.
//
// Each block serves one (sample, observation) and stages that sample's
// coefficient block into shared memory once (converted to the compute type),
// so every coefficient read in the step loop is a broadcast LDS.  Tables too
// large to share an SM comfortably (> kSmemLimit) are read from global memory
// through L1 instead (they fit L1 when shared memory is not carved out).
// FP64 is the parity path; FP32 is the optional fast mode (3-SE gate).
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "ad_body.cuh"

namespace smc {
namespace {

constexpr size_t kSmemLimit = 64 * 1024;   // tables up to here: 256-thread blocks, 2 per SM
constexpr size_t kSmemMax = 220 * 1024;    // larger tables: one 512-thread block per SM
constexpr size_t kSmemHard = 227 * 1024;
constexpr int kMaxDevices = 64;
// threads of the one-block-per-SM path for large staged tables (C5)
#ifndef SMC_BIG_BLOCK
#define SMC_BIG_BLOCK 512
#endif

// UNIT: the launch is in unit mode (sharded single-sample launches,
// kernels.h); a compile-time flag so the unsharded kernel carries none of it
// (as a runtime branch it cost C5 7 %: 4634 -> 4966 ms).
template <class T, bool SMEM, int kBlock, bool OM, bool UNIT>
__global__ void __launch_bounds__(kBlock, (512 / kBlock > 0 ? 512 / kBlock : 1)) ad_particles(const AdLaunch L) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // OM: grid (particle blocks, samples, observations longest first);
    // otherwise (particle blocks, observations, samples)
    const int obs = OM ? __ldg(L.obs_order + blockIdx.z) : static_cast<int>(blockIdx.y);
    const int sample = OM ? blockIdx.y : blockIdx.z;
    const LatticeImg& lat = L.vel.lat;
    const bool is_const = L.vel.is_constant;
    const double* gblock = lat.coef + static_cast<int64_t>(sample) * lat.sample_stride;
    T* sblock = reinterpret_cast<T*>(smem_raw);
    if constexpr (SMEM) {
        if (!is_const) {
            for (int64_t i = threadIdx.x; i < lat.sample_stride; i += kBlock) sblock[i] = T(gblock[i]);
            __syncthreads();
        }
    }
    int64_t local = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
    int64_t span = L.p_end - L.p_begin;
    if (local >= span) return;
    int ob = obs;
    if constexpr (UNIT) {  // sharded launch (kernels.h unit mode)
        if (!unit_coords(L, local, ob, local)) return;
        span = L.n_particles;
    }
    const T c1 = T(L.vel.c1), c2 = T(L.vel.c2);
    ad_particle<T, UNIT>(L, ob, sample, local, span, [&](T x1, T x2, T& v1, T& v2) {
        if (is_const) {
            v1 = c1;
            v2 = c2;
        } else if constexpr (SMEM) {
            velocity_lattice<T, T>(lat, sblock, x1, x2, v1, v2);
        } else {
            velocity_lattice<T, double>(lat, gblock, x1, x2, v1, v2);
        }
    });
}

template <class T, bool SMEM, int BS, bool OM, bool UNIT>
void go_om(const AdLaunch& L, int64_t nb, size_t smem, cudaStream_t s) {
    const dim3 grid = OM ? dim3(static_cast<unsigned>(nb), static_cast<unsigned>(L.n_samples),
                                static_cast<unsigned>(L.n_obs))
                         : dim3(static_cast<unsigned>(nb), static_cast<unsigned>(L.unit_cpo > 0 ? 1 : L.n_obs),
                                static_cast<unsigned>(L.n_samples));
    if constexpr (SMEM) {
        // once per instantiation and device (the attribute is per device)
        static std::once_flag flags[kMaxDevices];
        int dev = 0;
        cudaGetDevice(&dev);
        const auto configure = [] {
            cudaFuncSetAttribute(ad_particles<T, true, BS, OM, UNIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kSmemHard));
        };
        if (dev >= 0 && dev < kMaxDevices) std::call_once(flags[dev], configure);
        else configure();
    }
    ad_particles<T, SMEM, BS, OM, UNIT><<<grid, BS, smem, s>>>(L);
}

template <class T, bool SMEM, int BS>
void go(const AdLaunch& L, int64_t span, size_t smem, cudaStream_t s) {
    const int64_t nb = (span + BS - 1) / BS;
    if (L.unit_cpo > 0) go_om<T, SMEM, BS, false, true>(L, nb, smem, s);  // single-sample: grid order moot
    else if (batched_obs_major(L, nb)) go_om<T, SMEM, BS, true, false>(L, nb, smem, s);
    else go_om<T, SMEM, BS, false, false>(L, nb, smem, s);
}

template <class T>
cudaError_t launch(const AdLaunch& L, cudaStream_t s) {
    const int64_t span = L.p_end - L.p_begin;
    if (span <= 0) return cudaSuccess;
    const size_t smem = L.vel.is_constant ? 0 : static_cast<size_t>(L.vel.lat.sample_stride) * sizeof(T);
    if (std::getenv("SMC_LATTICE_GLOBAL") != nullptr || smem > kSmemMax) go<T, false, 256>(L, span, 0, s);
    else if (smem <= kSmemLimit) go<T, true, 256>(L, span, smem, s);
    else go<T, true, SMC_BIG_BLOCK>(L, span, smem, s);
    return cudaGetLastError();
}

}  // namespace

// Batched launches: observation-major with the longest observations first
// (their blocks start in the first wave, the short ones fill the tail) when
// the grid is a few waves; sample-major otherwise, so consecutive blocks
// share a sample's coefficient block in L2.  SMC_BATCH_ORDER=obs|sample
// forces one.
int batched_obs_major(const AdLaunch& L, int64_t blocks_per_obs) {
    const char* e = std::getenv("SMC_BATCH_ORDER");
    if (e && e[0] == 'o') return 1;
    if (e && e[0] == 's') return 0;
    if (L.n_samples <= 1) return 0;
    static const int sms = [] {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 148;
    }();
    // pCN-sized launches (100 chains x 9 obs x 2 blocks = 1 800 blocks):
    // 103 vs 117 us (K=2) and 266 vs 322 us (K=8) per chain step; C4 (147 456
    // blocks) keeps the sample-major order
    const int64_t blocks = blocks_per_obs * L.n_obs * static_cast<int64_t>(L.n_samples);
    return blocks <= 32LL * sms ? 1 : 0;
}

cudaError_t launch_ad_particles(const AdLaunch& L, cudaStream_t s) { return launch<double>(L, s); }
cudaError_t launch_ad_particles_fp32(const AdLaunch& L, cudaStream_t s) { return launch<float>(L, s); }

}  // namespace smc
