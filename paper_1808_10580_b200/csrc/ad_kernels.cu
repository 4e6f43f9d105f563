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

#include "ad_body.cuh"

namespace smc {
namespace {

constexpr size_t kSmemLimit = 64 * 1024;   // tables up to here: 256-thread blocks, 2 per SM
constexpr size_t kSmemMax = 220 * 1024;    // larger tables: one 512-thread block per SM
constexpr size_t kSmemHard = 227 * 1024;

template <class T, bool SMEM, int kBlock>
__global__ void __launch_bounds__(kBlock, 512 / kBlock) ad_particles(const AdLaunch L) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int obs = blockIdx.y;
    const int sample = blockIdx.z;
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
    const int64_t local = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const int64_t span = L.p_end - L.p_begin;
    if (local >= span) return;
    const T c1 = T(L.vel.c1), c2 = T(L.vel.c2);
    ad_particle<T>(L, obs, sample, local, span, [&](T x1, T x2, T& v1, T& v2) {
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

template <class T, bool SMEM, int BS>
void go(const AdLaunch& L, int64_t span, size_t smem, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((span + BS - 1) / BS), static_cast<unsigned>(L.n_obs),
                    static_cast<unsigned>(L.n_samples));
    if constexpr (SMEM) {
        static bool configured = false;
        if (!configured) {
            cudaFuncSetAttribute(ad_particles<T, true, BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kSmemHard));
            configured = true;
        }
    }
    ad_particles<T, SMEM, BS><<<grid, BS, smem, s>>>(L);
}

template <class T>
cudaError_t launch(const AdLaunch& L, cudaStream_t s) {
    const int64_t span = L.p_end - L.p_begin;
    if (span <= 0) return cudaSuccess;
    const size_t smem = L.vel.is_constant ? 0 : static_cast<size_t>(L.vel.lat.sample_stride) * sizeof(T);
    if (std::getenv("SMC_LATTICE_GLOBAL") != nullptr || smem > kSmemMax) go<T, false, 256>(L, span, 0, s);
    else if (smem <= kSmemLimit) go<T, true, 256>(L, span, smem, s);
    else go<T, true, 512>(L, span, smem, s);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_ad_particles(const AdLaunch& L, cudaStream_t s) { return launch<double>(L, s); }
cudaError_t launch_ad_particles_fp32(const AdLaunch& L, cudaStream_t s) { return launch<float>(L, s); }

}  // namespace smc
