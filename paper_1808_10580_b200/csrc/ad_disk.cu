// ad_disk.cu — K1 specialised at compile time for the full Fourier disk
// |k| <= K (K = 1..kDiskMaxK).
//
// The lattice velocity with every loop bound known: the
// powers P2[j] = e^{2 pi i j x2} and Q[j] = j P2[j] live in registers, each
// row's +/-j pairs unroll into 8 DFMAs on 4 coefficients, and every row folds
// into v through P1[k1] = e^{2 pi i k1 x1}.  Single-sample launches pass the
// coefficient block as a kernel parameter (FP64: uniform-register operands;
// FP32: packed FFMA2 form); batched launches stage one block per parameter
// sample in shared memory and read it with broadcast vector loads at
// compile-time offsets (grid order: launch_k).  disk_shape.h layout.  Modes
// absent from the caller's field are zero coefficients; the host only picks
// this kernel when the field fills most of its disk.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>

#include "ad_body.cuh"
#include "disk_velocity.cuh"

namespace smc {
namespace {

constexpr int kBlock = 128;

// Resident 128-thread blocks per SM for the tiled disk kernels (K > kDiskMaxK):
// 3 (168 registers, no spills) beats 4 (128 registers, 80 B of spills) on C4,
// 2 770 -> 2 709 ms (profiles/r02_ab_c4_tiled_minb.log).
#ifndef SMC_TILED_MINB
#define SMC_TILED_MINB 3
#endif

using namespace disk;

// FP32 with one particle per thread stages the packed FFMA2 block
// (PackedShape) — the same arithmetic as the kernel-parameter form, so batched
// and single-sample FP32 results are identical; otherwise the compute-type
// copy of the disk_shape.h block.
template <int K, class T, int P>
constexpr bool kPackedSmem = std::is_same<T, float>::value && P == 1;
template <int K, class T, int P>
constexpr int kStagedFloats = kPackedSmem<K, T, P> ? PackedShape<K>::n_padded : DiskShape<K>::n_coef;

template <int K, class T, int P>
__device__ __forceinline__ void stage_sample(T* dst, const double* src) {
    if constexpr (kPackedSmem<K, T, P>) {
        stage_packed<K>(dst, src, threadIdx.x, kBlock);
    } else {
        for (int i = threadIdx.x; i < DiskShape<K>::n_coef; i += kBlock) dst[i] = T(src[i]);
    }
}

template <int K, class T, int P, class Body>
__device__ __forceinline__ void with_smem_coef(const T* staged, Body&& body) {
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(staged));
    if constexpr (kPackedSmem<K, T, P>) body(PackedSmemCoef<K>{base});
    else body(SmemCoef<T>{base});
}

// UNIT: unit mode (a sharded single-sample launch, kernels.h; P = 1, grid
// y = 1) — the tiled disk kernels' form for group contexts (their parameter
// form reads its coefficients by run-time row offsets: 87.8 vs 72.2 ms).
template <int K, class T, int P, int MINB, bool UNIT = false>
__global__ void __launch_bounds__(kBlock, MINB) ad_particles_disk(const AdLaunch L, const double* coef) {
    // this sample's coefficient block -> shared memory (compute type)
    __shared__ __align__(16) T staged[kStagedFloats<K, T, P>];
    const int sample = UNIT ? 0 : (L.obs_major ? blockIdx.y : blockIdx.z);
    stage_sample<K, T, P>(staged, coef + static_cast<int64_t>(sample) * DiskShape<K>::n_coef);
    __syncthreads();
    int obs = UNIT ? 0 : __ldg(L.obs_order + (L.obs_major ? blockIdx.z : blockIdx.y));
    int64_t span = L.p_end - L.p_begin;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kBlock * P + threadIdx.x;
    if (base >= span) return;
    int64_t local[P];
#pragma unroll
    for (int p = 0; p < P; ++p) local[p] = base + static_cast<int64_t>(p) * kBlock;
    if constexpr (UNIT) {
        static_assert(P == 1, "unit mode: one particle per thread");
        if (!unit_coords(L, base, obs, local[0])) return;
        span = L.n_particles;
    }
    with_smem_coef<K, T, P>(staged, [&](const auto& C) {
        auto vel = [&](const T (&x1)[P], const T (&x2)[P], T (&v1)[P], T (&v2)[P], int) {
            if constexpr (P == 1) velocity_disk_any<K, T>(C, x1, x2, v1, v2);
            else velocity_disk<K, T, P>(C, x1, x2, v1, v2);
        };
        ad_particles_p<T, P, decltype(vel)&, false, UNIT>(L, obs, sample, local, span, vel);
    });
}

// Observation-major batched launches with >= 64 particles per observation
// (pCN: 100 chains x 160 particles): the threads of one observation run over
// the flattened (sample, particle) range, so every block is full (160
// particles per sample filled one 4-warp and one 1-warp block before) and
// stages the <= 3 consecutive sample blocks its threads touch.  Warps stay
// within one sample when the particle count is a multiple of 32.
template <int K, class T, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) ad_particles_disk_flat(const AdLaunch L, const double* coef) {
    constexpr int NC = DiskShape<K>::n_coef;   // doubles per sample in `coef`
    constexpr int NS = kStagedFloats<K, T, 1>;  // staged elements per sample
    constexpr int kMaxSamples = 3;
    __shared__ __align__(16) T staged[kMaxSamples * NS];
    const int64_t span = L.p_end - L.p_begin;
    const int64_t total = span * L.n_samples;
    const int64_t flat0 = static_cast<int64_t>(blockIdx.x) * kBlock;
    const int s0 = static_cast<int>(flat0 / span);
    const int64_t last = (flat0 + kBlock < total ? flat0 + kBlock : total) - 1;
    const int ns = static_cast<int>(last / span) - s0 + 1;
    for (int q = 0; q < ns; ++q) stage_sample<K, T, 1>(staged + q * NS, coef + static_cast<int64_t>(s0 + q) * NC);
    __syncthreads();
    const int64_t flat = flat0 + threadIdx.x;
    if (flat >= total) return;
    const int sample = static_cast<int>(flat / span);
    int64_t local[1] = {flat - static_cast<int64_t>(sample) * span};
    const int obs = __ldg(L.obs_order + blockIdx.y);
    with_smem_coef<K, T, 1>(staged + (sample - s0) * NS, [&](const auto& C) {
        auto vel = [&](const T (&x1)[1], const T (&x2)[1], T (&v1)[1], T (&v2)[1], int) {
            velocity_disk_any<K, T>(C, x1, x2, v1, v2);
        };
        ad_particles_p<T, 1, decltype(vel)&, false, false>(L, obs, sample, local, span, vel);  // never unit mode
    });
}

// Single-sample launches take the coefficient block as a KERNEL PARAMETER
// (constant bank 0, per launch, so concurrent contexts cannot race): the
// DFMAs then read their coefficient through uniform registers (LDCU), which
// frees the vector register file's operand bandwidth that the shared-memory
// version spends on it (C2 36.3 -> 31.7 ms).  The loads are indexed by a
// value that is 0 but varies with the step counter, so ptxas keeps them
// inside the loop instead of hoisting ~200 coefficients into spilled
// registers.
// FP64: DiskParam<K, double> read through ParamCoef; FP32: the packed
// FFMA2 block (PackedParam, disk_velocity.cuh).
template <int K, class T>
struct ParamBlock {
    using type = DiskParam<K, double>;
};
template <int K>
struct ParamBlock<K, float> {
    using type = PackedParam<K>;
};

template <int K, class T, int MINB>
__global__ void __launch_bounds__(kBlock, MINB)
    ad_particles_disk_param(const AdLaunch L, const typename ParamBlock<K, T>::type P) {
    int obs = blockIdx.y;
    int64_t span = L.p_end - L.p_begin;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
    if (base >= span) return;
    int64_t local[1] = {base};
    if (L.unit_cpo > 0) {  // sharded launch (kernels.h unit mode)
        if (!unit_coords(L, base, obs, local[0])) return;
        span = L.n_particles;
    }
    auto vel = [&](const T (&x1)[1], const T (&x2)[1], T (&v1)[1], T (&v2)[1], int zero) {
                             if constexpr (std::is_same<T, float>::value) {
                                 const PackedCoef<K> C{P};
                                 velocity_disk<K, T, 1>(C, x1, x2, v1, v2);
                             } else {
                                 const ParamCoef<K, T> C{P, zero};
                                 velocity_disk_any<K, T>(C, x1, x2, v1, v2);
                             }
                         };
    // FP32 takes the Philox round keys from the parameter bank too; FP64 does
    // not: the keys then occupy uniform registers that the step counter needs,
    // `zero` moves to a vector register and every coefficient load becomes a
    // per-thread LDC (C2 31.7 -> 43.2 ms measured)
    ad_particles_p<T, 1, decltype(vel)&, std::is_same<T, float>::value>(L, obs, 0, local, span, vel);
}

template <int K, class T>
cudaError_t launch_param(const AdLaunch& L, cudaStream_t s) {
    static_assert(DiskShape<K>::n_coef % 2 == 0, "coefficient pairs");
    typename ParamBlock<K, T>::type P;
    if constexpr (std::is_same<T, double>::value) {
        std::memcpy(&P, L.host_disk, sizeof(P));
    } else {  // float conversion as the shared-memory staging does it; pairs expanded for FFMA2
        const double* h = L.host_disk;
        float* dst = P.c;
        for (int i = 0; i < DiskShape<K>::n_pairs; ++i) {
            const float ar = float(h[4 * i]), ai = float(h[4 * i + 1]), br = float(h[4 * i + 2]),
                        bi = float(h[4 * i + 3]);
            const float e[8] = {ar, ai, br, bi, -bi, br, -ai, ar};
            for (int q = 0; q < 8; ++q) dst[8 * i + q] = e[q];
        }
        for (int i = DiskShape<K>::row0_offset; i < DiskShape<K>::n_coef; ++i)
            dst[i + PackedShape<K>::shift] = float(h[i]);
        for (int i = PackedShape<K>::n_coef; i < PackedShape<K>::n_padded; ++i) dst[i] = 0.0f;
    }
    const int64_t span = L.p_end - L.p_begin;
    const dim3 grid(static_cast<unsigned>((span + kBlock - 1) / kBlock),
                    static_cast<unsigned>(L.unit_cpo > 0 ? 1 : L.n_obs), 1);
    AdLaunch LK = L;
    LK.rk = make_round_keys(L.seed);
    // resident blocks per SM: FP64 with 5 <= K <= 8 runs 5 (96 registers; C2
    // 31.9 -> 31.5 ms; 6 blocks at 80 registers spill: 32.3 ms); 4 below (C1
    // is a small latency-bound launch: 0.34 ms at 4, 0.36 at 5) and for FP32
    // (the packed block spills 300 B at 96 registers)
    constexpr bool kFive = std::is_same<T, double>::value && K >= 5 && K <= 8;
    constexpr int kMinB = kFive ? 5 : (K <= 8 ? 4 : (K <= kDiskMaxK ? 3 : SMC_TILED_MINB));
    ad_particles_disk_param<K, T, kMinB><<<grid, kBlock, 0, s>>>(LK, P);
    return cudaGetLastError();
}

template <class T>
cudaError_t dispatch_param(const AdLaunch& L, int K, cudaStream_t s) {
    switch (K) {
        case 1: return launch_param<1, T>(L, s);
        case 2: return launch_param<2, T>(L, s);
        case 3: return launch_param<3, T>(L, s);
        case 4: return launch_param<4, T>(L, s);
        case 5: return launch_param<5, T>(L, s);
        case 6: return launch_param<6, T>(L, s);
        case 7: return launch_param<7, T>(L, s);
        case 8: return launch_param<8, T>(L, s);
        case 9: return launch_param<9, T>(L, s);
        case 10: return launch_param<10, T>(L, s);
        case 11: return launch_param<11, T>(L, s);
        case 12: return launch_param<12, T>(L, s);
        default:
            if constexpr (std::is_same<T, double>::value) {
                if (K == 25) return launch_param<25, T>(L, s);
            }
            return cudaErrorNotSupported;
    }
}

template <int K, class T, int P, int MINB>
cudaError_t launch_k(const AdLaunch& L, const double* coef, cudaStream_t s) {
    const int64_t span = L.p_end - L.p_begin;
    const int64_t per_block = static_cast<int64_t>(kBlock) * P;
    const int64_t nb = (span + per_block - 1) / per_block;
    if constexpr (P == 1 && K > kDiskMaxK) {
        if (L.unit_cpo > 0) {
            ad_particles_disk<K, T, 1, MINB, true><<<dim3(static_cast<unsigned>(nb), 1, 1), kBlock, 0, s>>>(L, coef);
            return cudaGetLastError();
        }
    }
    AdLaunch LB = L;
    LB.obs_major = batched_obs_major(L, nb);
    if constexpr (P == 1) {
        if (LB.obs_major && span >= 64 && std::getenv("SMC_NO_FLAT") == nullptr) {
            const int64_t total = span * L.n_samples;
            const dim3 fgrid(static_cast<unsigned>((total + kBlock - 1) / kBlock), static_cast<unsigned>(L.n_obs), 1);
            ad_particles_disk_flat<K, T, MINB><<<fgrid, kBlock, 0, s>>>(LB, coef);
            return cudaGetLastError();
        }
    }
    const dim3 grid = LB.obs_major ? dim3(static_cast<unsigned>(nb), static_cast<unsigned>(L.n_samples),
                                          static_cast<unsigned>(L.n_obs))
                                   : dim3(static_cast<unsigned>(nb), static_cast<unsigned>(L.n_obs),
                                          static_cast<unsigned>(L.n_samples));
    ad_particles_disk<K, T, P, MINB><<<grid, kBlock, 0, s>>>(LB, coef);
    return cudaGetLastError();
}

// Resident blocks per SM (register budget 65536 / (128 MINB)): two particles
// per thread need ~250 registers.
template <int K, int P>
struct MinBlocks {
    static constexpr int value = P == 2 ? 2 : (K <= 8 ? 4 : (K <= kDiskMaxK ? 3 : SMC_TILED_MINB));
};

template <class T, int P>
cudaError_t dispatch_p(const AdLaunch& L, int K, const double* c, cudaStream_t s) {
    switch (K) {
        case 1: return launch_k<1, T, P, MinBlocks<1, P>::value>(L, c, s);
        case 2: return launch_k<2, T, P, MinBlocks<2, P>::value>(L, c, s);
        case 3: return launch_k<3, T, P, MinBlocks<3, P>::value>(L, c, s);
        case 4: return launch_k<4, T, P, MinBlocks<4, P>::value>(L, c, s);
        case 5: return launch_k<5, T, P, MinBlocks<5, P>::value>(L, c, s);
        case 6: return launch_k<6, T, P, MinBlocks<6, P>::value>(L, c, s);
        case 7: return launch_k<7, T, P, MinBlocks<7, P>::value>(L, c, s);
        case 8: return launch_k<8, T, P, MinBlocks<8, P>::value>(L, c, s);
        case 9: return launch_k<9, T, P, MinBlocks<9, P>::value>(L, c, s);
        case 10: return launch_k<10, T, P, MinBlocks<10, P>::value>(L, c, s);
        case 11: return launch_k<11, T, P, MinBlocks<11, P>::value>(L, c, s);
        case 12: return launch_k<12, T, P, MinBlocks<12, P>::value>(L, c, s);
        default:
            if constexpr (std::is_same<T, double>::value && P == 1) {
                if (K == 25) return launch_k<25, T, 1, MinBlocks<25, 1>::value>(L, c, s);
            }
            return cudaErrorNotSupported;
    }
}

// Particles per thread: 1 by default; SMC_DISK_P=2 lets each staged
// coefficient load feed two particles and doubles the ILP of the Box-Muller /
// sincospi chains, but halves the threads.  Measured on C2 it lands within
// +-2.5% of P=1 depending on the box, and loses on small launches (C1, pCN).
template <class T>
cudaError_t dispatch(const AdLaunch& L, int K, const double* c, cudaStream_t s) {
    const char* e = std::getenv("SMC_DISK_P");
    const int P = (e && std::atoi(e) == 2 && K <= 11) ? 2 : 1;
    return P == 1 ? dispatch_p<T, 1>(L, K, c, s) : dispatch_p<T, 2>(L, K, c, s);
}

}  // namespace

cudaError_t launch_ad_disk(const AdLaunch& L, int K, const double* coef, cudaStream_t s) {
    if (L.p_end - L.p_begin <= 0) return cudaSuccess;
    // unit mode is single-sample with a host block: the kernel-parameter path only
    if (L.unit_cpo > 0 && (L.n_samples != 1 || !L.host_disk || L.seeds)) return cudaErrorInvalidValue;
    // one coefficient block with its host copy: the kernel-parameter path
    // (SMC_DISK_P=2 keeps the shared-memory kernel, which has the P=2 form)
    const char* pe = std::getenv("SMC_DISK_P");
    // The tiled disk kernels (K > kDiskMaxK) stay in shared memory, in unit
    // mode too: their parameter form reads run-time row offsets (K = 25
    // single sample: 87.8 vs 72.2 ms; SMC_DISK_PARAM=1 selects it for A/B).
    if (L.n_samples == 1 && L.host_disk && !L.seeds &&
        (K <= kDiskMaxK || std::getenv("SMC_DISK_PARAM") != nullptr) &&
        (L.unit_cpo > 0 || K > kDiskMaxK || !(pe && std::atoi(pe) == 2)))
        return L.precision == 1 ? dispatch_param<float>(L, K, s) : dispatch_param<double>(L, K, s);
    return L.precision == 1 ? dispatch<float>(L, K, coef, s) : dispatch<double>(L, K, coef, s);
}

}  // namespace smc
