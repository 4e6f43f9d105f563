// pcn_kernels.cu — device-resident multi-chain pCN (compiled with
// -fmad=false so the chain arithmetic keeps the reference's operation order).
//
// One pCN step of B chains (pcn_step, src/inference.cpp:136-166) is
//   propose (prior_draw + sqrt(1-b^2) u + b xi, prior norm of the proposal)
//   -> pack (u -> lattice coefficient blocks, velocity_from_coefficients,
//      inference.cpp:63-73, on the device)
//   -> K1 batched forward map + K3 reduction (LikelihoodSpec::misfit's
//      observe_ad, inference.cpp:93-104)
//   -> accept (Phi, the chain's uniform, min(1, e^{Phi - Phi'}), MAP tracking)
//   -> commit (state, MAP and thinned-sample copies).
// The chain randomness is each chain's own NormalStream{seed, 0xFFFFFFFF, 0}
// (inference.cpp:12, :175): the host tracks the stream's block counter and the
// uniform() cache (rng.cpp:85-94) — identical for every chain — and passes the
// block indices to the kernels, or (graph mode) the kernels derive them from a
// device step counter.
#define SMC_STRICT_TU 1
#include <cuda_runtime.h>

#include "../../include/scalarmc_b200.h"
#include "fastmath.cuh"
#include "kernels.h"
#include "smc_device.cuh"

namespace smc {
namespace {

constexpr uint32_t kChainTag = 0xFFFFFFFFu;  // inference.cpp:12

__device__ __forceinline__ void chain_normals(uint64_t seed, uint64_t block, double& z1, double& z2) {
    const Uniform2 u = uniform_block(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), kChainTag, 0u,
                                     block);
    const double r = sqrt(-2.0 * fm::log_pos(u.u0));
    double sn, cs;
    fm::sincospi(2.0 * u.u1, &sn, &cs);
    z1 = r * cs;
    z2 = r * sn;
}

// Per-step stream positions.  The host loop (capi.cu) draws M blocks per
// prior draw and one fresh uniform block every other step (the uniform()
// cache, rng.cpp:85-94), so after chain_init at block `base`:
//   blk0(it) = base + it M + ceil(it / 2),  ublk(it) = blk0(2 floor(it/2)) + M,
//   uhalf(it) = it & 1,  and the thinned-sample slot of iteration it + 1.
struct StepFields {
    uint64_t blk0, ublk;
    int32_t uhalf;
    int64_t step, sample_slot;
};

__device__ __forceinline__ StepFields step_fields(const PcnStep& S) {
    StepFields f;
    if (!S.it_dev) {
        f.blk0 = S.blk0;
        f.ublk = S.ublk;
        f.uhalf = S.uhalf;
        f.step = S.step;
        f.sample_slot = S.sample_slot;
        return f;
    }
    const int64_t it = *S.it_dev;
    const uint64_t M = static_cast<uint64_t>(S.M);
    f.blk0 = S.blk_base + static_cast<uint64_t>(it) * M + static_cast<uint64_t>((it + 1) / 2);
    const int64_t ev = it - (it & 1);
    f.ublk = S.blk_base + static_cast<uint64_t>(ev) * M + static_cast<uint64_t>((ev + 1) / 2) + M;
    f.uhalf = static_cast<int32_t>(it & 1);
    f.step = it;
    const int64_t iteration = it + 1;
    f.sample_slot = (iteration > S.burn_in && (iteration - S.burn_in - 1) % S.thin == 0)
                        ? (iteration - (S.burn_in > 0 ? S.burn_in : 0) - 1) / S.thin
                        : -1;
    return f;
}

// xi = prior_draw (stds[i] * normal(), normals pairwise, rng.cpp:74-83),
// Up = contraction * U + beta * xi (inference.cpp:141-144), and the prior
// norm 0.5 sum (Up_i / s_i)^2 (inference.cpp:75-83) in the reference's order.
__global__ void pcn_propose_kernel(PcnStep S) {
    const int64_t b = blockIdx.x;
    const uint64_t seed = S.seeds[b];
    const double* U = S.U + b * S.dim;
    double* Up = S.Up + b * S.dim;
    const uint64_t blk0 = step_fields(S).blk0;
    for (int64_t i = threadIdx.x; i < S.M; i += blockDim.x) {
        double z1, z2;
        chain_normals(seed, blk0 + static_cast<uint64_t>(i), z1, z2);
        const double s = S.stds[i];
        const double x1 = s * z1, x2 = s * z2;
        Up[2 * i] = S.contraction * U[2 * i] + S.beta * x1;
        Up[2 * i + 1] = S.contraction * U[2 * i + 1] + S.beta * x2;
    }
    __syncthreads();
    // prior norm: the squares in parallel, the sum in the reference's order
    // (one thread, shared-memory chunks) so the norm is bit-identical
    __shared__ double sq[1024];
    double acc = 0.0;
    for (int64_t base = 0; base < S.dim; base += 1024) {
        const int64_t n = S.dim - base < 1024 ? S.dim - base : 1024;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const double r = Up[base + i] / S.stds[(base + i) >> 1];
            sq[i] = r * r;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int64_t i = 0; i < n; ++i) acc += sq[i];
        __syncthreads();
    }
    if (threadIdx.x == 0) S.norm_prop[b] = 0.5 * acc;
}

// velocity_from_coefficients -> coefficient blocks through the host-built
// gather map (host_problem.h PackMap): the operations of lattice_fill /
// disk_fill, uncontracted (this TU is -fmad=false), so the blocks equal the
// host-filled ones bit for bit.  A non-finite coefficient raises *bad (the
// FourierVelocityField ctor check, fields.cpp:46-47).
__global__ void pcn_pack_kernel(PackDev M, const double* __restrict__ Up, int64_t dim, int64_t n_samples,
                                double* __restrict__ blocks, int* bad) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= M.stride) return;
    for (int64_t b = blockIdx.y; b < n_samples; b += gridDim.y) {  // gridDim.y <= 65535
    const double* u = Up + b * dim;
    const int32_t a = M.ip[q], c = M.im[q];
    const int ms = M.ms[q];
    double v = 0.0;
    if (a >= 0) {
        const double x = u[a];
        if (bad && !isfinite(x)) *bad = 1;
        v = 2.0 * x / M.kp[q];
    }
    if (ms != 0) {
        double g = 0.0;
        if (c >= 0) {
            const double x = u[c];
            if (bad && !isfinite(x)) *bad = 1;
            g = 2.0 * x / M.km[q];
        }
        v = ms > 0 ? v + g : v - g;
    }
    blocks[b * M.stride + q] = v;
    }
}

// misfit (inference.cpp:98-103), the chain's uniform, the accept rule
// (inference.cpp:154-165) and MAP tracking (inference.cpp:117-123).
__global__ void pcn_accept_kernel(PcnStep S, const smc_estimate* __restrict__ est) {
    const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= S.n_chains) return;
    double phi_prop = 0.0;
    if (!S.noise_inf) {
        double ss = 0.0;
        for (int64_t j = 0; j < S.n_obs; ++j) {
            const double r = S.data[j] - est[b * S.n_obs + j].mean;
            ss += r * r;
        }
        phi_prop = ss / (2.0 * S.noise_std * S.noise_std);
    }
    const StepFields F = step_fields(S);
    bool accept = false;
    if (S.init) {  // chain_init: the state is the proposal
        accept = true;
    } else {
        const Uniform2 u = uniform_block(static_cast<uint32_t>(S.seeds[b]), static_cast<uint32_t>(S.seeds[b] >> 32),
                                         kChainTag, 0u, F.ublk);
        const double uacc = F.uhalf ? u.u1 : u.u0;
        if (isfinite(phi_prop)) accept = uacc < exp(fmin(0.0, S.phi[b] - phi_prop));
    }
    if (accept) {
        S.phi[b] = phi_prop;
        S.norm_cur[b] = S.norm_prop[b];
        if (!S.init) S.accepted[b] += 1;
    }
    S.acc_flag[b] = accept ? 1 : 0;
    const double objective = S.phi[b] + S.norm_cur[b];
    const bool better = S.init || objective < S.map_obj[b];
    if (better) S.map_obj[b] = objective;
    S.map_flag[b] = better ? 1 : 0;
    if (!S.init && S.phi_trace) S.phi_trace[b * S.n_steps + F.step] = S.phi[b];
}

__global__ void pcn_commit_kernel(PcnStep S) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= S.dim) return;
    const int64_t slot = step_fields(S).sample_slot;
    for (int64_t b = blockIdx.y; b < S.n_chains; b += gridDim.y) {  // gridDim.y <= 65535
        double* U = S.U + b * S.dim;
        if (S.acc_flag[b]) U[i] = S.Up[b * S.dim + i];
        if (S.map_flag[b]) S.map_u[b * S.dim + i] = U[i];
        if (slot >= 0 && S.samples) S.samples[(b * S.n_samples + slot) * S.dim + i] = U[i];
    }
}

__global__ void pcn_advance_kernel(int64_t* it) { *it += 1; }

}  // namespace

cudaError_t launch_pcn_propose(const PcnStep& S, cudaStream_t s) {
    pcn_propose_kernel<<<static_cast<unsigned>(S.n_chains), 128, 0, s>>>(S);
    return cudaGetLastError();
}

cudaError_t launch_pack(const PackDev& M, const double* Up, int64_t dim, int64_t n_samples, double* blocks, int* bad,
                        cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((M.stride + 255) / 256),
                    static_cast<unsigned>(n_samples < 65535 ? n_samples : 65535));
    pcn_pack_kernel<<<grid, 256, 0, s>>>(M, Up, dim, n_samples, blocks, bad);
    return cudaGetLastError();
}

cudaError_t launch_pcn_accept(const PcnStep& S, const void* est, cudaStream_t s) {
    pcn_accept_kernel<<<static_cast<unsigned>((S.n_chains + 127) / 128), 128, 0, s>>>(
        S, static_cast<const smc_estimate*>(est));
    return cudaGetLastError();
}

cudaError_t launch_pcn_advance(int64_t* it_dev, cudaStream_t s) {
    pcn_advance_kernel<<<1, 1, 0, s>>>(it_dev);
    return cudaGetLastError();
}

cudaError_t launch_pcn_commit(const PcnStep& S, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((S.dim + 255) / 256),
                    static_cast<unsigned>(S.n_chains < 65535 ? S.n_chains : 65535));
    pcn_commit_kernel<<<grid, 256, 0, s>>>(S);
    return cudaGetLastError();
}

}  // namespace smc
