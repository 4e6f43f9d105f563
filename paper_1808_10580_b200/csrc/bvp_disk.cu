// bvp_disk.cu — K2 exit-time walkers with the compile-time disk velocity
// series (disk_velocity.cuh) for dense Fourier fields |k| <= K, K = 1..12:
// the Dirichlet problem with a C2-like velocity is FP64-bound in the series
// just like K1, and the runtime-tiled lattice loop reads its coefficients
// through L1 instead of broadcast shared-memory vector loads (C3b: 1.06e10
// -> 1.53e10 walker-steps/s).  Generic forcing evaluator (NB = 0: a 3-bump
// specialisation measured only 5 % more); FP64 fast path only.
#include <cuda_runtime.h>

#include "bvp_body.cuh"

namespace smc {

cudaError_t launch_bvp_disk(const BvpLaunch& L0, unsigned blocks, cudaStream_t s) {
    const BvpLaunch L = with_round_keys(L0);
    switch (L.disk_K) {
#define SMC_BVP_DISK_CASE(K) \
    case K: bvp_walkers<double, false, 0, 0, 0, false, K><<<blocks, kBvpBlock, 0, s>>>(L); break;
        SMC_BVP_DISK_CASE(1)
        SMC_BVP_DISK_CASE(2)
        SMC_BVP_DISK_CASE(3)
        SMC_BVP_DISK_CASE(4)
        SMC_BVP_DISK_CASE(5)
        SMC_BVP_DISK_CASE(6)
        SMC_BVP_DISK_CASE(7)
        SMC_BVP_DISK_CASE(8)
        SMC_BVP_DISK_CASE(9)
        SMC_BVP_DISK_CASE(10)
        SMC_BVP_DISK_CASE(11)
        SMC_BVP_DISK_CASE(12)
#undef SMC_BVP_DISK_CASE
        default: return cudaErrorNotSupported;
    }
    return cudaGetLastError();
}

}  // namespace smc
