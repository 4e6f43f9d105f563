// bvp_kernels.cu — K2 exit-time walkers, fast build (FP64 parity path and the
// FP32 mode).  The kernel body is in bvp_body.cuh.
#include <cuda_runtime.h>

#include "../../include/scalarmc_b200.h"
#include "bvp_body.cuh"

namespace smc {

cudaError_t launch_bvp_walkers(const BvpLaunch& L, int n_sms, cudaStream_t s) {
    // Persistent grid: enough resident warps to hide latency on every SM.
    const unsigned long long total = static_cast<unsigned long long>(L.n_obs) * L.n_particles;
    unsigned blocks = static_cast<unsigned>(n_sms) * 8u;
    const unsigned long long need = (total + kBvpBlock - 1) / kBvpBlock;
    if (need < blocks) blocks = static_cast<unsigned>(need > 0 ? need : 1);
    if (L.precision == SMC_FP32) bvp_walkers<float, false, 0><<<blocks, kBvpBlock, 0, s>>>(L);
    else bvp_walkers<double, false, 0><<<blocks, kBvpBlock, 0, s>>>(L);
    return cudaGetLastError();
}

}  // namespace smc
