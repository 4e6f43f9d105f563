// bvp_strict.cu — K2 exit-time walkers, strict FP64 diagnostic build
// (compiled with -fmad=false): the reference's operation order throughout, so
// per-walker results differ from the reference only where CUDA's libm rounds
// differently from glibc's.
#define SMC_STRICT_TU 1
#include <cuda_runtime.h>

#include "bvp_body.cuh"

namespace smc {

cudaError_t launch_bvp_walkers_strict(const BvpLaunch& L0, int n_sms, cudaStream_t s) {
    const BvpLaunch L = with_round_keys(L0);
    const unsigned long long total = static_cast<unsigned long long>(L.n_obs) * L.n_particles;
    unsigned blocks = static_cast<unsigned>(n_sms) * 8u;
    const unsigned long long need = (total + kBvpBlock - 1) / kBvpBlock;
    if (need < blocks) blocks = static_cast<unsigned>(need > 0 ? need : 1);
    const int K = L.vel.is_constant ? 0 : L.vel.K;
    if (K <= 8) bvp_walkers<double, true, 8><<<blocks, kBvpBlock, 0, s>>>(L);
    else if (K <= 32) bvp_walkers<double, true, 32><<<blocks, kBvpBlock, 0, s>>>(L);
    else if (K <= 128) bvp_walkers<double, true, 128><<<blocks, kBvpBlock, 0, s>>>(L);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace smc
