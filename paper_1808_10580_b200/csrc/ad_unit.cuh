// ad_unit.cuh — unit-mode indexing of K1 (kernels.h AdLaunch::unit_cpo):
// sharded single-sample launches over (observation, chunk) units.
#pragma once

#include "kernels.h"

namespace smc {

// Unit mode (kernels.h): the observation and particle of flat thread index
// `flat`; false for a thread past its observation's last particle.  The unit
// (hence the observation, its step count and the loop counter) is derived from
// the block's first index only: block sizes divide kChunk, so it is the same
// for every thread, and keeping it block-uniform keeps the step loop's counter
// in a uniform register (the disk kernel's coefficient loads depend on that,
// ad_disk.cu).
__device__ __forceinline__ bool unit_coords(const AdLaunch& L, int64_t flat, int& obs, int64_t& local) {
    const int64_t block_first = static_cast<int64_t>(blockIdx.x) * blockDim.x;
    const int64_t unit = L.unit0 + block_first / kChunk;
    const int64_t o = unit / L.unit_cpo;
    obs = static_cast<int>(o);
    local = (unit - o * L.unit_cpo) * kChunk + (flat % kChunk);
    return local < L.n_particles;
}

// Output slot of (sample, obs, local): [n_samples][n_obs][span] normally,
// values[flat] in unit mode.
__device__ __forceinline__ double* ad_out_row(const AdLaunch& L, int sample, int obs, int64_t span) {
    if (L.unit_cpo > 0)
        return L.values + static_cast<int64_t>(obs) * L.unit_cpo * kChunk - L.unit0 * kChunk;
    return L.values + (static_cast<int64_t>(sample) * L.n_obs + obs) * span;
}

}  // namespace smc
