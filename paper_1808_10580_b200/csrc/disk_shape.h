// disk_shape.h — compile-time lattice of the full Fourier disk |k| <= K.
//
// For the specialised K1 kernel (ad_disk.cu) every (k1, +/-j) pair of the disk
// is known at compile time, so the whole velocity series unrolls into
// straight-line DFMAs whose coefficient operands come from the kernel's
// parameter bank (constant bank 0) — no loads, no index arithmetic, no
// predication.  Layout of the coefficient block (doubles):
//   pairs:  for k1 = 1..K, j = 1..jmax(k1): (alpha_re, alpha_im, beta_re,
//           beta_im), alpha = g(k1,j) + g(k1,-j), beta = g(k1,j) - g(k1,-j)
//   row0:   for j = 1..K: g(0, j) (re, im)
//   g0:     for k1 = 1..K: g(k1, 0) (re, im)
// with g = 2 c / |k|.
// Shared by the host packer (capi.cu) and the kernels.
#pragma once

namespace smc {

template <int K>
struct DiskShape {
    static constexpr int jmax(int k1) {
        int j = 0;
        while ((j + 1) * (j + 1) + k1 * k1 <= K * K) ++j;
        return j;
    }
    static constexpr int pair_offset(int k1) {  // first pair of row k1 (k1 >= 1)
        int s = 0;
        for (int r = 1; r < k1; ++r) s += jmax(r);
        return s;
    }
    static constexpr int n_pairs = pair_offset(K + 1);
    static constexpr int row0_offset = 4 * n_pairs;
    static constexpr int g0_offset = row0_offset + 2 * K;
    static constexpr int n_coef = g0_offset + 2 * K;
    static constexpr int n_modes = 2 * n_pairs + K + K;  // (k1,+-j) pairs, (0,j), (k1,0)
};

// Largest K with the register-resident disk kernel.
constexpr int kDiskMaxK = 12;
// Tiled compile-time disk kernels (disk_velocity.cuh velocity_disk_tiled,
// FP64 K1 only) exist for these K above kDiskMaxK.
inline bool disk_tiled_instantiated(int K) { return K == 25; }
// Whether K1 has a compile-time disk kernel for a dense field of cutoff K.
inline bool disk_kernel_for(int K, bool fp64) { return K <= kDiskMaxK || (fp64 && disk_tiled_instantiated(K)); }

inline int disk_jmax(int K, int k1) {
    int j = 0;
    while ((j + 1) * (j + 1) + k1 * k1 <= K * K) ++j;
    return j;
}
inline int disk_n_pairs(int K) {
    int s = 0;
    for (int r = 1; r <= K; ++r) s += disk_jmax(K, r);
    return s;
}
inline int disk_n_coef(int K) { return 4 * disk_n_pairs(K) + 4 * K; }
inline int disk_n_modes(int K) { return 2 * disk_n_pairs(K) + 2 * K; }

}  // namespace smc
