// smc_device.cuh — device primitives of the particle forward map (sm_100a).
//
// Philox4x32-10 stream keyed exactly like the reference NormalStream
// (src/rng.cpp:13-72): key = (seed lo, seed hi), counter = (step lo, step hi,
// obs, particle), one block per Euler-Maruyama step, uniforms
// ((r >> 11) + 0.5) * 2^-53 built from words (r1:r0) and (r3:r2).  These
// functions are bit-identical to the reference on any input (integer work and
// exactly-rounded IEEE conversions); the transcendental parts (log, sin, cos)
// use CUDA's FP64 libdevice.
#pragma once

#include <cstdint>

#define SMC_HD __host__ __device__ __forceinline__

namespace smc {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

struct u32x4 {
    uint32_t x, y, z, w;
};

// Philox4x32-10 block (rng.cpp:24-41).  On the device each round is two
// IMAD.WIDE.U32 plus three LOP3 and the key bumps.
SMC_HD u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint64_t p0 = static_cast<uint64_t>(kPhiloxM0) * c.x;
        const uint64_t p1 = static_cast<uint64_t>(kPhiloxM1) * c.z;
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
        c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    return c;
}

// The same block with the 20 round keys precomputed on the host
// (k0 + r W0, k1 + r W1 for r = 0..9, mod 2^32 — identical words): when the
// keys sit in the kernel's parameter bank the XORs take them as uniform
// operands, instead of re-deriving the key schedule every step (20 uniform
// adds per block; the walker kernel is issue-bound).
struct RoundKeys {
    uint32_t k[20];
};
inline RoundKeys make_round_keys(uint64_t seed) {
    RoundKeys r;
    uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
    for (int round = 0; round < 10; ++round) {
        r.k[2 * round] = k0;
        r.k[2 * round + 1] = k1;
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    return r;
}
SMC_HD u32x4 philox4x32_10(u32x4 c, const RoundKeys& rk) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint64_t p0 = static_cast<uint64_t>(kPhiloxM0) * c.x;
        const uint64_t p1 = static_cast<uint64_t>(kPhiloxM1) * c.z;
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
        c = u32x4{hi1 ^ c.y ^ rk.k[2 * round], lo1, hi0 ^ c.w ^ rk.k[2 * round + 1], lo0};
    }
    return c;
}

// 53 random bits into (0,1): ((m) + 0.5) * 2^-53 with IEEE rounding of the
// add — bit-identical to rng.cpp:59-64.  m < 2^53, so the conversion is exact.
SMC_HD double u53_to_unit(uint64_t word) {
#ifdef __CUDA_ARCH__
    // the conversion of the 54-bit odd integer 2m + 1 is the one rounding of
    // the reference's RN(m + 0.5) (scaled by 2), and the power-of-two scale is
    // exact: I2F + DMUL by an immediate, no DADD and no constant registers
    return __dmul_rn(__ull2double_rn((word >> 10) | 1ull), 0x1p-54);
#else
    const uint64_t m = word >> 11;
    return (static_cast<double>(m) + 0.5) * 0x1p-53;
#endif
}

struct Uniform2 {
    double u0, u1;
};

// next_uniform_block for step `step` of stream (seed, obs, particle)
// (rng.cpp:53-65).
SMC_HD Uniform2 uniform_block(uint32_t k0, uint32_t k1, uint32_t obs, uint32_t particle,
                              uint64_t step) {
    const u32x4 r = philox4x32_10(
        u32x4{static_cast<uint32_t>(step), static_cast<uint32_t>(step >> 32), obs, particle}, k0, k1);
    const uint64_t a = (static_cast<uint64_t>(r.y) << 32) | r.x;
    const uint64_t b = (static_cast<uint64_t>(r.w) << 32) | r.z;
    return Uniform2{u53_to_unit(a), u53_to_unit(b)};
}

SMC_HD Uniform2 uniform_block(const RoundKeys& rk, uint32_t obs, uint32_t particle, uint64_t step) {
    const u32x4 r = philox4x32_10(
        u32x4{static_cast<uint32_t>(step), static_cast<uint32_t>(step >> 32), obs, particle}, rk);
    const uint64_t a = (static_cast<uint64_t>(r.y) << 32) | r.x;
    const uint64_t b = (static_cast<uint64_t>(r.w) << 32) | r.z;
    return Uniform2{u53_to_unit(a), u53_to_unit(b)};
}

constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 2.0 * 3.141592653589793;

// Complex helpers for the power recurrences.
struct cd {
    double re, im;
};

}  // namespace smc
