// velocity.cuh — FourierVelocityField::operator() on the device
// (src/fields.cpp:23-31, :71-89).  Included by each kernel translation unit
// so it inherits that unit's contraction mode.
//
// velocity_lattice<T>: the fast form.  Rows of constant k1;
// the +/-j pair of a row is one 8-FMA update on 4 coefficients against
// P2[j] = e^{2 pi i j x2} and Q[j] = j P2[j] held in registers (tiles of 8 j);
// each row folds into v through P1[k1] = e^{2 pi i k1 x1}.  4 FMA per mode;
// all coefficient loads are warp-uniform broadcasts (shared memory when the
// block can stage the table, else L1).
//
// velocity_strict<KCAP>: the reference's own loop — power tables by complex
// recurrence, (k1,k2)-sorted mode loop, w = 2 Re(v e), v += w d.
#pragma once

#include <cstdint>
#include <type_traits>

#include "fastmath.cuh"
#include "images.h"
#include "smc_device.cuh"

namespace smc {

constexpr int kLatticeTile = 8;

__device__ __forceinline__ void sincospi_t(double a, double* s, double* c) { fm::sincospi(a, s, c); }
// FP32 variant (3-SE gate): reduce to [-1, 1] and use the SFU sine/cosine
// (absolute error ~2^-21 on [-pi, pi]), which moves the work off the FMA pipe
// the FP32 kernels are bound by.
__device__ __forceinline__ void sincospi_t(float a, float* s, float* c) {
    const float r = fmaf(-2.0f, rintf(0.5f * a), a);  // a - 2 round(a / 2), exact
    __sincosf(3.14159265f * r, s, c);
}
// the quadrant by FP64 adds instead of FRND/F2I (issue-bound walker kernels)
__device__ __forceinline__ void sincospi_shift(double a, double* s, double* c) { fm::sincospi<true>(a, s, c); }
__device__ __forceinline__ void sincospi_shift(float a, float* s, float* c) { sincospi_t(a, s, c); }

// Four coefficients (alpha_re, alpha_im, beta_re, beta_im) of one pair.
template <class T>
__device__ __forceinline__ void load4(const double* p, T& a, T& b, T& c, T& d) {
    const double2 x = *reinterpret_cast<const double2*>(p);
    const double2 y = *reinterpret_cast<const double2*>(p + 2);
    a = T(x.x);
    b = T(x.y);
    c = T(y.x);
    d = T(y.y);
}
template <class T>
__device__ __forceinline__ void load4(const float* p, T& a, T& b, T& c, T& d) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    a = T(x.x);
    b = T(x.y);
    c = T(x.z);
    d = T(x.w);
}
template <class T, class CT>
__device__ __forceinline__ void load2(const CT* p, T& a, T& b) {
    a = T(p[0]);
    b = T(p[1]);
}

// Packed two-lane FP32 helpers (sm_100a fma.rn.f32x2 -> SASS FFMA2).
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
// acc += c * (s, s)   (ptxas folds the broadcast into the FFMA2 operand)
__device__ __forceinline__ void f2_fma_bcast(uint64_t& acc, uint64_t c, float s) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(c), "l"(f2_pack(s, s)));
}

// Generic tiled lattice evaluation (any K, any mode set).  `cf` points to one
// sample's coefficient block (shared or global memory) in the images.h layout.
template <class T, class CT>
__device__ __forceinline__ void velocity_lattice(const LatticeImg& L, const CT* __restrict__ cf, T x1, T x2, T& v1,
                                                 T& v2) {
    T s1, c1, s2, c2;
    sincospi_t(T(2) * x1, &s1, &c1);
    sincospi_t(T(2) * x2, &s2, &c2);
    T acc1 = T(0), acc2 = T(0);
    T qr0 = T(1), qi0 = T(0);  // P2 at the end of the previous tile
    for (int t = 0; t < L.n_tiles; ++t) {
        T pr[kLatticeTile], pi[kLatticeTile], qr[kLatticeTile], qi[kLatticeTile];
#pragma unroll
        for (int q = 0; q < kLatticeTile; ++q) {
            const T nr = fma(qr0, c2, -qi0 * s2);
            const T ni = fma(qr0, s2, qi0 * c2);
            qr0 = nr;
            qi0 = ni;
            pr[q] = nr;
            pi[q] = ni;
            const T j = T(kLatticeTile * t + q + 1);
            qr[q] = j * nr;
            qi[q] = j * ni;
        }
        // Row k1 = 0: modes (0, j), P1 = 1:  v1 -= sum (g_re qr - g_im qs)
        if (kLatticeTile * t < L.J0) {
            const CT* w = cf + L.row0_off + 2 * kLatticeTile * t;
#pragma unroll
            for (int q = 0; q < kLatticeTile; ++q) {
                T gr, gi;
                load2(w + 2 * q, gr, gi);
                acc1 = fma(gr, -qr[q], acc1);
                acc1 = fma(gi, qi[q], acc1);
            }
        }
        const int2 tl = L.tiles[t];
        T p1r = c1, p1i = s1;
        const CT* c = cf + tl.y;
        for (int k1 = 1; k1 <= tl.x; ++k1, c += 4 * kLatticeTile) {
            if (k1 > 1) {
                const T nr = fma(p1r, c1, -p1i * s1);
                p1i = fma(p1r, s1, p1i * c1);
                p1r = nr;
            }
            T Ar = T(0), Ai = T(0), Br = T(0), Bi = T(0);
            if (t == 0) load2(cf + L.g0_off + 2 * k1, Ar, Ai);
            if constexpr (std::is_same<T, float>::value && std::is_same<CT, float>::value) {
                // FP32 from a float table: four FFMA2 per pair on the loaded
                // coefficient pairs (ar, ai) and (br, bi) as they sit in the
                // LDS.128 registers; the cross terms accumulate separately,
                // D = sum (br, bi) pi and E = sum (ar, ai) qi, and fold in at
                // the row end: A += (-D.y, D.x), B' += (-E.y, E.x)
                uint64_t A = f2_pack(Ar, Ai), D = f2_pack(0.0f, 0.0f), B = D, E = D;
#pragma unroll
                for (int q = 0; q < kLatticeTile; ++q) {
                    const float4 v = *reinterpret_cast<const float4*>(c + 4 * q);
                    const uint64_t c01 = f2_pack(v.x, v.y), c23 = f2_pack(v.z, v.w);
                    f2_fma_bcast(A, c01, pr[q]);
                    f2_fma_bcast(D, c23, pi[q]);
                    f2_fma_bcast(B, c23, qr[q]);
                    f2_fma_bcast(E, c01, qi[q]);
                }
                float dr, di, er, ei;
                f2_unpack(A, Ar, Ai);
                f2_unpack(D, dr, di);
                f2_unpack(B, Br, Bi);
                f2_unpack(E, er, ei);
                Ar -= di;
                Ai += dr;
                Br -= ei;
                Bi += er;
            } else {
#pragma unroll
                for (int q = 0; q < kLatticeTile; ++q) {
                    T ar, ai, br, bi;
                    load4(c + 4 * q, ar, ai, br, bi);
                    Ar = fma(ar, pr[q], Ar);
                    Ai = fma(ai, pr[q], Ai);
                    Br = fma(br, qr[q], Br);
                    Bi = fma(bi, qr[q], Bi);
                    Ar = fma(bi, -pi[q], Ar);
                    Ai = fma(br, pi[q], Ai);
                    Br = fma(ai, -qi[q], Br);
                    Bi = fma(ar, qi[q], Bi);
                }
            }
            acc2 = fma(T(k1), fma(p1r, Ar, -p1i * Ai), acc2);
            acc1 = fma(-p1r, Br, fma(p1i, Bi, acc1));
        }
    }
    v1 = acc1;
    v2 = acc2;
}

template <int KCAP>
__device__ __forceinline__ void fill_powers_strict(cd* p, double x, int n) {
    p[0] = cd{1.0, 0.0};
    if (n == 0) return;
    const double a = kTwoPi * x;
    const cd e{cos(a), sin(a)};
    p[1] = e;
    for (int j = 2; j <= n; ++j) {
        const cd q = p[j - 1];
        p[j] = cd{q.re * e.re - q.im * e.im, q.re * e.im + q.im * e.re};
    }
}

// Reference-order evaluation; p1/p2 are per-thread scratch of KCAP+1 entries.
template <int KCAP>
__device__ __forceinline__ void velocity_strict(const VelImg& V, cd* p1, cd* p2, double x1, double x2, double& v1,
                                                double& v2) {
    if (V.is_constant) {
        v1 = V.c1;
        v2 = V.c2;
        return;
    }
    v1 = 0.0;
    v2 = 0.0;
    if (V.n_modes == 0) return;
    fill_powers_strict<KCAP>(p1, x1, V.K);
    fill_powers_strict<KCAP>(p2, x2, V.K);
    for (int m = 0; m < V.n_modes; ++m) {
        const ModeImg md = V.modes[m];
        const cd pa = p1[md.k1];
        cd pb = p2[md.k2 >= 0 ? md.k2 : -md.k2];
        if (md.k2 < 0) pb.im = -pb.im;
        const cd e{pa.re * pb.re - pa.im * pb.im, pa.re * pb.im + pa.im * pb.re};
        const double w = 2.0 * (md.re * e.re - md.im * e.im);
        v1 += w * md.d1;
        v2 += w * md.d2;
    }
}

}  // namespace smc
