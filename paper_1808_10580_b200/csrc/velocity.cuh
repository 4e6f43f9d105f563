// velocity.cuh — FourierVelocityField::operator() on the device
// (src/fields.cpp:23-31, :71-89).  Included by each kernel translation unit
// so it inherits that unit's contraction mode.
//
// velocity_lattice<T>: the fast form.  Rows of constant k1;
// the +/-j pair of a row is one 8-FMA update against P2[j] = e^{2 pi i j x2}
// held in registers (tiles of 8 j); each row folds into v through
// P1[k1] = e^{2 pi i k1 x1}.  4 FMA per mode; all coefficient loads are
// warp-uniform (one L1 broadcast per warp).
//
// velocity_strict<KCAP>: the reference's own loop — power tables by complex
// recurrence, (k1,k2)-sorted mode loop, w = 2 Re(v e), v += w d.
#pragma once

#include "images.h"
#include "smc_device.cuh"

namespace smc {

constexpr int kLatticeTile = 8;

__device__ __forceinline__ void sincospi_t(double a, double* s, double* c) { sincospi(a, s, c); }
__device__ __forceinline__ void sincospi_t(float a, float* s, float* c) { sincospif(a, s, c); }

template <class T>
__device__ __forceinline__ T ldc(const double* p) {
    return static_cast<T>(__ldg(p));
}

template <class T>
__device__ __forceinline__ void velocity_lattice(const LatticeImg& L, const double* __restrict__ coef,
                                                 const double* __restrict__ row0, const double* __restrict__ g0,
                                                 T x1, T x2, T& v1, T& v2) {
    T s1, c1, s2, c2;
    sincospi_t(T(2) * x1, &s1, &c1);
    sincospi_t(T(2) * x2, &s2, &c2);
    T acc1 = T(0), acc2 = T(0);
    T qr = T(1), qi = T(0);  // P2 at the end of the previous tile
    const int R1 = L.R + 1;
    for (int t = 0; t < L.n_tiles; ++t) {
        T r[kLatticeTile], s[kLatticeTile];
#pragma unroll
        for (int q = 0; q < kLatticeTile; ++q) {
            const T nr = fma(qr, c2, -qi * s2);
            const T ni = fma(qr, s2, qi * c2);
            qr = nr;
            qi = ni;
            r[q] = nr;
            s[q] = ni;
        }
        // Row k1 = 0: modes (0, j); P1 = 1 and only Re(B) feeds v1.
        const int j0 = kLatticeTile * t;
        const int n0 = min(kLatticeTile, L.J0 - j0);
        if (n0 > 0) {
            const double2* w = reinterpret_cast<const double2*>(row0) + j0;
#pragma unroll
            for (int q = 0; q < kLatticeTile; ++q) {
                if (q < n0) {
                    const double2 c = __ldg(w + q);
                    acc1 = fma(T(c.x), r[q], acc1);
                    acc1 = fma(T(c.y), s[q], acc1);
                }
            }
        }
        T p1r = T(1), p1i = T(0);
        const int rows = __ldg(L.tile_rows + t);
        for (int k1 = 1; k1 <= rows; ++k1) {
            const T nr = fma(p1r, c1, -p1i * s1);
            p1i = fma(p1r, s1, p1i * c1);
            p1r = nr;
            const int2 tr = __ldg(L.tile_row + t * R1 + k1);
            T Ar = T(0), Ai = T(0), Br = T(0), Bi = T(0);
            if (t == 0) {
                const double2 g = __ldg(reinterpret_cast<const double2*>(g0) + k1);
                Ar = T(g.x);
                Ai = T(g.y);
            }
            const double2* c = reinterpret_cast<const double2*>(coef + tr.x);
#pragma unroll
            for (int q = 0; q < kLatticeTile; ++q) {
                if (q < tr.y) {
                    const double2 a0 = __ldg(c + 4 * q + 0);
                    const double2 a1 = __ldg(c + 4 * q + 1);
                    const double2 b0 = __ldg(c + 4 * q + 2);
                    const double2 b1 = __ldg(c + 4 * q + 3);
                    Ar = fma(T(a0.x), r[q], Ar);
                    Ai = fma(T(a1.x), r[q], Ai);
                    Br = fma(T(b0.x), r[q], Br);
                    Bi = fma(T(b1.x), r[q], Bi);
                    Ar = fma(T(a0.y), s[q], Ar);
                    Ai = fma(T(a1.y), s[q], Ai);
                    Br = fma(T(b0.y), s[q], Br);
                    Bi = fma(T(b1.y), s[q], Bi);
                }
            }
            acc2 = fma(p1r, Ar, fma(-p1i, Ai, acc2));
            acc1 = fma(p1r, Br, fma(-p1i, Bi, acc1));
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
