// disk_velocity.cuh — the lattice velocity series for the full Fourier disk
// |k| <= K with every loop bound known at compile time:
// P2[j] = e^{2 pi i j x2} and Q[j] = j P2[j] in registers, each row's +/-j
// pairs unrolled into 8 DFMAs on 4 coefficients, every row folded into v
// through P1[k1] = e^{2 pi i k1 x1}.  Coefficients come from a block staged
// in shared memory (disk_shape.h layout), read with broadcast vector loads at
// compile-time offsets.  Used by K1 (ad_disk.cu) and the Dirichlet walkers
// (bvp_disk.cu).
#pragma once

#include <type_traits>
#include <utility>

#include "disk_shape.h"
#include "velocity.cuh"

namespace smc {
namespace disk {


// Coefficients staged in shared memory, read with volatile vector loads at
// compile-time offsets: one LDS.128 (broadcast) per two coefficients, kept
// inside the step loop (3-6 KB of loop-invariant values cannot live in
// registers, and hoisting part of them only produces register shuffles).
template <class T>
struct SmemCoef {
    uint32_t base;
    template <int O>
    __device__ __forceinline__ void get2(T& a, T& b) const;
};
template <>
template <int O>
__device__ __forceinline__ void SmemCoef<double>::get2(double& a, double& b) const {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(a), "=d"(b) : "r"(base), "n"(O * 8));
}
template <>
template <int O>
__device__ __forceinline__ void SmemCoef<float>::get2(float& a, float& b) const {
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2+%3];" : "=f"(a), "=f"(b) : "r"(base), "n"(O * 4));
}

// Coefficient block passed BY VALUE as a kernel parameter (constant bank 0):
// the DFMAs then take each coefficient from a uniform register (LDCU) instead
// of a vector register, freeing register-file operand bandwidth.  `zero` is 0
// but depends on a loop counter, so ptxas keeps the loads inside the loop
// instead of hoisting the whole block into (spilled) registers.
template <int K>
struct alignas(16) DiskParam {
    double2 c[DiskShape<K>::n_coef / 2];
};
template <int K, class T>
struct ParamCoef {
    const DiskParam<K>& P;
    int zero;  // 0, but loop-variant: keeps the loads inside the step loop
    template <int O>
    __device__ __forceinline__ void get2(T& a, T& b) const {
        const double2 v = P.c[zero + O / 2];
        a = T(v.x);
        b = T(v.y);
    }
};

struct NoDiskParam {};

template <int K, class T, int P>
struct Powers {
    T pr[P][K + 1], pi[P][K + 1];  // P2[j]
    T qr[P][K + 1], qi[P][K + 1];  // Q[j] = j P2[j]
};

template <int P, class T>
struct RowAcc {
    T Ar[P], Ai[P], Br[P], Bi[P];
};

// One (k1, +/-j) pair, alpha = g(k1,j) + g(k1,-j), beta = g(k1,j) - g(k1,-j):
//   A  += (ar r - bi s) + i (ai r + br s)
//   B' += (br qr - ai qs) + i (bi qr + ar qs)
template <int K, int K1, int J, class T, int P, class CA>
__device__ __forceinline__ void disk_pair(const CA& C, const Powers<K, T, P>& W, RowAcc<P, T>& a) {
    constexpr int o = 4 * (DiskShape<K>::pair_offset(K1) + J - 1);
    T ar, ai, br, bi;
    C.template get2<o>(ar, ai);
    C.template get2<o + 2>(br, bi);
#pragma unroll
    for (int p = 0; p < P; ++p) {
        a.Ar[p] = fma(ar, W.pr[p][J], a.Ar[p]);
        a.Ai[p] = fma(ai, W.pr[p][J], a.Ai[p]);
        a.Br[p] = fma(br, W.qr[p][J], a.Br[p]);
        a.Bi[p] = fma(bi, W.qr[p][J], a.Bi[p]);
        a.Ar[p] = fma(bi, -W.pi[p][J], a.Ar[p]);
        a.Ai[p] = fma(br, W.pi[p][J], a.Ai[p]);
        a.Br[p] = fma(ai, -W.qi[p][J], a.Br[p]);
        a.Bi[p] = fma(ar, W.qi[p][J], a.Bi[p]);
    }
}

template <int K, int K1, class T, int P, class CA, int... Js>
__device__ __forceinline__ void disk_row_pairs(const CA& C, const Powers<K, T, P>& W, RowAcc<P, T>& a,
                                               std::integer_sequence<int, Js...>) {
    (disk_pair<K, K1, Js + 1, T, P>(C, W, a), ...);
}

// Harmonics e^{i k theta} for k = 2..K.  FP64: the Chebyshev recurrence
// X_k = 2 cos(theta) X_{k-1} - X_{k-2} (2 DFMA per k instead of the 4 of a
// complex multiply; rounding error grows like eps k^2 — 1e-14 at k = 12,
// 1e-12 at k = 80, far inside the 1e-10 parity gate).  FP32 keeps the complex
// product (eps k^2 would be 4e-4 at k = 80).
template <class T>
constexpr bool kChebyshev = std::is_same<T, double>::value;

// Row k1 >= 1: P1 <- P1 e1 (k1 > 1), row sums A and B', then
//   v2 += k1 Re(P1 A),  v1 -= Re(P1 B').  (q1r, q1i) = P1[k1 - 1] for the
//   recurrence, tc1 = 2 cos(theta1).
template <int K, int K1, class T, int P, class CA>
__device__ __forceinline__ void disk_row(const CA& C, const Powers<K, T, P>& W, const T (&c1)[P],
                                         const T (&s1)[P], const T (&tc1)[P], T (&p1r)[P], T (&p1i)[P],
                                         T (&q1r)[P], T (&q1i)[P], T (&acc1)[P], T (&acc2)[P]) {
    using S = DiskShape<K>;
    if constexpr (K1 > 1) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            if constexpr (kChebyshev<T>) {
                const T nr = fma(tc1[p], p1r[p], -q1r[p]);
                const T ni = fma(tc1[p], p1i[p], -q1i[p]);
                q1r[p] = p1r[p];
                q1i[p] = p1i[p];
                p1r[p] = nr;
                p1i[p] = ni;
            } else {
                const T nr = fma(p1r[p], c1[p], -p1i[p] * s1[p]);
                p1i[p] = fma(p1r[p], s1[p], p1i[p] * c1[p]);
                p1r[p] = nr;
            }
        }
    }
    T g0r, g0i;
    C.template get2<S::g0_offset + 2 * (K1 - 1)>(g0r, g0i);
    RowAcc<P, T> a;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        a.Ar[p] = g0r;
        a.Ai[p] = g0i;
        a.Br[p] = T(0);
        a.Bi[p] = T(0);
    }
    disk_row_pairs<K, K1, T, P>(C, W, a, std::make_integer_sequence<int, S::jmax(K1)>{});
#pragma unroll
    for (int p = 0; p < P; ++p) {
        acc2[p] = fma(T(K1), fma(p1r[p], a.Ar[p], -p1i[p] * a.Ai[p]), acc2[p]);
        acc1[p] = fma(-p1r[p], a.Br[p], fma(p1i[p], a.Bi[p], acc1[p]));
    }
}

template <int K, class T, int P, class CA, int... K1s>
__device__ __forceinline__ void disk_rows(const CA& C, const Powers<K, T, P>& W, const T (&c1)[P],
                                          const T (&s1)[P], T (&acc1)[P], T (&acc2)[P],
                                          std::integer_sequence<int, K1s...>) {
    T p1r[P], p1i[P], q1r[P], q1i[P], tc1[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        p1r[p] = c1[p];
        p1i[p] = s1[p];
        q1r[p] = T(1);
        q1i[p] = T(0);
        tc1[p] = T(2) * c1[p];
    }
    (disk_row<K, K1s + 1, T, P>(C, W, c1, s1, tc1, p1r, p1i, q1r, q1i, acc1, acc2), ...);
}

// Row k1 = 0: modes (0, j) only (g- = 0), P1 = 1: v1 = -sum (g_re qr - g_im qs).
template <int K, int J, class T, int P, class CA>
__device__ __forceinline__ void disk_row0_term(const CA& C, const Powers<K, T, P>& W, T (&a0)[P],
                                               T (&a1)[P]) {
    T gr, gi;
    C.template get2<DiskShape<K>::row0_offset + 2 * J>(gr, gi);
#pragma unroll
    for (int p = 0; p < P; ++p) {
        a0[p] = fma(gr, -W.qr[p][J + 1], a0[p]);
        a1[p] = fma(gi, W.qi[p][J + 1], a1[p]);
    }
}

template <int K, class T, int P, class CA, int... Js>
__device__ __forceinline__ void disk_row0(const CA& C, const Powers<K, T, P>& W, T (&acc1)[P],
                                          std::integer_sequence<int, Js...>) {
    T a0[P], a1[P];
#pragma unroll
    for (int p = 0; p < P; ++p) a0[p] = a1[p] = T(0);
    (disk_row0_term<K, Js, T, P>(C, W, a0, a1), ...);
#pragma unroll
    for (int p = 0; p < P; ++p) acc1[p] = a0[p] + a1[p];
}

template <int K, class T, int P, class CA>
__device__ __forceinline__ void velocity_disk(const CA& C, const T (&x1)[P], const T (&x2)[P], T (&v1)[P],
                                              T (&v2)[P]) {
    T s1[P], c1[P];
    Powers<K, T, P> W;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        T s2, c2;
        sincospi_t(T(2) * x1[p], &s1[p], &c1[p]);
        sincospi_t(T(2) * x2[p], &s2, &c2);
        W.pr[p][1] = c2;
        W.pi[p][1] = s2;
        if constexpr (kChebyshev<T>) {
            const T tc = T(2) * c2;
            T rm = T(1), im = T(0);  // P2[j - 2]
#pragma unroll
            for (int j = 2; j <= K; ++j) {
                const T nr = fma(tc, W.pr[p][j - 1], -rm), ni = fma(tc, W.pi[p][j - 1], -im);
                rm = W.pr[p][j - 1];
                im = W.pi[p][j - 1];
                W.pr[p][j] = nr;
                W.pi[p][j] = ni;
            }
        } else {
            // P2[j] = P2[j/2] P2[j - j/2]: dependency depth log2(K) instead of K
#pragma unroll
            for (int j = 2; j <= K; ++j) {
                const int a = j / 2, b = j - j / 2;
                W.pr[p][j] = fma(W.pr[p][a], W.pr[p][b], -W.pi[p][a] * W.pi[p][b]);
                W.pi[p][j] = fma(W.pr[p][a], W.pi[p][b], W.pi[p][a] * W.pr[p][b]);
            }
        }
        W.qr[p][1] = c2;
        W.qi[p][1] = s2;
#pragma unroll
        for (int j = 2; j <= K; ++j) {
            W.qr[p][j] = T(j) * W.pr[p][j];
            W.qi[p][j] = T(j) * W.pi[p][j];
        }
    }
    T acc1[P], acc2[P];
    disk_row0<K, T, P>(C, W, acc1, std::make_integer_sequence<int, K>{});
#pragma unroll
    for (int p = 0; p < P; ++p) acc2[p] = T(0);
    disk_rows<K, T, P>(C, W, c1, s1, acc1, acc2, std::make_integer_sequence<int, K>{});
#pragma unroll
    for (int p = 0; p < P; ++p) {
        v1[p] = acc1[p];
        v2[p] = acc2[p];
    }
}

}  // namespace disk
}  // namespace smc
