// disk_velocity.cuh — the lattice velocity series for the full Fourier disk
// |k| <= K with every loop bound known at compile time:
// P2[j] = e^{2 pi i j x2} and Q[j] = j P2[j] in registers, each row's +/-j
// pairs unrolled into 8 DFMAs on 4 coefficients, every row folded into v
// through P1[k1] = e^{2 pi i k1 x1}.  The coefficient accessor is a template
// parameter: a block staged in shared memory (SmemCoef, broadcast vector
// loads at compile-time offsets), the kernel-parameter block read through
// uniform registers (ParamCoef, FP64), or the packed FP32 block whose pair
// updates are FFMA2s (PackedCoef).  Used by K1 (ad_disk.cu) and the Dirichlet
// walkers (bvp_disk.cu).
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
// The same block seen from a runtime offset of `off` elements (a row base in
// the tiled disk kernel's row loop).
template <class T>
__device__ __forceinline__ SmemCoef<T> shifted(const SmemCoef<T>& C, int off) {
    return SmemCoef<T>{C.base + static_cast<uint32_t>(off) * static_cast<uint32_t>(sizeof(T))};
}
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
// Four consecutive coefficients (O a multiple of 4): one 16-byte load for
// FP32, two for FP64.
template <int O, class T, class CA>
__device__ __forceinline__ void get4(const CA& C, T& a, T& b, T& c, T& d) {
    C.template get2<O>(a, b);
    C.template get2<O + 2>(c, d);
}
template <int O>
__device__ __forceinline__ void get4(const SmemCoef<float>& C, float& a, float& b, float& c, float& d) {
    static_assert(O % 4 == 0, "16-byte aligned");
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
                 : "r"(C.base), "n"(O * 4));
}

// Coefficient block passed BY VALUE as a kernel parameter (constant bank 0):
// the DFMAs then take each coefficient from a uniform register (LDCU) instead
// of a vector register, freeing register-file operand bandwidth.  `zero` is 0
// but depends on a loop counter, so ptxas keeps the loads inside the loop
// instead of hoisting the whole block into (spilled) registers.
// The block is stored in the compute type (FP32 launches convert it once on
// the host, exactly as the shared-memory staging does on the device).
template <class T>
struct Vec2Of;
template <>
struct Vec2Of<double> {
    using type = double2;
};
template <>
struct Vec2Of<float> {
    using type = float2;
};
template <int K, class T = double>
struct alignas(16) DiskParam {
    typename Vec2Of<T>::type c[DiskShape<K>::n_coef / 2];
};
template <int K, class T>
struct ParamCoef {
    const DiskParam<K, T>& P;
    int zero;  // 0, but loop-variant: keeps the loads inside the step loop
    // FP64 indexes by `zero` (LDCU.64 from a uniform-register address); FP32
    // uses immediate offsets, which ptxas turns into LDCU.128 (four
    // coefficients per issue slot — the FP32 kernel is issue-bound) and can
    // afford: hoisting part of the float block spills nothing, while the
    // double block spills at every K >= 4.
    template <int O>
    __device__ __forceinline__ void get2(T& a, T& b) const {
        const auto v = P.c[(std::is_same<T, double>::value ? zero : 0) + O / 2];
        a = v.x;
        b = v.y;
    }
};

template <int K, class T>
__device__ __forceinline__ ParamCoef<K, T> shifted(const ParamCoef<K, T>& C, int off) {  // off even
    return ParamCoef<K, T>{C.P, C.zero + off / 2};
}

template <int O, int K>
__device__ __forceinline__ void get4(const ParamCoef<K, float>& C, float& a, float& b, float& c, float& d) {
    static_assert(O % 4 == 0, "16-byte aligned");
    const float4 v = reinterpret_cast<const float4*>(C.P.c)[O / 4];
    a = v.x;
    b = v.y;
    c = v.z;
    d = v.w;
}

// FP32 packed form (FFMA2, sm_100a's fma.rn.f32x2): the pair update is four
// two-lane FMAs, (Ar, Ai) += (ar, ai) pr + (-bi, br) pi and
// (Br, Bi) += (br, bi) qr + (-ai, ar) qi, each taking a coefficient pair
// from a uniform register and the power as a broadcast scalar.  Per lane
// it is the same FMA sequence as the scalar form (identical results) in
// half the issue slots; the FP32 kernel is issue-bound, FFMA2 runs at the
// FFMA flop rate (tools/ubench_ffma2.cu).  The block stores each pair as
// (ar, ai, br, bi, -bi, br, -ai, ar); row0 and g0 follow as in disk_shape.h.
template <int K>
struct PackedShape {
    static constexpr int n_pairs = DiskShape<K>::n_pairs;
    static constexpr int shift = 4 * n_pairs;  // extra floats before row0
    static constexpr int n_coef = DiskShape<K>::n_coef + shift;
    static constexpr int n_padded = (n_coef + 3) / 4 * 4;
};
template <int K>
struct alignas(16) PackedParam {
    float c[PackedShape<K>::n_padded];
};
template <int K>
struct PackedCoef {
    const PackedParam<K>& P;
    template <int O>  // O: offset in the disk_shape.h layout (row0 / g0 only)
    __device__ __forceinline__ void get2(float& a, float& b) const {
        static_assert(O >= DiskShape<K>::row0_offset, "pairs use pair4");
        a = P.c[O + PackedShape<K>::shift];
        b = P.c[O + PackedShape<K>::shift + 1];
    }
    template <int I>  // the I-th pair's four coefficient pairs
    __device__ __forceinline__ void pair4(uint64_t& c0, uint64_t& c1, uint64_t& c2, uint64_t& c3) const {
        const ulonglong2* q = reinterpret_cast<const ulonglong2*>(P.c) + 2 * I;
        const ulonglong2 u = q[0], v = q[1];
        c0 = u.x;
        c1 = u.y;
        c2 = v.x;
        c3 = v.y;
    }
};
// The same packed block staged in shared memory (batched FP32 launches).
template <int K>
struct PackedSmemCoef {
    uint32_t base;  // shared-memory address of this sample's packed block
    template <int O>  // O: offset in the disk_shape.h layout (row0 / g0 only)
    __device__ __forceinline__ void get2(float& a, float& b) const {
        static_assert(O >= DiskShape<K>::row0_offset, "pairs use pair4");
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2+%3];"
                     : "=f"(a), "=f"(b)
                     : "r"(base), "n"((O + PackedShape<K>::shift) * 4));
    }
    template <int I>
    __device__ __forceinline__ void pair4(uint64_t& c0, uint64_t& c1, uint64_t& c2, uint64_t& c3) const {
        asm volatile("ld.shared.v2.u64 {%0, %1}, [%2+%3];" : "=l"(c0), "=l"(c1) : "r"(base), "n"(I * 32));
        asm volatile("ld.shared.v2.u64 {%0, %1}, [%2+%3];" : "=l"(c2), "=l"(c3) : "r"(base), "n"(I * 32 + 16));
    }
};
// Stage one sample's packed FP32 block (PackedShape layout) from its
// disk_shape.h double block; all threads of the block cooperate.
template <int K>
__device__ __forceinline__ void stage_packed(float* dst, const double* src, int tid, int nthreads) {
    for (int i = tid; i < DiskShape<K>::n_pairs; i += nthreads) {
        const float ar = float(src[4 * i]), ai = float(src[4 * i + 1]), br = float(src[4 * i + 2]),
                    bi = float(src[4 * i + 3]);
        float4* q = reinterpret_cast<float4*>(dst + 8 * i);
        q[0] = make_float4(ar, ai, br, bi);
        q[1] = make_float4(-bi, br, -ai, ar);
    }
    for (int i = DiskShape<K>::row0_offset + tid; i < DiskShape<K>::n_coef; i += nthreads)
        dst[i + PackedShape<K>::shift] = float(src[i]);
}

template <class CA>
struct IsPacked : std::false_type {};
template <int K>
struct IsPacked<PackedCoef<K>> : std::true_type {};
template <int K>
struct IsPacked<PackedSmemCoef<K>> : std::true_type {};

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
    get4<o>(C, ar, ai, br, bi);
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

template <int K, int K1, int J, class CA, class W_t>
__device__ __forceinline__ void disk_pair_packed(const CA& C, const W_t& W, uint64_t& A, uint64_t& B) {
    uint64_t c0, c1, c2, c3;
    C.template pair4<DiskShape<K>::pair_offset(K1) + J - 1>(c0, c1, c2, c3);
    f2_fma_bcast(A, c0, W.pr[0][J]);
    f2_fma_bcast(B, c1, W.qr[0][J]);
    f2_fma_bcast(A, c2, W.pi[0][J]);
    f2_fma_bcast(B, c3, W.qi[0][J]);
}

template <int K, int K1, class CA, class W_t, int... Js>
__device__ __forceinline__ void disk_row_pairs_packed(const CA& C, const W_t& W, uint64_t& A, uint64_t& B,
                                                      std::integer_sequence<int, Js...>) {
    (disk_pair_packed<K, K1, Js + 1>(C, W, A, B), ...);
}

template <int K, int K1, class T, int P, class CA, int... Js>
__device__ __forceinline__ void disk_row_pairs(const CA& C, const Powers<K, T, P>& W, RowAcc<P, T>& a,
                                               std::integer_sequence<int, Js...>) {
    (disk_pair<K, K1, Js + 1, T, P>(C, W, a), ...);
}

// Harmonics e^{i k theta} for k = 2..K: the Chebyshev recurrence
// X_k = 2 cos(theta) X_{k-1} - X_{k-2} (2 FMA per k instead of the 4 of a
// complex multiply).  Its rounding error grows like eps k^2: FP64 1e-14 at
// the disk kernels' K <= 12, far inside the 1e-10 parity gate; FP32 ~1e-5,
// two orders below the Monte Carlo standard error of any launch large enough
// to be worth the FP32 variant (the gate there is 3 SE).  The tiled generic
// kernel (K up to 80, where FP32 would reach 4e-4) keeps complex products.
template <class T>
constexpr bool kChebyshev = true;

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
    if constexpr (IsPacked<CA>::value) {
        static_assert(P == 1 && std::is_same<T, float>::value, "packed form: FP32, one particle per thread");
        uint64_t A = f2_pack(g0r, g0i), B = f2_pack(0.0f, 0.0f);
        disk_row_pairs_packed<K, K1>(C, W, A, B, std::make_integer_sequence<int, S::jmax(K1)>{});
        f2_unpack(A, a.Ar[0], a.Ai[0]);
        f2_unpack(B, a.Br[0], a.Bi[0]);
    } else {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            a.Ar[p] = g0r;
            a.Ai[p] = g0i;
            a.Br[p] = T(0);
            a.Bi[p] = T(0);
        }
        disk_row_pairs<K, K1, T, P>(C, W, a, std::make_integer_sequence<int, S::jmax(K1)>{});
    }
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

// ---------------------------------------------------------------------------
// Tiled disk series for kDiskMaxK < K (FP64 K1; disk_tiled_instantiated():
// the batched C4 prior has K = 25, M = 980).  Powers for every j no longer
// fit in registers, so the columns run in tiles of 8 (P2[j], Q[j] of one tile
// in registers, continued by complex products from the previous tile).  The
// shape is known at compile time: a tile's full rows (8 pairs) share one
// body in a run-time row loop, the partial rows at the disk's edge are
// unrolled with exactly their pairs, so unlike the generic tiled kernel
// (velocity.cuh) no pair slot is padding.  Same disk_shape.h coefficient
// layout as the K <= 12 kernel.  Per (tile, row): P1 <- P1 e1 (restarted
// each tile) and the fold v2 += k1 Re(P1 A), v1 -= Re(P1 B').  Measured and
// rejected: unrolling every row (instruction-fetch bound, C4 2969 vs 2763
// ms) and interleaving the pair updates of two rows (eight accumulator
// chains instead of four: 2974 -> 3032 ms).
#ifndef SMC_DISK_TILE
#define SMC_DISK_TILE 8
#endif
constexpr int kDiskTile = SMC_DISK_TILE;

template <int K, int T0>
struct DiskTile {
    static constexpr int j0 = kDiskTile * T0;
    static constexpr int w = (K - j0) < kDiskTile ? (K - j0) : kDiskTile;  // columns (row 0 reaches j = K)
    static constexpr int npair(int k1) {
        const int e = DiskShape<K>::jmax(k1) - j0;
        return e < 0 ? 0 : (e > kDiskTile ? kDiskTile : e);
    }
    static constexpr int rows() {  // k1 = 1..rows() have pairs here (jmax is non-increasing in k1)
        if (T0 == 0) return K;     // tile 0 also carries every row's (k1, 0) mode
        int r = 0;
        while (r < K && DiskShape<K>::jmax(r + 1) > j0) ++r;
        return r;
    }
};

template <int K>
constexpr int kDiskTiles = (K + kDiskTile - 1) / kDiskTile;

template <class T>
struct TilePowers {
    T pr[kDiskTile], pi[kDiskTile], qr[kDiskTile], qi[kDiskTile];
};

template <int K, int T0, int K1, int Q, class T, class CA>
__device__ __forceinline__ void tiled_pair(const CA& C, const TilePowers<T>& W, T& Ar, T& Ai, T& Br, T& Bi) {
    constexpr int o = 4 * (DiskShape<K>::pair_offset(K1) + DiskTile<K, T0>::j0 + Q);
    T ar, ai, br, bi;
    get4<o>(C, ar, ai, br, bi);
    Ar = fma(ar, W.pr[Q], Ar);
    Ai = fma(ai, W.pr[Q], Ai);
    Br = fma(br, W.qr[Q], Br);
    Bi = fma(bi, W.qr[Q], Bi);
    Ar = fma(bi, -W.pi[Q], Ar);
    Ai = fma(br, W.pi[Q], Ai);
    Br = fma(ai, -W.qi[Q], Br);
    Bi = fma(ar, W.qi[Q], Bi);
}

template <int K, int T0, int K1, class T, class CA, int... Qs>
__device__ __forceinline__ void tiled_pairs(const CA& C, const TilePowers<T>& W, T& Ar, T& Ai, T& Br, T& Bi,
                                            std::integer_sequence<int, Qs...>) {
    (tiled_pair<K, T0, K1, Qs>(C, W, Ar, Ai, Br, Bi), ...);
}

template <int K, int T0, int K1, class T, class CA>
__device__ __forceinline__ void tiled_row(const CA& C, const TilePowers<T>& W, T c1, T s1, T& p1r, T& p1i, T& acc1,
                                          T& acc2) {
    if constexpr (K1 > 1) {
        const T nr = fma(p1r, c1, -p1i * s1);
        p1i = fma(p1r, s1, p1i * c1);
        p1r = nr;
    }
    T Ar = T(0), Ai = T(0), Br = T(0), Bi = T(0);
    if constexpr (T0 == 0) C.template get2<DiskShape<K>::g0_offset + 2 * (K1 - 1)>(Ar, Ai);
    tiled_pairs<K, T0, K1>(C, W, Ar, Ai, Br, Bi, std::make_integer_sequence<int, DiskTile<K, T0>::npair(K1)>{});
    acc2 = fma(T(K1), fma(p1r, Ar, -p1i * Ai), acc2);
    acc1 = fma(-p1r, Br, fma(p1i, Bi, acc1));
}

template <int K, int T0, int Q, class T, class CA>
__device__ __forceinline__ void tiled_row0_term(const CA& C, const TilePowers<T>& W, T& a0, T& a1) {
    T gr, gi;
    C.template get2<DiskShape<K>::row0_offset + 2 * (DiskTile<K, T0>::j0 + Q)>(gr, gi);
    a0 = fma(gr, -W.qr[Q], a0);
    a1 = fma(gi, W.qi[Q], a1);
}

template <int K, int T0, class T, class CA, int... Qs>
__device__ __forceinline__ void tiled_row0(const CA& C, const TilePowers<T>& W, T& a0, T& a1,
                                           std::integer_sequence<int, Qs...>) {
    (tiled_row0_term<K, T0, Qs>(C, W, a0, a1), ...);
}

// Pair offsets of every row (4 doubles per pair) in the constant bank, for
// the runtime row loop over a tile's full rows.
template <int K>
struct DiskRowOffsets {
    int off[K + 2];
    constexpr DiskRowOffsets() : off() {
        for (int k1 = 1; k1 <= K + 1; ++k1) off[k1] = 4 * DiskShape<K>::pair_offset(k1);
    }
};
template <int K>
__constant__ DiskRowOffsets<K> c_disk_row_off = DiskRowOffsets<K>();

template <int K, int T0>
struct DiskTileFull {  // rows k1 = 1..full with all 8 pairs in this tile
    static constexpr int full() {
        int r = 0;
        while (r < K && DiskTile<K, T0>::npair(r + 1) == kDiskTile) ++r;
        return r;
    }
};

template <int K, int T0, int K1, class T, class CA, int... K1s>
__device__ __forceinline__ void tiled_rows_from(const CA& C, const TilePowers<T>& W, T c1, T s1, T& p1r, T& p1i,
                                                T& acc1, T& acc2, std::integer_sequence<int, K1s...>) {
    (tiled_row<K, T0, K1 + K1s>(C, W, c1, s1, p1r, p1i, acc1, acc2), ...);
}

// Rows of a tile: the full rows run through ONE 8-pair body
// in a runtime loop (row base from the constant-bank offset table), only the
// partial rows at the disk's edge are unrolled.  The fully unrolled form is
// ~5800 instructions per step at K = 25 and stalls on instruction fetch (ncu:
// no_instructions 44 % of samples).
template <int K, int T0, class T, class CA>
__device__ __forceinline__ void tiled_rows_hybrid(const CA& C, const TilePowers<T>& W, T c1, T s1, T& acc1,
                                                  T& acc2) {
    constexpr int F = DiskTileFull<K, T0>::full();
    constexpr int R = DiskTile<K, T0>::rows();
    T p1r = c1, p1i = s1;
#pragma unroll 1
    for (int k1 = 1; k1 <= F; ++k1) {
        if (k1 > 1) {
            const T nr = fma(p1r, c1, -p1i * s1);
            p1i = fma(p1r, s1, p1i * c1);
            p1r = nr;
        }
        T Ar = T(0), Ai = T(0), Br = T(0), Bi = T(0);
        if constexpr (T0 == 0) shifted(C, DiskShape<K>::g0_offset + 2 * (k1 - 1)).template get2<0>(Ar, Ai);
        // row k1's pairs j0+1..j0+8: the row-1 body (pair_offset(1) = 0) shifted to row k1
        tiled_pairs<K, T0, 1>(shifted(C, c_disk_row_off<K>.off[k1]), W, Ar, Ai, Br, Bi,
                              std::make_integer_sequence<int, kDiskTile>{});
        const T kd = T(k1);
        acc2 = fma(kd, fma(p1r, Ar, -p1i * Ai), acc2);
        acc1 = fma(-p1r, Br, fma(p1i, Bi, acc1));
    }
    if constexpr (R > F)
        tiled_rows_from<K, T0, F + 1>(C, W, c1, s1, p1r, p1i, acc1, acc2, std::make_integer_sequence<int, R - F>{});
}

template <int K, int T0, class T, class CA>
__device__ __forceinline__ void tiled_tile(const CA& C, T c1, T s1, T c2, T s2, T& p2r, T& p2i, T& a0, T& a1,
                                           T& acc1, T& acc2) {
    using Tl = DiskTile<K, T0>;
    TilePowers<T> W;
#pragma unroll
    for (int q = 0; q < Tl::w; ++q) {  // P2[j0 + q + 1] = P2[j0 + q] e2
        const T nr = fma(p2r, c2, -p2i * s2);
        p2i = fma(p2r, s2, p2i * c2);
        p2r = nr;
        W.pr[q] = p2r;
        W.pi[q] = p2i;
        W.qr[q] = T(Tl::j0 + q + 1) * p2r;
        W.qi[q] = T(Tl::j0 + q + 1) * p2i;
    }
    tiled_row0<K, T0>(C, W, a0, a1, std::make_integer_sequence<int, Tl::w>{});
    tiled_rows_hybrid<K, T0>(C, W, c1, s1, acc1, acc2);
}

template <int K, class T, class CA, int... Ts>
__device__ __forceinline__ void tiled_tiles(const CA& C, T c1, T s1, T c2, T s2, T& a0, T& a1, T& acc1, T& acc2,
                                            std::integer_sequence<int, Ts...>) {
    T p2r = T(1), p2i = T(0);
    (tiled_tile<K, Ts>(C, c1, s1, c2, s2, p2r, p2i, a0, a1, acc1, acc2), ...);
}

template <int K, class T, class CA>
__device__ __forceinline__ void velocity_disk_tiled(const CA& C, T x1, T x2, T& v1, T& v2) {
    T s1, c1, s2, c2;
    sincospi_t(T(2) * x1, &s1, &c1);
    sincospi_t(T(2) * x2, &s2, &c2);
    T a0 = T(0), a1 = T(0), acc1 = T(0), acc2 = T(0);
    tiled_tiles<K>(C, c1, s1, c2, s2, a0, a1, acc1, acc2, std::make_integer_sequence<int, kDiskTiles<K>>{});
    v1 = acc1 + (a0 + a1);
    v2 = acc2;
}

// Either disk form for P = 1.
template <int K, class T, class CA>
__device__ __forceinline__ void velocity_disk_any(const CA& C, const T (&x1)[1], const T (&x2)[1], T (&v1)[1],
                                                  T (&v2)[1]) {
    if constexpr (K > kDiskMaxK) velocity_disk_tiled<K, T>(C, x1[0], x2[0], v1[0], v2[0]);
    else velocity_disk<K, T, 1>(C, x1, x2, v1, v2);
}

}  // namespace disk
}  // namespace smc
