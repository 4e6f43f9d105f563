// ubench_dfma.cu — FP64 pipe microbenchmarks on B200 (sm_100a): what limits a
// DFMA-dense kernel?  Variants:
//   uniform : a[q] = fma(a[q], b, c), b/c warp-uniform (the peak recipe)
//   regs3   : a[q] = fma(x[q], y[q], a[q]), three distinct register operands
//   pairs   : the K1 lattice pair update: 4 accumulators, coefficients from
//             shared memory (LDS.128 broadcast), powers in registers
// each at several warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_dfma tools/ubench_dfma.cu
#include <cstdint>
#include <cstdio>
#include <utility>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_uniform(int iters, double b, double c, double* sink) {
    double a[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) a[q] = 1.0 + 1e-9 * (threadIdx.x + q);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int q = 0; q < CH; ++q) a[q] = fma(a[q], b, c);
    double s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += a[q];
    if (s == 12345.0) sink[blockIdx.x] = s;
}

template <int CH>
__global__ void k_regs3(int iters, double* sink) {
    double a[CH], x[CH], y[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        a[q] = 1.0 + 1e-9 * (threadIdx.x + q);
        x[q] = 0.999999 + 1e-12 * q * threadIdx.x;
        y[q] = 1e-12 * (q + 1);
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int q = 0; q < CH; ++q) a[q] = fma(a[q], x[q], y[(q + 1) % CH]);
    double s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += a[q];
    if (s == 12345.0) sink[blockIdx.x] = s;
}

// K1-like: J powers in registers, 4 accumulators per row, 4 coefs per pair from smem
template <int J>
__global__ void k_pairs(int iters, const double* coef_g, double* sink) {
    __shared__ __align__(16) double coef[4 * J * 8];
    for (int i = threadIdx.x; i < 4 * J * 8; i += blockDim.x) coef[i] = coef_g[i];
    __syncthreads();
    const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(coef));
    double pr[J], pi[J], qr[J], qi[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        pr[j] = 0.5 + 1e-3 * j + 1e-9 * threadIdx.x;
        pi[j] = 0.25 - 1e-3 * j;
        qr[j] = (j + 1) * pr[j];
        qi[j] = (j + 1) * pi[j];
    }
    double acc1 = 0, acc2 = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int row = 0; row < 8; ++row) {
            double Ar = 0, Ai = 0, Br = 0, Bi = 0;
#pragma unroll
            for (int j = 0; j < J; ++j) {
                double ar, ai, br, bi;
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(ar), "=d"(ai) : "r"(base + 32 * (row * J + j)));
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(br), "=d"(bi) : "r"(base + 32 * (row * J + j) + 16));
                Ar = fma(ar, pr[j], Ar);
                Ai = fma(ai, pr[j], Ai);
                Br = fma(br, qr[j], Br);
                Bi = fma(bi, qr[j], Bi);
                Ar = fma(bi, -pi[j], Ar);
                Ai = fma(br, pi[j], Ai);
                Br = fma(ai, -qi[j], Br);
                Bi = fma(ar, qi[j], Bi);
            }
            acc2 = fma(Ar, 0.3, fma(Ai, -0.2, acc2));
            acc1 = fma(Br, 0.7, fma(Bi, 0.1, acc1));
        }
#pragma unroll
        for (int j = 0; j < J; ++j) pr[j] = fma(pr[j], 1e-17, acc1 * 1e-300);
    }
    if (acc1 + acc2 == 12345.0) sink[blockIdx.x] = acc1;
}

// same DFMA pattern, coefficients from registers (no shared-memory loads)
template <int J>
__global__ void k_pairs_reg(int iters, const double* coef_g, double* sink) {
    double cr[4 * J];
#pragma unroll
    for (int i = 0; i < 4 * J; ++i) cr[i] = coef_g[i] + 1e-9 * threadIdx.x;
    double pr[J], pi[J], qr[J], qi[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        pr[j] = 0.5 + 1e-3 * j + 1e-9 * threadIdx.x;
        pi[j] = 0.25 - 1e-3 * j;
        qr[j] = (j + 1) * pr[j];
        qi[j] = (j + 1) * pi[j];
    }
    double acc1 = 0, acc2 = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int row = 0; row < 8; ++row) {
            double Ar = 0, Ai = 0, Br = 0, Bi = 0;
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const double ar = cr[4 * j] * (1 + row), ai = cr[4 * j + 1], br = cr[4 * j + 2], bi = cr[4 * j + 3];
                Ar = fma(ar, pr[j], Ar);
                Ai = fma(ai, pr[j], Ai);
                Br = fma(br, qr[j], Br);
                Bi = fma(bi, qr[j], Bi);
                Ar = fma(bi, -pi[j], Ar);
                Ai = fma(br, pi[j], Ai);
                Br = fma(ai, -qi[j], Br);
                Bi = fma(ar, qi[j], Bi);
            }
            acc2 = fma(Ar, 0.3, fma(Ai, -0.2, acc2));
            acc1 = fma(Br, 0.7, fma(Bi, 0.1, acc1));
        }
#pragma unroll
        for (int j = 0; j < J; ++j) pr[j] = fma(pr[j], 1e-17, acc1 * 1e-300);
    }
    if (acc1 + acc2 == 12345.0) sink[blockIdx.x] = acc1;
}

// shared-memory coefficients with 64-bit loads
template <int J>
__global__ void k_pairs64(int iters, const double* coef_g, double* sink) {
    __shared__ __align__(16) double coef[4 * J * 8];
    for (int i = threadIdx.x; i < 4 * J * 8; i += blockDim.x) coef[i] = coef_g[i];
    __syncthreads();
    const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(coef));
    double pr[J], pi[J], qr[J], qi[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        pr[j] = 0.5 + 1e-3 * j + 1e-9 * threadIdx.x;
        pi[j] = 0.25 - 1e-3 * j;
        qr[j] = (j + 1) * pr[j];
        qi[j] = (j + 1) * pi[j];
    }
    double acc1 = 0, acc2 = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int row = 0; row < 8; ++row) {
            double Ar = 0, Ai = 0, Br = 0, Bi = 0;
#pragma unroll
            for (int j = 0; j < J; ++j) {
                double ar, ai, br, bi;
                const unsigned a = base + 32 * (row * J + j);
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(ar) : "r"(a));
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(ai) : "r"(a + 8));
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(br) : "r"(a + 16));
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(bi) : "r"(a + 24));
                Ar = fma(ar, pr[j], Ar);
                Ai = fma(ai, pr[j], Ai);
                Br = fma(br, qr[j], Br);
                Bi = fma(bi, qr[j], Bi);
                Ar = fma(bi, -pi[j], Ar);
                Ai = fma(br, pi[j], Ai);
                Br = fma(ai, -qi[j], Br);
                Bi = fma(ar, qi[j], Bi);
            }
            acc2 = fma(Ar, 0.3, fma(Ai, -0.2, acc2));
            acc1 = fma(Br, 0.7, fma(Bi, 0.1, acc1));
        }
#pragma unroll
        for (int j = 0; j < J; ++j) pr[j] = fma(pr[j], 1e-17, acc1 * 1e-300);
    }
    if (acc1 + acc2 == 12345.0) sink[blockIdx.x] = acc1;
}

// coefficients replicated across the 128 TMEM lanes; each pair's 4 doubles
// come back with one tcgen05.ld.32x32b.x8 (next pair's load overlaps this
// pair's DFMAs).  1 CTA/SM, 512 threads, 512 TMEM columns.
__device__ __forceinline__ void tm_ld8(uint32_t taddr, double& a, double& b, double& c, double& d) {
    uint32_t r0, r1, r2, r3, r4, r5, r6, r7;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(r4), "=r"(r5), "=r"(r6), "=r"(r7)
                 : "r"(taddr));
    a = __hiloint2double(r1, r0);
    b = __hiloint2double(r3, r2);
    c = __hiloint2double(r5, r4);
    d = __hiloint2double(r7, r6);
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void tm_ldn(uint32_t taddr, double (&d)[N / 2]);
template <>
__device__ __forceinline__ void tm_ldn<16>(uint32_t taddr, double (&d)[8]) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = __hiloint2double(r[2 * i + 1], r[2 * i]);
}
template <>
__device__ __forceinline__ void tm_ldn<32>(uint32_t taddr, double (&d)[16]) {
    uint32_t r[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) d[i] = __hiloint2double(r[2 * i + 1], r[2 * i]);
}

// PPL pairs per tcgen05.ld (4 doubles = 8 columns per pair); 8 rows x 8 pairs
template <int PPL>
__global__ void __launch_bounds__(512, 1) k_pairs_tmem(int iters, const double* coef_g, double* sink) {
    constexpr int J = 8;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t taddr0 = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    if (warp < 4) {
        for (int col = 0; col < 8 * J * 8; col += 8) {
            uint32_t w[8];
            for (int q = 0; q < 8; ++q) {
                const int word = col + q;
                const unsigned long long bits = __double_as_longlong(coef_g[(word >> 1) % 1024]);
                w[q] = (word & 1) ? static_cast<uint32_t>(bits >> 32) : static_cast<uint32_t>(bits);
            }
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                             taddr0 + col),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    double pr[J], pi[J], qr[J], qi[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        pr[j] = 0.5 + 1e-3 * j + 1e-9 * threadIdx.x;
        pi[j] = 0.25 - 1e-3 * j;
        qr[j] = (j + 1) * pr[j];
        qi[j] = (j + 1) * pi[j];
    }
    constexpr int NL = 8 * J / PPL;  // loads per sweep
    double acc1 = 0, acc2 = 0;
    for (int it = 0; it < iters; ++it) {
        double cur[4 * PPL], nxt[4 * PPL];
        tm_ldn<8 * PPL>(taddr0, cur);
        tm_wait_ld();
        double Ar = 0, Ai = 0, Br = 0, Bi = 0;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            if (l + 1 < NL) tm_ldn<8 * PPL>(taddr0 + 8 * PPL * (l + 1), nxt);
#pragma unroll
            for (int q = 0; q < PPL; ++q) {
                const int j = (l * PPL + q) % J;
                const double ar = cur[4 * q], ai = cur[4 * q + 1], br = cur[4 * q + 2], bi = cur[4 * q + 3];
                Ar = fma(ar, pr[j], Ar);
                Ai = fma(ai, pr[j], Ai);
                Br = fma(br, qr[j], Br);
                Bi = fma(bi, qr[j], Bi);
                Ar = fma(bi, -pi[j], Ar);
                Ai = fma(br, pi[j], Ai);
                Br = fma(ai, -qi[j], Br);
                Bi = fma(ar, qi[j], Bi);
                if (j == J - 1) {
                    acc2 = fma(Ar, 0.3, fma(Ai, -0.2, acc2));
                    acc1 = fma(Br, 0.7, fma(Bi, 0.1, acc1));
                    Ar = Ai = Br = Bi = 0;
                }
            }
            tm_wait_ld();
#pragma unroll
            for (int q = 0; q < 4 * PPL; ++q) cur[q] = nxt[q];
        }
#pragma unroll
        for (int j = 0; j < J; ++j) pr[j] = fma(pr[j], 1e-17, acc1 * 1e-300);
    }
    if (acc1 + acc2 == 12345.0) sink[blockIdx.x] = acc1;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
}

__constant__ double c_coef[4 * 7 * 8];

template <int O>
__device__ __forceinline__ void ldc2(double& a, double& b) {
    asm volatile("ld.const.v2.f64 {%0, %1}, [c_coef+%2];" : "=d"(a), "=d"(b) : "n"(O * 8));
}

template <int J, int ROW, int JJ>
__device__ __forceinline__ void pc_pair(const double* pr, const double* pi, const double* qr, const double* qi,
                                        double& Ar, double& Ai, double& Br, double& Bi) {
    constexpr int o = 4 * (ROW * J + JJ);
    double ar, ai, br, bi;
    ldc2<o>(ar, ai);
    ldc2<o + 2>(br, bi);
    Ar = fma(ar, pr[JJ], Ar);
    Ai = fma(ai, pr[JJ], Ai);
    Br = fma(br, qr[JJ], Br);
    Bi = fma(bi, qr[JJ], Bi);
    Ar = fma(bi, -pi[JJ], Ar);
    Ai = fma(br, pi[JJ], Ai);
    Br = fma(ai, -qi[JJ], Br);
    Bi = fma(ar, qi[JJ], Bi);
}

template <int J, int ROW, int... JJ>
__device__ __forceinline__ void pc_row(const double* pr, const double* pi, const double* qr, const double* qi,
                                       double& acc1, double& acc2, std::integer_sequence<int, JJ...>) {
    double Ar = 0, Ai = 0, Br = 0, Bi = 0;
    (pc_pair<J, ROW, JJ>(pr, pi, qr, qi, Ar, Ai, Br, Bi), ...);
    acc2 = fma(Ar, 0.3, fma(Ai, -0.2, acc2));
    acc1 = fma(Br, 0.7, fma(Bi, 0.1, acc1));
}

template <int J, int... ROWS>
__device__ __forceinline__ void pc_rows(const double* pr, const double* pi, const double* qr, const double* qi,
                                        double& acc1, double& acc2, std::integer_sequence<int, ROWS...>) {
    (pc_row<J, ROWS>(pr, pi, qr, qi, acc1, acc2, std::make_integer_sequence<int, J>{}), ...);
}

// coefficients from the constant bank (uniform datapath loads), volatile so
// they stay inside the loop
template <int J>
__global__ void k_pairs_const(int iters, double* sink) {
    double pr[J], pi[J], qr[J], qi[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        pr[j] = 0.5 + 1e-3 * j + 1e-9 * threadIdx.x;
        pi[j] = 0.25 - 1e-3 * j;
        qr[j] = (j + 1) * pr[j];
        qi[j] = (j + 1) * pi[j];
    }
    double acc1 = 0, acc2 = 0;
    for (int it = 0; it < iters; ++it) {
        pc_rows<J>(pr, pi, qr, qi, acc1, acc2, std::make_integer_sequence<int, 8>{});
#pragma unroll
        for (int j = 0; j < J; ++j) pr[j] = fma(pr[j], 1e-17, acc1 * 1e-300);
    }
    if (acc1 + acc2 == 12345.0) sink[blockIdx.x] = acc1;
}

// two particles share each shared-memory coefficient load
template <int J>
__global__ void k_pairs2(int iters, const double* coef_g, double* sink) {
    __shared__ __align__(16) double coef[4 * J * 8];
    for (int i = threadIdx.x; i < 4 * J * 8; i += blockDim.x) coef[i] = coef_g[i];
    __syncthreads();
    const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(coef));
    double pr[2][J], pi[2][J], qr[2][J], qi[2][J];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int j = 0; j < J; ++j) {
        pr[p][j] = 0.5 + 1e-3 * j + 1e-9 * threadIdx.x + p;
        pi[p][j] = 0.25 - 1e-3 * j;
        qr[p][j] = (j + 1) * pr[p][j];
        qi[p][j] = (j + 1) * pi[p][j];
    }
    double acc1[2] = {0, 0}, acc2[2] = {0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int row = 0; row < 8; ++row) {
            double Ar[2] = {0, 0}, Ai[2] = {0, 0}, Br[2] = {0, 0}, Bi[2] = {0, 0};
#pragma unroll
            for (int j = 0; j < J; ++j) {
                double ar, ai, br, bi;
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(ar), "=d"(ai) : "r"(base + 32 * (row * J + j)));
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(br), "=d"(bi) : "r"(base + 32 * (row * J + j) + 16));
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    Ar[p] = fma(ar, pr[p][j], Ar[p]);
                    Ai[p] = fma(ai, pr[p][j], Ai[p]);
                    Br[p] = fma(br, qr[p][j], Br[p]);
                    Bi[p] = fma(bi, qr[p][j], Bi[p]);
                    Ar[p] = fma(bi, -pi[p][j], Ar[p]);
                    Ai[p] = fma(br, pi[p][j], Ai[p]);
                    Br[p] = fma(ai, -qi[p][j], Br[p]);
                    Bi[p] = fma(ar, qi[p][j], Bi[p]);
                }
            }
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                acc2[p] = fma(Ar[p], 0.3, fma(Ai[p], -0.2, acc2[p]));
                acc1[p] = fma(Br[p], 0.7, fma(Bi[p], 0.1, acc1[p]));
            }
        }
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int j = 0; j < J; ++j) pr[p][j] = fma(pr[p][j], 1e-17, acc1[p] * 1e-300);
    }
    if (acc1[0] + acc2[1] == 12345.0) sink[blockIdx.x] = acc1[0];
}

template <class F>
double time_kernel(F launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    cudaMalloc(&sink, 1 << 20);
    double* coef;
    cudaMalloc(&coef, 8 * 4096);
    cudaMemset(coef, 0, 8 * 4096);
    const int iters = 20000;
    for (int warps : {4, 8, 16, 32, 64}) {
        const int threads = 128, blocks = sms * warps * 32 / threads;
        double ms = time_kernel([&] { k_uniform<8><<<blocks, threads>>>(iters, 0.999999999, 1e-12, sink); });
        double fl = 2.0 * 8 * iters * double(blocks) * threads;
        printf("uniform ch8  warps/SM=%2d  %.2f TFLOP/s\n", warps, fl / ms / 1e9);
        ms = time_kernel([&] { k_uniform<4><<<blocks, threads>>>(iters, 0.999999999, 1e-12, sink); });
        fl = 2.0 * 4 * iters * double(blocks) * threads;
        printf("uniform ch4  warps/SM=%2d  %.2f TFLOP/s\n", warps, fl / ms / 1e9);
        ms = time_kernel([&] { k_regs3<8><<<blocks, threads>>>(iters, sink); });
        fl = 2.0 * 8 * iters * double(blocks) * threads;
        printf("regs3 ch8    warps/SM=%2d  %.2f TFLOP/s\n", warps, fl / ms / 1e9);
        ms = time_kernel([&] { k_pairs<7><<<blocks, threads>>>(iters / 20, coef, sink); });
        fl = 2.0 * (8 * (8 * 7 + 4) + 7) * (iters / 20) * double(blocks) * threads;
        printf("pairs J=7    warps/SM=%2d  %.2f TFLOP/s\n", warps, fl / ms / 1e9);
        ms = time_kernel([&] { k_pairs_reg<7><<<blocks, threads>>>(iters / 20, coef, sink); });
        printf("pairs_reg    warps/SM=%2d  %.2f TFLOP/s\n", warps, fl / ms / 1e9);
        ms = time_kernel([&] { k_pairs64<7><<<blocks, threads>>>(iters / 20, coef, sink); });
        printf("pairs_lds64  warps/SM=%2d  %.2f TFLOP/s\n", warps, fl / ms / 1e9);
    }
    {
        const int blocks = sms, threads = 512;
        double fl = 2.0 * (8 * (8 * 8 + 4) + 8) * (iters / 20) * double(blocks) * threads;
        double ms = time_kernel([&] { k_pairs_tmem<2><<<blocks, threads>>>(iters / 20, coef, sink); });
        printf("pairs_tmem x16 (2 pairs/ld) %.2f TFLOP/s  (%s)\n", fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        ms = time_kernel([&] { k_pairs_tmem<4><<<blocks, threads>>>(iters / 20, coef, sink); });
        printf("pairs_tmem x32 (4 pairs/ld) %.2f TFLOP/s  (%s)\n", fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
