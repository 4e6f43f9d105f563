// ubench_dmma.cu — does FP64 tensor-core MMA (mma.sync .f64) run beside the
// DFMA pipe on B200 (sm_100a)?  If it does, the particle kernels could put
// the velocity mode sums (a batched GEMV) on DMMA and keep
// Box-Muller / Euler-Maruyama on DFMA.
//   dmma<shape>  : CH independent accumulators per warp, back-to-back MMAs
//   dfma         : 8 independent DFMA chains per thread
//   mixed        : each warp interleaves MMAs and DFMAs (ratio R DFMA per MMA)
//   split        : even warps MMA only, odd warps DFMA only (same SM)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_dmma tools/ubench_dmma.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

// shape 0: m8n8k4 (512 flop), 1: m16n8k4 (1024), 2: m16n8k8 (2048), 3: m16n8k16 (4096)
template <int SH>
struct Mma;
template <>
struct Mma<0> {
    static constexpr int NA = 1, NB = 1, NC = 2, FLOP = 512;
    __device__ static void run(double (&c)[NC], const double (&a)[NA], const double (&b)[NB]) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[0]), "+d"(c[1])
                     : "d"(a[0]), "d"(b[0]));
    }
};
template <>
struct Mma<1> {
    static constexpr int NA = 2, NB = 1, NC = 4, FLOP = 1024;
    __device__ static void run(double (&c)[NC], const double (&a)[NA], const double (&b)[NB]) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                     : "d"(a[0]), "d"(a[1]), "d"(b[0]));
    }
};
template <>
struct Mma<2> {
    static constexpr int NA = 4, NB = 2, NC = 4, FLOP = 2048;
    __device__ static void run(double (&c)[NC], const double (&a)[NA], const double (&b)[NB]) {
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    }
};
template <>
struct Mma<3> {
    static constexpr int NA = 8, NB = 4, NC = 4, FLOP = 4096;
    __device__ static void run(double (&c)[NC], const double (&a)[NA], const double (&b)[NB]) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
            "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
            : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
              "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
};

// MODE 0: MMA only; 1: DFMA only; 2: both in every warp; 3: split by warp parity
template <int SH, int CH, int MODE, int R>
__global__ void __launch_bounds__(256) kbench(int iters, double* sink) {
    using M = Mma<SH>;
    double a[M::NA], b[M::NB], c[CH][M::NC];
#pragma unroll
    for (int i = 0; i < M::NA; ++i) a[i] = 1e-3 * (threadIdx.x + i);
#pragma unroll
    for (int i = 0; i < M::NB; ++i) b[i] = 1e-3 * (threadIdx.x - i);
#pragma unroll
    for (int q = 0; q < CH; ++q)
#pragma unroll
        for (int i = 0; i < M::NC; ++i) c[q][i] = 0.0;
    double f[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) f[q] = 1.0 + 1e-9 * (threadIdx.x + q);
    const double fb = 0.9999999, fc = 1e-7;
    const bool do_mma = MODE == 0 || MODE == 2 || (MODE == 3 && (threadIdx.x / 32) % 2 == 0);
    const bool do_fma = MODE == 1 || MODE == 2 || (MODE == 3 && (threadIdx.x / 32) % 2 == 1);
    if (do_mma && do_fma) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                M::run(c[q], a, b);
#pragma unroll
                for (int r = 0; r < R; ++r) f[r % 8] = fma(f[r % 8], fb, fc);
            }
        }
    } else if (do_mma) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int q = 0; q < CH; ++q) M::run(c[q], a, b);
    } else if (do_fma) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int q = 0; q < CH; ++q)
#pragma unroll
                for (int r = 0; r < R; ++r) f[r % 8] = fma(f[r % 8], fb, fc);
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q)
#pragma unroll
        for (int i = 0; i < M::NC; ++i) s += c[q][i];
#pragma unroll
    for (int q = 0; q < 8; ++q) s += f[q];
    if (s == 12345.0) sink[blockIdx.x] = s;
}

template <int SH, int CH, int MODE, int R>
int run(const char* name, int blocks_per_sm, int threads, int iters) {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    double* sink;
    CK(cudaMalloc(&sink, 1 << 20));
    const int grid = sms * blocks_per_sm;
    kbench<SH, CH, MODE, R><<<grid, threads>>>(2, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kbench<SH, CH, MODE, R><<<grid, threads>>>(iters, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = double(grid) * threads / 32;
    const double warps_mma = MODE == 3 ? warps / 2 : (MODE == 1 ? 0 : warps);
    const double warps_fma = MODE == 3 ? warps / 2 : (MODE == 0 ? 0 : warps);
    const double mma_flop = warps_mma * double(iters) * CH * Mma<SH>::FLOP;
    const double fma_flop = warps_fma * 32.0 * double(iters) * CH * R * 2;
    std::printf("%-34s %2d blk/SM x %3d thr: %8.3f ms  mma %6.2f TF/s  dfma %6.2f TF/s  total %6.2f TF/s\n", name,
                blocks_per_sm, threads, ms, mma_flop / ms / 1e9, fma_flop / ms / 1e9, (mma_flop + fma_flop) / ms / 1e9);
    cudaFree(sink);
    return 0;
}

int main() {
    const int it = 20000;
    run<0, 4, 0, 8>("mma m8n8k4 only", 2, 256, it);
    run<1, 4, 0, 8>("mma m16n8k4 only", 2, 256, it);
    run<2, 4, 0, 8>("mma m16n8k8 only", 2, 256, it);
    run<3, 4, 0, 8>("mma m16n8k16 only", 2, 256, it / 2);
    run<3, 2, 0, 8>("mma m16n8k16 only CH2", 2, 256, it / 2);
    run<3, 4, 0, 8>("mma m16n8k16 only 1blk", 1, 256, it / 2);
    run<3, 4, 0, 8>("mma m16n8k16 only 4blk", 4, 256, it / 2);
    run<2, 4, 1, 8>("dfma only (8/iter)", 2, 256, it);
    // m16n8k8: 2048 flop per warp-MMA = 1024 DFMA-lane-equivalents = 32 DFMA per thread
    run<2, 4, 2, 8>("mixed k8, 8 dfma/mma", 2, 256, it);
    run<2, 4, 2, 16>("mixed k8, 16 dfma/mma", 2, 256, it);
    run<2, 4, 2, 32>("mixed k8, 32 dfma/mma", 2, 256, it / 2);
    run<3, 4, 2, 16>("mixed k16, 16 dfma/mma", 2, 256, it / 2);
    run<3, 4, 2, 32>("mixed k16, 32 dfma/mma", 2, 256, it / 2);
    run<3, 4, 2, 64>("mixed k16, 64 dfma/mma", 2, 256, it / 4);
    run<2, 4, 3, 16>("split k8 / 16 dfma", 2, 256, it);
    run<3, 4, 3, 32>("split k16 / 32 dfma", 2, 256, it / 2);
    return 0;
}
