// ubench_ffma2.cu — FP32 issue-rate microbenchmarks on B200 (sm_100a) for the
// FP32 variant of K1: FFMA with three vector-register operands, FFMA with a
// uniform-register operand, and the packed FFMA2 (fma.rn.f32x2, sm_100a),
// each with 8 independent chains per thread at 16 and 32 warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_ffma2 tools/ubench_ffma2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;

__device__ __forceinline__ uint64_t pack(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float lo_of(uint64_t v) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return a + b;
}
__device__ __forceinline__ void fma2(uint64_t& acc, uint64_t x, uint64_t y) {
    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(x), "l"(y));
}

// a[q] = fma(a[q], b, c): b, c kernel parameters (uniform registers)
__global__ void k_uniform(int iters, float b, float c, float* sink) {
    float a[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) a[q] = 1.0f + 1e-6f * float(threadIdx.x + q);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int q = 0; q < CH; ++q) a[q] = fmaf(a[q], b, c);
    float s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += a[q];
    if (s == 12345.0f) sink[blockIdx.x] = s;
}

// a[q] = fma(x[q], y[q'], a[q]): three vector registers
__global__ void k_regs3(int iters, float* sink) {
    float a[CH], x[CH], y[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        a[q] = 1.0f + 1e-6f * float(threadIdx.x + q);
        x[q] = 0.9999f + 1e-9f * float(q * threadIdx.x);
        y[q] = 1e-9f * float(q + 1);
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int q = 0; q < CH; ++q) a[q] = fmaf(x[q], y[(q + 1) % CH], a[q]);
    float s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += a[q] + x[q];
    if (s == 12345.0f) sink[blockIdx.x] = s;
}

// packed: acc[q] (2 floats) += x[q] * y[q'] (2 floats each): 2 FMAs per instruction
__global__ void k_ffma2(int iters, float* sink) {
    uint64_t a[CH], x[CH], y[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        a[q] = pack(1.0f + 1e-6f * float(threadIdx.x + q), 1.0f);
        x[q] = pack(0.9999f + 1e-9f * float(q * threadIdx.x), 0.9998f);
        y[q] = pack(1e-9f * float(q + 1), 2e-9f);
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int q = 0; q < CH; ++q) fma2(a[q], x[q], y[(q + 1) % CH]);
    float s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += lo_of(a[q]) + lo_of(x[q]);
    if (s == 12345.0f) sink[blockIdx.x] = s;
}

// packed with one operand a uniform pair (kernel parameter)
__global__ void k_ffma2_uniform(int iters, uint64_t b, float* sink) {
    uint64_t a[CH], x[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        a[q] = pack(1.0f + 1e-6f * float(threadIdx.x + q), 1.0f);
        x[q] = pack(0.9999f + 1e-9f * float(q * threadIdx.x), 0.9998f);
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int q = 0; q < CH; ++q) fma2(a[q], x[q], b);
    float s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += lo_of(a[q]) + lo_of(x[q]);
    if (s == 12345.0f) sink[blockIdx.x] = s;
}

// packed with a broadcast scalar: acc[q] += x[q] * (s, s), s a per-thread register
__global__ void k_ffma2_bcast(int iters, float* sink) {
    uint64_t a[CH], x[CH];
    float sv[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        a[q] = pack(1.0f + 1e-6f * float(threadIdx.x + q), 1.0f);
        x[q] = pack(0.9999f + 1e-9f * float(q * threadIdx.x), 0.9998f);
        sv[q] = 1e-9f * float(q + threadIdx.x);
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int q = 0; q < CH; ++q) fma2(a[q], x[q], pack(sv[(q + 1) % CH], sv[(q + 1) % CH]));
    float s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += lo_of(a[q]) + lo_of(x[q]) + sv[q];
    if (s == 12345.0f) sink[blockIdx.x] = s;
}

template <class F>
double run(const char* name, int blocks, int threads, double flops_per_iter_thread, F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 1 << 16;
    launch(blocks, threads, 64);
    cudaEventRecord(e0);
    launch(blocks, threads, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = flops_per_iter_thread * iters * double(blocks) * threads / (ms * 1e-3) / 1e12;
    printf("%-16s warps/SM %2d: %7.2f TFLOP/s (%s)\n", name, blocks / 148 * threads / 32, tf,
           cudaGetErrorString(cudaGetLastError()));
    return tf;
}

int main() {
    float* sink;
    cudaMalloc(&sink, 1 << 20);
    for (int wps : {16, 32}) {
        const int threads = 256, blocks = 148 * wps * 32 / threads;
        run("ffma uniform", blocks, threads, 2.0 * CH, [&](int b, int t, int it) { k_uniform<<<b, t>>>(it, 0.9999999f, 1e-9f, sink); });
        run("ffma 3-reg", blocks, threads, 2.0 * CH, [&](int b, int t, int it) { k_regs3<<<b, t>>>(it, sink); });
        run("ffma2 3-reg", blocks, threads, 4.0 * CH, [&](int b, int t, int it) { k_ffma2<<<b, t>>>(it, sink); });
        run("ffma2 bcast", blocks, threads, 4.0 * CH, [&](int b, int t, int it) { k_ffma2_bcast<<<b, t>>>(it, sink); });
        run("ffma2 uniform", blocks, threads, 4.0 * CH, [&](int b, int t, int it) {
            k_ffma2_uniform<<<b, t>>>(it, 0x3f7fffff3f7fffffull, sink);
        });
    }
    return 0;
}
