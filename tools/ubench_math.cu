// ubench_math.cu — throughput and accuracy of fastmath.cuh vs libdevice on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1808_10580_b200/csrc -o tools/ubench_math tools/ubench_math.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "fastmath.cuh"

template <int MODE>
__global__ void k_tp(int iters, double* sink) {
    double a = 0.1 + 1e-7 * (blockIdx.x * blockDim.x + threadIdx.x), acc = 0.0, b = 0.3;
    for (int it = 0; it < iters; ++it) {
        double s, c;
        if (MODE == 0) sincospi(a, &s, &c);
        else if (MODE == 1) smc::fm::sincospi(a, &s, &c);
        else if (MODE == 2) { s = log(a); c = log(b); }
        else { s = smc::fm::log_pos(a); c = smc::fm::log_pos(b); }
        acc += s + c;
        a = fma(a, 1.0000001, 1e-9);
        b = fma(b, 0.9999999, 1e-9);
    }
    if (acc == 12345.0) sink[0] = acc;
}

__global__ void k_acc(int n, double* err) {  // max |fast - libdevice| in ulp of libdevice
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double a = 2.0 * (i + 0.37) / n;
    double s0, c0, s1, c1;
    sincospi(a, &s0, &c0);
    smc::fm::sincospi(a, &s1, &c1);
    const double u = (i + 0.5) / n;
    const double l0 = log(u), l1 = smc::fm::log_pos(u);
    const double tiny = 1e-300;
    err[3 * i] = fabs(s1 - s0) / fmax(fabs(s0) * 1.1102230246251565e-16, tiny * 0 + 4.9e-324);
    err[3 * i + 1] = fabs(c1 - c0) / fmax(fabs(c0) * 1.1102230246251565e-16, 4.9e-324);
    err[3 * i + 2] = fabs(l1 - l0) / fmax(fabs(l0) * 1.1102230246251565e-16, 4.9e-324);
}

int main() {
    double* sink;
    cudaMalloc(&sink, 8);
    const char* names[] = {"libdevice sincospi", "fm::sincospi", "libdevice log x2", "fm::log_pos x2"};
    for (int mode = 0; mode < 4; ++mode) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int blocks = 148 * 8, threads = 256, iters = 2000;
        auto go = [&] {
            if (mode == 0) k_tp<0><<<blocks, threads>>>(iters, sink);
            if (mode == 1) k_tp<1><<<blocks, threads>>>(iters, sink);
            if (mode == 2) k_tp<2><<<blocks, threads>>>(iters, sink);
            if (mode == 3) k_tp<3><<<blocks, threads>>>(iters, sink);
        };
        go();
        cudaEventRecord(a);
        go();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-20s %.3f ms  %.3g calls/s\n", names[mode], ms, double(blocks) * threads * iters / (ms * 1e-3));
    }
    const int n = 1 << 22;
    double* err;
    cudaMalloc(&err, sizeof(double) * 3 * n);
    k_acc<<<(n + 255) / 256, 256>>>(n, err);
    double* h = new double[3 * (size_t)n];
    cudaMemcpy(h, err, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost);
    double m[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k)
            if (h[3 * i + k] > m[k]) m[k] = h[3 * i + k];
    printf("max rel diff vs libdevice in units of 2^-53: sin %.2f cos %.2f log %.2f\n", m[0], m[1], m[2]);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
