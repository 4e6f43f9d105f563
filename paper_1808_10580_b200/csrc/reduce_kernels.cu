// reduce_kernels.cu — K3: deterministic per-observation reduction
// (compiled with -fmad=false).
//
// Reproduces reduce_observation (src/executor.cpp:87-117) bit for bit given
// the same per-particle values.  pairwise_sum (executor.cpp:11-26) is an
// adjacent-pair tree with odd-tail carry; at level L its node i is exactly the
// sum of the aligned range [i 2^L, min((i+1) 2^L, n)), so it equals a full
// binary tree over the values padded with -0.0 (x + -0.0 == x for every x,
// including -0.0).  Each pass sums aligned 1024-leaf chunks: 4 leaves per
// thread, a shuffle-down tree over the warp (offsets 1..16 pair aligned
// neighbours), and a fixed 8-way tree over the warps.  Passes compose, so the
// chunk partials of disjoint particle shards (multi-GPU) finish into the same
// bits as one device would produce.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.h"
#include "../../include/scalarmc_b200.h"

namespace smc {
namespace {

constexpr int kThreads = 256;  // 4 leaves per thread -> 1024-leaf chunk

// One aligned 1024-leaf chunk tree: leaves src[i] for i < n (the rest -0.0),
// mode 1 squares their deviation from c.  The sum is valid on thread 0.
__device__ __forceinline__ double chunk_tree(const double* __restrict__ src, int64_t n, double c, int mode) {
    const int64_t base = 4 * static_cast<int64_t>(threadIdx.x);
    double leaf[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t i = base + q;
        if (i < n) {
            double v = src[i];
            if (mode == 1) {
                const double d = v - c;
                v = d * d;
            }
            leaf[q] = v;
        } else {
            leaf[q] = -0.0;
        }
    }
    double v = (leaf[0] + leaf[1]) + (leaf[2] + leaf[3]);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = v + __shfl_down_sync(0xffffffffu, v, off);
    __shared__ double warp_sum[kThreads / 32];
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = v;
    __syncthreads();
    const double* w = warp_sum;
    return ((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7]));
}

__global__ void __launch_bounds__(kThreads) tree_pass_kernel(const double* __restrict__ in, int64_t in_stride,
                                                             const int64_t* __restrict__ counts, int64_t n_uniform,
                                                             double* __restrict__ out, int64_t out_stride,
                                                             const double* __restrict__ center, int mode) {
    const int64_t seg = blockIdx.y;
    const int64_t n = counts ? counts[seg] : n_uniform;
    const int64_t first = static_cast<int64_t>(blockIdx.x) * kChunk;
    const double c = (mode == 1) ? center[seg] : 0.0;
    const double sum = chunk_tree(in + seg * in_stride + first, n - first, c, mode);
    if (threadIdx.x == 0) out[seg * out_stride + blockIdx.x] = sum;
}

// Sharded AD (kernels.h unit mode): block b reduces the chunk of unit
// unit0 + b, values[b * 1024 ...], whose first min(1024, n - chunk * 1024)
// leaves are particles — exactly the first tree pass's partial for that
// (observation, chunk).  mode 1: deviations from center[observation].
__global__ void __launch_bounds__(kThreads) unit_partials_kernel(const double* __restrict__ values, int64_t unit0,
                                                                 int64_t cpo, int64_t n_particles,
                                                                 const double* __restrict__ center, int mode,
                                                                 double* __restrict__ out) {
    const int64_t unit = unit0 + blockIdx.x;
    const int64_t obs = unit / cpo;
    const int64_t first = (unit - obs * cpo) * kChunk;
    const double c = (mode == 1) ? center[obs] : 0.0;
    const double sum = chunk_tree(values + static_cast<int64_t>(blockIdx.x) * kChunk, n_particles - first, c, mode);
    if (threadIdx.x == 0) out[blockIdx.x] = sum;
}

__global__ void divide_kernel(const double* sums, const int64_t* counts, int64_t n_uniform, int64_t n_seg,
                              double* means) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_seg) return;
    const int64_t n = counts ? counts[i] : n_uniform;
    means[i] = sums[i] / static_cast<double>(n);
}

__global__ void estimates_kernel(const double* means, const double* sumsq, const double* sumaux,
                                 const int64_t* counts, int64_t n_uniform, int64_t n_particles, int64_t n_seg,
                                 smc_estimate* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_seg) return;
    const int64_t nv = counts ? counts[i] : n_uniform;
    const double n = static_cast<double>(nv);
    double se = 0.0;
    if (nv > 1) {
        const double var = sumsq[i] / (n - 1.0);
        se = sqrt(var / n);
    }
    smc_estimate e;
    e.mean = means[i];
    e.std_error = se;
    e.n_particles = n_particles;
    e.n_failed = n_particles - nv;
    e.aux_mean = sumaux ? sumaux[i] / n : 0.0;
    out[i] = e;
}


// ---- stable compaction of valid walkers (executor.cpp:93-101) -------------
__global__ void __launch_bounds__(kThreads) count_valid_kernel(const uint8_t* __restrict__ failed, int64_t n,
                                                               int64_t n_chunks, int64_t* __restrict__ chunk_counts) {
    const int64_t seg = blockIdx.y;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kChunk + 4 * threadIdx.x;
    const uint8_t* f = failed + seg * n;
    int c = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t i = base + q;
        if (i < n && !f[i]) ++c;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_down_sync(0xffffffffu, c, off);
    __shared__ int wsum[kThreads / 32];
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int k = 0; k < kThreads / 32; ++k) t += wsum[k];
        chunk_counts[seg * n_chunks + blockIdx.x] = t;
    }
}

// Exclusive scan of chunk counts per segment (one thread per segment; at most
// 2^22 chunks, sequential is fine next to the walkers).
__global__ void scan_chunks_kernel(const int64_t* chunk_counts, int64_t n_chunks, int64_t n_seg,
                                   int64_t* chunk_offsets, int64_t* counts) {
    const int64_t seg = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (seg >= n_seg) return;
    int64_t acc = 0;
    for (int64_t c = 0; c < n_chunks; ++c) {
        chunk_offsets[seg * n_chunks + c] = acc;
        acc += chunk_counts[seg * n_chunks + c];
    }
    counts[seg] = acc;
}

__global__ void __launch_bounds__(kThreads) compact_kernel(const double* __restrict__ values,
                                                           const double* __restrict__ aux,
                                                           const uint8_t* __restrict__ failed, int64_t n,
                                                           int64_t n_chunks, const int64_t* __restrict__ chunk_offsets,
                                                           double* __restrict__ cvalues, double* __restrict__ caux) {
    const int64_t seg = blockIdx.y;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kChunk + 4 * threadIdx.x;
    const uint8_t* f = failed + seg * n;
    bool ok[4];
    int c = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t i = base + q;
        ok[q] = i < n && !f[i];
        c += ok[q];
    }
    // block-wide exclusive scan of c (thread order == particle order)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int inc = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += y;
    }
    __shared__ int wtot[kThreads / 32];
    if (lane == 31) wtot[wid] = inc;
    __syncthreads();
    int wbase = 0;
    for (int k = 0; k < wid; ++k) wbase += wtot[k];
    int64_t pos = chunk_offsets[seg * n_chunks + blockIdx.x] + wbase + (inc - c);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (ok[q]) {
            cvalues[seg * n + pos] = values[seg * n + base + q];
            caux[seg * n + pos] = aux[seg * n + base + q];
            ++pos;
        }
    }
}

// ---- sharded Dirichlet reduction: aligned dyadic blocks --
// A rank holding the compacted valid walkers [off, off + cnt) of an
// observation's global compacted order sends the tree sums of the canonical
// (greedy, maximal) decomposition of that interval into aligned blocks
// [i 2^L, (i+1) 2^L) — at most 2 per level.  Every such block is a node of
// the reference's pairwise tree (executor.cpp:11-26, see the header), so the
// receiver rebuilds the root exactly by merging sibling nodes in order and
// promoting the last one through the -0.0 padding.

// Greedy decomposition of [a, b): block k = (level lv[k], first leaf st[k]).
__device__ __forceinline__ int dyadic_decompose(int64_t a, int64_t b, int* lv, int64_t* st) {
    int nb = 0;
    int64_t p = a;
    while (p < b) {
        int L = p == 0 ? 62 : __ffsll(static_cast<long long>(p)) - 1;
        while ((int64_t(1) << L) > b - p) --L;
        lv[nb] = L;
        st[nb] = p;
        ++nb;
        p += int64_t(1) << L;
    }
    return nb;
}

// Canonical tree over one value per thread of a 1024-thread CTA (pad with
// -0.0); the root on every thread.
__device__ __forceinline__ double cta_tree(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = v + __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double w = red[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) w = w + __shfl_down_sync(0xffffffffu, w, off);
        if (lane == 0) red[32] = w;
    }
    __syncthreads();
    const double r = red[32];
    __syncthreads();
    return r;
}

constexpr int kDyThreads = 1024;

// One CTA per (observation, quantity).  vals: [nq][n_obs][vstride] compacted
// local values (quantity q at vals + q * qstride); gcounts: [world][n_obs]
// valid counts of every rank (this rank's interval starts after the lower
// ranks'); mode 1 squares deviations from center[obs] (quantity 0 only).
// rec: [n_obs][nq][kDyadicSlots] block sums in decomposition order.
// scratch: [n_obs][nq][sstride] (>= cnt / 1024 doubles per row).
__global__ void __launch_bounds__(kDyThreads) dyadic_blocks_kernel(const double* __restrict__ vals, int64_t qstride,
                                                                   int64_t vstride, const int64_t* __restrict__ gcounts,
                                                                   int world, int rank, int64_t n_obs,
                                                                   const double* __restrict__ center, int mode,
                                                                   double* __restrict__ rec, double* scratch,
                                                                   int64_t sstride) {
    __shared__ double red[33];
    __shared__ int lv[kDyadicSlots];
    __shared__ int64_t st[kDyadicSlots];
    __shared__ int nb_s;
    const int64_t j = blockIdx.x;
    const int q = blockIdx.y, nq = gridDim.y;
    int64_t off = 0;
    for (int r = 0; r < rank; ++r) off += gcounts[r * n_obs + j];
    const int64_t cnt = gcounts[rank * n_obs + j];
    if (threadIdx.x == 0) nb_s = dyadic_decompose(off, off + cnt, lv, st);
    __syncthreads();
    const int nb = nb_s;
    const double* src0 = vals + q * qstride + j * vstride - off;  // indexed by global compacted position
    double* scr = scratch + (j * nq + q) * sstride;
    const double c = (mode == 1) ? center[j] : 0.0;
    const int t = threadIdx.x;
    auto leaf = [&](int64_t pos) {
        double v = src0[pos];
        if (mode == 1) {
            const double d = v - c;
            v = d * d;
        }
        return v;
    };
    for (int k = 0; k < nb; ++k) {
        const int64_t len = int64_t(1) << lv[k], start = st[k];
        double sum;
        if (len <= kDyThreads) {
            sum = cta_tree(t < len ? leaf(start + t) : -0.0, red);
        } else {
            int64_t n = len >> 10;
            for (int64_t w = 0; w < n; ++w) {
                const double s = cta_tree(leaf(start + w * kDyThreads + t), red);
                if (t == 0) scr[w] = s;
            }
            __syncthreads();
            while (n > kDyThreads) {  // in place: window w is written after it is read, at w < 1024 w
                const int64_t m = n >> 10;
                for (int64_t w = 0; w < m; ++w) {
                    const double s = cta_tree(scr[w * kDyThreads + t], red);
                    if (t == 0) scr[w] = s;
                }
                __syncthreads();
                n = m;
            }
            sum = cta_tree(t < n ? scr[t] : -0.0, red);
        }
        if (t == 0) rec[(j * nq + q) * kDyadicSlots + k] = sum;
    }
}

// One thread per (observation, quantity): merge every rank's blocks in rank
// order into the root of the tree over all valid walkers.  sums: [nq][n_obs];
// counts_total (optional): [n_obs] valid walkers; means (optional): sums of
// quantity 0 / counts (IEEE division, executor.cpp:103).
__global__ void dyadic_finish_kernel(const double* __restrict__ rec, const int64_t* __restrict__ gcounts, int world,
                                     int64_t n_obs, int nq, double* __restrict__ sums,
                                     int64_t* __restrict__ counts_total, double* __restrict__ means) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_obs * nq) return;
    const int64_t j = i % n_obs;
    const int q = static_cast<int>(i / n_obs);
    int lvl[kDyadicSlots + 2];
    int64_t idx[kDyadicSlots + 2];
    double val[kDyadicSlots + 2];
    int top = 0;
    int blv[kDyadicSlots];
    int64_t bst[kDyadicSlots];
    int64_t off = 0;
    auto merge = [&]() {
        while (top >= 2 && lvl[top - 1] == lvl[top - 2] && idx[top - 2] % 2 == 0 && idx[top - 1] == idx[top - 2] + 1) {
            val[top - 2] = val[top - 2] + val[top - 1];
            lvl[top - 2] += 1;
            idx[top - 2] >>= 1;
            --top;
        }
    };
    for (int r = 0; r < world; ++r) {
        const int64_t cnt = gcounts[r * n_obs + j];
        const int nb = dyadic_decompose(off, off + cnt, blv, bst);
        const double* rr = rec + static_cast<int64_t>(r) * n_obs * nq * kDyadicSlots + (j * nq + q) * kDyadicSlots;
        for (int k = 0; k < nb; ++k) {
            lvl[top] = blv[k];
            idx[top] = bst[k] >> blv[k];
            val[top] = rr[k];
            ++top;
            merge();
        }
        off += cnt;
    }
    // promote the trailing left children through the -0.0 padding (x + -0.0 == x)
    while (top > 1) {
        lvl[top - 1] += 1;
        idx[top - 1] >>= 1;
        merge();
    }
    const double total = top ? val[0] : 0.0;  // pairwise_sum of nothing is +0.0
    sums[q * n_obs + j] = total;
    if (q == 0) {
        if (counts_total) counts_total[j] = off;
        if (means) means[j] = total / static_cast<double>(off);
    }
}

}  // namespace

// Segments index gridDim.y (<= 65535): larger segment counts run as several
// launches over pointer-offset segment groups (results unchanged).
constexpr int64_t kMaxGridY = 65535;

cudaError_t launch_tree_pass(const double* in, int64_t in_stride, const int64_t* counts, int64_t n_uniform,
                             int64_t n_seg, double* out, int64_t out_stride, const double* center, int mode,
                             cudaStream_t s) {
    // n_uniform is the max count when counts is given.
    const int64_t chunks = (n_uniform + kChunk - 1) / kChunk;
    if (chunks <= 0 || n_seg <= 0) return cudaSuccess;
    for (int64_t g = 0; g < n_seg; g += kMaxGridY) {
        const int64_t ng = std::min(kMaxGridY, n_seg - g);
        const dim3 grid(static_cast<unsigned>(chunks), static_cast<unsigned>(ng));
        tree_pass_kernel<<<grid, kThreads, 0, s>>>(in + g * in_stride, in_stride, counts ? counts + g : nullptr,
                                                   n_uniform, out + g * out_stride, out_stride,
                                                   center ? center + g : nullptr, mode);
    }
    return cudaGetLastError();
}

cudaError_t launch_unit_partials(const double* values, int64_t n_units, int64_t unit0, int64_t cpo,
                                 int64_t n_particles, const double* center, int mode, double* out, cudaStream_t s) {
    if (n_units <= 0) return cudaSuccess;
    unit_partials_kernel<<<static_cast<unsigned>(n_units), kThreads, 0, s>>>(values, unit0, cpo, n_particles, center,
                                                                             mode, out);
    return cudaGetLastError();
}

cudaError_t launch_dyadic_blocks(const double* vals, int64_t qstride, int nq, int64_t vstride, const int64_t* gcounts,
                                 int world, int rank, int64_t n_obs, const double* center, int mode, double* rec,
                                 double* scratch, int64_t sstride, cudaStream_t s) {
    if (n_obs <= 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>(n_obs), static_cast<unsigned>(nq));
    dyadic_blocks_kernel<<<grid, kDyThreads, 0, s>>>(vals, qstride, vstride, gcounts, world, rank, n_obs, center,
                                                     mode, rec, scratch, sstride);
    return cudaGetLastError();
}

cudaError_t launch_dyadic_finish(const double* rec, const int64_t* gcounts, int world, int64_t n_obs, int nq,
                                 double* sums, int64_t* counts_total, double* means, cudaStream_t s) {
    const int64_t n = n_obs * nq;
    if (n <= 0) return cudaSuccess;
    dyadic_finish_kernel<<<static_cast<unsigned>((n + 63) / 64), 64, 0, s>>>(rec, gcounts, world, n_obs, nq, sums,
                                                                            counts_total, means);
    return cudaGetLastError();
}

cudaError_t tree_reduce(const double* in, int64_t in_stride, const int64_t* counts, int64_t n, int64_t n_seg,
                        double* sums, const double* center, int mode, double* scratch, cudaStream_t s,
                        int* launches) {
    // Pass 1 reads the leaves (optionally per-segment counts, optional square).
    int64_t m = (n + kChunk - 1) / kChunk;
    if (m <= 0) m = 1;
    double* a = scratch;
    double* b = scratch + n_seg * m;
    cudaError_t e;
    if (n == 0) {
        // Empty segments sum to +0.0 (pairwise_sum of nothing, executor.cpp:12).
        return cudaMemsetAsync(sums, 0, sizeof(double) * n_seg, s);
    }
    e = launch_tree_pass(in, in_stride, counts, n, n_seg, (m == 1) ? sums : a, (m == 1) ? 1 : m, center, mode, s);
    if (launches) ++*launches;
    if (e != cudaSuccess || m == 1) return e;
    // Later passes: the chunk partials.  Every segment has its own count of
    // partials when counts are given: ceil(count / 1024); trailing partial
    // slots beyond it must be excluded (they would be -0.0 anyway, so using
    // the uniform count is exact).
    double* cur = a;
    int64_t len = m;
    while (len > 1) {
        const int64_t nxt = (len + kChunk - 1) / kChunk;
        double* dst = (nxt == 1) ? sums : ((cur == a) ? b : a);
        e = launch_tree_pass(cur, len, nullptr, len, n_seg, dst, (nxt == 1) ? 1 : nxt, nullptr, 0, s);
        if (launches) ++*launches;
        if (e != cudaSuccess) return e;
        cur = dst;
        len = nxt;
    }
    return cudaSuccess;
}

cudaError_t launch_divide(const double* sums, const int64_t* counts, int64_t n_uniform, int64_t n_seg,
                          double* means, cudaStream_t s) {
    divide_kernel<<<static_cast<unsigned>((n_seg + 127) / 128), 128, 0, s>>>(sums, counts, n_uniform, n_seg, means);
    return cudaGetLastError();
}

cudaError_t launch_estimates(const double* means, const double* sumsq, const double* sumaux, const int64_t* counts,
                             int64_t n_uniform, int64_t n_particles, int64_t n_seg, void* out, cudaStream_t s) {
    estimates_kernel<<<static_cast<unsigned>((n_seg + 127) / 128), 128, 0, s>>>(
        means, sumsq, sumaux, counts, n_uniform, n_particles, n_seg, static_cast<smc_estimate*>(out));
    return cudaGetLastError();
}

cudaError_t compact_valid(const double* values, const double* aux, const uint8_t* failed, int64_t n, int64_t n_seg,
                          double* cvalues, double* caux, int64_t* counts, int64_t* chunk_tmp, cudaStream_t s) {
    const int64_t chunks = (n + kChunk - 1) / kChunk;
    if (chunks <= 0 || n_seg <= 0) return cudaSuccess;
    int64_t* chunk_counts = chunk_tmp;
    int64_t* chunk_offsets = chunk_tmp + n_seg * chunks;
    for (int64_t g = 0; g < n_seg; g += kMaxGridY) {
        const int64_t ng = std::min(kMaxGridY, n_seg - g);
        const dim3 grid(static_cast<unsigned>(chunks), static_cast<unsigned>(ng));
        count_valid_kernel<<<grid, kThreads, 0, s>>>(failed + g * n, n, chunks, chunk_counts + g * chunks);
    }
    scan_chunks_kernel<<<static_cast<unsigned>((n_seg + 63) / 64), 64, 0, s>>>(chunk_counts, chunks, n_seg,
                                                                              chunk_offsets, counts);
    for (int64_t g = 0; g < n_seg; g += kMaxGridY) {
        const int64_t ng = std::min(kMaxGridY, n_seg - g);
        const dim3 grid(static_cast<unsigned>(chunks), static_cast<unsigned>(ng));
        compact_kernel<<<grid, kThreads, 0, s>>>(values + g * n, aux + g * n, failed + g * n, n, chunks,
                                                 chunk_offsets + g * chunks, cvalues + g * n, caux + g * n);
    }
    return cudaGetLastError();
}

}  // namespace smc
