// geometry.cuh — Domain::contains and Domain::boundary_exit on the device
// (src/geometry.cpp:22-31, :47-114).  Included per translation unit so the
// strict build keeps the reference's exact operation order.
#pragma once

#include "images.h"

namespace smc {

struct DomainImg {
    int32_t kind;  // smc_domain_kind
    int32_t pad_;
    double lo1, lo2, hi1, hi2;  // box
    double c1, c2, r, r2;       // disk (r2 = r * r)
};

// KIND: 0 = the kind read at run time; 1 (box) / 2 (disk) compile the test
// for that kind only (the walker kernels' box instantiation).
template <class T, int KIND = 0>
__device__ __forceinline__ bool domain_contains(const DomainImg& d, T x1, T x2) {
    if constexpr (KIND == 1) return (x1 > T(d.lo1)) & (x1 < T(d.hi1)) & (x2 > T(d.lo2)) & (x2 < T(d.hi2));
    // both tests evaluated, then selected: no branch on the (uniform) kind in
    // the walker loop, so the step stays one basic block
    const bool in_box = (x1 > T(d.lo1)) & (x1 < T(d.hi1)) & (x2 > T(d.lo2)) & (x2 < T(d.hi2));
    const T q1 = x1 - T(d.c1), q2 = x2 - T(d.c2);
    const bool in_disk = q1 * q1 + q2 * q2 < T(d.r2);
    return d.kind == 1 ? in_box : (d.kind == 2 ? in_disk : true);
}

template <class T>
__device__ __forceinline__ T face_crossing(T from, T to, T c) {  // geometry.cpp:47-52
    const T d = to - from;
    if (d == T(0)) return T(INFINITY);
    const T t = (c - from) / d;
    return (t >= T(0) && t <= T(1)) ? t : T(INFINITY);
}

template <class T>
__device__ __forceinline__ T clamp_ref(T v, T lo, T hi) {  // std::clamp
    return v < lo ? lo : (hi < v ? hi : v);
}

// Crossing of segment inside->outside with the boundary; returns the fraction
// and writes the crossing point (geometry.cpp:56-114).
template <class T>
__device__ __forceinline__ T boundary_exit(const DomainImg& d, T in1, T in2, T out1, T out2, T& p1, T& p2) {
    if (d.kind == 1) {
        const T d1 = out1 - in1, d2 = out2 - in2;
        T best_t = T(INFINITY), best_val = T(0);
        int best_axis = -1;
        const T faces[2][2] = {{T(d.lo1), T(d.hi1)}, {T(d.lo2), T(d.hi2)}};
#pragma unroll
        for (int axis = 0; axis < 2; ++axis) {
            const T from = axis == 0 ? in1 : in2;
            const T to = axis == 0 ? out1 : out2;
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                const T t = face_crossing(from, to, faces[axis][f]);
                if (t < best_t) {
                    best_t = t;
                    best_axis = axis;
                    best_val = faces[axis][f];
                }
            }
        }
        T x = in1 + best_t * d1, y = in2 + best_t * d2;
        if (best_axis == 0) {
            x = best_val;
            y = clamp_ref(y, T(d.lo2), T(d.hi2));
        } else {
            y = best_val;
            x = clamp_ref(x, T(d.lo1), T(d.hi1));
        }
        p1 = x;
        p2 = y;
        return best_t;
    }
    // disk: |(inside - c) + t d|^2 = r^2, root in [0,1], then radial projection.
    const T q1 = in1 - T(d.c1), q2 = in2 - T(d.c2);
    const T d1 = out1 - in1, d2 = out2 - in2;
    const T a = d1 * d1 + d2 * d2;
    const T bq = T(2) * (q1 * d1 + q2 * d2);
    const T c = (q1 * q1 + q2 * q2) - T(d.r) * T(d.r);
    const T disc = bq * bq - T(4) * a * c;
    const T t = (-bq + sqrt(disc)) / (T(2) * a);
    const T tc = clamp_ref(t, T(0), T(1));
    T x = in1 + tc * d1, y = in2 + tc * d2;
    const T r1 = x - T(d.c1), r2 = y - T(d.c2);
    const T rn = hypot(r1, r2);
    if (rn > T(0)) {
        const T s = T(d.r) / rn;
        x = T(d.c1) + s * r1;
        y = T(d.c2) + s * r2;
    }
    p1 = x;
    p2 = y;
    return tc;
}

}  // namespace smc
