// scalar_eval.cuh — ScalarField::operator() on the device
// (src/fields.cpp:235-253).  Included by each kernel translation unit so it
// inherits that unit's contraction mode (-fmad=false for the strict path).
#pragma once

#include "fastmath.cuh"
#include "images.h"
#include "../../include/scalarmc_b200.h"

namespace smc {

// The strict translation units keep libdevice exp; the fast ones use the
// constant-bank fastmath version.
#ifdef SMC_STRICT_TU
#define SMC_SCALAR_EXP exp
#else
#define SMC_SCALAR_EXP fm::exp_
#endif

__device__ __forceinline__ double scalar_eval(const ScalarImg& f, double x1, double x2) {
    switch (f.kind) {
        case SMC_SCALAR_COSINE: {
            double s = 0.0;
            for (int i = 0; i < f.n; ++i) {
                const double dot = __ldg(f.freq + 2 * i) * x1 + __ldg(f.freq + 2 * i + 1) * x2;
                s += __ldg(f.amp + i) * cos(dot + __ldg(f.phase + i));
            }
            return s;
        }
        case SMC_SCALAR_BUMPS: {
            double s = 0.0;
            for (int i = 0; i < f.n; ++i) {
                const double d1 = x1 - __ldg(f.center + 2 * i), d2 = x2 - __ldg(f.center + 2 * i + 1);
                s += __ldg(f.amp + i) * SMC_SCALAR_EXP(f.neg_sharpness * (d1 * d1 + d2 * d2));
            }
            return s;
        }
        case SMC_SCALAR_LINEAR:
            return f.constant + (f.g0 * x1 + f.g1 * x2);
        default:
            return f.constant;
    }
}

// Single-precision evaluation for the FP32 particle kernel.
__device__ __forceinline__ float scalar_eval_f32(const ScalarImg& f, float x1, float x2) {
    switch (f.kind) {
        case SMC_SCALAR_COSINE: {
            float s = 0.0f;
            for (int i = 0; i < f.n; ++i) {
                const float dot = float(__ldg(f.freq + 2 * i)) * x1 + float(__ldg(f.freq + 2 * i + 1)) * x2;
                s += float(__ldg(f.amp + i)) * cosf(dot + float(__ldg(f.phase + i)));
            }
            return s;
        }
        case SMC_SCALAR_BUMPS: {
            float s = 0.0f;
            for (int i = 0; i < f.n; ++i) {
                const float d1 = x1 - float(__ldg(f.center + 2 * i)), d2 = x2 - float(__ldg(f.center + 2 * i + 1));
                s += float(__ldg(f.amp + i)) * expf(float(f.neg_sharpness) * (d1 * d1 + d2 * d2));
            }
            return s;
        }
        case SMC_SCALAR_LINEAR:
            return float(f.constant) + (float(f.g0) * x1 + float(f.g1) * x2);
        default:
            return float(f.constant);
    }
}

}  // namespace smc
