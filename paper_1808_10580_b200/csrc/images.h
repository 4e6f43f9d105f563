// images.h — device-side problem images (POD, shared by host packer and
// kernels).  All pointers are device pointers into the context's image
// buffer.  Layout rationale is in DESIGN.md §3.
#pragma once

#include <cstdint>

#include <vector_types.h>

namespace smc {

// ScalarField (include/scalarmc/fields.hpp:121-164) — SoA term arrays.
struct ScalarImg {
    int32_t kind;  // smc_scalar_kind
    int32_t n;
    double constant;
    double g0, g1;  // linear gradient
    double neg_sharpness;  // -a for bumps (negation is exact)
    const double* amp;     // [n]
    const double* freq;    // [n][2]
    const double* phase;   // [n]
    const double* center;  // [n][2]
};

// One AD observation: start point and the reference's step schedule
// (sde.cpp:42-45): n steps of dt, the last one shortened to dt_last.
struct AdObsImg {
    double x1, x2;
    int64_t n_steps;
    double dt, dt_last;
    double rdt, rdt_last;  // sqrt(dt), sqrt(dt_last)
    double sr, sr_last;    // sigma * sqrt(dt), sigma * sqrt(dt_last)
};

// Canonical sorted mode (fields.hpp:56-60) for the strict kernel.
struct ModeImg {
    int32_t k1, k2;
    double re, im, d1, d2;
};

// Tiled lattice coefficients for the generic fast kernels.
// Columns j are processed in tiles of 8 (j = 8t+1 .. 8t+8); tile t covers rows
// k1 = 1..rows_t.  Per-sample block of doubles (sample_stride apart):
//   [tile data][row0][g0]
//   tile data: for t, for k1 = 1..rows_t: 8 pairs x (alpha_re, alpha_im,
//              beta_re, beta_im), zero-padded past the row's last mode
//   row0:      8 n_tiles x (g_re, g_im) of modes (0, j)
//   g0:        (R+1) x (g_re, g_im) of modes (k1, 0)
// with g = 2 c / |k|, alpha = g(k1,j) + g(k1,-j), beta = g(k1,j) - g(k1,-j).
struct LatticeImg {
    int64_t sample_stride;  // doubles per sample block
    int32_t K;
    int32_t R;          // largest k1 with any mode
    int32_t J0;         // largest j with a row-0 mode
    int32_t n_tiles;
    int32_t row0_off;   // offsets (doubles) inside a sample block
    int32_t g0_off;
    const int2* tiles;  // [n_tiles]: (rows_t, data offset in doubles)
    const double* coef; // sample 0 block
};

struct VelImg {
    int32_t is_constant;
    int32_t n_modes;
    double c1, c2;
    int32_t K;
    int32_t pad_;
    const ModeImg* modes;  // strict kernel
    LatticeImg lat;        // fast kernels
};

}  // namespace smc
