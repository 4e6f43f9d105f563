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

// Lattice coefficient image for the fast kernels.
//   v2 = sum_{k1>=1} Re(P1[k1] * A(k1)),  v1 = Re(B(0)) + sum_{k1>=1} Re(P1[k1] * B(k1))
//   A(k1) = k1 g_{k1,0} + sum_j [8-coefficient pair update with P2[j]]
// Tiles cover j in [8t+1, 8t+8].  For tile t and row k1 in [1, rows[t]],
// tile_row[t*(R+1)+k1] = (offset into coef, pair count n <= 8); the pair
// coefficients are 8 doubles each.  Row 0 (k1 = 0) keeps 2 doubles per j.
struct LatticeImg {
    int64_t sample_stride;  // doubles between consecutive samples' coef/row0/g0 (batched)
    int32_t K;        // max_wavenumber
    int32_t R;        // largest k1 with any mode (rows 1..R)
    int32_t J;        // largest |k2| with any mode
    int32_t J0;       // largest j with a row-0 mode
    int32_t n_tiles;  // ceil(J / 8)
    int32_t pad_;
    const int32_t* tile_rows;   // [n_tiles]: last row with pairs in tile t
    const int2* tile_row;       // [n_tiles][R+1]: (offset, count)
    const double* coef;         // pair coefficients
    const double* row0;         // [J0][2]: (-j g_re, j g_im) for (0, j)
    const double* g0;           // [R+1][2]: k1 * g_{k1,0}
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
