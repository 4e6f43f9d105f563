// host_problem.h — host side of the C ABI: validation with the reference's
// messages, field canonicalisation, step schedules and device-image packing.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/scalarmc_b200.h"
#include "images.h"

namespace smc {

struct Error {
    int code;
    std::string msg;
};
[[noreturn]] void raise(int code, const std::string& msg);

// FourierVelocityField after its constructor (src/fields.cpp:35-69).
struct HostMode {
    int k1, k2;
    double re, im;
};
struct PreparedVelocity {
    bool is_constant = true;
    double c1 = 0.0, c2 = 0.0;
    int K = 0;
    std::vector<HostMode> modes;  // canonical, (k1,k2)-sorted
};
PreparedVelocity prepare_velocity(const smc_velocity& v);
double amplitude_bound(const PreparedVelocity& v);  // fields.cpp:109-113, :140-142

void check_kappa(double kappa);                      // fields.cpp:158-160
void check_scalar(const smc_scalar_field& f);        // fields.cpp:224-232
void check_domain(const smc_domain& d);              // geometry.cpp:10-19

double ad_resolved_dt(const smc_ad_problem& p);      // forward_ad.cpp:10-15
void ad_validate(const smc_ad_problem& p);           // forward_ad.cpp:17-28
double bvp_resolved_dt(const smc_bvp_problem& p, const PreparedVelocity& v);  // forward_bvp.cpp:9-18
void bvp_validate(const smc_bvp_problem& p);         // forward_bvp.cpp:20-32
bool domain_contains(const smc_domain& d, double x1, double x2);  // geometry.cpp:22-31

// Tiled lattice layout (images.h) for one mode set.
struct LatticeHost {
    int K = 0, R = 0, J0 = 0, n_tiles = 1;
    std::vector<int2> tiles;      // (rows_t, offset)
    int64_t row0_off = 0, g0_off = 0, stride = 0;
};
// Structure only (which (k1,k2) slots exist) from a mode list.
LatticeHost lattice_structure(const PreparedVelocity& v);
// Coefficients of `v` (same mode set as the structure): stride doubles at dst.
void lattice_fill(const LatticeHost& s, const PreparedVelocity& v, double* dst);

// Coefficient block of the compile-time disk kernel (disk_shape.h layout).
void disk_fill(int K, const PreparedVelocity& v, double* dst);

// PriorSpec::modes (src/inference.cpp:24-40).
std::vector<HostMode> prior_modes(int cutoff);

// Gather map u (prior order, velocity_from_coefficients, inference.cpp:63-73)
// -> coefficient block (disk or tiled-lattice layout), so the blocks of many
// parameter samples are packed on the device.  Slot q of a block is
//   v = (ip[q] >= 0 ? 2 u[ip[q]] / kp[q] : 0);
//   if (ms[q] != 0) v = v +/- (im[q] >= 0 ? 2 u[im[q]] / km[q] : 0)
// evaluated without contraction: the same operations lattice_fill/disk_fill
// perform on the field built from u, so the blocks are bit-identical.
struct PackMap {
    int64_t stride = 0;
    std::vector<int32_t> ip, im;
    std::vector<double> kp, km;
    std::vector<int8_t> ms;  // +1: alpha (g+ + g-), -1: beta (g+ - g-), 0: single mode
};
PackMap pack_map(int cutoff, bool disk, const LatticeHost* lattice);
// Full prior disk as a mode list (coefficients 1), for the layout structure.
PreparedVelocity prior_structure(int cutoff);

// Step schedule of one AD observation (sde.cpp:42-45).
// ---- spectral Galerkin reference solver (src/galerkin.cpp) ----------------
struct GalerkinModes {
    std::vector<int> k1, k2;  // basis order: k1 = -L..L outer, k2 = -L..L inner (galerkin.cpp:20-33)
    int max_abs = 0;
    int64_t size() const { return static_cast<int64_t>(k1.size()); }
};
GalerkinModes galerkin_modes(const smc_galerkin_basis& b);
// Dense system A (galerkin.cpp:108-142), row-major, complex interleaved
// (2 nb^2 doubles), built with the reference's complex arithmetic.
std::vector<double> galerkin_assemble(double kappa, const PreparedVelocity& v, const GalerkinModes& m);
double galerkin_radius(const std::vector<double>& A, int64_t nb);  // max_l sum_m |A_lm|
// vector_coefficients (fields.cpp:112-123) on a dense (2K+1)^2 grid for the
// device assembly: 4 doubles per cell [c1re, c1im, c2re, c2im] + present flags.
struct VhatGrid {
    int K = 0;
    std::vector<double> c;
    std::vector<unsigned char> present;
};
VhatGrid galerkin_vhat_grid(const PreparedVelocity& v);
// Exact projection of a constant or integer-mode cosine theta_0
// (galerkin.cpp:43-81) into theta (2 nb doubles); false: needs quadrature.
bool galerkin_project_exact(const smc_scalar_field& f, const GalerkinModes& m, std::vector<double>& theta);

AdObsImg make_ad_obs(double t, double x1, double x2, double dt, double sigma);

}  // namespace smc
