// host_problem.cpp — validation, canonicalisation and packing on the host.
// Messages and exception classes follow the reference exactly so the C++ shim
// (host/scalarmc_forward_gpu.cpp) can rethrow the same std:: types.
#include "host_problem.h"

#include "disk_shape.h"

#include <algorithm>
#include <complex>
#include <cmath>
#include <limits>

namespace smc {

void raise(int code, const std::string& msg) { throw Error{code, msg}; }

namespace {
bool is_canonical(int k1, int k2) { return k1 > 0 || (k1 == 0 && k2 > 0); }  // fields.cpp:15
}  // namespace

PreparedVelocity prepare_velocity(const smc_velocity& v) {
    PreparedVelocity out;
    if (v.is_constant) {
        out.is_constant = true;
        out.c1 = v.constant[0];
        out.c2 = v.constant[1];
        return out;
    }
    out.is_constant = false;
    if (v.max_wavenumber <= 0) raise(SMC_EINVAL, "FourierVelocityField: max_wavenumber must be positive");
    out.K = v.max_wavenumber;
    if (v.n_modes < 0) raise(SMC_EINVAL, "FourierVelocityField: negative mode count");
    out.modes.reserve(static_cast<size_t>(v.n_modes));
    for (int64_t i = 0; i < v.n_modes; ++i) {
        HostMode m{v.k[2 * i], v.k[2 * i + 1], v.coeff[2 * i], v.coeff[2 * i + 1]};
        if (m.k1 == 0 && m.k2 == 0) raise(SMC_EINVAL, "FourierVelocityField: k = (0,0) is not allowed");
        const double kn2 = double(m.k1) * m.k1 + double(m.k2) * m.k2;
        if (kn2 > double(out.K) * out.K + 1e-9) raise(SMC_EINVAL, "FourierVelocityField: |k| exceeds max_wavenumber");
        if (!std::isfinite(m.re) || !std::isfinite(m.im))
            raise(SMC_EINVAL, "FourierVelocityField: non-finite coefficient");
        if (!is_canonical(m.k1, m.k2)) m = HostMode{-m.k1, -m.k2, -m.re, m.im};  // v_k = -conj(v_-k)
        out.modes.push_back(m);
    }
    std::sort(out.modes.begin(), out.modes.end(), [](const HostMode& a, const HostMode& b) {
        return a.k1 != b.k1 ? a.k1 < b.k1 : a.k2 < b.k2;
    });
    for (size_t i = 1; i < out.modes.size(); ++i)
        if (out.modes[i].k1 == out.modes[i - 1].k1 && out.modes[i].k2 == out.modes[i - 1].k2)
            raise(SMC_EINVAL, "FourierVelocityField: duplicate mode (both members of a +/-k pair given?)");
    return out;
}

double amplitude_bound(const PreparedVelocity& v) {
    if (v.is_constant) return std::hypot(v.c1, v.c2);
    double s = 0.0;
    for (const auto& m : v.modes) s += 2.0 * std::hypot(m.re, m.im);
    return s;
}

void check_kappa(double kappa) {
    if (!(kappa >= 0.0)) raise(SMC_EINVAL, "DiffusionModel: kappa must be >= 0");
}

void check_scalar(const smc_scalar_field& f) {
    if (f.kind < SMC_SCALAR_CONSTANT || f.kind > SMC_SCALAR_LINEAR) raise(SMC_EINVAL, "ScalarField: unknown kind");
    if (f.n_terms < 0) raise(SMC_EINVAL, "ScalarField: negative term count");
    if (f.kind == SMC_SCALAR_BUMPS && !(f.sharpness > 0.0))
        raise(SMC_EINVAL, "ScalarField: sharpness must be positive");
    if (f.kind == SMC_SCALAR_COSINE && f.n_terms > 0 && (!f.amplitude || !f.freq || !f.phase))
        raise(SMC_EINVAL, "ScalarField: cosine terms need amplitude, freq and phase arrays");
    if (f.kind == SMC_SCALAR_BUMPS && f.n_terms > 0 && (!f.amplitude || !f.center))
        raise(SMC_EINVAL, "ScalarField: bumps need amplitude and center arrays");
}

void check_domain(const smc_domain& d) {
    if (d.kind == SMC_DOMAIN_BOX && !(d.lower[0] < d.upper[0] && d.lower[1] < d.upper[1]))
        raise(SMC_EINVAL, "Domain::box: lower corner must be strictly below upper");
    if (d.kind == SMC_DOMAIN_DISK && !(d.radius > 0.0)) raise(SMC_EINVAL, "Domain::disk: radius must be positive");
    if (d.kind < SMC_DOMAIN_TORUS || d.kind > SMC_DOMAIN_DISK) raise(SMC_EINVAL, "Domain: unknown kind");
}

double ad_resolved_dt(const smc_ad_problem& p) {
    if (p.dt > 0.0) return p.dt;
    double t_min = std::numeric_limits<double>::infinity();
    for (int64_t j = 0; j < p.n_obs; ++j) t_min = std::min(t_min, p.obs_t[j]);
    return t_min / 200.0;
}

void ad_validate(const smc_ad_problem& p) {
    if (p.n_obs <= 0) raise(SMC_EINVAL, "AdProblemSpec: no observations");
    for (int64_t j = 0; j < p.n_obs; ++j) {
        const double t = p.obs_t[j], x1 = p.obs_x[2 * j], x2 = p.obs_x[2 * j + 1];
        if (!(t > 0.0)) raise(SMC_EINVAL, "AdProblemSpec: observation times must be positive");
        if (!std::isfinite(x1) || !std::isfinite(x2)) raise(SMC_EINVAL, "AdProblemSpec: non-finite observation point");
        if (x1 < 0.0 || x1 >= 1.0 || x2 < 0.0 || x2 >= 1.0)
            raise(SMC_EINVAL, "AdProblemSpec: observation points must lie in [0,1)^2");
    }
    if (p.n_particles < 2) raise(SMC_EINVAL, "AdProblemSpec: need at least two particles");
    if (p.scheme != SMC_EULER_MARUYAMA && p.scheme != SMC_MILSTEIN) raise(SMC_EINVAL, "AdProblemSpec: unknown scheme");
    if (p.precision < SMC_FP64 || p.precision > SMC_FP64_STRICT) raise(SMC_EINVAL, "AdProblemSpec: unknown precision");
}

bool domain_contains(const smc_domain& d, double x1, double x2) {
    if (d.kind == SMC_DOMAIN_BOX) return x1 > d.lower[0] && x1 < d.upper[0] && x2 > d.lower[1] && x2 < d.upper[1];
    if (d.kind == SMC_DOMAIN_DISK) {
        const double q1 = x1 - d.center[0], q2 = x2 - d.center[1];
        return q1 * q1 + q2 * q2 < d.radius * d.radius;
    }
    return true;
}

double bvp_resolved_dt(const smc_bvp_problem& p, const PreparedVelocity& v) {
    if (p.dt > 0.0) return p.dt;
    double diam;
    if (p.domain.kind == SMC_DOMAIN_BOX) diam = std::hypot(p.domain.upper[0] - p.domain.lower[0], p.domain.upper[1] - p.domain.lower[1]);
    else if (p.domain.kind == SMC_DOMAIN_DISK) diam = 2.0 * p.domain.radius;
    else diam = 1.4142135623730951;
    const double speed = amplitude_bound(v);
    const double denom = 2.0 * p.kappa + speed * diam;
    const double raw = denom > 0.0 ? 1e-3 * diam * diam / denom : 1e-2;
    return std::clamp(raw, 1e-6, 1e-2);
}

void bvp_validate(const smc_bvp_problem& p) {
    if (p.domain.kind == SMC_DOMAIN_TORUS) raise(SMC_EINVAL, "BvpProblemSpec: domain must be bounded");
    if (p.n_obs <= 0) raise(SMC_EINVAL, "BvpProblemSpec: no observations");
    for (int64_t j = 0; j < p.n_obs; ++j) {
        const double x1 = p.obs_x[2 * j], x2 = p.obs_x[2 * j + 1];
        if (!std::isfinite(x1) || !std::isfinite(x2)) raise(SMC_EINVAL, "BvpProblemSpec: non-finite observation point");
        if (!domain_contains(p.domain, x1, x2))
            raise(SMC_EINVAL, "BvpProblemSpec: observation points must be strictly interior");
    }
    if (p.n_particles < 2) raise(SMC_EINVAL, "BvpProblemSpec: need at least two particles");
    if (p.max_steps < 1) raise(SMC_EINVAL, "BvpProblemSpec: max_steps must be positive");
    if (p.scheme != SMC_EULER_MARUYAMA && p.scheme != SMC_MILSTEIN) raise(SMC_EINVAL, "BvpProblemSpec: unknown scheme");
    if (p.precision < SMC_FP64 || p.precision > SMC_FP64_STRICT) raise(SMC_EINVAL, "BvpProblemSpec: unknown precision");
}

// ---------------------------------------------------------------------------
// Lattice packing.  For mode (k1,k2) with coefficient c, g = 2 c / |k|; the
// velocity is v1 = sum -k2 Re(g E), v2 = sum k1 Re(g E), E = P1[k1] P2[k2].
// A +/-j pair of row k1 with P2[j] = r + i s and Q[j] = j P2[j] contributes,
// with alpha = g+ + g-, beta = g+ - g-:
//   A  += (alpha_re r - beta_im s) + i (alpha_im r + beta_re s)   v2 += k1 Re(P1 A)
//   B' += (beta_re qr - alpha_im qs) + i (beta_im qr + alpha_re qs) v1 -= Re(P1 B')
// ---------------------------------------------------------------------------
namespace {

struct Slot {
    double gr = 0.0, gi = 0.0;
};

struct Grid {
    int K, R = 0, J = 0, J0 = 0;
    std::vector<Slot> g;  // [(K+1)][(2K+1)], index k1*(2K+1) + (k2+K)
    std::vector<int> jrow;
    explicit Grid(int K_) : K(K_), g(static_cast<size_t>(K_ + 1) * (2 * K_ + 1)), jrow(static_cast<size_t>(K_ + 1), 0) {}
    Slot& at(int k1, int k2) { return g[static_cast<size_t>(k1) * (2 * K + 1) + (k2 + K)]; }
};

Grid make_grid(const PreparedVelocity& v, bool with_values) {
    Grid gr(v.K);
    for (const auto& m : v.modes) {
        if (with_values) {
            const double kn = std::sqrt(double(m.k1) * m.k1 + double(m.k2) * m.k2);
            gr.at(m.k1, m.k2) = Slot{2.0 * m.re / kn, 2.0 * m.im / kn};
        }
        const int j = m.k2 >= 0 ? m.k2 : -m.k2;
        if (m.k1 == 0) gr.J0 = std::max(gr.J0, j);
        else {
            gr.R = std::max(gr.R, m.k1);
            gr.jrow[static_cast<size_t>(m.k1)] = std::max(gr.jrow[static_cast<size_t>(m.k1)], j);
            gr.J = std::max(gr.J, j);
        }
    }
    return gr;
}

constexpr int kTileW = 8;

}  // namespace

LatticeHost lattice_structure(const PreparedVelocity& v) {
    LatticeHost L;
    const Grid gr = make_grid(v, false);
    L.K = v.K;
    L.R = gr.R;
    L.J0 = gr.J0;
    const int jmax = std::max(gr.J, gr.J0);
    L.n_tiles = std::max(1, (jmax + kTileW - 1) / kTileW);
    int64_t off = 0;
    for (int t = 0; t < L.n_tiles; ++t) {
        int rows = (t == 0) ? L.R : 0;  // tile 0 folds every row's k2 = 0 term
        for (int k1 = 1; k1 <= L.R; ++k1)
            if (gr.jrow[static_cast<size_t>(k1)] > kTileW * t) rows = std::max(rows, k1);
        L.tiles.push_back(int2{rows, static_cast<int>(off)});
        off += static_cast<int64_t>(rows) * kTileW * 4;
    }
    L.row0_off = off;
    off += 2 * kTileW * L.n_tiles;
    L.g0_off = off;
    off += 2 * (L.R + 1);
    L.stride = (off + 1) & ~int64_t(1);  // keep blocks 16-byte aligned
    return L;
}

void lattice_fill(const LatticeHost& s, const PreparedVelocity& v, double* dst) {
    Grid gr = make_grid(v, true);
    std::fill(dst, dst + s.stride, 0.0);
    for (int t = 0; t < s.n_tiles; ++t) {
        const int2 tl = s.tiles[static_cast<size_t>(t)];
        for (int k1 = 1; k1 <= tl.x; ++k1) {
            double* c = dst + tl.y + static_cast<int64_t>(k1 - 1) * kTileW * 4;
            for (int q = 0; q < kTileW; ++q) {
                const int j = kTileW * t + q + 1;
                if (j > gr.K) break;
                const Slot gp = gr.at(k1, j), gm = gr.at(k1, -j);
                c[4 * q + 0] = gp.gr + gm.gr;  // alpha
                c[4 * q + 1] = gp.gi + gm.gi;
                c[4 * q + 2] = gp.gr - gm.gr;  // beta
                c[4 * q + 3] = gp.gi - gm.gi;
            }
        }
    }
    double* row0 = dst + s.row0_off;
    for (int j = 1; j <= s.J0; ++j) {
        const Slot g = gr.at(0, j);
        row0[2 * (j - 1)] = g.gr;
        row0[2 * (j - 1) + 1] = g.gi;
    }
    double* g0 = dst + s.g0_off;
    for (int k1 = 1; k1 <= s.R; ++k1) {
        const Slot g = gr.at(k1, 0);
        g0[2 * k1] = g.gr;
        g0[2 * k1 + 1] = g.gi;
    }
}

void disk_fill(int K, const PreparedVelocity& v, double* dst) {
    Grid gr = make_grid(v, true);
    const int n_pairs = disk_n_pairs(K);
    double* pairs = dst;
    double* row0 = dst + 4 * n_pairs;
    double* g0 = row0 + 2 * K;
    int p = 0;
    for (int k1 = 1; k1 <= K; ++k1) {
        for (int j = 1; j <= disk_jmax(K, k1); ++j, ++p) {
            const Slot gp = gr.at(k1, j), gm = gr.at(k1, -j);
            double* c = pairs + 4 * p;
            c[0] = gp.gr + gm.gr;  // alpha
            c[1] = gp.gi + gm.gi;
            c[2] = gp.gr - gm.gr;  // beta
            c[3] = gp.gi - gm.gi;
        }
    }
    for (int j = 1; j <= K; ++j) {
        const Slot g = gr.at(0, j);
        row0[2 * (j - 1)] = g.gr;
        row0[2 * (j - 1) + 1] = g.gi;
    }
    for (int k1 = 1; k1 <= K; ++k1) {
        const Slot g = gr.at(k1, 0);
        g0[2 * (k1 - 1)] = g.gr;
        g0[2 * (k1 - 1) + 1] = g.gi;
    }
}

std::vector<HostMode> prior_modes(int cutoff) {
    std::vector<HostMode> out;
    for (int k1 = -cutoff; k1 <= cutoff; ++k1)
        for (int k2 = -cutoff; k2 <= cutoff; ++k2) {
            if (!is_canonical(k1, k2)) continue;
            if (double(k1) * k1 + double(k2) * k2 > double(cutoff) * cutoff) continue;
            out.push_back({k1, k2, 0.0, 0.0});
        }
    std::sort(out.begin(), out.end(), [](const HostMode& a, const HostMode& b) {
        const double na = double(a.k1) * a.k1 + double(a.k2) * a.k2;
        const double nb = double(b.k1) * b.k1 + double(b.k2) * b.k2;
        if (na != nb) return na < nb;
        return a.k1 != b.k1 ? a.k1 < b.k1 : a.k2 < b.k2;
    });
    return out;
}

PreparedVelocity prior_structure(int cutoff) {
    PreparedVelocity v;
    v.is_constant = false;
    v.K = cutoff;
    for (const auto& m : prior_modes(cutoff)) v.modes.push_back(HostMode{m.k1, m.k2, 1.0, 0.0});
    std::sort(v.modes.begin(), v.modes.end(), [](const HostMode& a, const HostMode& b) {
        return a.k1 != b.k1 ? a.k1 < b.k1 : a.k2 < b.k2;
    });
    return v;
}

PackMap pack_map(int K, bool disk, const LatticeHost* lattice) {
    const std::vector<HostMode> pm = prior_modes(K);
    std::vector<int32_t> idx(static_cast<size_t>((K + 1) * (2 * K + 1)), -1);
    auto at = [&](int k1, int k2) -> int32_t& { return idx[static_cast<size_t>(k1 * (2 * K + 1) + k2 + K)]; };
    for (size_t i = 0; i < pm.size(); ++i) at(pm[i].k1, pm[i].k2) = static_cast<int32_t>(i);
    auto kn = [](int k1, int k2) { return std::sqrt(double(k1) * k1 + double(k2) * k2); };
    PackMap m;
    m.stride = disk ? disk_n_coef(K) : lattice->stride;
    const size_t n = static_cast<size_t>(m.stride);
    m.ip.assign(n, -1);
    m.im.assign(n, -1);
    m.kp.assign(n, 1.0);
    m.km.assign(n, 1.0);
    m.ms.assign(n, 0);
    auto present = [&](int k1, int k2) { return k1 >= 0 && k2 >= -K && k2 <= K && at(k1, k2) >= 0; };
    // single mode (k1, k2), real or imaginary part
    auto single = [&](int64_t slot, int k1, int k2, int part) {
        if (!present(k1, k2)) return;
        m.ip[slot] = 2 * at(k1, k2) + part;
        m.kp[slot] = kn(k1, k2);
    };
    // the 4 slots of a +/-j pair: alpha_re, alpha_im, beta_re, beta_im
    auto pair = [&](int64_t base, int k1, int j) {
        for (int q = 0; q < 4; ++q) {
            const int part = q & 1;
            single(base + q, k1, j, part);
            m.ms[base + q] = q < 2 ? 1 : -1;
            if (present(k1, -j)) {
                m.im[base + q] = 2 * at(k1, -j) + part;
                m.km[base + q] = kn(k1, -j);
            }
        }
    };
    if (disk) {  // disk_fill's slot order
        int64_t p = 0;
        for (int k1 = 1; k1 <= K; ++k1)
            for (int j = 1; j <= disk_jmax(K, k1); ++j, ++p) pair(4 * p, k1, j);
        const int64_t row0 = 4 * disk_n_pairs(K), g0 = row0 + 2 * K;
        for (int j = 1; j <= K; ++j) {
            single(row0 + 2 * (j - 1), 0, j, 0);
            single(row0 + 2 * (j - 1) + 1, 0, j, 1);
        }
        for (int k1 = 1; k1 <= K; ++k1) {
            single(g0 + 2 * (k1 - 1), k1, 0, 0);
            single(g0 + 2 * (k1 - 1) + 1, k1, 0, 1);
        }
    } else {  // lattice_fill's slot order
        const LatticeHost& s = *lattice;
        for (int t = 0; t < s.n_tiles; ++t) {
            const int2 tl = s.tiles[static_cast<size_t>(t)];
            for (int k1 = 1; k1 <= tl.x; ++k1)
                for (int q = 0; q < kTileW; ++q) {
                    const int j = kTileW * t + q + 1;
                    if (j > K) break;
                    pair(tl.y + static_cast<int64_t>(k1 - 1) * kTileW * 4 + 4 * q, k1, j);
                }
        }
        for (int j = 1; j <= s.J0; ++j) {
            single(s.row0_off + 2 * (j - 1), 0, j, 0);
            single(s.row0_off + 2 * (j - 1) + 1, 0, j, 1);
        }
        for (int k1 = 1; k1 <= s.R; ++k1) {
            single(s.g0_off + 2 * k1, k1, 0, 0);
            single(s.g0_off + 2 * k1 + 1, k1, 0, 1);
        }
    }
    return m;
}

GalerkinModes galerkin_modes(const smc_galerkin_basis& b) {
    const int L = b.cutoff;
    if (L < 1) raise(SMC_EINVAL, "GalerkinBasis: cutoff must be >= 1");
    if (b.kind != 0 && b.kind != 1) raise(SMC_EINVAL, "GalerkinBasis: unknown kind");
    GalerkinModes m;
    for (int k1 = -L; k1 <= L; ++k1)
        for (int k2 = -L; k2 <= L; ++k2) {
            if (b.kind == 1 && double(k1) * k1 + double(k2) * k2 > double(L) * L) continue;
            m.k1.push_back(k1);
            m.k2.push_back(k2);
            m.max_abs = std::max({m.max_abs, std::abs(k1), std::abs(k2)});
        }
    return m;
}

std::vector<double> galerkin_assemble(double kappa, const PreparedVelocity& v, const GalerkinModes& m) {
    using cd = std::complex<double>;
    const double two_pi = 2.0 * 3.14159265358979323846;
    const int64_t nb = m.size();
    std::vector<cd> A(static_cast<size_t>(nb * nb), cd(0.0, 0.0));
    const cd i2pi(0.0, two_pi);
    if (v.is_constant) {
        for (int64_t l = 0; l < nb; ++l)
            A[static_cast<size_t>(l * nb + l)] -= i2pi * (v.c1 * double(m.k1[l]) + v.c2 * double(m.k2[l]));
    } else {
        // vector_coefficients (fields.cpp:112-123) on a dense (2K+1)^2 grid
        const int K = v.K, W = 2 * K + 1;
        std::vector<cd> c1(static_cast<size_t>(W * W)), c2(static_cast<size_t>(W * W));
        std::vector<char> has(static_cast<size_t>(W * W), 0);
        auto put = [&](int k1, int k2, cd a, cd b) {
            const size_t i = static_cast<size_t>((k1 + K) * W + (k2 + K));
            c1[i] = a;
            c2[i] = b;
            has[i] = 1;
        };
        for (const auto& md : v.modes) {
            const double kn = std::sqrt(double(md.k1) * md.k1 + double(md.k2) * md.k2);
            const double d1 = -double(md.k2) / kn, d2 = double(md.k1) / kn;
            const cd c(md.re, md.im);
            put(md.k1, md.k2, c * d1, c * d2);
            const cd cm = -std::conj(c);
            put(-md.k1, -md.k2, cm * (-d1), cm * (-d2));
        }
        for (int64_t l = 0; l < nb; ++l)
            for (int64_t j = 0; j < nb; ++j) {
                const int d1 = m.k1[l] - m.k1[j], d2 = m.k2[l] - m.k2[j];
                if (d1 < -K || d1 > K || d2 < -K || d2 > K) continue;
                const size_t i = static_cast<size_t>((d1 + K) * W + (d2 + K));
                if (!has[i]) continue;
                A[static_cast<size_t>(l * nb + j)] -= (c1[i] * double(m.k1[j]) + c2[i] * double(m.k2[j])) * i2pi;
            }
    }
    for (int64_t l = 0; l < nb; ++l) {
        const double ksq = two_pi * two_pi * (double(m.k1[l]) * m.k1[l] + double(m.k2[l]) * m.k2[l]);
        A[static_cast<size_t>(l * nb + l)] -= kappa * ksq;
    }
    std::vector<double> out(static_cast<size_t>(2 * nb * nb));
    for (size_t i = 0; i < A.size(); ++i) {
        out[2 * i] = A[i].real();
        out[2 * i + 1] = A[i].imag();
    }
    return out;
}

VhatGrid galerkin_vhat_grid(const PreparedVelocity& v) {
    using cd = std::complex<double>;
    VhatGrid g;
    g.K = v.is_constant ? 0 : v.K;
    const int W = 2 * g.K + 1;
    g.c.assign(static_cast<size_t>(4 * W * W), 0.0);
    g.present.assign(static_cast<size_t>(W * W), 0);
    if (v.is_constant) return g;
    auto put = [&](int k1, int k2, cd a, cd b) {
        const size_t i = static_cast<size_t>((k1 + g.K) * W + (k2 + g.K));
        g.c[4 * i] = a.real();
        g.c[4 * i + 1] = a.imag();
        g.c[4 * i + 2] = b.real();
        g.c[4 * i + 3] = b.imag();
        g.present[i] = 1;
    };
    for (const auto& md : v.modes) {
        const double kn = std::sqrt(double(md.k1) * md.k1 + double(md.k2) * md.k2);
        const double d1 = -double(md.k2) / kn, d2 = double(md.k1) / kn;
        const cd c(md.re, md.im);
        put(md.k1, md.k2, c * d1, c * d2);
        const cd cm = -std::conj(c);
        put(-md.k1, -md.k2, cm * (-d1), cm * (-d2));
    }
    return g;
}

double galerkin_radius(const std::vector<double>& A, int64_t nb) {
    double r = 0.0;
    for (int64_t l = 0; l < nb; ++l) {
        double s = 0.0;
        for (int64_t j = 0; j < nb; ++j) {
            const size_t i = static_cast<size_t>(l * nb + j);
            s += std::hypot(A[2 * i], A[2 * i + 1]);
        }
        r = std::max(r, s);
    }
    return r;
}

bool galerkin_project_exact(const smc_scalar_field& f, const GalerkinModes& m, std::vector<double>& theta) {
    const double two_pi = 2.0 * 3.14159265358979323846;
    const int64_t nb = m.size();
    theta.assign(static_cast<size_t>(2 * nb), 0.0);
    const int L = std::max(m.max_abs, 0);
    auto place = [&](int k1, int k2, double re, double im) {
        if (k1 < -L || k1 > L || k2 < -L || k2 > L) return;  // outside cutoff: truncated
        for (int64_t i = 0; i < nb; ++i)
            if (m.k1[i] == k1 && m.k2[i] == k2) {
                theta[2 * i] += re;
                theta[2 * i + 1] += im;
                return;
            }
    };
    if (f.kind == SMC_SCALAR_CONSTANT) {
        place(0, 0, f.constant, 0.0);
        return true;
    }
    if (f.kind != SMC_SCALAR_COSINE) return false;
    for (int64_t t = 0; t < f.n_terms; ++t) {
        const double k1d = f.freq[2 * t] / two_pi, k2d = f.freq[2 * t + 1] / two_pi;
        if (std::abs(k1d - std::round(k1d)) > 1e-12 || std::abs(k2d - std::round(k2d)) > 1e-12) return false;
    }
    for (int64_t t = 0; t < f.n_terms; ++t) {
        const int k1 = static_cast<int>(std::lround(f.freq[2 * t] / two_pi));
        const int k2 = static_cast<int>(std::lround(f.freq[2 * t + 1] / two_pi));
        // a cos(2 pi k.x + phi) = (a/2) e^{i phi} e_k + (a/2) e^{-i phi} e_{-k}
        const double hr = 0.5 * f.amplitude[t] * std::cos(f.phase[t]);
        const double hi = 0.5 * f.amplitude[t] * std::sin(f.phase[t]);
        if (k1 == 0 && k2 == 0) {
            place(0, 0, 2.0 * hr, 0.0);
        } else {
            place(k1, k2, hr, hi);
            place(-k1, -k2, hr, -hi);
        }
    }
    return true;
}

AdObsImg make_ad_obs(double t, double x1, double x2, double dt, double sigma) {
    AdObsImg o;
    o.x1 = x1;
    o.x2 = x2;
    o.n_steps = static_cast<int64_t>(std::ceil(t / dt));
    o.dt = dt;
    o.dt_last = t - double(o.n_steps - 1) * dt;
    o.rdt = std::sqrt(dt);
    o.rdt_last = std::sqrt(o.dt_last);
    o.sr = sigma * o.rdt;
    o.sr_last = sigma * o.rdt_last;
    return o;
}

}  // namespace smc
