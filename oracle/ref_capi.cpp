// ref_capi.cpp — extern "C" harness over the REAL reference library (TEST
// INFRASTRUCTURE ONLY).
//
// Compiled (oracle/Makefile) against the reference's public headers
// (/root/reference/proj/include) and linked with the reference's own hot-path
// sources, compiled in place from /root/reference/proj/src into oracle/_ref/.
// Nothing is copied.  It translates the C-ABI POD structs of
// include/scalarmc_b200.h into the reference's C++ types and calls the
// reference's public API, so that tests/ and bench.py (cpu_baseline and
// --impl reference) can run the unmodified reference on the same inputs as the
// CUDA path.  The product never links this file.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "scalarmc/executor.hpp"
#include "scalarmc/fields.hpp"
#include "scalarmc/forward_ad.hpp"
#include "scalarmc/forward_bvp.hpp"
#include "scalarmc/galerkin.hpp"
#include "scalarmc/geometry.hpp"
#include "scalarmc/inference.hpp"
#include "scalarmc/optimize.hpp"
#include "scalarmc/rng.hpp"
#include "scalarmc/sde.hpp"

#include "../include/scalarmc_b200.h"

using namespace scalarmc;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SMC_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SMC_EINVAL;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return SMC_ERANGE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SMC_ERUNTIME;
    }
}

ScalarField to_scalar(const smc_scalar_field& f) {
    switch (f.kind) {
        case SMC_SCALAR_CONSTANT:
            return ScalarField::constant(f.constant);
        case SMC_SCALAR_COSINE: {
            std::vector<ScalarField::CosineTerm> t;
            for (int i = 0; i < f.n_terms; ++i)
                t.push_back({f.amplitude[i], {f.freq[2 * i], f.freq[2 * i + 1]}, f.phase[i]});
            return ScalarField::cosine_series(std::move(t));
        }
        case SMC_SCALAR_BUMPS: {
            std::vector<ScalarField::Bump> b;
            for (int i = 0; i < f.n_terms; ++i)
                b.push_back({f.amplitude[i], {f.center[2 * i], f.center[2 * i + 1]}});
            return ScalarField::gaussian_bumps(std::move(b), f.sharpness);
        }
        case SMC_SCALAR_LINEAR:
            return ScalarField::affine(f.constant, {f.gradient[0], f.gradient[1]});
    }
    throw std::invalid_argument("ref_capi: unknown scalar kind");
}

VelocityField to_velocity(const smc_velocity& v) {
    if (v.is_constant) return VelocityField::constant({v.constant[0], v.constant[1]});
    std::vector<VelocityMode> modes;
    for (int64_t i = 0; i < v.n_modes; ++i)
        modes.push_back({v.k[2 * i], v.k[2 * i + 1], {v.coeff[2 * i], v.coeff[2 * i + 1]}});
    return VelocityField::fourier(FourierVelocityField(std::move(modes), v.max_wavenumber));
}

Domain to_domain(const smc_domain& d) {
    if (d.kind == SMC_DOMAIN_BOX) return Domain::box({d.lower[0], d.lower[1]}, {d.upper[0], d.upper[1]});
    if (d.kind == SMC_DOMAIN_DISK) return Domain::disk({d.center[0], d.center[1]}, d.radius);
    return Domain::unit_torus();
}

AdProblemSpec to_ad(const smc_ad_problem& p) {
    AdProblemSpec s;
    s.velocity = to_velocity(p.velocity);
    s.diffusion = DiffusionModel::isotropic(p.kappa);
    s.initial_condition = to_scalar(p.initial_condition);
    for (int64_t j = 0; j < p.n_obs; ++j)
        s.observations.push_back({p.obs_t[j], {p.obs_x[2 * j], p.obs_x[2 * j + 1]}});
    s.dt = p.dt;
    s.n_particles = p.n_particles;
    s.scheme = p.scheme == SMC_MILSTEIN ? StepScheme::milstein : StepScheme::euler_maruyama;
    return s;
}

BvpProblemSpec to_bvp(const smc_bvp_problem& p) {
    BvpProblemSpec s;
    s.velocity = to_velocity(p.velocity);
    s.diffusion = DiffusionModel::isotropic(p.kappa);
    s.forcing = to_scalar(p.forcing);
    s.boundary_data = to_scalar(p.boundary_data);
    s.domain = to_domain(p.domain);
    for (int64_t j = 0; j < p.n_obs; ++j) s.observations.push_back({p.obs_x[2 * j], p.obs_x[2 * j + 1]});
    s.dt = p.dt;
    s.n_particles = p.n_particles;
    s.scheme = p.scheme == SMC_MILSTEIN ? StepScheme::milstein : StepScheme::euler_maruyama;
    s.max_steps = p.max_steps;
    return s;
}

void put(const ParticleEstimate& e, smc_estimate* o) {
    o->mean = e.mean;
    o->std_error = e.std_error;
    o->n_particles = e.n_particles;
    o->n_failed = e.n_failed;
    o->aux_mean = e.aux_mean;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_philox4x32(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    const auto r = detail::philox4x32({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
    for (int i = 0; i < 4; ++i) out[i] = r[i];
}

void ref_normal_pairs(uint64_t seed, uint64_t obs, uint64_t particle, int64_t n, double* out) {
    NormalStream s(StreamKey{seed, obs, particle});
    for (int64_t i = 0; i < n; ++i) {
        const Vec2 z = s.normal_pair();
        out[2 * i] = z.x1;
        out[2 * i + 1] = z.x2;
    }
}

int64_t ref_stream_draws(uint64_t seed, uint64_t obs, uint64_t particle, int64_t n, const int32_t* ops,
                         double* out) {
    NormalStream s(StreamKey{seed, obs, particle});
    int64_t w = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (ops[i] == 0) out[w++] = s.normal();
        else if (ops[i] == 1) out[w++] = s.uniform();
        else {
            const Vec2 z = s.normal_pair();
            out[w++] = z.x1;
            out[w++] = z.x2;
        }
    }
    return w;
}

int ref_velocity_eval(const smc_velocity* v, int64_t n, const double* x, double* out) {
    return guarded([&] {
        const VelocityField f = to_velocity(*v);
        for (int64_t i = 0; i < n; ++i) {
            const Vec2 r = f({x[2 * i], x[2 * i + 1]});
            out[2 * i] = r.x1;
            out[2 * i + 1] = r.x2;
        }
    });
}

int ref_scalar_eval(const smc_scalar_field* f, int64_t n, const double* x, double* out) {
    return guarded([&] {
        const ScalarField s = to_scalar(*f);
        for (int64_t i = 0; i < n; ++i) out[i] = s({x[2 * i], x[2 * i + 1]});
    });
}

double ref_pairwise_sum(const double* v, int64_t n) {
    return pairwise_sum(std::span<const double>(v, static_cast<std::size_t>(n)));
}

int ref_ad_observe(const smc_ad_problem* p, uint64_t seed, int workers, smc_estimate* out) {
    return guarded([&] {
        const auto est = observe_ad(to_ad(*p), seed, workers);
        for (std::size_t j = 0; j < est.size(); ++j) put(est[j], &out[j]);
    });
}

int ref_ad_observe_single(const smc_ad_problem* p, uint64_t obs_index, uint64_t seed, int workers,
                          smc_estimate* out) {
    return guarded([&] { put(observe_ad_single(to_ad(*p), obs_index, seed, workers), out); });
}

int ref_ad_resolved_dt(const smc_ad_problem* p, double* out) {
    return guarded([&] { *out = to_ad(*p).resolved_dt(); });
}

int ref_bvp_resolved_dt(const smc_bvp_problem* p, double* out) {
    return guarded([&] { *out = to_bvp(*p).resolved_dt(); });
}

// Per-particle theta_0(X_T) through the reference's own simulate_to_time.
int ref_ad_particle_values(const smc_ad_problem* p, uint64_t obs_index, uint64_t seed, int64_t n,
                           double* out, double* terminal) {
    return guarded([&] {
        const AdProblemSpec s = to_ad(*p);
        const PathContext ctx{s.velocity, s.diffusion, s.scheme, s.resolved_dt()};
        const Domain torus = Domain::unit_torus();
        const AdObservation o = s.observations[obs_index];
        for (int64_t i = 0; i < n; ++i) {
            NormalStream rng(StreamKey{seed, obs_index, static_cast<std::uint64_t>(i)});
            const PathResult r = simulate_to_time(o.x, o.t, ctx, torus, rng);
            out[i] = s.initial_condition(r.terminal);
            if (terminal) {
                terminal[2 * i] = r.terminal.x1;
                terminal[2 * i + 1] = r.terminal.x2;
            }
        }
    });
}

int ref_bvp_observe(const smc_bvp_problem* p, uint64_t seed, int workers, smc_estimate* out) {
    return guarded([&] {
        const auto est = observe_bvp(to_bvp(*p), seed, workers);
        for (std::size_t j = 0; j < est.size(); ++j) put(est[j], &out[j]);
    });
}

int ref_bvp_particle_values(const smc_bvp_problem* p, uint64_t obs_index, uint64_t seed, int64_t n,
                            double* values, double* aux, uint8_t* failed, int64_t* steps) {
    return guarded([&] {
        const BvpProblemSpec s = to_bvp(*p);
        const PathContext ctx{s.velocity, s.diffusion, s.scheme, s.resolved_dt()};
        const Point2 x0 = s.observations[obs_index];
        for (int64_t i = 0; i < n; ++i) {
            NormalStream rng(StreamKey{seed, obs_index, static_cast<std::uint64_t>(i)});
            const PathResult r = simulate_to_exit(x0, ctx, s.domain, s.forcing, s.max_steps, rng);
            failed[i] = r.failed ? 1 : 0;
            values[i] = r.failed ? 0.0 : s.boundary_data(r.terminal) - r.f_integral;
            aux[i] = r.failed ? 0.0 : *r.exit_time;
            if (steps) steps[i] = r.steps_taken;
        }
    });
}

int64_t ref_prior_modes(int cutoff, int32_t* out, int64_t cap) {
    const PriorSpec prior{cutoff, 1.0, 2.5};
    const auto m = prior.modes();
    for (std::size_t i = 0; i < m.size() && static_cast<int64_t>(i) < cap; ++i) {
        out[2 * i] = m[i].k1;
        out[2 * i + 1] = m[i].k2;
    }
    return static_cast<int64_t>(m.size());
}

int64_t ref_prior_draw(const smc_prior* prior, uint64_t seed, uint64_t obs, uint64_t particle, double* out,
                       int64_t cap) {
    const PriorSpec ps{prior->cutoff, prior->s0, prior->alpha};
    NormalStream rng(StreamKey{seed, obs, particle});
    const auto u = prior_draw(ps, rng);
    for (std::size_t i = 0; i < u.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = u[i];
    return static_cast<int64_t>(u.size());
}

// observe_ad for the field velocity_from_coefficients(prior, u): exactly the
// forward map LikelihoodSpec::misfit evaluates (inference.cpp:93-104).
int ref_ad_observe_u(const smc_ad_problem* base, const smc_prior* prior, const double* u, uint64_t seed,
                     int workers, smc_estimate* out) {
    return guarded([&] {
        const PriorSpec ps{prior->cutoff, prior->s0, prior->alpha};
        AdProblemSpec s = to_ad(*base);
        const std::size_t dim = static_cast<std::size_t>(ps.dimension());
        s.velocity = VelocityField::fourier(velocity_from_coefficients(ps, std::span<const double>(u, dim)));
        const auto est = observe_ad(s, seed, workers);
        for (std::size_t j = 0; j < est.size(); ++j) put(est[j], &out[j]);
    });
}

// LikelihoodSpec::misfit (inference.cpp:93-104), unchanged reference code.
int ref_misfit(const smc_ad_problem* base, const smc_prior* prior, const double* u, const double* data,
               double noise_std, uint64_t forward_seed, int workers, double* out) {
    return guarded([&] {
        const PriorSpec ps{prior->cutoff, prior->s0, prior->alpha};
        LikelihoodSpec like;
        if (base) {  // base == nullptr: run_chain(..., likelihood = nullptr) — Phi == 0
            like.forward = to_ad(*base);
            like.data.assign(data, data + base->n_obs);
            like.noise_std = noise_std;
            like.forward_seed = forward_seed;
            like.workers = workers;
        }
        *out = like.misfit(ps, std::span<const double>(u, static_cast<std::size_t>(ps.dimension())));
    });
}

// forcing_cost (optimize.cpp:161-173), unchanged reference code.
int ref_forcing_cost(const smc_bvp_problem* base, int64_t n_bumps, const double* amplitudes,
                     const double* centers, double sharpness, const double* target, uint64_t seed,
                     int workers, double* out) {
    return guarded([&] {
        ForcingControl c;
        for (int64_t j = 0; j < n_bumps; ++j) {
            c.initial_amplitudes.push_back(amplitudes[j]);
            c.centers.push_back({centers[2 * j], centers[2 * j + 1]});
        }
        c.sharpness = sharpness;
        const BvpProblemSpec b = to_bvp(*base);
        c.observation_points = b.observations;
        c.target.assign(target, target + base->n_obs);
        *out = forcing_cost(std::span<const double>(amplitudes, static_cast<std::size_t>(n_bumps)), c, b,
                            seed, workers);
    });
}

// run_chain (inference.cpp:170-194), unchanged reference code.  Outputs:
// phi_trace [n_steps], samples [n_samples][dim], final_u [dim], map_u [dim],
// scalars[0..2] = (final phi, map objective, accepted).
int ref_run_chain(const smc_ad_problem* base, const smc_prior* prior, const double* data, double noise_std,
                  uint64_t forward_seed, int64_t n_steps, double beta, int64_t burn_in, int64_t thin, uint64_t seed,
                  const double* u0, int workers, double* phi_trace, double* samples, double* final_u, double* map_u,
                  double* scalars) {
    return guarded([&] {
        const PriorSpec ps{prior->cutoff, prior->s0, prior->alpha};
        LikelihoodSpec like;
        if (base) {  // base == nullptr: run_chain(..., likelihood = nullptr) — Phi == 0
            like.forward = to_ad(*base);
            like.data.assign(data, data + base->n_obs);
            like.noise_std = noise_std;
            like.forward_seed = forward_seed;
            like.workers = workers;
        }
        ChainConfig cc;
        cc.n_steps = n_steps;
        cc.beta = beta;
        cc.burn_in = burn_in;
        cc.thin = thin;
        cc.seed = seed;
        std::optional<std::vector<double>> start;
        const std::size_t dim = static_cast<std::size_t>(ps.dimension());
        if (u0) start = std::vector<double>(u0, u0 + dim);
        const ChainResult r = run_chain(cc, ps, base ? &like : nullptr, start);
        for (std::size_t i = 0; i < r.phi_trace.size(); ++i) phi_trace[i] = r.phi_trace[i];
        for (std::size_t k = 0; k < r.samples.size(); ++k)
            for (std::size_t i = 0; i < dim; ++i) samples[k * dim + i] = r.samples[k][i];
        for (std::size_t i = 0; i < dim; ++i) {
            final_u[i] = r.final_state.u[i];
            map_u[i] = r.map_u[i];
        }
        scalars[0] = r.final_state.phi;
        scalars[1] = r.map_objective;
        scalars[2] = static_cast<double>(r.final_state.accepted);
    });
}

// optimize_forcing (optimize.cpp:175-185), unchanged reference code.
// out: argmin [n_bumps], scalars = (min_value, iterations); reason: >= 16 chars.
int ref_optimize_forcing(const smc_bvp_problem* base, int64_t n_bumps, const double* initial, const double* centers,
                         double sharpness, const double* target, double x_tol, double f_tol, int max_iter,
                         double initial_step, uint64_t seed, int workers, double* argmin, double* scalars,
                         char* reason) {
    return guarded([&] {
        ForcingControl c;
        for (int64_t j = 0; j < n_bumps; ++j) {
            c.initial_amplitudes.push_back(initial[j]);
            c.centers.push_back({centers[2 * j], centers[2 * j + 1]});
        }
        c.sharpness = sharpness;
        const BvpProblemSpec b = to_bvp(*base);
        c.observation_points = b.observations;
        c.target.assign(target, target + base->n_obs);
        NelderMeadOptions o;
        o.x_tol = x_tol;
        o.f_tol = f_tol;
        o.max_iter = max_iter;
        o.initial_step = initial_step;
        const NelderMeadResult r = optimize_forcing(c, b, o, seed, workers);
        for (int64_t j = 0; j < n_bumps; ++j) argmin[j] = r.argmin[static_cast<std::size_t>(j)];
        scalars[0] = r.min_value;
        scalars[1] = r.iterations;
        std::snprintf(reason, 16, "%s", r.stop_reason.c_str());
    });
}

int ref_resolve_workers(int requested) { return resolve_workers(requested); }

// ---- spectral Galerkin reference solver (src/galerkin.cpp, built against
// eigen_shim/Eigen/Dense) --------------------------------------------------
static GalerkinBasis to_basis(const smc_galerkin_basis& b) {
    return GalerkinBasis{b.kind == 1 ? GalerkinBasis::Kind::disk : GalerkinBasis::Kind::box, b.cutoff};
}

int ref_galerkin_spectral_radius(const smc_ad_problem* p, const smc_galerkin_basis* b, double* out) {
    return guarded([&] { *out = galerkin_spectral_radius(to_ad(*p), to_basis(*b)); });
}

// out->observation_values [n_obs]; out->coefficients_at_observations
// [n_obs][nb][2] and out->final_coefficients [nb][2] when non-null; modes
// [nb][2] when non-null (capacity nb_cap modes).
int ref_galerkin_solve_ad(const smc_ad_problem* p, const smc_galerkin_basis* b, double dt_ref,
                          smc_galerkin_result* out, int32_t* modes, int64_t nb_cap) {
    return guarded([&] {
        const GalerkinResult r = galerkin_solve_ad(to_ad(*p), to_basis(*b), dt_ref);
        const std::size_t nb = r.basis_modes.size();
        if (static_cast<int64_t>(nb) > nb_cap) throw std::out_of_range("ref_galerkin_solve_ad: mode capacity");
        for (std::size_t j = 0; j < r.observation_values.size(); ++j) out->observation_values[j] = r.observation_values[j];
        if (out->coefficients_at_observations)
            for (std::size_t j = 0; j < r.coefficients_at_observations.size(); ++j)
                for (std::size_t l = 0; l < nb; ++l) {
                    out->coefficients_at_observations[2 * (j * nb + l)] = r.coefficients_at_observations[j][l].real();
                    out->coefficients_at_observations[2 * (j * nb + l) + 1] = r.coefficients_at_observations[j][l].imag();
                }
        if (out->final_coefficients)
            for (std::size_t l = 0; l < nb; ++l) {
                out->final_coefficients[2 * l] = r.final_coefficients[l].real();
                out->final_coefficients[2 * l + 1] = r.final_coefficients[l].imag();
            }
        if (modes)
            for (std::size_t l = 0; l < nb; ++l) {
                modes[2 * l] = r.basis_modes[l].first;
                modes[2 * l + 1] = r.basis_modes[l].second;
            }
        out->dt_used = r.dt_used;
        out->steps = r.steps;
    });
}

int ref_galerkin_field_grid(int64_t nb, const int32_t* modes, const double* coefficients, int32_t n,
                            double* grid) {
    return guarded([&] {
        GalerkinResult r;
        for (int64_t l = 0; l < nb; ++l) {
            r.basis_modes.emplace_back(modes[2 * l], modes[2 * l + 1]);
            r.final_coefficients.emplace_back(coefficients[2 * l], coefficients[2 * l + 1]);
        }
        const std::vector<double> g = galerkin_field_grid(r, n);
        std::copy(g.begin(), g.end(), grid);
    });
}

}  // extern "C"
