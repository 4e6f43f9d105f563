// scalarmc_forward_gpu.cpp — C++ drop-in for the reference forward maps.
//
// Replaces proj/src/forward_ad.cpp and proj/src/forward_bvp.cpp of the
// reference library scalarmc: it defines the same symbols with the same
// signatures, declared by the reference's own headers,
//
//   std::vector<ParticleEstimate> observe_ad(const AdProblemSpec&, uint64_t, int)   forward_ad.hpp:39-40
//   ParticleEstimate observe_ad_single(const AdProblemSpec&, size_t, uint64_t, int) forward_ad.hpp:43-44
//   double AdProblemSpec::resolved_dt() const / void validate() const              forward_ad.hpp:32-33
//   std::vector<ParticleEstimate> observe_bvp(const BvpProblemSpec&, uint64_t, int) forward_bvp.hpp:35-36
//   double BvpProblemSpec::resolved_dt() const / void validate() const             forward_bvp.hpp:28-29
//
// and runs them on the GPU through the C ABI (include/scalarmc_b200.h).  Every
// caller above the boundary — LikelihoodSpec::misfit (inference.cpp:93-104),
// forcing_cost (optimize.cpp:161-173), the CLI, the benchmark — links
// unchanged.  Exceptions keep the reference's types and messages
// (std::invalid_argument / std::out_of_range / std::runtime_error).
//
// Build: compile against the reference's include directory and
// link libscalarmc_b200.so instead of forward_ad.o and forward_bvp.o.
// `workers` (the reference's thread count, executor.cpp:45-85) is ignored:
// the parallelism is the GPU set.  SCALARMC_DEVICES=0,1,...,7 makes the forward
// maps shard over those GPUs of the box (smc_create_multi: NCCL exchange,
// results bit-identical to one GPU, so run_chain and every other caller scale
// unchanged); otherwise one device, SCALARMC_DEVICE (default LOCAL_RANK, else 0).  SCALARMC_PRECISION=fp32|fp64_strict selects the
// optional FP32 mode or the strict diagnostic build.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "scalarmc/forward_ad.hpp"
#include "scalarmc/forward_bvp.hpp"
#include "scalarmc_b200.h"

namespace scalarmc {
namespace {

[[noreturn]] void rethrow(smc_status st) {
    const std::string msg = smc_last_error();
    if (st == SMC_EINVAL) throw std::invalid_argument(msg);
    if (st == SMC_ERANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

void check(smc_status st) {
    if (st != SMC_OK) rethrow(st);
}

// One context per process (the device of this rank); calls are serialised,
// matching the reference's synchronous contract.
struct Device {
    std::once_flag once;
    std::mutex mu;
    smc_ctx* ctx = nullptr;
    smc_status init_status = SMC_OK;
};

Device& device() {
    static Device d;
    std::call_once(d.once, [&] {
        if (const char* list = std::getenv("SCALARMC_DEVICES")) {
            std::vector<int> devs;
            for (const char* p = list; *p;) {
                char* end = nullptr;
                const long v = std::strtol(p, &end, 10);
                if (end == p) break;
                devs.push_back(static_cast<int>(v));
                p = (*end == ',') ? end + 1 : end;
            }
            if (!devs.empty()) {
                d.init_status = smc_create_multi(static_cast<int>(devs.size()), devs.data(), &d.ctx);
                return;
            }
        }
        int dev = 0;
        if (const char* e = std::getenv("SCALARMC_DEVICE")) dev = std::atoi(e);
        else if (const char* r = std::getenv("LOCAL_RANK")) dev = std::atoi(r);
        d.init_status = smc_create(dev, &d.ctx);
    });
    if (d.init_status != SMC_OK) rethrow(d.init_status);
    return d;
}

int32_t precision() {
    const char* e = std::getenv("SCALARMC_PRECISION");
    if (!e) return SMC_FP64;
    if (std::strcmp(e, "fp32") == 0) return SMC_FP32;
    if (std::strcmp(e, "fp64_strict") == 0) return SMC_FP64_STRICT;
    return SMC_FP64;
}

// POD views of the reference's types; the vectors own the SoA arrays.
struct ScalarPod {
    smc_scalar_field f{};
    std::vector<double> amp, freq, phase, center;
    explicit ScalarPod(const ScalarField& s) {
        switch (s.kind()) {
            case ScalarField::Kind::constant:
                f.kind = SMC_SCALAR_CONSTANT;
                f.constant = s.constant_value();
                break;
            case ScalarField::Kind::linear:
                f.kind = SMC_SCALAR_LINEAR;
                f.constant = s.constant_value();
                f.gradient[0] = s.gradient().x1;
                f.gradient[1] = s.gradient().x2;
                break;
            case ScalarField::Kind::cosine:
                f.kind = SMC_SCALAR_COSINE;
                for (const auto& t : s.cosine_terms()) {
                    amp.push_back(t.amplitude);
                    freq.push_back(t.freq.x1);
                    freq.push_back(t.freq.x2);
                    phase.push_back(t.phase);
                }
                f.n_terms = static_cast<int32_t>(amp.size());
                f.amplitude = amp.data();
                f.freq = freq.data();
                f.phase = phase.data();
                break;
            case ScalarField::Kind::bumps:
                f.kind = SMC_SCALAR_BUMPS;
                f.sharpness = s.sharpness();
                for (const auto& b : s.bumps()) {
                    amp.push_back(b.amplitude);
                    center.push_back(b.center.x1);
                    center.push_back(b.center.x2);
                }
                f.n_terms = static_cast<int32_t>(amp.size());
                f.amplitude = amp.data();
                f.center = center.data();
                break;
        }
    }
};

struct VelocityPod {
    smc_velocity v{};
    std::vector<int32_t> k;
    std::vector<double> coeff;
    explicit VelocityPod(const VelocityField& vf) {
        if (vf.is_constant()) {
            v.is_constant = 1;
            v.constant[0] = vf.constant_value().x1;
            v.constant[1] = vf.constant_value().x2;
            return;
        }
        const FourierVelocityField& f = vf.fourier_field();
        if (f.empty() && f.max_wavenumber() == 0) {  // default-constructed zero field
            v.is_constant = 1;
            return;
        }
        v.is_constant = 0;
        v.max_wavenumber = f.max_wavenumber();
        for (const auto& m : f.modes()) {
            k.push_back(m.k1);
            k.push_back(m.k2);
            coeff.push_back(m.coeff.real());
            coeff.push_back(m.coeff.imag());
        }
        v.n_modes = static_cast<int64_t>(f.modes().size());
        v.k = k.data();
        v.coeff = coeff.data();
    }
};

double kappa_of(const DiffusionModel& d) {
    if (!d.is_isotropic())
        throw std::invalid_argument(
            "scalarmc_b200: state-dependent (std::function) diffusion has no device representation");
    return d.kappa();
}

struct AdPod {
    VelocityPod vel;
    ScalarPod theta0;
    std::vector<double> t, x;
    smc_ad_problem p{};
    explicit AdPod(const AdProblemSpec& s) : vel(s.velocity), theta0(s.initial_condition) {
        for (const auto& o : s.observations) {
            t.push_back(o.t);
            x.push_back(o.x.x1);
            x.push_back(o.x.x2);
        }
        p.velocity = vel.v;
        p.kappa = kappa_of(s.diffusion);
        p.initial_condition = theta0.f;
        p.n_obs = static_cast<int64_t>(t.size());
        p.obs_t = t.data();
        p.obs_x = x.data();
        p.dt = s.dt;
        p.n_particles = s.n_particles;
        p.scheme = s.scheme == StepScheme::milstein ? SMC_MILSTEIN : SMC_EULER_MARUYAMA;
        p.precision = precision();
    }
};

struct BvpPod {
    VelocityPod vel;
    ScalarPod forcing, bc;
    std::vector<double> x;
    smc_bvp_problem p{};
    explicit BvpPod(const BvpProblemSpec& s) : vel(s.velocity), forcing(s.forcing), bc(s.boundary_data) {
        for (const auto& o : s.observations) {
            x.push_back(o.x1);
            x.push_back(o.x2);
        }
        p.velocity = vel.v;
        p.kappa = kappa_of(s.diffusion);
        p.forcing = forcing.f;
        p.boundary_data = bc.f;
        if (const auto* b = s.domain.as_box()) {
            p.domain.kind = SMC_DOMAIN_BOX;
            p.domain.lower[0] = b->lower.x1;
            p.domain.lower[1] = b->lower.x2;
            p.domain.upper[0] = b->upper.x1;
            p.domain.upper[1] = b->upper.x2;
        } else if (const auto* d = s.domain.as_disk()) {
            p.domain.kind = SMC_DOMAIN_DISK;
            p.domain.center[0] = d->center.x1;
            p.domain.center[1] = d->center.x2;
            p.domain.radius = d->radius;
        } else {
            p.domain.kind = SMC_DOMAIN_TORUS;
        }
        p.n_obs = static_cast<int64_t>(s.observations.size());
        p.obs_x = x.data();
        p.dt = s.dt;
        p.n_particles = s.n_particles;
        p.scheme = s.scheme == StepScheme::milstein ? SMC_MILSTEIN : SMC_EULER_MARUYAMA;
        p.precision = precision();
        p.max_steps = s.max_steps;
    }
};

ParticleEstimate from(const smc_estimate& e) {
    return ParticleEstimate{e.mean, e.std_error, e.n_particles, e.n_failed, e.aux_mean};
}

}  // namespace

double AdProblemSpec::resolved_dt() const {
    const AdPod pod(*this);
    double dt = 0.0;
    check(smc_ad_resolved_dt(&pod.p, &dt));
    return dt;
}

void AdProblemSpec::validate() const {
    const AdPod pod(*this);
    check(smc_ad_validate(&pod.p));
    if (scheme == StepScheme::milstein && !diffusion.has_derivative())
        throw std::invalid_argument("AdProblemSpec: Milstein requires diffusion derivatives");
}

std::vector<ParticleEstimate> observe_ad(const AdProblemSpec& spec, std::uint64_t seed, int /*workers*/) {
    spec.validate();
    const AdPod pod(spec);
    std::vector<smc_estimate> out(spec.observations.size());
    Device& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    check(smc_ad_observe(d.ctx, &pod.p, seed, out.data()));
    std::vector<ParticleEstimate> r;
    r.reserve(out.size());
    for (const auto& e : out) r.push_back(from(e));
    return r;
}

ParticleEstimate observe_ad_single(const AdProblemSpec& spec, std::size_t obs_index, std::uint64_t seed,
                                   int /*workers*/) {
    spec.validate();
    if (obs_index >= spec.observations.size())
        throw std::out_of_range("observe_ad_single: observation index out of range");
    const AdPod pod(spec);
    smc_estimate out{};
    Device& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    check(smc_ad_observe_single(d.ctx, &pod.p, obs_index, seed, &out));
    return from(out);
}

double BvpProblemSpec::resolved_dt() const {
    const BvpPod pod(*this);
    double dt = 0.0;
    check(smc_bvp_resolved_dt(&pod.p, &dt));
    return dt;
}

void BvpProblemSpec::validate() const {
    const BvpPod pod(*this);
    check(smc_bvp_validate(&pod.p));
    if (scheme == StepScheme::milstein && !diffusion.has_derivative())
        throw std::invalid_argument("BvpProblemSpec: Milstein requires diffusion derivatives");
}

std::vector<ParticleEstimate> observe_bvp(const BvpProblemSpec& spec, std::uint64_t seed, int /*workers*/) {
    spec.validate();
    const BvpPod pod(spec);
    std::vector<smc_estimate> out(spec.observations.size());
    Device& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    check(smc_bvp_observe(d.ctx, &pod.p, seed, out.data()));
    std::vector<ParticleEstimate> r;
    r.reserve(out.size());
    for (const auto& e : out) r.push_back(from(e));
    return r;
}

}  // namespace scalarmc
