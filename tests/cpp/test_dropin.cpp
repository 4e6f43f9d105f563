// test_dropin.cpp — the C++ drop-in under the reference's own callers.
//
// Linked against the reference's UNCHANGED inference.cpp / optimize.cpp (and
// the rng/fields/geometry/sde/executor objects they need, compiled in place
// into oracle/_ref) plus paper_1808_10580_b200/host/scalarmc_forward_gpu.cpp in
// place of forward_ad.cpp / forward_bvp.cpp.  Every forward map below runs on
// the GPU.  Prints one JSON object per check; tests/test_dropin_cpp.py compares
// the numbers with the golden fixtures of the real reference and requires
// every "ok" to be true.
#include <cmath>
#include <cstdio>
#include <numbers>
#include <stdexcept>
#include <string>
#include <vector>

#include "scalarmc/forward_ad.hpp"
#include "scalarmc/forward_bvp.hpp"
#include "scalarmc/inference.hpp"
#include "scalarmc/optimize.hpp"

using namespace scalarmc;

namespace {

constexpr double kPi = std::numbers::pi;

void emit_estimates(const char* name, const std::vector<ParticleEstimate>& est) {
    std::printf("{\"check\": \"%s\", \"estimates\": [", name);
    for (std::size_t j = 0; j < est.size(); ++j)
        std::printf("%s{\"mean\": \"%a\", \"std_error\": \"%a\", \"n_particles\": %lld, \"n_failed\": %lld, "
                    "\"aux_mean\": \"%a\"}",
                    j ? ", " : "", est[j].mean, est[j].std_error, static_cast<long long>(est[j].n_particles),
                    static_cast<long long>(est[j].n_failed), est[j].aux_mean);
    std::printf("]}\n");
}

void emit_value(const char* name, double v) { std::printf("{\"check\": \"%s\", \"value\": \"%a\"}\n", name, v); }

void emit_ok(const char* name, bool ok, const std::string& detail = "") {
    std::printf("{\"check\": \"%s\", \"ok\": %s, \"detail\": \"%s\"}\n", name, ok ? "true" : "false", detail.c_str());
}

template <class E, class F>
void expect_throw(const char* name, F&& f, const std::string& message) {
    try {
        f();
        emit_ok(name, false, "no exception");
    } catch (const E& e) {
        emit_ok(name, message.empty() || message == e.what(), e.what());
    } catch (const std::exception& e) {
        emit_ok(name, false, std::string("wrong type: ") + e.what());
    }
}

AdProblemSpec two_mode() {  // forward_ad_two_mode.json
    AdProblemSpec s;
    s.velocity = VelocityField::fourier(FourierVelocityField({{1, 0, {0.3, 0.2}}, {0, 1, {-0.1, 0.25}}}, 1));
    s.diffusion = DiffusionModel::isotropic(0.05);
    s.initial_condition = ScalarField::cosine_series(
        {{1.0, {2 * kPi, 0.0}, 0.0}, {0.6, {0.0, 2 * kPi}, 0.7}, {0.4, {2 * kPi, 2 * kPi}, -0.3}});
    s.observations = {{0.1, {0.5, 0.5}}, {0.15, {0.25, 0.75}}, {0.2, {0.0, 0.0}}};
    s.n_particles = 10000;
    return s;
}

BvpProblemSpec paper_bvp(std::int64_t n) {  // forward_bvp_box.json
    BvpProblemSpec s;
    s.velocity = VelocityField::constant({1.0, 1.0});
    s.diffusion = DiffusionModel::isotropic(0.282);
    s.forcing = ScalarField::gaussian_bumps({{0.0, {0.68, 0.4}}, {0.0, {0.4, 0.68}}, {0.0, {0.82, 0.82}}}, 4.0);
    s.boundary_data =
        ScalarField::cosine_series({{0.5, {kPi / 2, 0.0}, 0.0}, {0.5, {0.0, kPi / 2}, 0.0}});
    s.observations = {{0.88, 0.6}, {0.6, 0.88}, {0.94, 0.94}};
    s.n_particles = n;
    s.dt = 0.00015;
    return s;
}

}  // namespace

int main() {
    // 1. observe_ad on the shipped two-mode config (golden c1).
    const AdProblemSpec c1 = two_mode();
    const auto est = observe_ad(c1, 7, 8);
    emit_estimates("c1", est);

    // 2. observe_ad_single slot equivalence and range error (forward_ad.cpp:62-69).
    bool same = true;
    for (std::size_t j = 0; j < c1.observations.size(); ++j) {
        const auto s = observe_ad_single(c1, j, 7);
        same = same && s.mean == est[j].mean && s.std_error == est[j].std_error;
    }
    emit_ok("single_equals_all", same);
    expect_throw<std::out_of_range>("single_out_of_range", [&] { observe_ad_single(c1, 3, 7); },
                                    "observe_ad_single: observation index out of range");

    // 3. validation errors with the reference's types and messages.
    AdProblemSpec bad;
    expect_throw<std::invalid_argument>("no_observations", [&] { observe_ad(bad, 0); },
                                        "AdProblemSpec: no observations");
    bad.observations = {{0.0, {0.5, 0.5}}};
    expect_throw<std::invalid_argument>("t_positive", [&] { observe_ad(bad, 0); },
                                        "AdProblemSpec: observation times must be positive");
    bad.observations = {{0.5, {1.5, 0.5}}};
    expect_throw<std::invalid_argument>("x_in_torus", [&] { observe_ad(bad, 0); },
                                        "AdProblemSpec: observation points must lie in [0,1)^2");
    emit_ok("resolved_dt", c1.resolved_dt() == 0.1 / 200.0);

    // 4. LikelihoodSpec::misfit, the reference's own code, over the GPU map
    //    (sample_k2.json shape; golden "misfit").
    {
        const PriorSpec prior{2, 0.6, 2.5};
        NormalStream rng(StreamKey{31337, 0xFFFFFFFFull, 0});
        const auto u = prior_draw(prior, rng);
        LikelihoodSpec like;
        like.data = {-0.9065, -0.7528, -0.6665, -0.8091, -0.6508, -0.5135, -0.5185, -0.4553, -0.4066};
        like.noise_std = 0.05;
        like.forward_seed = 1234;
        AdProblemSpec f;
        f.diffusion = DiffusionModel::isotropic(0.01);
        f.initial_condition = ScalarField::cosine_mode(1, 0, 1.0);
        for (double t : {0.1, 0.2, 0.3})
            for (Point2 x : {Point2{0.25, 0.25}, Point2{0.75, 0.5}, Point2{0.5, 0.75}}) f.observations.push_back({t, x});
        f.dt = 0.006;
        f.n_particles = 160;
        like.forward = f;
        emit_value("misfit", like.misfit(prior, u));
        // a short pCN chain through the unchanged run_chain (inference.cpp:170-194)
        ChainConfig cc;
        cc.n_steps = 20;
        cc.beta = 0.22;
        cc.seed = 31337;
        const auto res = run_chain(cc, prior, &like);
        emit_ok("pcn_chain_runs", res.phi_trace.size() == 20 && std::isfinite(res.map_objective));
        emit_value("pcn_map_objective", res.map_objective);
        emit_value("pcn_acceptance_rate", res.acceptance_rate);
        emit_value("pcn_last_phi", res.phi_trace.back());
    }

    // 5. observe_bvp and forcing_cost (optimize.cpp:161-173) over the GPU map.
    emit_estimates("bvp_box", observe_bvp(paper_bvp(16000), 606));
    {
        ForcingControl c;
        c.initial_amplitudes = {1.0, -0.5, 2.0};
        c.centers = {{0.68, 0.4}, {0.4, 0.68}, {0.82, 0.82}};
        c.sharpness = 4.0;
        c.target = {0.0, 0.0, 0.0};
        c.observation_points = {{0.88, 0.6}, {0.6, 0.88}, {0.94, 0.94}};
        const std::vector<double> F = {1.0, -0.5, 2.0};
        emit_value("forcing_cost", forcing_cost(F, c, paper_bvp(400), 606));
    }
    BvpProblemSpec torus = paper_bvp(10);
    torus.domain = Domain::unit_torus();
    expect_throw<std::invalid_argument>("bvp_bounded", [&] { observe_bvp(torus, 1); },
                                        "BvpProblemSpec: domain must be bounded");
    return 0;
}
