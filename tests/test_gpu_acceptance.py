"""The reference's own acceptance criteria (tests/acceptance.cpp of scalarmc)
run on the B200 path, with the reference's configurations, seeds and
tolerances: 2, 4, 7, 8, 9 here.  Criteria covered elsewhere: 1 heat (test_gpu_parity
test_heat_matches_reference_and_analytic), 3 manufactured Dirichlet
(test_bvp_manufactured_solution), 5 Milstein == EM
(test_milstein_equals_euler_maruyama_for_isotropic_diffusion), 6 determinism
(test_single_slot_equivalence_and_determinism, the sharded bit-identity
tests), 10 optimal forcing (test_gpu_forcing), 12 maximum principle
(test_maximum_principle_property).  Criterion 11 (CPU cost-scaling
benchmark) is the reference's harness, not part of this path.
"""
import math

import numpy as np
import pytest

import paper_1808_10580_b200 as S
import specs

pytestmark = pytest.mark.gpu
PI = math.pi


def test_criterion2_particles_vs_spectral_reference(ctx):
    """acceptance.cpp:67-86: the shipped two-mode flow, particles (seed 77)
    against galerkin_solve_ad(spec, 16, dt/10) within 3 SE + 5 (dt + dt_ref)."""
    spec = specs.c1_two_mode(n_particles=10000)
    dt = spec.resolved_dt()
    dt_ref = dt / 10.0
    particle = S.observe_ad(spec, 77, ctx=ctx)
    reference = S.galerkin_solve_ad(spec, 16, dt_ref, ctx=ctx)
    for e, g in zip(particle, reference.observation_values):
        assert abs(e.mean - g) <= 3.0 * e.std_error + 5.0 * (dt + dt_ref), (e.mean, g)


def test_criterion4_walkers_vs_finite_differences(ctx):
    """acceptance.cpp:120-142: the paper's Dirichlet setup (kappa 0.282,
    v = (1, 1)), 20 000 walkers at dt 2e-5 (seed 140) against the
    finite-difference solution on 513^2 nodes within 3 SE + 2 |FD257 - FD513|
    (oracle/fd_oracle.py restates fd_bvp.cpp; Eigen is absent here)."""
    from oracle.fd_oracle import fd_solve_bvp
    spec = S.BvpProblemSpec(velocity=S.VelocityField.constant((1.0, 1.0)), diffusion=S.DiffusionModel.isotropic(0.282),
                            forcing=S.ScalarField.constant(0.0),
                            boundary_data=S.ScalarField.cosine_series([(0.5, (PI / 2, 0.0), 0.0),
                                                                       (0.5, (0.0, PI / 2), 0.0)]),
                            observations=[(0.25, 0.65), (0.5, 0.5), (0.75, 0.35)], n_particles=20000, dt=2e-5)
    particle = S.observe_bvp(spec, 140, ctx=ctx)
    _, coarse = fd_solve_bvp(spec, 257)
    _, fine = fd_solve_bvp(spec, 513)
    for e, c, f in zip(particle, coarse, fine):
        assert e.n_failed == 0
        assert abs(e.mean - f) <= 3.0 * e.std_error + 2.0 * abs(c - f), (e.mean, f, e.std_error)


def test_criterion7_monte_carlo_law(ctx):
    """acceptance.cpp:191-207: SE(4e4) / (SE(1e4) / 2) within 15 % of 1 on
    the heat problem (seed 2718)."""
    spec = S.AdProblemSpec(diffusion=S.DiffusionModel.isotropic(0.01),
                           initial_condition=S.ScalarField.cosine_mode(1, 0, 1.0),
                           observations=[S.AdObservation(0.5, S.Vec2(0.0, 0.0))], dt=1e-3, n_particles=10000)
    small = S.observe_ad(spec, 2718, ctx=ctx)[0]
    spec.n_particles = 40000
    large = S.observe_ad(spec, 2718, ctx=ctx)[0]
    assert abs(large.std_error / (0.5 * small.std_error) - 1.0) <= 0.15


def test_criterion8_pcn_preserves_the_prior(ctx, reference):
    """acceptance.cpp:211-233: run_chain with no likelihood (Phi == 0),
    100 000 steps at beta 0.8 (seed 888): acceptance exactly 1 and every
    component's sample variance within 5 % of its prior variance.  The chain
    is also the reference's own run_chain, state for state."""
    prior = S.PriorSpec(4, 1.0, 2.5)
    cfg = S.ChainConfig(n_steps=100000, beta=0.8, burn_in=0, thin=1)
    res = S.run_chains(cfg, prior, None, [888], ctx=ctx)
    assert res["accepted"][0] == cfg.n_steps
    samples = res["samples"][0]
    stds = prior.component_stds()
    var = np.mean(samples * samples, axis=0)
    assert np.max(np.abs(var / stds ** 2 - 1.0)) <= 0.05
    ref = reference.run_chain(None, prior, 2000, 0.8, 0, 1, 888)
    assert ref["accepted"] == 2000
    assert np.allclose(samples[:2000], ref["samples"], rtol=0, atol=1e-12)


def test_criterion9_bayesian_recovery(ctx):
    """acceptance.cpp:236-291: synthetic truth u* from the prior (stream
    424242/0/0), data = the fixed-seed forward map at u* + 0.05 noise (stream
    424242/1/0), 200 000 pCN steps (beta 0.12, burn-in 20 000, thin 20, seed
    31337): the central 95 % posterior interval covers u* in >= 90 % of the
    components."""
    prior = S.PriorSpec(2, 0.6, 2.5)
    forward = S.AdProblemSpec(
        diffusion=S.DiffusionModel.isotropic(0.05),
        initial_condition=S.ScalarField.cosine_series([(1.0, (2 * PI, 0.0), 0.0), (0.8, (0.0, 2 * PI), 0.0),
                                                       (0.6, (2 * PI, 2 * PI), 0.0)]),
        observations=[S.AdObservation(t, S.Vec2(*x)) for t in (0.06, 0.12, 0.18)
                      for x in ((0.25, 0.25), (0.75, 0.5), (0.5, 0.75))],
        n_particles=160, dt=6e-3)
    truth = S.prior_draw(prior, 424242, 0, 0, ctx)
    data_spec = S.AdProblemSpec(**{**forward.__dict__})
    data_spec.velocity = S.VelocityField.fourier(S.velocity_from_coefficients(prior, truth))
    clean = S.observe_ad(data_spec, 1234, ctx=ctx)
    noise = S.normal_pairs_device(424242, 1, 0, 5, ctx).reshape(-1)  # normal(): pairs in order
    data = [e.mean + 0.05 * z for e, z in zip(clean, noise)]
    like = S.LikelihoodSpec(data=data, noise_std=0.05, forward=forward, forward_seed=1234)
    cfg = S.ChainConfig(n_steps=200000, beta=0.12, burn_in=20000, thin=20)
    res = S.run_chains(cfg, prior, like, [31337], keep_trace=False, ctx=ctx)
    samples = np.sort(res["samples"][0], axis=0)
    lo = samples[int(0.025 * len(samples))]
    hi = samples[min(int(0.975 * len(samples)), len(samples) - 1)]
    covered = np.sum((truth >= lo) & (truth <= hi))
    assert covered / prior.dimension() >= 0.90, (covered, prior.dimension(), res["acceptance_rate"])
