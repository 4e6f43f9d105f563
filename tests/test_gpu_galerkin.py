"""Device Galerkin reference solver (smc_galerkin_*)
against the reference's own src/galerkin.cpp (compiled into oracle/_ref
against oracle/eigen_shim, its absent Eigen dependency restated), against the
numpy restatement (oracle/galerkin_oracle.py, pinned by closed forms and by
the compiled reference in tests/test_galerkin_oracle.py) and against the
particle forward map (the paper's Fig. 8 comparison)."""
import math

import numpy as np
import pytest

import paper_1808_10580_b200 as S
from oracle import galerkin_oracle as G
import specs

pytestmark = pytest.mark.gpu
TP = 2 * math.pi


def ad_spec(velocity, kappa=0.02, ic=None, obs=None):
    ic = ic or S.ScalarField.cosine_series([(1.0, (TP, 0.0), 0.0), (0.6, (0.0, TP), 0.7), (0.4, (TP, TP), -0.3)])
    obs = obs or [(0.1, (0.5, 0.5)), (0.15, (0.25, 0.75)), (0.0437, (0.0, 0.0)), (0.1, (0.9, 0.3))]
    return S.AdProblemSpec(velocity=velocity, diffusion=S.DiffusionModel.isotropic(kappa), initial_condition=ic,
                           observations=[S.AdObservation(t, S.Vec2(*x)) for t, x in obs], n_particles=1000)


def fourier(K=3, seed=4, scale=0.3):
    f = specs.random_fourier(np.random.default_rng(seed), 6, K)
    modes = [S.VelocityMode(int(k1), int(k2), complex(scale * re, scale * im))
             for (k1, k2), (re, im) in zip(f.k.tolist(), f.coeff.tolist())]
    return S.VelocityField.fourier(S.FourierVelocityField(modes, K))


def stable_dt(spec, kind, L, cap):
    A = G.assemble(spec.velocity, spec.diffusion.kappa(), G.basis_modes(kind, L))
    return min(cap, 1.0 / np.abs(A).sum(axis=1).max())


CASES = {
    "fourier_box": (lambda: ad_spec(fourier()), "box", 6, 2e-4),
    "fourier_disk": (lambda: ad_spec(fourier(K=2, seed=9)), "disk", 7, 2e-4),
    "constant": (lambda: ad_spec(S.VelocityField.constant((0.8, -0.3))), "box", 4, 1e-3),
    "bumps_quadrature": (lambda: ad_spec(fourier(K=2, seed=1), ic=S.ScalarField.gaussian_bumps(
        [S.Bump(1.0, S.Vec2(0.5, 0.5)), S.Bump(-0.5, S.Vec2(0.2, 0.7))], 6.0)), "box", 5, 2e-4),
}


@pytest.mark.parametrize("name", list(CASES))
def test_matches_oracle(ctx, name):
    make, kind, L, cap = CASES[name]
    spec = make()
    dt = stable_dt(spec, kind, L, cap)
    res = S.galerkin_solve_ad(spec, S.GalerkinBasis(kind, L), dt, keep_observation_coefficients=True, ctx=ctx)
    vals, theta, steps, modes = G.solve(spec, kind, L, dt)
    assert res.steps == steps and res.dt_used == dt and res.basis_modes == modes
    scale = max(1.0, np.max(np.abs(vals)))
    assert np.max(np.abs(res.observation_values - vals)) <= 1e-10 * scale, (res.observation_values, vals)
    assert np.max(np.abs(res.final_coefficients - theta)) <= 1e-10 * max(1.0, np.max(np.abs(theta)))
    last = int(np.argmax([o.t for o in spec.observations]))
    assert np.max(np.abs(res.coefficients_at_observations[last] - res.final_coefficients)) == 0.0


@pytest.mark.parametrize("name", list(CASES))
def test_matches_compiled_reference(ctx, reference, name):
    make, kind, L, cap = CASES[name]
    spec = make()
    dt = stable_dt(spec, kind, L, cap)
    res = S.galerkin_solve_ad(spec, S.GalerkinBasis(kind, L), dt, keep_observation_coefficients=True, ctx=ctx)
    want = reference.galerkin_solve_ad(spec, kind, L, dt)
    assert res.steps == want["steps"] and res.dt_used == want["dt_used"] and res.basis_modes == want["basis_modes"]
    vals = want["observation_values"]
    assert np.max(np.abs(res.observation_values - vals)) <= 1e-10 * max(1.0, np.max(np.abs(vals)))
    th = want["final_coefficients"]
    assert np.max(np.abs(res.final_coefficients - th)) <= 1e-10 * max(1.0, np.max(np.abs(th)))
    cat = want["coefficients_at_observations"]
    assert np.max(np.abs(res.coefficients_at_observations - cat)) <= 1e-10 * max(1.0, np.max(np.abs(cat)))
    radius = S.galerkin_spectral_radius(spec, S.GalerkinBasis(kind, L), ctx=ctx)
    assert abs(radius - reference.galerkin_spectral_radius(spec, kind, L)) <= 1e-12 * radius
    grid = S.galerkin_field_grid(res, 11, ctx=ctx)
    assert np.max(np.abs(grid - reference.galerkin_field_grid(res.final_coefficients, res.basis_modes, 11))) < 1e-11


def test_field_grid(ctx):
    spec = ad_spec(fourier())
    res = S.galerkin_solve_ad(spec, 5, stable_dt(spec, "box", 5, 2e-4), ctx=ctx)
    grid = S.galerkin_field_grid(res, 17, ctx=ctx)
    want = G.field_grid(res.final_coefficients, res.basis_modes, 17)
    assert np.max(np.abs(grid - want)) < 1e-11
    with pytest.raises(ValueError, match="n must be >= 2"):
        S.galerkin_field_grid(res, 1, ctx=ctx)


def test_errors(ctx):
    spec = ad_spec(fourier())
    with pytest.raises(ValueError, match="dt_ref must be positive"):
        S.galerkin_solve_ad(spec, 4, 0.0, ctx=ctx)
    with pytest.raises(ValueError, match="cutoff must be >= 1"):
        S.galerkin_solve_ad(spec, 0, 1e-3, ctx=ctx)
    radius = S.galerkin_spectral_radius(spec, 6, ctx=ctx)
    A = G.assemble(spec.velocity, 0.02, G.basis_modes("box", 6))
    assert abs(radius - np.abs(A).sum(axis=1).max()) <= 1e-12 * radius
    with pytest.raises(RuntimeError, match=r"violates the stability estimate; suggest dt_ref <= "):
        S.galerkin_solve_ad(spec, 6, 3.0 / radius, ctx=ctx)
    bad = ad_spec(fourier(), obs=[(0.0, (0.5, 0.5))])
    with pytest.raises(ValueError):
        S.galerkin_solve_ad(bad, 4, 1e-3, ctx=ctx)


def test_particles_agree_with_galerkin(ctx):
    """The paper's Fig. 8 check: the particle estimate of theta(t, x) and the
    spectral reference agree within the Monte Carlo error."""
    spec = ad_spec(fourier(K=2, seed=3), kappa=0.03)
    spec.n_particles = 200_000
    spec.dt = 2.5e-4
    ref = S.galerkin_solve_ad(spec, 12, stable_dt(spec, "box", 12, 5e-5), ctx=ctx).observation_values
    est = S.observe_ad(spec, 2024, ctx=ctx)
    for e, g in zip(est, ref):
        assert abs(e.mean - g) < 5 * e.std_error + 2e-3, (e.mean, g, e.std_error)
