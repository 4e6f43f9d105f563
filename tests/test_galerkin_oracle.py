"""Pin the numpy Galerkin restatement (oracle/galerkin_oracle.py) — the
reference's galerkin.cpp needs Eigen, absent here — with closed forms: for
zero or constant velocity A is diagonal, A_ll = -2 pi i v.l - kappa (2 pi |l|)^2,
so explicit Euler gives Theta_l(t) = Theta_l(0) prod_i (1 + dt_i A_ll)."""
import math

import numpy as np
import pytest

import paper_1808_10580_b200 as S
from oracle import galerkin_oracle as G


def spec(velocity, kappa, terms, obs):
    return S.AdProblemSpec(velocity=velocity, diffusion=S.DiffusionModel.isotropic(kappa),
                           initial_condition=S.ScalarField.cosine_series(terms),
                           observations=[S.AdObservation(t, S.Vec2(*x)) for t, x in obs], n_particles=100)


@pytest.mark.parametrize("vel", [(0.0, 0.0), (0.7, -0.4)])
def test_diagonal_closed_form(vel):
    tp = 2 * math.pi
    terms = [(1.0, (tp, 0.0), 0.3), (0.5, (tp * 2, -tp), -1.1), (0.25, (0.0, 0.0), 0.0)]
    sp = spec(S.VelocityField.constant(vel), 0.03, terms, [(0.05, (0.3, 0.6)), (0.0123, (0.9, 0.1))])
    dt = 0.001
    vals, theta, steps, modes = G.solve(sp, "box", 3, dt)
    # the step schedule of galerkin.cpp:193-210
    t, dts = 0.0, []
    for target in sorted(o.t for o in sp.observations):
        while t < target - 1e-15:
            d = min(dt, target - t)
            dts.append(d)
            t += d
    assert steps == len(dts)
    th0 = G.project(sp.initial_condition, modes)
    for i, (l1, l2) in enumerate(modes):
        a = -2j * math.pi * (vel[0] * l1 + vel[1] * l2) - 0.03 * (2 * math.pi) ** 2 * (l1 * l1 + l2 * l2)
        want = th0[i] * np.prod([1 + d * a for d in dts])
        assert abs(theta[i] - want) <= 1e-13 * max(1.0, abs(want))
    # the solution at the observation is the analytic Euler iterate evaluated there
    x = sp.observations[0].x
    assert abs(vals[0] - sum(
        (th0[i] * np.prod([1 + d * (-2j * math.pi * (vel[0] * l1 + vel[1] * l2)
                                    - 0.03 * (2 * math.pi) ** 2 * (l1 * l1 + l2 * l2))
                           for d in dts]) * np.exp(2j * math.pi * (l1 * x[0] + l2 * x[1]))).real
        for i, (l1, l2) in enumerate(modes))) < 1e-12


def test_projection_exact_and_quadrature_agree():
    tp = 2 * math.pi
    terms = [(1.0, (tp, tp), 0.4), (0.3, (0.0, 3 * tp), 0.0)]
    modes = G.basis_modes("box", 4)
    exact = G.project(S.ScalarField.cosine_series(terms), modes)
    # a non-integer frequency forces the quadrature path; perturb by 1e-9 of a mode
    quad = G.project(S.ScalarField.cosine_series([(1.0, (tp * (1 + 1e-13), tp), 0.4), (0.3, (0.0, 3 * tp), 0.0)]),
                     modes)
    assert np.max(np.abs(exact - quad)) < 1e-10


def test_basis_modes():
    assert len(G.basis_modes("box", 2)) == 25 and len(G.basis_modes("disk", 2)) == 13
    assert G.basis_modes("box", 1)[0] == (-1, -1)
    with pytest.raises(ValueError, match="cutoff must be >= 1"):
        G.basis_modes("box", 0)
    assert S.GalerkinBasis("disk", 5).modes() == G.basis_modes("disk", 5)
    assert S.GalerkinBasis("box", 4).modes() == G.basis_modes("box", 4)


# ---- the reference's own galerkin.cpp (compiled against oracle/eigen_shim) ----
def _fourier(K=3, seed=4, scale=0.3):
    import specs
    f = specs.random_fourier(np.random.default_rng(seed), 6, K)
    modes = [S.VelocityMode(int(k1), int(k2), complex(scale * re, scale * im))
             for (k1, k2), (re, im) in zip(f.k.tolist(), f.coeff.tolist())]
    return S.VelocityField.fourier(S.FourierVelocityField(modes, K))


REF_CASES = {
    "fourier_box": (lambda: _fourier(), "box", 5, [(1.0, (2 * math.pi, 0.0), 0.0), (0.6, (0.0, 2 * math.pi), 0.7)]),
    "fourier_disk": (lambda: _fourier(K=2, seed=9), "disk", 6, [(0.4, (2 * math.pi, 2 * math.pi), -0.3)]),
    "constant_box": (lambda: S.VelocityField.constant((0.8, -0.3)), "box", 4, [(1.0, (2 * math.pi, 0.0), 0.2)]),
}


@pytest.mark.parametrize("name", list(REF_CASES))
def test_restatement_matches_compiled_reference(reference, name):
    """The numpy restatement against the reference's galerkin.cpp itself:
    same basis order, step count, observation values and coefficients (to
    rounding: the shim's GEMV and numpy sum in different orders)."""
    make, kind, L, terms = REF_CASES[name]
    sp = spec(make(), 0.02, terms, [(0.02, (0.5, 0.5)), (0.0437, (0.25, 0.75)), (0.01, (0.9, 0.3))])
    A = G.assemble(sp.velocity, 0.02, G.basis_modes(kind, L))
    radius = np.abs(A).sum(axis=1).max()
    assert abs(reference.galerkin_spectral_radius(sp, kind, L) - radius) <= 1e-13 * radius
    dt = min(2e-4, 1.0 / radius)
    want = reference.galerkin_solve_ad(sp, kind, L, dt)
    vals, theta, steps, modes = G.solve(sp, kind, L, dt)
    assert want["basis_modes"] == modes and want["steps"] == steps and want["dt_used"] == dt
    assert np.max(np.abs(want["observation_values"] - vals)) <= 1e-12 * max(1.0, np.max(np.abs(vals)))
    assert np.max(np.abs(want["final_coefficients"] - theta)) <= 1e-12 * max(1.0, np.max(np.abs(theta)))
    grid = reference.galerkin_field_grid(want["final_coefficients"], modes, 9)
    assert np.max(np.abs(grid - G.field_grid(want["final_coefficients"], modes, 9))) <= 1e-12


def test_compiled_reference_errors(reference):
    sp = spec(_fourier(), 0.02, [(1.0, (2 * math.pi, 0.0), 0.0)], [(0.02, (0.5, 0.5))])
    with pytest.raises(ValueError, match="dt_ref must be positive"):
        reference.galerkin_solve_ad(sp, "box", 4, 0.0)
    with pytest.raises(ValueError, match="cutoff must be >= 1"):
        reference.galerkin_solve_ad(sp, "box", 0, 1e-3)
    radius = reference.galerkin_spectral_radius(sp, "box", 6)
    with pytest.raises(RuntimeError, match="violates the stability estimate; suggest dt_ref <= "):
        reference.galerkin_solve_ad(sp, "box", 6, 3.0 / radius)
