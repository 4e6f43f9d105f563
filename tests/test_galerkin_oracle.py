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
