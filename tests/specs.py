"""Problem specs shared by tests, golden generation and bench.py.

Each builder restates a configuration from the reference (file:line cited) or
from BASELINE.json / SURVEY.md §8(d) (C1..C5).
"""
from __future__ import annotations

import math

import numpy as np

import paper_1808_10580_b200 as S

TP = 2.0 * math.pi


def c1_two_mode(n_particles: int = 10000, precision=S.Precision.fp64) -> S.AdProblemSpec:
    """proj/configs/forward_ad_two_mode.json (BASELINE config 1; acceptance.cpp:53-66)."""
    return S.AdProblemSpec(
        velocity=S.VelocityField.fourier(
            S.FourierVelocityField([S.VelocityMode(1, 0, 0.3 + 0.2j), S.VelocityMode(0, 1, -0.1 + 0.25j)], 1)),
        diffusion=S.DiffusionModel.isotropic(0.05),
        initial_condition=S.ScalarField.cosine_series([
            S.CosineTerm(1.0, S.Vec2(TP, 0.0), 0.0),
            S.CosineTerm(0.6, S.Vec2(0.0, TP), 0.7),
            S.CosineTerm(0.4, S.Vec2(TP, TP), -0.3)]),
        observations=[S.AdObservation(0.1, S.Vec2(0.5, 0.5)), S.AdObservation(0.15, S.Vec2(0.25, 0.75)),
                      S.AdObservation(0.2, S.Vec2(0.0, 0.0))],
        n_particles=n_particles, precision=precision)


def heat_spec(kappa: float, t: float, x, n_particles: int, dt: float) -> S.AdProblemSpec:
    """test_forward.cpp:15-24."""
    return S.AdProblemSpec(diffusion=S.DiffusionModel.isotropic(kappa),
                           initial_condition=S.ScalarField.cosine_mode(1, 0, 1.0),
                           observations=[S.AdObservation(t, S.Vec2(*x))], n_particles=n_particles, dt=dt)


C2_PRIOR = S.PriorSpec(8, 1.0, 2.5)
C4_PRIOR = S.PriorSpec(25, 1.0, 2.5)


def c2_spec(u: np.ndarray, n_particles: int = 100000, precision=S.Precision.fp64) -> S.AdProblemSpec:
    """K=8 (M=98) prior-draw velocity, kappa 0.01,
    theta_0 = cos 2 pi x1, 9 observations on {0.25,0.5,0.75}^2 at t=1, dt 1e-3."""
    obs = [S.AdObservation(1.0, S.Vec2(a, b)) for a in (0.25, 0.5, 0.75) for b in (0.25, 0.5, 0.75)]
    return S.AdProblemSpec(velocity=S.VelocityField.fourier(S.velocity_from_coefficients(C2_PRIOR, u)),
                           diffusion=S.DiffusionModel.isotropic(0.01),
                           initial_condition=S.ScalarField.cosine_mode(1, 0, 1.0), observations=obs, dt=1e-3,
                           n_particles=n_particles, precision=precision)


def c4_base(n_particles: int = 1024, precision=S.Precision.fp64) -> S.AdProblemSpec:
    """9 observations {(0.25,0.25),(0.75,0.5),(0.5,0.75)} x
    t in {0.1,0.2,0.3}, kappa 0.01, theta_0 = cos 2 pi x1, dt 1e-3."""
    pts = [(0.25, 0.25), (0.75, 0.5), (0.5, 0.75)]
    obs = [S.AdObservation(t, S.Vec2(*p)) for t in (0.1, 0.2, 0.3) for p in pts]
    return S.AdProblemSpec(diffusion=S.DiffusionModel.isotropic(0.01),
                           initial_condition=S.ScalarField.cosine_mode(1, 0, 1.0), observations=obs, dt=1e-3,
                           n_particles=n_particles, precision=precision)


def paper_bvp(n_particles: int = 16000, amplitudes=(0.0, 0.0, 0.0), observations=None, dt: float = 0.00015,
              precision=S.Precision.fp64, velocity=None) -> S.BvpProblemSpec:
    """proj/configs/forward_bvp_box.json and PAPER Eq. (bvp:ex1): box, v=(1,1),
    kappa 0.282, theta_bc = (cos(pi x/2) + cos(pi y/2)) / 2, 3 Gaussian bumps."""
    h = math.pi / 2
    centers = [(0.68, 0.4), (0.4, 0.68), (0.82, 0.82)]
    return S.BvpProblemSpec(
        velocity=velocity or S.VelocityField.constant((1.0, 1.0)),
        diffusion=S.DiffusionModel.isotropic(0.282),
        forcing=S.ScalarField.gaussian_bumps([S.Bump(a, S.Vec2(*c)) for a, c in zip(amplitudes, centers)], 4.0),
        boundary_data=S.ScalarField.cosine_series([S.CosineTerm(0.5, S.Vec2(h, 0.0), 0.0),
                                                   S.CosineTerm(0.5, S.Vec2(0.0, h), 0.0)]),
        observations=observations or [(0.88, 0.6), (0.6, 0.88), (0.94, 0.94)],
        n_particles=n_particles, dt=dt, precision=precision)


def c3_spec(n_particles: int = 1_000_000, precision=S.Precision.fp64) -> S.BvpProblemSpec:
    """paper BVP with F = (1.0, -0.5, 2.0), 25 observations
    on {0.1,...,0.9}^2, dt 1.5e-4, seed 606."""
    obs = [(a, b) for a in (0.1, 0.3, 0.5, 0.7, 0.9) for b in (0.1, 0.3, 0.5, 0.7, 0.9)]
    return paper_bvp(n_particles, amplitudes=(1.0, -0.5, 2.0), observations=obs, precision=precision)


def random_fourier(rng: np.random.Generator, n_modes: int, max_k: int) -> S.FourierVelocityField:
    """test_fields.cpp:24-41 style random field (any sign convention)."""
    modes: list = []
    while len(modes) < n_modes:
        k1, k2 = (int(v) for v in rng.integers(-max_k, max_k + 1, size=2))
        if k1 == 0 and k2 == 0:
            continue
        if k1 * k1 + k2 * k2 > max_k * max_k:
            continue
        if any((m.k1, m.k2) in ((k1, k2), (-k1, -k2)) for m in modes):
            continue
        modes.append(S.VelocityMode(k1, k2, complex(rng.normal(), rng.normal())))
    return S.FourierVelocityField(modes, max_k)
