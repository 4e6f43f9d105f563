"""numpy restatement of the reference's spectral Galerkin solver
(TEST INFRASTRUCTURE ONLY — the checker for smc_galerkin_*).

This restatement follows src/galerkin.cpp line by line (cited per function)
with numpy complex128 in place of Eigen::MatrixXcd.  It is pinned two ways
(tests/test_galerkin_oracle.py): by closed forms (the heat equation and any
constant velocity make A diagonal, so explicit Euler gives
Theta_l(t) = Theta_l(0) prod_i (1 + dt_i A_ll) exactly), and against the
reference's own galerkin.cpp, which oracle/Makefile compiles into
oracle/_ref against oracle/eigen_shim/Eigen/Dense (a restatement of the
small dense Eigen subset it uses; Eigen itself is absent here).
"""
from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi


def basis_modes(kind: str, L: int) -> list[tuple[int, int]]:
    """basis_mode_list (galerkin.cpp:20-33)."""
    if L < 1:
        raise ValueError("GalerkinBasis: cutoff must be >= 1")
    out = []
    for k1 in range(-L, L + 1):
        for k2 in range(-L, L + 1):
            if kind == "disk" and float(k1) * k1 + float(k2) * k2 > float(L) * L:
                continue
            out.append((k1, k2))
    return out


def _canonical_modes(field) -> list[tuple[int, int, complex]]:
    """FourierVelocityField ctor canonicalisation (fields.cpp:49-52)."""
    out = []
    for (k1, k2), (re, im) in zip(field.k.tolist(), field.coeff.tolist()):
        c = complex(re, im)
        if not (k1 > 0 or (k1 == 0 and k2 > 0)):
            k1, k2, c = -k1, -k2, -c.conjugate()
        out.append((k1, k2, c))
    return out


def vector_coefficients(field) -> dict:
    """FourierVelocityField::vector_coefficients (fields.cpp:112-123)."""
    vhat = {}
    for k1, k2, c in _canonical_modes(field):
        kn = math.sqrt(float(k1) * k1 + float(k2) * k2)
        d1, d2 = -float(k2) / kn, float(k1) / kn
        vhat[(k1, k2)] = (c * d1, c * d2)
        cm = -c.conjugate()
        vhat[(-k1, -k2)] = (cm * (-d1), cm * (-d2))
    return vhat


def assemble(velocity, kappa: float, modes) -> np.ndarray:
    """assemble_system (galerkin.cpp:108-142)."""
    nb = len(modes)
    A = np.zeros((nb, nb), dtype=np.complex128)
    i2pi = complex(0.0, TWO_PI)
    if velocity.is_constant:
        v1, v2 = velocity.constant_value
        for l, (l1, l2) in enumerate(modes):
            A[l, l] -= i2pi * (v1 * l1 + v2 * l2)
    else:
        vhat = vector_coefficients(velocity.fourier_field)
        for l, (l1, l2) in enumerate(modes):
            for m, (m1, m2) in enumerate(modes):
                c = vhat.get((l1 - m1, l2 - m2))
                if c is not None:
                    A[l, m] -= (c[0] * m1 + c[1] * m2) * i2pi
    for l, (l1, l2) in enumerate(modes):
        A[l, l] -= kappa * (TWO_PI * TWO_PI * (float(l1) * l1 + float(l2) * l2))
    return A


def project(theta0, modes) -> np.ndarray:
    """project_initial_condition (galerkin.cpp:38-104)."""
    index = {m: i for i, m in enumerate(modes)}
    theta = np.zeros(len(modes), dtype=np.complex128)

    def place(k1, k2, c):
        i = index.get((k1, k2))
        if i is not None:
            theta[i] += c

    kind = theta0.kind
    from oracle import pods as A
    if kind == A.SCALAR_CONSTANT:
        place(0, 0, theta0.constant_value)
        return theta
    if kind == A.SCALAR_COSINE:
        ks = [(t.freq[0] / TWO_PI, t.freq[1] / TWO_PI) for t in theta0.terms]
        if all(abs(a - round(a)) <= 1e-12 and abs(b - round(b)) <= 1e-12 for a, b in ks):
            for t in theta0.terms:
                k1, k2 = int(round(t.freq[0] / TWO_PI)), int(round(t.freq[1] / TWO_PI))
                half = complex(0.5 * t.amplitude * math.cos(t.phase), 0.5 * t.amplitude * math.sin(t.phase))
                if k1 == 0 and k2 == 0:
                    place(0, 0, 2.0 * half.real)
                else:
                    place(k1, k2, half)
                    place(-k1, -k2, half.conjugate())
            return theta
    max_abs = max(max(abs(a), abs(b)) for a, b in modes)
    n = max(128, 4 * (max_abs + 1))
    g = np.arange(n) / n
    samples = np.array([[theta0((x1, x2)) for x2 in g] for x1 in g])
    j = np.arange(n)[:, None]
    k = np.arange(n)[None, :]
    for i, (l1, l2) in enumerate(modes):
        ph = -TWO_PI * (float(l1) * j / n + float(l2) * k / n)
        theta[i] = np.sum(samples * np.exp(1j * ph)) / n / n
    return theta


def solve(spec, kind: str, L: int, dt_ref: float):
    """galerkin_solve_ad (galerkin.cpp:159-231) -> (observation values,
    final coefficients, steps)."""
    modes = basis_modes(kind, L)
    A = assemble(spec.velocity, spec.diffusion.kappa(), modes)
    radius = np.abs(A).sum(axis=1).max()
    if radius * dt_ref >= 2.0:
        raise RuntimeError("stability")
    theta = project(spec.initial_condition, modes)
    order = sorted(range(len(spec.observations)), key=lambda i: spec.observations[i].t)
    vals = np.zeros(len(spec.observations))
    t, steps = 0.0, 0
    k1 = np.array([m[0] for m in modes], dtype=np.float64)
    k2 = np.array([m[1] for m in modes], dtype=np.float64)
    for oi in order:
        target = spec.observations[oi].t
        while t < target - 1e-15:
            dt = min(dt_ref, target - t)
            theta = theta + dt * (A @ theta)
            t += dt
            steps += 1
        x1, x2 = spec.observations[oi].x
        vals[oi] = float(np.sum(theta * np.exp(1j * TWO_PI * (k1 * x1 + k2 * x2))).real)
    return vals, theta, steps, modes


def field_grid(coeffs, modes, n: int) -> np.ndarray:
    """galerkin_field_grid (galerkin.cpp:233-250)."""
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    grid = np.zeros((n, n))
    for c, (l1, l2) in zip(coeffs, modes):
        grid += (c * np.exp(1j * TWO_PI * (float(l1) * i / n + float(l2) * j / n))).real
    return grid.reshape(-1)
