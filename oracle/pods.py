"""The checkers' own view of the C-ABI POD structs (include/scalarmc_b200.h)
and the BASELINE workloads built from them (TEST INFRASTRUCTURE ONLY).

The oracle libraries (liboracle.so, _ref/libscalarmc_ref.so) take the same
POD structs as the product library.  This module restates the layouts and the
C1..C5 workload builders without importing paper_1808_10580_b200, so
bench.py's reference arm times the reference with nothing of the product in
the process (tests/test_oracle_pods.py checks the layouts and the built PODs
against the package's, field for field).  Builders follow SURVEY.md §8(d) and
tests/specs.py (which builds the same problems with the package's types).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

SMC_OK, SMC_EINVAL, SMC_ERANGE, SMC_ERUNTIME, SMC_ECUDA = range(5)
SCALAR_CONSTANT, SCALAR_COSINE, SCALAR_BUMPS, SCALAR_LINEAR = range(4)
DOMAIN_TORUS, DOMAIN_BOX, DOMAIN_DISK = range(3)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class smc_estimate(C.Structure):
    _fields_ = [("mean", C.c_double), ("std_error", C.c_double), ("n_particles", C.c_int64),
                ("n_failed", C.c_int64), ("aux_mean", C.c_double)]


class smc_scalar_field(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_terms", C.c_int32), ("constant", C.c_double),
                ("gradient", C.c_double * 2), ("sharpness", C.c_double), ("amplitude", _dp),
                ("freq", _dp), ("phase", _dp), ("center", _dp)]


class smc_velocity(C.Structure):
    _fields_ = [("is_constant", C.c_int32), ("max_wavenumber", C.c_int32),
                ("constant", C.c_double * 2), ("n_modes", C.c_int64), ("k", _ip), ("coeff", _dp)]


class smc_ad_problem(C.Structure):
    _fields_ = [("velocity", smc_velocity), ("kappa", C.c_double),
                ("initial_condition", smc_scalar_field), ("n_obs", C.c_int64), ("obs_t", _dp),
                ("obs_x", _dp), ("dt", C.c_double), ("n_particles", C.c_int64),
                ("scheme", C.c_int32), ("precision", C.c_int32)]


class smc_domain(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("lower", C.c_double * 2),
                ("upper", C.c_double * 2), ("center", C.c_double * 2), ("radius", C.c_double)]


class smc_bvp_problem(C.Structure):
    _fields_ = [("velocity", smc_velocity), ("kappa", C.c_double), ("forcing", smc_scalar_field),
                ("boundary_data", smc_scalar_field), ("domain", smc_domain), ("n_obs", C.c_int64),
                ("obs_x", _dp), ("dt", C.c_double), ("n_particles", C.c_int64),
                ("scheme", C.c_int32), ("precision", C.c_int32), ("max_steps", C.c_int64)]


class smc_prior(C.Structure):
    _fields_ = [("cutoff", C.c_int32), ("pad_", C.c_int32), ("s0", C.c_double), ("alpha", C.c_double)]


def _arr(x, dtype=np.float64):
    return np.ascontiguousarray(x, dtype=dtype)


def _p(a: np.ndarray | None, t=_dp):
    return a.ctypes.data_as(t) if a is not None and a.size else t()


class Prior:
    """PriorSpec (inference.hpp:22-38) as the checkers need it."""

    def __init__(self, cutoff: int, s0: float, alpha: float):
        self.cutoff, self.s0, self.alpha = int(cutoff), float(s0), float(alpha)

    def _pod(self) -> smc_prior:
        return smc_prior(self.cutoff, 0, self.s0, self.alpha)

    def dimension(self) -> int:
        return 2 * sum(1 for k1 in range(-self.cutoff, self.cutoff + 1) for k2 in range(-self.cutoff, self.cutoff + 1)
                       if 0 < k1 * k1 + k2 * k2 <= self.cutoff * self.cutoff and (k1 > 0 or (k1 == 0 and k2 > 0)))


def _scalar_cosine(terms):
    """terms: [(amplitude, (f1, f2), phase)] -> (pod, keep)."""
    amp = _arr([t[0] for t in terms])
    freq = _arr([[t[1][0], t[1][1]] for t in terms]).reshape(-1, 2)
    ph = _arr([t[2] for t in terms])
    f = smc_scalar_field()
    f.kind, f.n_terms, f.sharpness = SCALAR_COSINE, len(terms), 4.0  # the package default (unused)
    f.amplitude, f.freq, f.phase = _p(amp), _p(freq), _p(ph)
    return f, [amp, freq, ph]


def _scalar_bumps(amplitudes, centers, sharpness):
    amp = _arr(amplitudes)
    cen = _arr(centers).reshape(-1, 2)
    f = smc_scalar_field()
    f.kind, f.n_terms, f.sharpness = SCALAR_BUMPS, len(amplitudes), float(sharpness)
    f.amplitude, f.center = _p(amp), _p(cen)
    return f, [amp, cen]


class AdSpec:
    """AdProblemSpec (forward_ad.hpp:23-34) as a POD builder.  modes: None
    (empty velocity slot: observe_ad_u supplies the field from u),
    'constant' vector, or [(k1, k2, complex)] with max_wavenumber K."""

    def __init__(self, kappa, theta0_terms, observations, dt, n_particles, modes=None, K=0, constant=None):
        self.kappa, self.theta0_terms = float(kappa), list(theta0_terms)
        self.observations = [(float(t), (float(x[0]), float(x[1]))) for t, x in observations]
        self.dt, self.n_particles = float(dt), int(n_particles)
        self.modes, self.K, self.constant = modes, int(K), constant

    def _pod(self):
        p = smc_ad_problem()
        keep = []
        v = smc_velocity()
        if self.modes:
            k = _arr([[m[0], m[1]] for m in self.modes], np.int32).reshape(-1, 2)
            c = _arr([[complex(m[2]).real, complex(m[2]).imag] for m in self.modes]).reshape(-1, 2)
            v.is_constant, v.max_wavenumber, v.n_modes = 0, self.K, len(self.modes)
            v.k, v.coeff = _p(k, _ip), _p(c)
            keep += [k, c]
        else:
            v.is_constant = 1
            v.constant[:] = self.constant or (0.0, 0.0)
        p.velocity = v
        p.kappa = self.kappa
        f, fk = _scalar_cosine(self.theta0_terms)
        p.initial_condition = f
        t = _arr([o[0] for o in self.observations])
        x = _arr([[o[1][0], o[1][1]] for o in self.observations]).reshape(-1, 2)
        keep += fk + [t, x]
        p.n_obs, p.obs_t, p.obs_x = len(self.observations), _p(t), _p(x)
        p.dt, p.n_particles = self.dt, self.n_particles
        return p, keep


class BvpSpec:
    """BvpProblemSpec (forward_bvp.hpp:16-30): box domain, constant velocity,
    Gaussian-bump forcing, cosine boundary data."""

    def __init__(self, kappa, velocity, bumps, centers, sharpness, bc_terms, observations, dt, n_particles,
                 max_steps=10_000_000, lower=(0.0, 0.0), upper=(1.0, 1.0)):
        self.kappa, self.velocity = float(kappa), tuple(velocity)
        self.bumps, self.centers, self.sharpness = list(bumps), list(centers), float(sharpness)
        self.bc_terms, self.observations = list(bc_terms), [tuple(o) for o in observations]
        self.dt, self.n_particles, self.max_steps = float(dt), int(n_particles), int(max_steps)
        self.lower, self.upper = lower, upper

    def _pod(self):
        p = smc_bvp_problem()
        v = smc_velocity()
        v.is_constant = 1
        v.constant[:] = self.velocity
        p.velocity = v
        p.kappa = self.kappa
        f, fk = _scalar_bumps(self.bumps, self.centers, self.sharpness)
        b, bk = _scalar_cosine(self.bc_terms)
        p.forcing, p.boundary_data = f, b
        d = smc_domain()
        d.kind = DOMAIN_BOX
        d.lower[:], d.upper[:] = self.lower, self.upper
        p.domain = d
        x = _arr([[o[0], o[1]] for o in self.observations]).reshape(-1, 2)
        p.n_obs, p.obs_x = len(self.observations), _p(x)
        p.dt, p.n_particles, p.max_steps = self.dt, self.n_particles, self.max_steps
        return p, fk + bk + [x]


TP = 2.0 * math.pi
C2_PRIOR = Prior(8, 1.0, 2.5)
C4_PRIOR = Prior(25, 1.0, 2.5)
C5_PRIOR = Prior(80, 1.0, 2.5)
COS_X1 = [(1.0, (TP, 0.0), 0.0)]  # ScalarField::cosine_mode(1, 0, 1.0)


def c1(n_particles: int = 10_000) -> AdSpec:
    """proj/configs/forward_ad_two_mode.json (tests/specs.py c1_two_mode)."""
    return AdSpec(0.05, [(1.0, (TP, 0.0), 0.0), (0.6, (0.0, TP), 0.7), (0.4, (TP, TP), -0.3)],
                  [(0.1, (0.5, 0.5)), (0.15, (0.25, 0.75)), (0.2, (0.0, 0.0))], 0.0, n_particles,
                  modes=[(1, 0, 0.3 + 0.2j), (0, 1, -0.1 + 0.25j)], K=1)


def c2_base(n_particles: int = 100_000) -> AdSpec:
    """C2 without its velocity (observe_ad_u builds it from u)."""
    obs = [(1.0, (a, b)) for a in (0.25, 0.5, 0.75) for b in (0.25, 0.5, 0.75)]
    return AdSpec(0.01, COS_X1, obs, 1e-3, n_particles)


def c4_base(n_particles: int = 1024) -> AdSpec:
    pts = [(0.25, 0.25), (0.75, 0.5), (0.5, 0.75)]
    return AdSpec(0.01, COS_X1, [(t, p) for t in (0.1, 0.2, 0.3) for p in pts], 1e-3, n_particles)


def c5_theta0_terms():
    """C5's 100-term cosine series (|k| <= 8, random amplitudes; bench.py c5_spec)."""
    rng = np.random.default_rng(5)
    terms = []
    for k1 in range(-8, 9):
        for k2 in range(-8, 9):
            if len(terms) < 100 and 0 < k1 * k1 + k2 * k2 <= 64:
                terms.append((float(rng.normal()) / (k1 * k1 + k2 * k2), (2 * math.pi * k1, 2 * math.pi * k2),
                              float(rng.random() * 2 * math.pi)))
    return terms


def c5_base(n_particles: int = 32768) -> AdSpec:
    obs = [(t / 16.0, (j / 8.0, j / 8.0)) for j in range(8) for t in range(1, 9)]
    return AdSpec(3e-5, c5_theta0_terms(), obs, 5e-4, n_particles)


def paper_bvp(n_particles: int = 16000, amplitudes=(0.0, 0.0, 0.0), observations=None, dt: float = 0.00015) -> BvpSpec:
    h = math.pi / 2
    return BvpSpec(0.282, (1.0, 1.0), amplitudes, [(0.68, 0.4), (0.4, 0.68), (0.82, 0.82)], 4.0,
                   [(0.5, (h, 0.0), 0.0), (0.5, (0.0, h), 0.0)],
                   observations or [(0.88, 0.6), (0.6, 0.88), (0.94, 0.94)], dt, n_particles)


def c3(n_particles: int = 1_000_000) -> BvpSpec:
    obs = [(a, b) for a in (0.1, 0.3, 0.5, 0.7, 0.9) for b in (0.1, 0.3, 0.5, 0.7, 0.9)]
    return paper_bvp(n_particles, amplitudes=(1.0, -0.5, 2.0), observations=obs)


class smc_galerkin_basis(C.Structure):
    _fields_ = [("kind", C.c_int32), ("cutoff", C.c_int32)]


class smc_galerkin_result(C.Structure):
    _fields_ = [("observation_values", C.POINTER(C.c_double)), ("coefficients_at_observations", C.POINTER(C.c_double)),
                ("final_coefficients", C.POINTER(C.c_double)), ("dt_used", C.c_double), ("steps", C.c_int64)]
