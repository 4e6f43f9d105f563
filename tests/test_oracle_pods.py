"""oracle/pods.py — the checkers' own copy of the C-ABI POD layouts and of the
BASELINE workload builders (used by bench.py's reference arm so that no
product code is loaded there) — against the package's, field for field."""
import ctypes as C
import math

import numpy as np
import pytest

import paper_1808_10580_b200 as S
from paper_1808_10580_b200 import _abi as A
from oracle import pods as P
import specs


@pytest.mark.parametrize("name", ["smc_estimate", "smc_scalar_field", "smc_velocity", "smc_ad_problem",
                                  "smc_domain", "smc_bvp_problem", "smc_prior"])
def test_struct_layouts_equal(name):
    a, b = getattr(A, name), getattr(P, name)
    assert C.sizeof(a) == C.sizeof(b)
    for (fa, ta), (fb, tb) in zip(a._fields_, b._fields_):
        assert fa == fb and C.sizeof(ta) == C.sizeof(tb) and getattr(a, fa).offset == getattr(b, fb).offset


def _deref(ptr, n, ctype=C.c_double):
    if not ptr or n == 0:
        return []
    return [ptr[i] for i in range(n)]


def scalar_view(f):
    n = f.n_terms
    return (f.kind, n, f.constant, tuple(f.gradient), f.sharpness, _deref(f.amplitude, n), _deref(f.freq, 2 * n),
            _deref(f.phase, n), _deref(f.center, 2 * n))


def velocity_view(v):
    m = v.n_modes
    return (v.is_constant, v.max_wavenumber if not v.is_constant else 0, tuple(v.constant) if v.is_constant else (),
            m, _deref(v.k, 2 * m), _deref(v.coeff, 2 * m))


def ad_view(p):
    return (velocity_view(p.velocity), p.kappa, scalar_view(p.initial_condition), p.n_obs,
            _deref(p.obs_t, p.n_obs), _deref(p.obs_x, 2 * p.n_obs), p.dt, p.n_particles, p.scheme, p.precision)


def bvp_view(p):
    d = p.domain
    return (velocity_view(p.velocity), p.kappa, scalar_view(p.forcing), scalar_view(p.boundary_data),
            (d.kind, tuple(d.lower), tuple(d.upper)), p.n_obs, _deref(p.obs_x, 2 * p.n_obs), p.dt,
            p.n_particles, p.scheme, p.precision, p.max_steps)


def test_c1_pod_equal():
    a, ka = specs.c1_two_mode(n_particles=10_000)._pod()
    b, kb = P.c1(10_000)._pod()
    assert ad_view(a) == ad_view(b)


def test_c2_c4_bases_equal():
    u = np.linspace(-1, 1, specs.C2_PRIOR.dimension())
    a, ka = specs.c2_spec(u, n_particles=100_000)._pod()
    b, kb = P.c2_base(100_000)._pod()
    va, vb = ad_view(a), ad_view(b)
    assert va[1:] == vb[1:]  # the velocity comes from u (observe_ad_u) on the reference arm
    a, ka = specs.c4_base(n_particles=1024)._pod()
    b, kb = P.c4_base(1024)._pod()
    assert ad_view(a) == ad_view(b)
    assert P.C2_PRIOR.dimension() == specs.C2_PRIOR.dimension() == 196
    assert P.C4_PRIOR.dimension() == specs.C4_PRIOR.dimension()


def test_c5_base_equal():
    import bench
    u = np.zeros(S.PriorSpec(80, 1.0, 2.5).dimension())
    a, ka = bench.c5_spec(S, u)._pod()
    b, kb = P.c5_base()._pod()
    assert ad_view(a)[1:] == ad_view(b)[1:]
    assert P.C5_PRIOR.dimension() == 20080


def test_c3_pod_equal():
    a, ka = specs.c3_spec(n_particles=1_000_000)._pod()
    b, kb = P.c3(1_000_000)._pod()
    assert bvp_view(a) == bvp_view(b)
