"""Affine-in-F Dirichlet evaluation and the
Nelder–Mead optimal-forcing driver on top of it, against the reference.

* forcing_basis: one pass gives E[theta_bc] and E[int phi_k]; its means for any
  amplitude vector F must equal observe_bvp with that forcing (the reference's
  G(F)) within the FP64 gate — G is linear in F under common random numbers.
* optimize_forcing: Nelder–Mead over the basis must retrace the reference's
  optimize_forcing (optimize.cpp:175-185): same iterations and stop reason,
  same argmin.
"""
import numpy as np
import pytest

import paper_1808_10580_b200 as S
import specs
from conftest import est_from, unhex

pytestmark = pytest.mark.gpu

CENTERS = [(0.68, 0.4), (0.4, 0.68), (0.82, 0.82)]


def control(target=(0.0, 0.0, 0.0), initial=(0.0, 0.0, 0.0)):
    return S.ForcingControl(initial_amplitudes=list(initial), centers=CENTERS, sharpness=4.0, target=list(target),
                            observation_points=[(0.88, 0.6), (0.6, 0.88), (0.94, 0.94)])


@pytest.mark.parametrize("F", [(1.0, -0.5, 2.0), (0.0, 0.0, 0.0), (-3.0, 0.25, 7.5)])
def test_basis_reproduces_observe_bvp(ctx, F):
    base = specs.paper_bvp(n_particles=4000)
    fb = S.forcing_basis(control(), base, 606, ctx)
    direct = S.observe_bvp(S.api._control_spec(control(), base, F), 606, ctx=ctx)
    means = fb.means(F)
    for m, e in zip(means, direct):
        assert abs(m - e.mean) <= 1e-10 * max(abs(e.mean), 1.0)
    assert np.allclose(fb.exit_time, [e.aux_mean for e in direct], rtol=1e-12)


def test_basis_matches_reference_forcing_cost(ctx, golden):
    for rec in golden["forcing_cost"]:
        c = control(target=rec["target"])
        fb = S.forcing_basis(c, specs.paper_bvp(n_particles=400), rec["seed"], ctx)
        r = np.asarray(rec["target"]) - fb.means(rec["F"])
        cost = float(np.sqrt(np.sum(r * r)))
        ref = float.fromhex(rec["cost"])
        assert abs(cost - ref) <= 1e-9 * max(ref, 1.0)


def test_optimize_forcing_retraces_reference(ctx, golden):
    opts = S.NelderMeadOptions(x_tol=0.005, f_tol=1e-4, max_iter=250, initial_step=1.0)
    for rec in golden["optimize"]:
        res = S.optimize_forcing(control(target=rec["target"]), specs.paper_bvp(n_particles=300), opts, 606, ctx)
        assert res["iterations"] == rec["iterations"]
        assert res["stop_reason"] == rec["stop_reason"]
        assert np.allclose(res["argmin"], unhex(rec["argmin"]), rtol=1e-8, atol=1e-10)
        ref = float.fromhex(rec["min_value"])
        assert abs(res["min_value"] - ref) <= 1e-8 * max(ref, 1e-3)


def test_basis_validation(ctx):
    base = specs.paper_bvp(n_particles=100)
    spec = S.api._control_spec(control(), base, [1.0, 1.0, 1.0])
    spec.forcing = S.ScalarField.constant(1.0)
    p, keep = spec._pod()
    import ctypes as C
    from paper_1808_10580_b200 import _abi as A
    rc = ctx.lib.smc_bvp_forcing_basis(ctx.handle, C.byref(p), C.c_uint64(1), A.dptr(None), A.dptr(None),
                                       A.dptr(None), None)
    assert rc == A.SMC_EINVAL
