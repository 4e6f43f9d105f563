"""Optimal-forcing control of the Dirichlet problem: ForcingControl, the
affine-in-F forcing basis (one walker pass per optimisation) and the
reference's Nelder-Mead (include/scalarmc/optimize.hpp, src/optimize.cpp;
SURVEY.md §8(f) rank 2)."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np

from . import _abi as A
from .api import (Bump, BvpProblemSpec, Context, ScalarField, Vec2, _check, default_context, observe_bvp)

@dataclass
class ForcingControl:
    """ForcingControl (optimize.hpp:45-54)."""
    initial_amplitudes: list
    centers: list
    sharpness: float = 4.0
    target: list = field(default_factory=list)
    observation_points: list = field(default_factory=list)

    def validate(self) -> None:
        if not self.centers:
            raise ValueError("ForcingControl: no forcing centers")
        if len(self.initial_amplitudes) != len(self.centers):
            raise ValueError("ForcingControl: amplitude/center count mismatch")
        if len(self.target) != len(self.observation_points):
            raise ValueError("ForcingControl: target and observation lengths must match")
        if not self.sharpness > 0.0:
            raise ValueError("ForcingControl: sharpness must be positive")


def _control_spec(control: ForcingControl, base: BvpProblemSpec, amplitudes: Sequence[float]) -> BvpProblemSpec:
    """control_spec (optimize.cpp:147-157)."""
    return replace(base, forcing=ScalarField.gaussian_bumps(
        [Bump(float(a), Vec2(*c)) for a, c in zip(amplitudes, control.centers)], control.sharpness),
        observations=list(control.observation_points))


@dataclass(frozen=True)
class ForcingBasis:
    """One Dirichlet pass under common random numbers, linear in the bump
    amplitudes F: mean_j(F) = bc[j] - basis[j] . F (smc_bvp_forcing_basis)."""
    bc: np.ndarray        # [n_obs] E[theta_bc(X_tau)]
    basis: np.ndarray     # [n_obs][n_bumps] E[int phi_k(X_t) dt]
    exit_time: np.ndarray # [n_obs]
    n_failed: np.ndarray  # [n_obs]

    def means(self, amplitudes: Sequence[float]) -> np.ndarray:
        return self.bc - self.basis @ np.asarray(amplitudes, dtype=np.float64)


def forcing_basis(control: ForcingControl, base: BvpProblemSpec, seed: int, ctx: Context | None = None) -> ForcingBasis:
    ctx = ctx or default_context()
    control.validate()
    spec = _control_spec(control, base, [1.0] * len(control.centers))
    p, keep = spec._pod()
    nb, no = len(control.centers), len(control.observation_points)
    bc, tau = np.zeros(no), np.zeros(no)
    basis = np.zeros((no, nb))
    nf = np.zeros(no, dtype=np.int64)
    _check(ctx.lib.smc_bvp_forcing_basis(ctx.handle, C.byref(p), C.c_uint64(seed), A.dptr(bc), A.dptr(basis),
                                         A.dptr(tau), nf.ctypes.data_as(C.POINTER(C.c_int64))))
    return ForcingBasis(bc, basis, tau, nf)


@dataclass
class NelderMeadOptions:
    """NelderMeadOptions (optimize.hpp:13-21)."""
    x_tol: float = 1e-6
    f_tol: float = 1e-9
    max_iter: int = 2000
    initial_step: float = 1.0


def nelder_mead(objective, x0: Sequence[float], options: NelderMeadOptions = NelderMeadOptions()) -> dict:
    """nelder_mead (optimize.cpp:37-134): coefficients (1, 2, 0.5, 0.5),
    non-finite values as +inf, stops on simplex diameter < x_tol, value spread
    < f_tol, or max_iter (the reference's algorithm, restated on the host)."""
    dim = len(x0)
    if dim == 0:
        raise ValueError("nelder_mead: empty start point")
    if not all(math.isfinite(v) for v in x0):
        raise ValueError("nelder_mead: non-finite start point")

    def guarded(x):
        v = objective(x)
        return v if math.isfinite(v) else math.inf

    verts = [list(map(float, x0)) for _ in range(dim + 1)]
    for i in range(dim):
        verts[i + 1][i] += options.initial_step
    vals = [guarded(v) for v in verts]

    def sort_simplex():
        nonlocal verts, vals
        order = sorted(range(dim + 1), key=lambda i: vals[i])  # stable, like std::stable_sort
        verts = [verts[i] for i in order]
        vals = [vals[i] for i in order]

    def diameter():
        d = 0.0
        for i in range(1, dim + 1):
            s = 0.0
            for c in range(dim):
                diff = verts[i][c] - verts[0][c]
                s += diff * diff
            d = max(d, math.sqrt(s))
        return d

    sort_simplex()
    trace = [(0, vals[0], list(verts[0]))]
    it, reason = 0, "max_iter"
    while it < options.max_iter:
        if diameter() < options.x_tol:
            reason = "x_tol"
            break
        if math.isfinite(vals[dim]) and vals[dim] - vals[0] < options.f_tol:
            reason = "f_tol"
            break
        centroid = [0.0] * dim
        for i in range(dim):
            for c in range(dim):
                centroid[c] += verts[i][c] / float(dim)

        def along(t):
            return [centroid[c] + t * (centroid[c] - verts[dim][c]) for c in range(dim)]

        refl = along(1.0)
        f_refl = guarded(refl)
        if f_refl < vals[0]:
            exp_ = along(2.0)
            f_exp = guarded(exp_)
            if f_exp < f_refl:
                verts[dim], vals[dim] = exp_, f_exp
            else:
                verts[dim], vals[dim] = refl, f_refl
        elif f_refl < vals[dim - 1]:
            verts[dim], vals[dim] = refl, f_refl
        else:
            outside = f_refl < vals[dim]
            con = along(0.5 if outside else -0.5)
            f_con = guarded(con)
            if f_con < min(vals[dim], f_refl):
                verts[dim], vals[dim] = con, f_con
            else:
                for i in range(1, dim + 1):
                    verts[i] = [verts[0][c] + 0.5 * (verts[i][c] - verts[0][c]) for c in range(dim)]
                    vals[i] = guarded(verts[i])
        sort_simplex()
        it += 1
        trace.append((it, vals[0], list(verts[0])))
    return {"argmin": verts[0], "min_value": vals[0], "iterations": it, "stop_reason": reason, "trace": trace}


def optimize_forcing(control: ForcingControl, base: BvpProblemSpec, options: NelderMeadOptions, seed: int,
                     ctx: Context | None = None) -> dict:
    """optimize_forcing (optimize.cpp:175-185) with every Nelder-Mead vertex
    evaluated from ONE device pass (forcing_basis): under the fixed seed the
    objective |Y - G(F)|_2 is exactly the reference's forcing_cost up to
    summation order (G is linear in F)."""
    control.validate()
    fb = forcing_basis(control, base, seed, ctx)
    Y = np.asarray(control.target, dtype=np.float64)

    def cost(F):
        r = Y - fb.means(F)
        return math.sqrt(float(np.sum(r * r)))
    res = nelder_mead(cost, control.initial_amplitudes, options)
    res["basis"] = fb
    return res


def forcing_cost(amplitudes: Sequence[float], control: ForcingControl, base: BvpProblemSpec, seed: int,
                 workers: int = 1) -> float:
    """|Y - G(F)|_2 with G = observe_bvp under a fixed seed (optimize.cpp:161-173)."""
    control.validate()
    if len(amplitudes) != len(control.centers):
        raise ValueError("forcing_cost: amplitude count mismatch")
    est = observe_bvp(_control_spec(control, base, amplitudes), seed, workers)
    ss = 0.0
    for y, e in zip(control.target, est):
        r = y - e.mean
        ss += r * r
    return math.sqrt(ss)
