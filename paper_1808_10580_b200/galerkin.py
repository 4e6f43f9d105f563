"""Spectral Galerkin reference solver of the advection-diffusion problem
(include/scalarmc/galerkin.hpp, src/galerkin.cpp)."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np

from . import _abi as A
from .api import AdProblemSpec, Context, _check, default_context

# ---------------------------------------------------------------------------
# spectral Galerkin reference solver
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class GalerkinBasis:
    """GalerkinBasis (galerkin.hpp:14-18): `box` keeps max(|l1|,|l2|) <= cutoff,
    `disk` keeps |l|_2 <= cutoff."""
    kind: str = "box"
    cutoff: int = 8

    def _pod(self) -> A.smc_galerkin_basis:
        if self.kind not in ("box", "disk"):
            raise ValueError("GalerkinBasis: kind must be 'box' or 'disk'")
        return A.smc_galerkin_basis(0 if self.kind == "box" else 1, int(self.cutoff))

    def modes(self) -> list[tuple[int, int]]:
        lib = A.load_library()
        b = self._pod()
        n = int(lib.smc_galerkin_n_basis(C.byref(b)))
        if n < 0:
            _check(lib.smc_galerkin_modes(C.byref(b), None))
        out = np.zeros((n, 2), dtype=np.int32)
        _check(lib.smc_galerkin_modes(C.byref(b), out.ctypes.data_as(C.POINTER(C.c_int32))))
        return [(int(a), int(c)) for a, c in out]


@dataclass
class GalerkinResult:
    """GalerkinResult (galerkin.hpp:20-27)."""
    observation_values: np.ndarray
    coefficients_at_observations: np.ndarray | None
    final_coefficients: np.ndarray
    basis_modes: list
    dt_used: float
    steps: int


def _basis(basis) -> GalerkinBasis:
    return basis if isinstance(basis, GalerkinBasis) else GalerkinBasis("box", int(basis))


def galerkin_spectral_radius(spec: AdProblemSpec, basis, ctx: Context | None = None) -> float:
    """galerkin_spectral_radius (galerkin.cpp:151-157)."""
    ctx = ctx or default_context()
    p, keep = spec._pod()
    b = _basis(basis)._pod()
    out = C.c_double()
    _check(ctx.lib.smc_galerkin_spectral_radius(ctx.handle, C.byref(p), C.byref(b), C.byref(out)))
    return out.value


def galerkin_solve_ad(spec: AdProblemSpec, basis, dt_ref: float, keep_observation_coefficients: bool = False,
                      ctx: Context | None = None) -> GalerkinResult:
    """galerkin_solve_ad (galerkin.hpp:36-40, galerkin.cpp:159-231) on the
    device; `basis` is a GalerkinBasis or a box cutoff (the int overload)."""
    ctx = ctx or default_context()
    b = _basis(basis)
    modes = b.modes()
    nb = len(modes)
    p, keep = spec._pod()
    vals = np.zeros(len(spec.observations))
    final = np.zeros((nb, 2))
    cat = np.zeros((len(spec.observations), nb, 2)) if keep_observation_coefficients else None
    r = A.smc_galerkin_result(A.dptr(vals), A.dptr(cat), A.dptr(final), 0.0, 0)
    _check(ctx.lib.smc_galerkin_solve_ad(ctx.handle, C.byref(p), C.byref(b._pod()), C.c_double(dt_ref), C.byref(r)))
    to_c = (lambda a: a[..., 0] + 1j * a[..., 1])
    return GalerkinResult(vals, to_c(cat) if cat is not None else None, to_c(final), modes, r.dt_used, int(r.steps))


def galerkin_field_grid(result: GalerkinResult, n: int, basis=None, ctx: Context | None = None) -> np.ndarray:
    """galerkin_field_grid (galerkin.cpp:233-250): n x n grid, row-major,
    x2 fastest (result.basis_modes must be the basis' mode order)."""
    ctx = ctx or default_context()
    if basis is None:
        L = max(max(abs(a), abs(c)) for a, c in result.basis_modes)
        box = len(result.basis_modes) == (2 * L + 1) ** 2
        basis = GalerkinBasis("box" if box else "disk", L)
    b = _basis(basis)._pod()
    c = np.ascontiguousarray(np.stack([result.final_coefficients.real, result.final_coefficients.imag], axis=-1))
    out = np.zeros(int(n) * int(n)) if n >= 2 else np.zeros(1)
    _check(ctx.lib.smc_galerkin_field_grid(ctx.handle, C.byref(b), A.dptr(c), int(n), A.dptr(out)))
    return out
