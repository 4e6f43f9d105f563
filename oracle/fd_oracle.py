"""scipy restatement of the reference's finite-difference Dirichlet solver
(src/fd_bvp.cpp, TEST INFRASTRUCTURE ONLY): the oracle of the reference's
acceptance criterion 4 (tests/acceptance.cpp:120-142) for the device walkers.

fd_bvp.cpp builds the same upwind 5-point system and solves it with Eigen's
BiCGSTAB + ILUT to 1e-12; here it is solved directly (SuperLU), i.e. to
rounding, which only tightens the comparison.  Constant velocity only (the
acceptance criterion's setup); boundary and forcing fields are evaluated on
the host by paper_1808_10580_b200.ScalarField.__call__.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def fd_solve_bvp(spec, n: int):
    """fd_solve_bvp (fd_bvp.cpp:26-106) -> (values [n*n], observation values)."""
    if n < 33:
        raise ValueError("fd_solve_bvp: n must be >= 33")
    lo, hi = spec.domain.lower, spec.domain.upper
    kappa = spec.diffusion.kappa()
    if not spec.velocity.is_constant:
        raise ValueError("fd oracle: constant velocity only")
    v1, v2 = spec.velocity.constant_value
    h1 = (hi[0] - lo[0]) / (n - 1)
    h2 = (hi[1] - lo[1]) / (n - 1)
    total = n * n
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    i, j = i.ravel(), j.ravel()
    row = i * n + j
    x1, x2 = lo[0] + i * h1, lo[1] + j * h2
    bnd = (i == 0) | (i == n - 1) | (j == 0) | (j == n - 1)
    rhs = np.zeros(total)
    rhs[bnd] = [spec.boundary_data((a, b)) for a, b in zip(x1[bnd], x2[bnd])]
    inner = ~bnd
    rhs[inner] = [-spec.forcing((a, b)) for a, b in zip(x1[inner], x2[inner])]
    center = 2.0 * kappa / (h1 * h1) + 2.0 * kappa / (h2 * h2)
    west = east = -kappa / (h1 * h1)
    south = north = -kappa / (h2 * h2)
    if v1 >= 0.0:
        center += v1 / h1
        west -= v1 / h1
    else:
        center -= v1 / h1
        east += v1 / h1
    if v2 >= 0.0:
        center += v2 / h2
        south -= v2 / h2
    else:
        center -= v2 / h2
        north += v2 / h2
    r = row[inner]
    rows = np.concatenate([row[bnd], r, r, r, r, r])
    cols = np.concatenate([row[bnd], r - n, r + n, r - 1, r + 1, r])
    m = r.size
    vals = np.concatenate([np.ones(bnd.sum()), np.full(m, west), np.full(m, east), np.full(m, south),
                           np.full(m, north), np.full(m, center)])
    A = sp.csr_matrix((vals, (rows, cols)), shape=(total, total))
    sol = spla.spsolve(A.tocsc(), rhs)

    def value_at(x):  # FdSolution::value_at (fd_bvp.cpp:12-24), bilinear
        s = min(max((x[0] - lo[0]) / h1, 0.0), float(n - 1))
        t = min(max((x[1] - lo[1]) / h2, 0.0), float(n - 1))
        i = min(int(s), n - 2)
        j = min(int(t), n - 2)
        a, b = s - i, t - j
        at = lambda ii, jj: sol[ii * n + jj]  # noqa: E731
        return ((1 - a) * (1 - b) * at(i, j) + a * (1 - b) * at(i + 1, j) + (1 - a) * b * at(i, j + 1)
                + a * b * at(i + 1, j + 1))
    return sol, [value_at(x) for x in spec.observations]
