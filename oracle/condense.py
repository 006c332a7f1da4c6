"""Oracle static condensation (TEST INFRASTRUCTURE; see oracle/__init__.py).

SURVEY §8(f) NEXT-3, the supplement's "Static Condensation": with the
element-interior nodes i (nodes on no element face, one element each) and the
skeleton nodes b, the Dirichlet-eliminated system A_FF u_F = b_F splits into

    [A_bb A_bi] [u_b]   [b_b]
    [A_ib A_ii] [u_i] = [b_i]

and the condensed system (eq for phi_b in the supplement) is

    S u_b = g,   S = A_bb - A_bi A_ii^{-1} A_ib,   g = b_b - A_bi A_ii^{-1} b_i,

after which the interior values follow from A_ii u_i = b_i - A_ib u_b.
A_ii is block diagonal (one block per element).  Plain definitions with SciPy
sparse algebra; the solution equals the full system's exactly (block
elimination), which the pins check.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from . import refelem as R
from . import sem


def interior_nodes(level: sem.Level) -> np.ndarray:
    """Global ids of element-interior nodes: local lattice (i, j, k >= 1, 0 < l < q)."""
    p, q = level.p, level.pz
    _, ijl = R.prism_nodes(p, level.q)
    i, j, l = ijl[:, 0], ijl[:, 1], ijl[:, 2]
    k = p - i - j
    loc = np.nonzero((i > 0) & (j > 0) & (k > 0) & (l > 0) & (l < q))[0]
    return np.unique(level.conn[:, loc].ravel())


def condensed_system(level: sem.Level, phi_D: np.ndarray, rhs: np.ndarray | None = None):
    """(S, g, split) on the free skeleton nodes (free-node numbering of dirichlet_lift)."""
    AFF, bF = sem.dirichlet_lift(level, phi_D, rhs)
    F = level.free
    fid = -np.ones(level.n, dtype=np.int64)
    fid[F] = np.arange(len(F))
    I = fid[interior_nodes(level)]
    assert np.all(I >= 0), "an interior node is Dirichlet"
    isin = np.zeros(len(F), dtype=bool)
    isin[I] = True
    B = np.nonzero(~isin)[0]
    A = AFF.tocsr()
    Abb, Abi = A[B][:, B], A[B][:, I]
    Aib, Aii = A[I][:, B], A[I][:, I].tocsc()
    lu = splu(Aii) if len(I) else None
    S = (Abb - sp.csr_matrix(Abi @ lu.solve(Aib.toarray()))) if len(I) else Abb
    g = bF[B] - (Abi @ lu.solve(bF[I]) if len(I) else 0.0)
    return sp.csr_matrix(S), g, (B, I, lu, Aib, bF)


def solve_condensed(level: sem.Level, phi_D: np.ndarray, rhs: np.ndarray | None = None):
    """phi from the condensed system: S u_b = g (sparse direct), then the interior
    values A_ii u_i = b_i - A_ib u_b."""
    S, g, (B, I, lu, Aib, bF) = condensed_system(level, phi_D, rhs)
    ub = splu(S.tocsc()).solve(g)
    uF = np.zeros(len(bF))
    uF[B] = ub
    if len(I):
        uF[I] = lu.solve(bF[I] - Aib @ ub)
    phi = phi_D.copy()
    phi[~level.dirichlet] = 0.0
    phi[level.free] = uF
    return phi, S
