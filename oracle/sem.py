"""Oracle SEM discretisation on prisms (TEST INFRASTRUCTURE; see oracle/__init__.py).

Follows PAPER.md §3.1 step by step:

* nodes x_j^p of V^p: the element nodes of every prism mapped by the
  workload's nodal map, merged by coordinates (O-7: KD-tree, 1e-9 tolerance);
* geometry (O-5, O7): J = sum_n X_n (x) grad l_n of the FINEST-order nodal map
   at the level's cubature; G = w detJ J^{-1} J^{-T};
* element matrix A_e = sum_q gradl^T G_q gradl; global A = sum_e Q_e^T A_e Q_e,
  i.e. A = -L of P:161 (reading O3: the sign that makes the system SPD);
* Dirichlet = nodes on faces tagged 1 (free surface; reading O8
  lift-and-eliminate); Neumann natural.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components
from scipy.spatial import cKDTree

from . import refelem as R


@dataclasses.dataclass
class Level:
    p: int
    conn: np.ndarray          # [E][N] global node ids (oracle numbering)
    xyz: np.ndarray           # [n][3] node coordinates
    dirichlet: np.ndarray     # [n] bool
    G: np.ndarray | None = None   # [E][Q][3][3]
    A: sp.csr_matrix | None = None
    q: int | None = None      # vertical order (None = p, the isotropic space)

    @property
    def pz(self):
        return self.p if self.q is None else self.q

    @property
    def n(self):
        return self.xyz.shape[0]

    @property
    def free(self):
        return np.nonzero(~self.dirichlet)[0]


def number_nodes(pts: np.ndarray, tol: float = 1e-9):
    """Merge coincident element nodes: pts [E][N][3] -> (conn [E][N], xyz [n][3]).
    Canonical order: lexicographic in (x, y, z) of the merged node."""
    E, N, _ = pts.shape
    flat = pts.reshape(-1, 3)
    diam = float(np.max(np.ptp(flat, axis=0)))
    tree = cKDTree(flat)
    pairs = tree.query_pairs(r=tol * max(diam, 1.0), output_type="ndarray")
    g = sp.coo_matrix((np.ones(len(pairs)), (pairs[:, 0], pairs[:, 1])), shape=(len(flat),) * 2)
    ncomp, lab = connected_components(g, directed=False)
    # representative coordinate = first occurrence
    first = np.full(ncomp, -1, dtype=np.int64)
    order = np.arange(len(flat))[::-1]
    first[lab[order]] = order
    rep = flat[first]
    key = np.round(rep, 9)
    perm = np.lexsort((key[:, 2], key[:, 1], key[:, 0]))
    rank = np.empty(ncomp, dtype=np.int64)
    rank[perm] = np.arange(ncomp)
    conn = rank[lab].reshape(E, N)
    return conn, rep[perm]


def mesh_pz(mesh):
    """Vertical order of the mesh's finest nodal map (default its p)."""
    return getattr(mesh, "pz", None) or mesh.p


def build_level(mesh, p: int, q: int | None = None) -> Level:
    rst, _ = R.prism_nodes(p, q)
    pts = mesh.node_xyz(rst)
    conn, xyz = number_nodes(pts)
    dirichlet = np.zeros(xyz.shape[0], dtype=bool)
    fn = R.face_nodes(p, q)
    for f in range(5):
        tagged = np.nonzero(mesh.face_tag[:, f] == 1)[0]
        if len(tagged):
            dirichlet[conn[np.ix_(tagged, fn[f])].ravel()] = True
    return Level(p=p, conn=conn, xyz=xyz, dirichlet=dirichlet, q=q)


def geometry(mesh, p_geo: int, p: int, elems=None, q_geo: int | None = None, q: int | None = None):
    """G = w detJ J^{-1} J^{-T} [e][Q][3][3] at the order-(p, q) cubature from the
    order-(p_geo, q_geo) nodal map (O-5).  Raises on detJ <= 0."""
    rst_geo, _ = R.prism_nodes(p_geo, q_geo)
    X = mesh.node_xyz(rst_geo, elems)                   # [e][Ng][3]
    pts, w = R.prism_cubature(p, q)
    _, dgeo = R.prism_basis(p_geo, pts, q_geo)          # [3][Q][Ng]
    # J[e][q][i][c] = sum_n X[e][n][i] * dgeo[c][q][n]
    # (optimize=True only lets numpy contract through BLAS: same formula, summation order only)
    J = np.einsum("eni,cqn->eqic", X, dgeo, optimize=True)
    det = np.linalg.det(J)
    if np.any(det <= 0):
        raise ValueError("invalid element: detJ <= 0")
    Ji = np.linalg.inv(J)
    G = np.einsum("q,eq,eqij,eqkj->eqik", w, det, Ji, Ji, optimize=True)
    return G


def element_matrices(G: np.ndarray, p: int, q: int | None = None):
    """A_e[i][j] = sum_q sum_cd dl_i^c(q) G_q[c][d] dl_j^d(q)   [e][N][N]."""
    pts, _ = R.prism_cubature(p, q)
    _, D = R.prism_basis(p, pts, q)                     # [3][Q][N]
    return np.einsum("cqi,eqcd,dqj->eij", D, G, D)


def assemble(level: Level, Ae: np.ndarray) -> sp.csr_matrix:
    E, N, _ = Ae.shape
    rows = np.repeat(level.conn, N, axis=1).ravel()
    cols = np.tile(level.conn, (1, N)).ravel()
    return sp.coo_matrix((Ae.ravel(), (rows, cols)), shape=(level.n, level.n)).tocsr()


def build_system(mesh, p: int, p_geo: int | None = None, q: int | None = None, q_geo: int | None = None) -> Level:
    """Assembled Neumann stiffness A (= -L) of order (p, q) with geometry from
    the order-(p_geo, q_geo) map (default: the mesh's finest orders)."""
    if p_geo is None:
        p_geo, q_geo = mesh.p, mesh_pz(mesh)
    lev = build_level(mesh, p, q)
    lev.G = geometry(mesh, p_geo, p, q_geo=q_geo, q=q)
    lev.A = assemble(lev, element_matrices(lev.G, p, q))
    return lev


def apply_streamed(mesh, level: Level, u: np.ndarray, p_geo: int | None = None, chunk: int = 4096,
                   elems: np.ndarray | None = None):
    """y = sum_e Q_e^T D^T (G (.) D Q_e u) without forming element matrices
    (SURVEY §8(c) tier (a) for configs too large to assemble).  u: [n] or [n][k]
    (k vectors at once); elems: the elements summed (default all; level.conn is
    indexed by position in elems when given)."""
    p = level.p
    pts, _ = R.prism_cubature(p)
    _, D = R.prism_basis(p, pts)                        # [3][Q][N]
    u2 = u.reshape(u.shape[0], -1)
    y = np.zeros((level.n, u2.shape[1]))
    all_el = np.arange(level.conn.shape[0]) if elems is None else np.asarray(elems)
    for c0 in range(0, len(all_el), chunk):
        pos = np.arange(c0, min(len(all_el), c0 + chunk))
        G = geometry(mesh, p_geo or mesh.p, p, all_el[pos])   # [e][Q][3][3]
        ue = u2[level.conn[pos]]                        # [e][N][k]
        g = np.einsum("cqn,enk->eqck", D, ue, optimize=True)
        f = np.einsum("eqcd,eqdk->eqck", G, g, optimize=True)
        ye = np.einsum("cqn,eqck->enk", D, f, optimize=True)
        np.add.at(y, level.conn[pos].ravel(), ye.reshape(-1, u2.shape[1]))
    return y.reshape(u.shape)


def apply_sampled(mesh, level: Level, u: np.ndarray, rows: np.ndarray, p_geo: int | None = None):
    """(A u)_i for selected global rows i only: sums the element contributions of
    the elements containing each node (used on configurations too large to
    assemble or stream in the test time budget)."""
    p = level.p
    pts, _ = R.prism_cubature(p)
    _, D = R.prism_basis(p, pts)
    rows = np.asarray(rows)
    hit = np.isin(level.conn, rows)
    el = np.nonzero(hit.any(axis=1))[0]
    G = geometry(mesh, p_geo or mesh.p, p, el)
    ue = u[level.conn[el]]
    g = np.einsum("cqn,en->eqc", D, ue)
    f = np.einsum("eqcd,eqd->eqc", G, g)
    ye = np.einsum("cqn,eqc->en", D, f)
    out = dict.fromkeys(rows.tolist(), 0.0)
    for k, e in enumerate(el):
        for n in np.nonzero(hit[e])[0]:
            out[int(level.conn[e, n])] += ye[k, n]
    return np.array([out[int(r)] for r in rows])


def dirichlet_lift(level: Level, phi_D: np.ndarray, rhs: np.ndarray | None = None):
    """Reduced system A_FF u_F = b_F - A_FD phi_D (lift-and-eliminate, O8)."""
    F = level.free
    D = np.nonzero(level.dirichlet)[0]
    b = np.zeros(level.n) if rhs is None else rhs.copy()
    bF = b[F] - level.A[F][:, D] @ phi_D[D]
    AFF = level.A[F][:, F].tocsc()
    return AFF, bF


def solve_direct(level: Level, phi_D: np.ndarray, rhs: np.ndarray | None = None):
    """phi = u_F (+) phi_D with u_F = A_FF^{-1} b_F by SuperLU (O-9)."""
    from scipy.sparse.linalg import splu
    AFF, bF = dirichlet_lift(level, phi_D, rhs)
    phi = phi_D.copy()
    phi[~level.dirichlet] = 0.0
    phi[level.free] = splu(AFF).solve(bF)
    return phi
