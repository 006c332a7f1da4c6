"""Oracle fast-diagonalisation (FDM) local solves of the Schwarz smoother
(TEST INFRASTRUCTURE; see oracle/__init__.py).

Reading O33.  The paper's smoother (eq 4.4) inverts the
principal submatrix B_k = R_k A R_k^T exactly.  Its own source for the additive
Schwarz method, Lottes & Fischer [FL05], replaces each local block by
a separable operator that is inverted by fast diagonalisation.  On layered
prism meshes (every config) the subdomain of element k is a product of a
horizontal node patch H_k and a vertical node range V_k, and

    B~_k = K_h[H,H] (x) M_v[V,V]  +  M_h[H,H] (x) K_v[V,V]

where K_h, M_h are the 2D stiffness and mass matrices of the P_p triangle
space on the footprint mesh (x, y affine per triangle) and K_v, M_v the 1D
GLL P_q stiffness and mass matrices of element k's column (q = the vertical
order: q = p on isotropic levels, the P_z of the paper's (P_xy, P_z) pairs,
P:450, otherwise), layer j having the mean thickness d_j of its three vertical
edges.  B~_k = B_k exactly when the
prisms are straight with flat layers (config 1: A = K_h (x) M_v + M_h (x) K_v).

Definitions written out here (the library computes the same operator by a
generalised eigendecomposition; this oracle inverts the Kronecker box with
numpy.linalg.inv):

* line structure: 3D nodes with equal (x, y) form one vertical line h (2D
  node); the z-index of a node is its rank by z on its line;
* column of element k: its footprint triangle (2D labels of its bottom nodes);
  layer j: its lowest z-index / q;
* H_k: 2D nodes within 2D lattice-graph distance `overlap` of the triangle's
  nodes (reading O15 restricted to one level: lattice neighbours inside a
  common triangle);
* V_k: z-indices [max(0, jq - o), min(Z_c, jq + q + o)] of the column (Z_c =
  q x layers), without the z-levels at which all of the column's own nodes
  are Dirichlet (the free surface);
* local solve: (B~_k^{-1}) restricted to the box entries that exist and are
  free; W from the subdomain counts (eq 4.6).

Reading O35 (hybrid): the separable form is only used where the box is a
regular product -- every footprint triangle with a node in H_k widened by one
element ring carries a column with as many layers as element k's own (so K_h,
M_h are the true horizontal operators at every height of the box, and the
sloped bilge rows next to a body keep the exact inverse).  Next to a body (config 5)
the patch mixes columns of different heights and the geometry is far from
separable; those subdomains keep the paper's exact local inverse of eq 4.4 on
their reading-O15 node set.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components
from scipy.spatial import cKDTree

from . import refelem as R
from . import sem


def line_structure(level: sem.Level, tol: float = 1e-9):
    """(hl [n] 2D label of each node, zi [n] z-index on its line, xy [nh][2],
    node_at [nh][Zmax+1] 3D id or -1)."""
    xy = level.xyz[:, :2]
    diam = float(max(np.ptp(xy[:, 0]), np.ptp(xy[:, 1]), 1.0))
    pairs = cKDTree(xy).query_pairs(r=tol * diam, output_type="ndarray")
    g = sp.coo_matrix((np.ones(len(pairs)), (pairs[:, 0], pairs[:, 1])), shape=(level.n,) * 2)
    nh, hl = connected_components(g, directed=False)
    order = np.lexsort((level.xyz[:, 2], hl))          # by line, then by z
    zi = np.empty(level.n, dtype=np.int64)
    start = np.searchsorted(hl[order], np.arange(nh))
    zi[order] = np.arange(level.n) - start[hl[order]]
    node_at = np.full((nh, int(zi.max()) + 1), -1, dtype=np.int64)
    node_at[hl, zi] = np.arange(level.n)
    xy2 = np.zeros((nh, 2))
    xy2[hl] = xy
    return hl, zi, xy2, node_at


def tri_matrices(p: int, xy3: np.ndarray):
    """2D stiffness and mass of the order-p triangle with vertices xy3 [3][2]
    (v0, v1, v2 at (r,s) = (-1,-1), (1,-1), (-1,1)), collapsed cubature (O-4)."""
    r, s, w = R.tri_cubature(p)
    L, Lr, Ls = R.tri_lagrange(p, r, s)
    J = 0.5 * np.array([[xy3[1, 0] - xy3[0, 0], xy3[2, 0] - xy3[0, 0]],
                        [xy3[1, 1] - xy3[0, 1], xy3[2, 1] - xy3[0, 1]]])
    det = np.linalg.det(J)
    Ji = np.linalg.inv(J)                               # d(r,s)/d(x,y)
    Lx = Lr * Ji[0, 0] + Ls * Ji[1, 0]
    Ly = Lr * Ji[0, 1] + Ls * Ji[1, 1]
    wd = w * abs(det)
    K = Lx.T @ (wd[:, None] * Lx) + Ly.T @ (wd[:, None] * Ly)
    M = L.T @ (wd[:, None] * L)
    return K, M


def line_matrices(p: int):
    """Reference 1D GLL P_p stiffness and mass on [-1,1] (GL(p+1), exact)."""
    x, w = R.gauss_legendre(p + 1)
    h, dh = R.lagrange1d(R.lgl(p)[0], x)
    return dh.T @ (w[:, None] * dh), h.T @ (w[:, None] * h)


class Columns:
    """Footprint triangles, element layers and the 2D / 1D operators of a level."""

    def __init__(self, mesh, level: sem.Level):
        p, q = level.p, level.pz          # horizontal / vertical order (q = p isotropic)
        Nt = R.n_tri(p)
        self.p, self.q = p, q
        self.hl, self.zi, self.xy, self.node_at = line_structure(level)
        E = level.conn.shape[0]
        elem_h = self.hl[level.conn[:, :Nt]]            # [E][Nt] labels of the bottom-level nodes
        z_lo = self.zi[level.conn].min(axis=1)
        if np.any(z_lo % q):
            raise ValueError("mesh is not layered")
        self.layer = z_lo // q
        keys = {}
        self.col = np.empty(E, dtype=np.int64)
        for e in range(E):
            self.col[e] = keys.setdefault(tuple(sorted(elem_h[e, [0, p, Nt - 1]])), len(keys))
        nc = len(keys)
        self.tri_h = np.zeros((nc, Nt), dtype=np.int64)
        self.tri_h[self.col] = elem_h                    # the same for every layer of a column
        self.nlayer = np.bincount(self.col, minlength=nc)
        # vertical thickness d_j of every element: mean of its three vertical edges
        corners = np.array([[-1, -1, -1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1], [1, -1, 1], [-1, 1, 1]], float)
        cz = mesh.node_xyz(corners)[:, :, 2]             # [E][6]
        self.d = (cz[:, 3:] - cz[:, :3]).mean(axis=1)
        self.col_elems = [np.nonzero(self.col == c)[0] for c in range(nc)]
        for c, el in enumerate(self.col_elems):
            self.col_elems[c] = el[np.argsort(self.layer[el])]
            assert np.array_equal(self.layer[self.col_elems[c]], np.arange(len(el))), "gap in a column"
        # 2D operators over the footprint mesh
        nh = self.xy.shape[0]
        rows, cols, kv, mv = [], [], [], []
        for c in range(nc):
            hh = self.tri_h[c]
            K, M = tri_matrices(p, self.xy[hh[[0, p, Nt - 1]]])
            rows.append(np.repeat(hh, Nt))
            cols.append(np.tile(hh, Nt))
            kv.append(K.ravel())
            mv.append(M.ravel())
        rows, cols = np.concatenate(rows), np.concatenate(cols)
        self.K2 = sp.coo_matrix((np.concatenate(kv), (rows, cols)), shape=(nh, nh)).tocsr()
        self.M2 = sp.coo_matrix((np.concatenate(mv), (rows, cols)), shape=(nh, nh)).tocsr()
        # 2D lattice graph (O15 on one level)
        lat = np.array(R.tri_lattice(p))
        i, j = lat[:, 0], lat[:, 1]
        k = p - i - j
        step = (np.abs(i[:, None] - i[None, :]) + np.abs(j[:, None] - j[None, :]) +
                np.abs(k[:, None] - k[None, :])) == 2
        a, b = np.nonzero(step)
        ar = self.tri_h[:, a].ravel()
        br = self.tri_h[:, b].ravel()
        self.adj = sp.csr_matrix((np.ones(ar.size), (ar, br)), shape=(nh, nh))
        self.Kref, self.Mref = line_matrices(q)

    def column_line_matrices(self, c: int):
        """K_v, M_v [Z_c+1][Z_c+1] of column c (layers of mean thickness d_j)."""
        q = self.q
        el = self.col_elems[c]
        Z = q * len(el)
        Kv = np.zeros((Z + 1, Z + 1))
        Mv = np.zeros((Z + 1, Z + 1))
        for j, e in enumerate(el):
            s = slice(j * q, j * q + q + 1)
            Kv[s, s] += (2.0 / self.d[e]) * self.Kref
            Mv[s, s] += (self.d[e] / 2.0) * self.Mref
        return Kv, Mv

    def patch(self, c: int, overlap: int):
        cur = np.unique(self.tri_h[c])
        for _ in range(overlap):
            cur = np.union1d(cur, self.adj[cur].indices)
        return cur


def regular(cols: Columns, overlap: int):
    """[E] bool: reading O35 -- every column whose footprint triangle has a node
    within lattice distance overlap + p of element k's triangle (its patch widened
    by one element ring) has as many layers as k's column."""
    nh = cols.xy.shape[0]
    touch = [[] for _ in range(nh)]                     # 2D node -> columns holding it
    for c in range(cols.tri_h.shape[0]):
        for h in cols.tri_h[c]:
            touch[h].append(c)
    out = np.zeros(len(cols.col), dtype=bool)
    cache = {}
    for k in range(len(cols.col)):
        c = int(cols.col[k])
        if c not in cache:
            H = cols.patch(c, overlap + cols.p)
            cache[c] = all(cols.nlayer[t] == cols.nlayer[c] for h in H for t in touch[h])
        out[k] = cache[c]
    return out


def fdm_blocks(mesh, level: sem.Level, overlap: int, cols: Columns | None = None, elems=None,
               inverses: bool = True):
    """Per element k (all, or those in `elems`): (global 3D ids of the subdomain's
    free nodes, dense local inverse (B~_k^{-1}) restricted to them, or None when
    inverses=False)."""
    cols = cols or Columns(mesh, level)
    q = level.pz
    out = []
    cache = {}
    for k in (range(level.conn.shape[0]) if elems is None else elems):
        c = int(cols.col[k])
        if c not in cache:
            H = cols.patch(c, overlap)
            Kv, Mv = cols.column_line_matrices(c)
            Zc = Kv.shape[0] - 1
            own = cols.node_at[cols.tri_h[c]]                    # [Nt][Zmax+1]
            dz = [z for z in range(Zc + 1) if np.all(level.dirichlet[own[:, z]])]
            cache[c] = (H, Kv, Mv, Zc, set(dz), cols.K2[H][:, H].toarray(), cols.M2[H][:, H].toarray())
        H, Kv, Mv, Zc, dz, Kh, Mh = cache[c]
        j = int(cols.layer[k])
        V = [z for z in range(max(0, j * q - overlap), min(Zc, j * q + q + overlap) + 1) if z not in dz]
        V = np.array(V)
        ids = cols.node_at[np.repeat(H, len(V)), np.tile(V, len(H))]    # box order (h outer, z inner)
        keep = ids >= 0
        keep[keep] = ~level.dirichlet[ids[keep]]
        if not inverses:
            out.append((ids[keep], None))
            continue
        B = np.kron(Kh, Mv[np.ix_(V, V)]) + np.kron(Mh, Kv[np.ix_(V, V)])
        Binv = np.linalg.inv(B)
        out.append((ids[keep], Binv[np.ix_(keep, keep)]))
    return out
