"""Oracle geometric p-multigrid (TEST INFRASTRUCTURE; see oracle/__init__.py).

Written in the paper's order and notation:

* prolongation P_{p-1}^p: interpolation between nested spaces,
  P[j][i] = N_i^c(x_j^f), the coarse cardinal function at the fine node;
  restriction R = P^T (eq 4.3);
* additive Schwarz smoother (eq 4.2-4.6):
  S^{-1} = W sum_k R_k^T (R_k A R_k^T)^{-1} R_k,  W = (sum_k R_k R_k^T)^{-1},
  subdomain k = element k's nodes plus every node within node-graph distance
  `overlap` (reading O15), Dirichlet nodes excluded;
  post-smoothing uses the transpose S^{-T} (reading O14) unless `literal=True`;
* V-cycle Alg 4.1 with readings O10 (recurse to the next level,
  exact solve when that level is P=1) and O11;
* PDC Alg 4.2 (reading O13) and PCG Alg 4.3 (reading O12),
  stop test ||r||_2 <= rtol ||f||_2 + atol over free nodes (O21).

All operators act on the Dirichlet-eliminated (free-node) systems.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from . import fdm
from . import refelem as R
from . import sem


def prolongation(fine: sem.Level, coarse: sem.Level) -> sp.csr_matrix:
    """P[j][i] = N_i^c(x_j^f) assembled from one element containing x_j^f."""
    rst_f, _ = R.prism_nodes(fine.p, fine.q)
    I, _ = R.prism_basis(coarse.p, rst_f, coarse.q)     # [Nf][Nc]
    E, Nf = fine.conn.shape
    owner_e = np.full(fine.n, -1, dtype=np.int64)
    owner_l = np.full(fine.n, -1, dtype=np.int64)
    flat = fine.conn.ravel()
    idx = np.arange(flat.size)[::-1]
    owner_e[flat[idx]] = idx // Nf
    owner_l[flat[idx]] = idx % Nf
    Nc = coarse.conn.shape[1]
    rows = np.repeat(np.arange(fine.n), Nc)
    cols = coarse.conn[owner_e].ravel()
    vals = I[owner_l].ravel()
    keep = vals != 0.0
    return sp.csr_matrix((vals[keep], (rows[keep], cols[keep])), shape=(fine.n, coarse.n))


def lattice_adjacency(level: sem.Level) -> sp.csr_matrix:
    """Node graph of reading O15: distinct nodes a, b are adjacent iff an element
    holds both with |dl| <= 1 and triangular-lattice offset in {0, +-(1,-1,0),
    +-(1,0,-1), +-(0,1,-1)} of the barycentric indices (i, j, k=p-i-j)."""
    p = level.p
    _, ijl = R.prism_nodes(p, level.q)
    i, j, l = ijl[:, 0], ijl[:, 1], ijl[:, 2]
    k = p - i - j
    di = i[:, None] - i[None, :]
    dj = j[:, None] - j[None, :]
    dk = k[:, None] - k[None, :]
    dl = l[:, None] - l[None, :]
    horiz = (np.abs(di) + np.abs(dj) + np.abs(dk)) <= 2   # 0 or one lattice step
    pat = horiz & (np.abs(dl) <= 1)
    np.fill_diagonal(pat, False)
    a, b = np.nonzero(pat)
    rows = level.conn[:, a].ravel()
    cols = level.conn[:, b].ravel()
    A = sp.csr_matrix((np.ones(rows.size), (rows, cols)), shape=(level.n, level.n))
    A.data[:] = 1.0
    return A


def schwarz_sets(level: sem.Level, overlap: int):
    """Per element k: sorted global ids of subdomain k's free nodes."""
    adj = lattice_adjacency(level) if overlap > 0 else None
    sets = []
    for e in range(level.conn.shape[0]):
        cur = np.unique(level.conn[e])
        for _ in range(overlap):
            nb = adj[cur].indices
            cur = np.union1d(cur, nb)
        cur = cur[~level.dirichlet[cur]]
        sets.append(cur)
    return sets


@dataclasses.dataclass
class Smoother:
    sets: list          # in free-node numbering
    inv: list           # dense (R_k A R_k^T)^{-1}
    W: np.ndarray       # [nF]

    def apply(self, r: np.ndarray, transpose: bool = False) -> np.ndarray:
        """S^{-1} r (pre) or S^{-T} r (post, reading O14)."""
        rr = self.W * r if transpose else r
        z = np.zeros_like(r)
        for I, Bi in zip(self.sets, self.inv):
            z[I] += Bi @ rr[I]
        return z if transpose else self.W * z


def build_smoother(level: sem.Level, AFF: sp.csr_matrix, overlap: int) -> Smoother:
    F = level.free
    fid = np.full(level.n, -1, dtype=np.int64)
    fid[F] = np.arange(len(F))
    sets = [fid[s] for s in schwarz_sets(level, overlap)]
    count = np.zeros(len(F))
    inv = []
    Ad = AFF.tocsr()
    for I in sets:
        count[I] += 1.0
        B = Ad[I][:, I].toarray()
        inv.append(np.linalg.inv(B))
    return Smoother(sets=sets, inv=inv, W=1.0 / count)


def hybrid_sets(mesh, level: sem.Level, overlap: int):
    """Node sets (global ids) of the FDM smoother's subdomains: the product box
    where it is regular, the O15 set elsewhere (reading O35)."""
    cols = fdm.Columns(mesh, level)
    reg = fdm.regular(cols, overlap)
    dense = schwarz_sets(level, overlap) if not reg.all() else None
    return [np.sort(ids) if reg[k] else dense[k]
            for k, (ids, _) in enumerate(fdm.fdm_blocks(mesh, level, overlap, cols, inverses=False))], reg


def build_fdm_smoother(mesh, level: sem.Level, overlap: int, AFF: sp.csr_matrix | None = None) -> Smoother:
    """eq 4.4 with the FDM local inverses of reading O33 (oracle/fdm.py) on the
    regular subdomains and the exact (R_k A R_k^T)^{-1} on the others (O35)."""
    F = level.free
    fid = np.full(level.n, -1, dtype=np.int64)
    fid[F] = np.arange(len(F))
    cols = fdm.Columns(mesh, level)
    reg = fdm.regular(cols, overlap)
    dense_sets = schwarz_sets(level, overlap) if not reg.all() else None
    Ad = AFF.tocsr() if AFF is not None else None
    sets, inv = [], []
    count = np.zeros(len(F))
    for k, (ids, Binv) in enumerate(fdm.fdm_blocks(mesh, level, overlap, cols)):
        if not reg[k]:
            I = fid[dense_sets[k]]
            Binv = np.linalg.inv(Ad[I][:, I].toarray())
        else:
            I = fid[ids]
        sets.append(I)
        inv.append(Binv)
        count[I] += 1.0
    return Smoother(sets=sets, inv=inv, W=1.0 / count)


@dataclasses.dataclass
class MGLevel:
    level: sem.Level
    A: sp.csr_matrix            # free-free operator
    smoother: Smoother | None = None
    P: sp.csr_matrix | None = None   # from the next coarser level (free x free)
    coarse_lu: object = None


class PMG:
    """Hierarchy of Alg 4.1 built from the oracle discretisation."""

    def __init__(self, mesh, p: int | None = None, schedule=None, overlap: int = 1,
                 nu1: int = 3, nu2: int = 3, literal: bool = False, local_solve: str = "dense"):
        p = p or mesh.p
        self.schedule = list(schedule) if schedule else R.level_schedule(p)
        self.nu1, self.nu2, self.literal = nu1, nu2, literal
        self.levels = []
        for pl in self.schedule:
            # a level is an order p, or a pair (P_xy, P_z)
            pp, qq = (pl, None) if np.isscalar(pl) else (int(pl[0]), int(pl[1]))
            lev = sem.build_system(mesh, pp, q=qq if qq != pp else None)
            F = lev.free
            AFF = lev.A[F][:, F].tocsr()
            self.levels.append(MGLevel(level=lev, A=AFF))
        for li in range(len(self.levels) - 1):
            f, c = self.levels[li], self.levels[li + 1]
            Pfull = prolongation(f.level, c.level)
            f.P = Pfull[f.level.free][:, c.level.free].tocsr()
        for li, ml in enumerate(self.levels):
            if li == len(self.levels) - 1:
                ml.coarse_lu = splu(ml.A.tocsc())
            else:
                ov = overlap if overlap >= 0 else (ml.level.p + 2) // 2   # refined: ceil((P+1)/2)
                if local_solve == "fdm":
                    ml.smoother = build_fdm_smoother(mesh, ml.level, ov, ml.A)
                else:
                    ml.smoother = build_smoother(ml.level, ml.A, ov)

    def smooth(self, li, u, f, nu, post):
        ml = self.levels[li]
        for _ in range(nu):
            # eq 4.2: u <- u - S^{-1}(A u - f)
            u = u + ml.smoother.apply(f - ml.A @ u, transpose=(post and not self.literal))
        return u

    def vcycle(self, f: np.ndarray, li: int = 0) -> np.ndarray:
        """MultigridCycle(p, 0, A_p, f, nu1, nu2) of Alg 4.1 (free-node vectors)."""
        ml = self.levels[li]
        if ml.coarse_lu is not None:          # single-level hierarchy (O26)
            return ml.coarse_lu.solve(f)
        u = np.zeros_like(f)
        u = self.smooth(li, u, f, self.nu1, post=False)          # line 1
        r = f - ml.A @ u                                          # line 2
        rc = ml.P.T @ r                                           # line 3, R = P^T
        nxt = self.levels[li + 1]
        if nxt.coarse_lu is not None:
            uc = nxt.coarse_lu.solve(rc)                          # line 4 (O10)
        else:
            uc = self.vcycle(rc, li + 1)                          # line 6
        u = u + ml.P @ uc                                         # lines 7-8
        u = self.smooth(li, u, f, self.nu2, post=True)            # line 9
        return u


def pcg(mg: PMG, f: np.ndarray, rtol: float, atol: float = 0.0, imax: int = 200, u0=None):
    """Alg 4.3 with q <- A p (O12).  The loop test of line 4 is evaluated right
    after r is updated; the V-cycle of that iteration is skipped when it passes
    (its z is never used), which leaves every iterate u unchanged."""
    A = mg.levels[0].A
    u = np.zeros_like(f) if u0 is None else u0.copy()
    r = f - A @ u
    nf = np.linalg.norm(f)
    hist = [np.linalg.norm(r)]
    vcycles = 0
    it = 0
    if hist[-1] <= rtol * nf + atol:
        return u, dict(iters=0, vcycles=0, res=hist)
    pdir = mg.vcycle(r)
    vcycles += 1
    delta = pdir @ r
    while it < imax:
        q = A @ pdir
        alpha = delta / (pdir @ q)
        u = u + alpha * pdir
        r = r - alpha * q
        it += 1
        hist.append(np.linalg.norm(r))
        if hist[-1] <= rtol * nf + atol:
            break
        z = mg.vcycle(r)
        vcycles += 1
        beta = (z @ r) / delta
        pdir = z + beta * pdir
        delta = z @ r
    return u, dict(iters=it, vcycles=vcycles, res=hist)


def pdc(mg: PMG, f: np.ndarray, rtol: float, atol: float = 0.0, imax: int = 200):
    """Alg 4.2 (r computed before the loop test, O13): u <- u - MG(-r)."""
    A = mg.levels[0].A
    u = np.zeros_like(f)
    nf = np.linalg.norm(f)
    r = f - A @ u
    hist = [np.linalg.norm(r)]
    it = 0
    while it < imax and hist[-1] > rtol * nf + atol:
        delta = mg.vcycle(-r)
        u = u - delta
        r = f - A @ u
        hist.append(np.linalg.norm(r))
        it += 1
    return u, dict(iters=it, vcycles=it, res=hist)
