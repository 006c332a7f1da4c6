"""Oracle reference element (TEST INFRASTRUCTURE; see oracle/__init__.py).

Plain definitions, written to be checked by eye:

* LGL rule of order p: nodes = {-1, roots of P_p', +1}, weights 2/(p(p+1)P_p(x)^2)
  (nodal set of P:209).
* Gauss-Legendre GL(n) = numpy.polynomial.legendre.leggauss; Gauss-Jacobi(1,0)(n)
  = scipy.special.roots_jacobi(n, 1, 0) (library primitives, O-1 / O-4).
* Triangle nodes: Blyth-Pozrikidis closed form built from LGL (reading O1; the
  paper's Fekete table P:541 is not given).
* Triangle basis: Dubiner/Koornwinder polynomials psi_ij(r,s) =
  P_i(a) P_j^{(2i+1,0)}(b) (1-b)^i, a = 2(1+r)/(1-s)-1, b = s; Lagrange
  (cardinal) basis = psi(x) V^{-1} with V[n][m] = psi_m(x_n).
* Prism: P_p(triangle) x P_p(t) (reading O2), local node n = m + Nt*l.
* Cubature (reading O6): collapsed GL(p+1) x GJ(1,0)(p+1) on the triangle
  (w = w_a w_b / 2, r = (1+a)(1-b)/2 - 1, s = b) times GL(p+1) in t.

Reference prism: {r,s >= -1, r+s <= 0} x [-1,1]; bottom vertices v0,v1,v2 at
(r,s) = (-1,-1), (1,-1), (-1,1), t = -1; top v3,v4,v5 above them at t = +1.
"""
from __future__ import annotations

import functools
import math

import numpy as np
from numpy.polynomial import legendre as L
from scipy.special import eval_jacobi, roots_jacobi


# ------------------------------------------------------------------ 1D rules
@functools.lru_cache(maxsize=None)
def lgl(p: int):
    """LGL nodes/weights of order p (p+1 points). S:41-49."""
    if p < 1:
        raise ValueError("order must be >= 1")
    c = np.zeros(p + 1)
    c[p] = 1.0
    if p == 1:
        x = np.array([-1.0, 1.0])
    else:
        dc = L.legder(c)
        inner = np.sort(L.legroots(dc).real)
        ddc = L.legder(dc)
        for _ in range(8):  # Newton polish of the library roots
            inner = inner - L.legval(inner, dc) / L.legval(inner, ddc)
        x = np.concatenate([[-1.0], inner, [1.0]])
    w = 2.0 / (p * (p + 1) * L.legval(x, c) ** 2)
    return x, w


@functools.lru_cache(maxsize=None)
def gauss_legendre(n: int):
    return L.leggauss(n)


@functools.lru_cache(maxsize=None)
def gauss_jacobi10(n: int):
    """Gauss-Jacobi rule for weight (1-x)^1 (1+x)^0 on [-1,1]."""
    x, w = roots_jacobi(n, 1.0, 0.0)
    return np.asarray(x, dtype=np.float64), np.asarray(w, dtype=np.float64)


def lagrange1d(nodes: np.ndarray, x: np.ndarray):
    """Values h_l(x) and derivatives h_l'(x) of the 1D Lagrange cardinal basis
    on `nodes`, by the product formula.  Returns ([len(x)][n], [len(x)][n])."""
    nodes = np.asarray(nodes, dtype=np.float64)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = len(nodes)
    V = np.ones((len(x), n))
    D = np.zeros((len(x), n))
    for l in range(n):
        others = [m for m in range(n) if m != l]
        den = np.prod([nodes[l] - nodes[m] for m in others])
        V[:, l] = np.prod([x - nodes[m] for m in others], axis=0) / den if others else 1.0
        acc = np.zeros(len(x))
        for k in others:
            acc += np.prod([x - nodes[m] for m in others if m != k], axis=0) if len(others) > 1 else 1.0
        D[:, l] = acc / den
    return V, D


# ------------------------------------------------------------------ triangle
@functools.lru_cache(maxsize=None)
def tri_lattice(p: int):
    """Local triangle node order: for j in 0..p, for i in 0..p-j -> (i, j),
    k = p-i-j.  i counts toward v1, j toward v2, k toward v0."""
    return tuple((i, j) for j in range(p + 1) for i in range(p + 1 - j))


@functools.lru_cache(maxsize=None)
def tri_nodes(p: int):
    """Blyth-Pozrikidis triangle nodes (reading O1). Returns r, s arrays [Nt]."""
    x, _ = lgl(p)
    v = (1.0 + x) / 2.0
    r, s = [], []
    for (i, j) in tri_lattice(p):
        k = p - i - j
        lam1 = (1.0 + 2.0 * v[i] - v[j] - v[k]) / 3.0
        lam2 = (1.0 + 2.0 * v[j] - v[i] - v[k]) / 3.0
        r.append(2.0 * lam1 - 1.0)
        s.append(2.0 * lam2 - 1.0)
    return np.array(r), np.array(s)


def _jacobi(n, alpha, beta, x):
    return eval_jacobi(n, alpha, beta, x)


def _djacobi(n, alpha, beta, x):
    if n == 0:
        return np.zeros_like(x)
    return 0.5 * (n + alpha + beta + 1) * eval_jacobi(n - 1, alpha + 1, beta + 1, x)


def dubiner(p: int, r: np.ndarray, s: np.ndarray):
    """Dubiner polynomials psi_ij and their r/s derivatives at points (r,s).
    Returns (psi, dpsi_dr, dpsi_ds), each [npts][Nt]."""
    r = np.asarray(r, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    top = np.isclose(s, 1.0, atol=1e-14, rtol=0)
    denom = np.where(top, 1.0, 1.0 - s)
    a = np.where(top, -1.0, 2.0 * (1.0 + r) / denom - 1.0)
    b = s
    cols, cr, cs = [], [], []
    for (i, j) in [(i, j) for i in range(p + 1) for j in range(p + 1 - i)]:
        Pi, dPi = _jacobi(i, 0, 0, a), _djacobi(i, 0, 0, a)
        Qj, dQj = _jacobi(j, 2 * i + 1, 0, b), _djacobi(j, 2 * i + 1, 0, b)
        om = (1.0 - b)
        om_i = om ** i
        om_im1 = om ** (i - 1) if i >= 1 else np.zeros_like(b)
        cols.append(Pi * Qj * om_i)
        cr.append(2.0 * dPi * Qj * om_im1)
        cs.append(dPi * Qj * om_im1 * (1.0 + a) + Pi * (dQj * om_i - i * Qj * om_im1))
    return np.stack(cols, 1), np.stack(cr, 1), np.stack(cs, 1)


@functools.lru_cache(maxsize=None)
def _tri_vinv(p: int):
    r, s = tri_nodes(p)
    V, _, _ = dubiner(p, r, s)
    return np.linalg.inv(V)


def tri_lagrange(p: int, r, s):
    """Triangle cardinal basis L_m and derivatives at points: ([np][Nt],)*3."""
    Vi = _tri_vinv(p)
    psi, pr, ps = dubiner(p, np.atleast_1d(r), np.atleast_1d(s))
    return psi @ Vi, pr @ Vi, ps @ Vi


# ------------------------------------------------------------------ prism
def n_tri(p):
    return (p + 1) * (p + 2) // 2


def n_prism(p, q=None):
    """Nodes of P_p(triangle) x P_q(t) (q = p: the isotropic space of reading O2)."""
    return n_tri(p) * ((p if q is None else q) + 1)


@functools.lru_cache(maxsize=None)
def prism_nodes(p: int, q: int | None = None):
    """Reference coordinates [N][3] of local prism nodes n = m + Nt*l and the
    lattice coordinates [N][3] = (i, j, l).  Horizontal order p (triangle nodes),
    vertical order q (LGL(q) in t; default q = p).  SURVEY NEXT-2: the paper's
    (P_xy, P_z) pairs."""
    q = p if q is None else q
    r, s = tri_nodes(p)
    t, _ = lgl(q)
    lat = tri_lattice(p)
    Nt = n_tri(p)
    rst = np.zeros((Nt * (q + 1), 3))
    ijl = np.zeros((Nt * (q + 1), 3), dtype=np.int64)
    for l in range(q + 1):
        for m in range(Nt):
            n = m + Nt * l
            rst[n] = (r[m], s[m], t[l])
            ijl[n] = (lat[m][0], lat[m][1], l)
    return rst, ijl


def prism_basis(p: int, pts: np.ndarray, q: int | None = None):
    """Prism cardinal basis of P_p(triangle) x P_q(t) (default q = p) at points
    [np][3]: values [np][N] and gradient [3][np][N] (d/dr, d/ds, d/dt)."""
    q = p if q is None else q
    pts = np.atleast_2d(pts)
    Lt, Lr, Ls = tri_lagrange(p, pts[:, 0], pts[:, 1])
    h, dh = lagrange1d(lgl(q)[0], pts[:, 2])
    Nt = n_tri(p)
    npt = pts.shape[0]
    val = np.zeros((npt, Nt * (q + 1)))
    grad = np.zeros((3, npt, Nt * (q + 1)))
    for l in range(q + 1):
        sl = slice(Nt * l, Nt * (l + 1))
        val[:, sl] = Lt * h[:, l:l + 1]
        grad[0][:, sl] = Lr * h[:, l:l + 1]
        grad[1][:, sl] = Ls * h[:, l:l + 1]
        grad[2][:, sl] = Lt * dh[:, l:l + 1]
    return val, grad


@functools.lru_cache(maxsize=None)
def tri_cubature(p: int):
    """Collapsed rule exact to degree 2p+1 on the reference triangle (O-4)."""
    a, wa = gauss_legendre(p + 1)
    b, wb = gauss_jacobi10(p + 1)
    r, s, w = [], [], []
    for jb in range(p + 1):
        for ia in range(p + 1):
            r.append((1.0 + a[ia]) * (1.0 - b[jb]) / 2.0 - 1.0)
            s.append(b[jb])
            w.append(wa[ia] * wb[jb] / 2.0)
    return np.array(r), np.array(s), np.array(w)


@functools.lru_cache(maxsize=None)
def prism_cubature(p: int, q: int | None = None):
    """Cubature points [Q][3] and weights [Q], point q = ta + Qt*qv: the collapsed
    triangle rule of order p times GL(q+1) in t (default q = p; reading O6)."""
    q = p if q is None else q
    r, s, wt = tri_cubature(p)
    t, wv = gauss_legendre(q + 1)
    Qt = len(r)
    pts = np.zeros((Qt * (q + 1), 3))
    w = np.zeros(Qt * (q + 1))
    for qv in range(q + 1):
        for ta in range(Qt):
            q = ta + Qt * qv
            pts[q] = (r[ta], s[ta], t[qv])
            w[q] = wt[ta] * wv[qv]
    return pts, w


def face_nodes(p: int, q: int | None = None):
    """Local node lists of the 5 prism faces (bot, top, q01, q12, q20)."""
    q = p if q is None else q
    _, ijl = prism_nodes(p, q)
    i, j, l = ijl[:, 0], ijl[:, 1], ijl[:, 2]
    return [np.nonzero(l == 0)[0], np.nonzero(l == q)[0], np.nonzero(j == 0)[0],
            np.nonzero(i + j == p)[0], np.nonzero(i == 0)[0]]


def level_schedule_pq(p: int, q: int):
    """Coarsening of (P_xy, P_z) (reading O19): semi-coarsen the larger
    order first, to max(smaller, ceil((larger+1)/2)), until the orders are equal
    ("until polynomial orders in all directions are equal"), then the
    isotropic rule of level_schedule."""
    out = [(p, q)]
    while out[-1][0] != out[-1][1]:
        a, b = out[-1]
        if a > b:
            out.append((max(b, math.ceil((a + 1) / 2) if math.ceil((a + 1) / 2) < a else a - 1), b))
        else:
            out.append((a, max(a, math.ceil((b + 1) / 2) if math.ceil((b + 1) / 2) < b else b - 1)))
    return out + [(c, c) for c in level_schedule(out[-1][0])[1:]]


def level_schedule(p: int):
    """Default coarsening P -> ceil((P+1)/2) with a strict-decrease guard, down
    to 1 (reading O18)."""
    out = [p]
    while out[-1] > 1:
        c = math.ceil((out[-1] + 1) / 2)
        if c >= out[-1]:
            c = out[-1] - 1
        out.append(c)
    return out
