"""Synthetic workload of BASELINE.json config 5: unstructured basin with a body.

Recipe (readings O29, O31, O34):

* Domain [0,Lx]x[0,Ly] (default 64 x 32), depth h = 1.  A fixed box hull with
  footprint 8 x 2 centred at (Lx/2, Ly/2), draft 0.6 and a rounded bilge of
  radius 0.2 is cut out of the fluid volume.
* Horizontal mesh: seeded jittered Delaunay triangulation
  (scipy.spatial.Delaunay) of a point set graded 4x finer near the hull:
  lattice spacing hf inside the ring hull +- 2 m, 2 hf inside hull +- 4 m, 4 hf
  elsewhere (the finer lattice includes the coarser one's points on the ring
  boundaries).  Interior points are jittered by U(-0.15, 0.15) x local spacing;
  points on the domain boundary or the hull footprint slide only along it;
  corners are fixed.  The triangulation conforms to the footprint rectangle
  (checked).  Default hf = 1/12 gives ~61 k triangles (reading O29: the ~50 M
  DOF target at p = 6 needs ~57 k triangles, not 100 k).
* Vertical layering (reading O31): columns under the footprint have 5 layers
  from z = -1 up to the hull bottom z_h(x, y); every other column has 5 layers
  from -1 up to s, then 3 layers from s up to the free surface eta(x, y).  The
  bilge is a circular arc of radius 0.2 truncated at 75 degrees and continued
  by its tangent to the footprint edge, where it reaches s = z_h(edge) = -0.4264
  (a vertical tangent would make the layered columns degenerate); the outer
  split height s is that edge height, so the nodes on the footprint boundary
  are shared by both column types.
* Faces: bottom and domain walls Neumann, hull bottom (top of the footprint
  columns) and hull walls (lateral faces of the outer columns' upper 3 layers
  on the footprint edge) Neumann, free surface Dirichlet.
* Dirichlet data: a linear focused wave group at focus time: 32 components,
  k_i uniform in [0.5, 2] k_p, k_p = 5.6 (k_p h of P:448 with h = 1),
  Gaussian amplitude spectrum normalised to sum a_i = 0.03, direction 0.1745
  rad, all crests at the hull centre:
  eta = sum a_i cos(k_i . (x - x_f)), phi = sum (g a_i / w_i) cosh(k_i(z+h)) /
  cosh(k_i h) sin(k_i . (x - x_f)), w_i^2 = g k_i tanh(k_i h), g = 9.81.
  The wave data is deterministic (no random draws); the jitter uses
  numpy.random.default_rng(seed).

No arithmetic of the method lives here (no basis, cubature or operator).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np
from scipy.spatial import Delaunay

from .configs import G_ACC

DRAFT, BILGE, TRUNC_DEG = 0.6, 0.2, 75.0
FOOT = (8.0, 2.0)


def _bilge_profile():
    """z_h(delta), delta = distance inside the footprint from its nearest edge."""
    th = math.radians(TRUNC_DEG)
    d75 = BILGE - BILGE * math.sin(th)
    z75 = -DRAFT + BILGE * (1.0 - math.cos(th))
    slope = math.tan(th)                       # dz/d(-delta) of the tangent at 75 degrees
    z_edge = z75 + slope * d75

    def zh(delta):
        delta = np.asarray(delta, dtype=np.float64)
        out = np.full(delta.shape, -DRAFT)
        arc = (delta < BILGE) & (delta >= d75)
        # arc point at angle t: delta = R - R sin t, z = -D + R (1 - cos t)
        t = np.arcsin(np.clip((BILGE - delta[arc]) / BILGE, -1.0, 1.0))
        out[arc] = -DRAFT + BILGE * (1.0 - np.cos(t))
        lin = delta < d75
        out[lin] = z75 + slope * (d75 - delta[lin])
        return out

    return zh, z_edge


@dataclasses.dataclass
class HullMesh:
    name: str
    p: int
    vertices: np.ndarray          # [n_vert][3]
    prisms: np.ndarray            # [E][6] int32
    face_tag: np.ndarray          # [E][5] uint8
    vert2d: np.ndarray            # [nv2][2]
    tri: np.ndarray               # [T][3]
    elem_tri: np.ndarray          # [E] footprint triangle of every prism
    elem_layer: np.ndarray        # [E] layer (0 = bottom)
    tri_inside: np.ndarray        # [T] bool: triangle under the hull
    h: float
    s_split: float
    meta: dict

    @property
    def n_elem(self) -> int:
        return int(self.prisms.shape[0])

    def eta(self, x, y):
        return _group(self.meta)[0](x, y)

    def phi(self, x, y, z):
        return _group(self.meta)[1](x, y, z)

    def z_hull(self, x, y):
        zh, _ = _bilge_profile()
        x0, y0, x1, y1 = self.meta["foot"]
        delta = np.minimum(np.minimum(x - x0, x1 - x), np.minimum(y - y0, y1 - y))
        return zh(np.maximum(delta, 0.0))

    def node_xyz(self, rst: np.ndarray, elems: Optional[np.ndarray] = None) -> np.ndarray:
        """Element node coordinates [E][N][3] for the caller's reference nodes rst
        (same reference prism as PrismMesh.node_xyz): x, y affine per triangle, z
        from the layered map of reading O31 evaluated at the node's (x, y)."""
        rst = np.asarray(rst, dtype=np.float64)
        if elems is None:
            elems = np.arange(self.n_elem)
        elems = np.asarray(elems)
        t = self.elem_tri[elems]
        lay = self.elem_layer[elems]
        A, B, C = (self.vert2d[self.tri[t, i]] for i in range(3))
        l1 = (1.0 + rst[:, 0]) * 0.5
        l2 = (1.0 + rst[:, 1]) * 0.5
        l0 = 1.0 - l1 - l2
        x = A[:, None, 0] * l0 + B[:, None, 0] * l1 + C[:, None, 0] * l2
        y = A[:, None, 1] * l0 + B[:, None, 1] * l1 + C[:, None, 1] * l2
        tt = (1.0 + rst[None, :, 2]) * 0.5
        inside = self.tri_inside[t][:, None]
        low = lay[:, None] < 5
        top5 = np.where(inside, self.z_hull(x, y), self.s_split)
        z_low = -self.h + ((lay[:, None] + tt) / 5.0) * (top5 + self.h)
        sig3 = (lay[:, None] - 5 + tt) / 3.0
        z_up = self.s_split + sig3 * (self.eta(x, y) - self.s_split)
        z = np.where(low, z_low, z_up)
        return np.stack([x, y, z], axis=-1)


def _group(meta):
    a = np.asarray(meta["a"])
    k = np.asarray(meta["k"])
    th = meta["theta"]
    xf, yf = meta["focus"]
    h = 1.0
    om = np.sqrt(G_ACC * k * np.tanh(k * h))
    kx, ky = k * math.cos(th), k * math.sin(th)

    def eta(x, y):
        x = np.asarray(x, dtype=np.float64)
        out = np.zeros(np.broadcast(x, y).shape)
        for i in range(len(a)):
            out += a[i] * np.cos(kx[i] * (x - xf) + ky[i] * (y - yf))
        return out

    def phi(x, y, z):
        x = np.asarray(x, dtype=np.float64)
        out = np.zeros(np.broadcast(x, y, z).shape)
        for i in range(len(a)):
            out += (G_ACC * a[i] / om[i]) * np.cosh(k[i] * (z + h)) / np.cosh(k[i] * h) \
                * np.sin(kx[i] * (x - xf) + ky[i] * (y - yf))
        return out

    return eta, phi


def _points(Lx, Ly, foot, hf, rng, jitter):
    x0, y0, x1, y1 = foot
    rings = [(x0 - 2, y0 - 2, x1 + 2, y1 + 2), (x0 - 4, y0 - 4, x1 + 4, y1 + 4), (0.0, 0.0, Lx, Ly)]

    def inside(px, py, r, strict=False):
        if strict:
            return (px > r[0]) & (px < r[2]) & (py > r[1]) & (py < r[3])
        return (px >= r[0] - 1e-9) & (px <= r[2] + 1e-9) & (py >= r[1] - 1e-9) & (py <= r[3] + 1e-9)

    pts, spacing = [], []
    for k, R in enumerate(rings):
        sp = hf * 2 ** k
        xs = np.arange(round(R[0] / sp), round(R[2] / sp) + 1) * sp
        ys = np.arange(round(R[1] / sp), round(R[3] / sp) + 1) * sp
        X, Y = np.meshgrid(xs, ys)
        X, Y = X.ravel(), Y.ravel()
        keep = inside(X, Y, R)
        if k > 0:
            keep &= ~inside(X, Y, rings[k - 1], strict=True)
        pts.append(np.stack([X[keep], Y[keep]], 1))
        spacing.append(np.full(int(keep.sum()), sp))
    P = np.concatenate(pts)
    S = np.concatenate(spacing)
    key = np.round(P / (hf * 1e-3)).astype(np.int64)
    _, first = np.unique(key[:, 0] * 10 ** 9 + key[:, 1], return_index=True)
    first = np.sort(first)
    P, S = P[first], S[first]
    # jitter: interior free; domain boundary / footprint boundary tangential only; corners fixed
    d = rng.uniform(-1.0, 1.0, size=P.shape) * jitter * S[:, None]
    eps = 1e-9
    on_x = (np.abs(P[:, 0]) < eps) | (np.abs(P[:, 0] - Lx) < eps)
    on_y = (np.abs(P[:, 1]) < eps) | (np.abs(P[:, 1] - Ly) < eps)
    fx = ((np.abs(P[:, 0] - x0) < eps) | (np.abs(P[:, 0] - x1) < eps)) & (P[:, 1] >= y0 - eps) & (P[:, 1] <= y1 + eps)
    fy = ((np.abs(P[:, 1] - y0) < eps) | (np.abs(P[:, 1] - y1) < eps)) & (P[:, 0] >= x0 - eps) & (P[:, 0] <= x1 + eps)
    d[on_x | fx, 0] = 0.0
    d[on_y | fy, 1] = 0.0
    # points on a footprint edge keep their position along the other footprint edge's corner
    corner = (fx & fy) | (on_x & on_y)
    d[corner] = 0.0
    # footprint-edge points only slide within the edge (keep away from its corners)
    return P + d, S


def config5(p: int = 6, hf: float = 1.0 / 12.0, Lx: float = 64.0, Ly: float = 32.0, seed: int = 5,
            jitter: float = 0.15, n_comp: int = 32, hull: bool = True, amp: float = 0.03) -> HullMesh:
    """Unstructured basin with a body (BASELINE.json config 5).  Scaled replicas:
    a smaller domain around the same hull and/or a larger hf."""
    rng = np.random.default_rng(seed)
    xc, yc = Lx / 2.0, Ly / 2.0
    foot = (xc - FOOT[0] / 2, yc - FOOT[1] / 2, xc + FOOT[0] / 2, yc + FOOT[1] / 2)
    P, _ = _points(Lx, Ly, foot, hf, rng, jitter)
    tri = Delaunay(P).simplices.astype(np.int32)
    a2 = P[tri]
    area = 0.5 * ((a2[:, 1, 0] - a2[:, 0, 0]) * (a2[:, 2, 1] - a2[:, 0, 1]) -
                  (a2[:, 2, 0] - a2[:, 0, 0]) * (a2[:, 1, 1] - a2[:, 0, 1]))
    tri[area < 0] = tri[area < 0][:, [0, 2, 1]]
    area = np.abs(area)
    assert area.min() > 1e-3 * hf * hf, "degenerate triangle"
    cen = a2.mean(axis=1)
    x0, y0, x1, y1 = foot
    tin = (cen[:, 0] > x0) & (cen[:, 0] < x1) & (cen[:, 1] > y0) & (cen[:, 1] < y1)
    if not hull:  # study variant: the same graded mesh without the body
        tin[:] = False
    eps = 1e-9
    vin = (P[:, 0] >= x0 - eps) & (P[:, 0] <= x1 + eps) & (P[:, 1] >= y0 - eps) & (P[:, 1] <= y1 + eps)
    vout = ~((P[:, 0] > x0 + eps) & (P[:, 0] < x1 - eps) & (P[:, 1] > y0 + eps) & (P[:, 1] < y1 - eps))
    assert np.all(vin[tri[tin]]) and (not hull or np.all(vout[tri[~tin]])), "triangulation does not conform"
    if not hull:
        vout[:] = True
    # wave group (deterministic)
    kp = 5.6
    k = np.linspace(0.5, 2.0, n_comp) * kp
    a = np.exp(-0.5 * ((k - kp) / (0.25 * kp)) ** 2)
    a = amp * a / a.sum()
    meta = dict(a=a.tolist(), k=k.tolist(), theta=0.1745, focus=(xc, yc), foot=foot, hf=hf, seed=seed,
                Lx=Lx, Ly=Ly)
    zh, z_edge = _bilge_profile()
    eta = _group(meta)[0]
    nv2, T = P.shape[0], tri.shape[0]
    # vertical lines of 3D vertices: outer-or-edge vertices 9 levels, strictly-inside ones 6
    nlev = np.where(vout, 9, 6)
    voff = np.concatenate([[0], np.cumsum(nlev)])
    verts = np.zeros((voff[-1], 3))
    foot_delta = np.minimum(np.minimum(P[:, 0] - x0, x1 - P[:, 0]), np.minimum(P[:, 1] - y0, y1 - P[:, 1]))
    top5 = np.where(vout, z_edge, zh(np.maximum(foot_delta, 0.0)))
    et = eta(P[:, 0], P[:, 1])
    for lv in range(9):
        has = nlev > lv
        idx = voff[:-1][has] + lv
        verts[idx, 0] = P[has, 0]
        verts[idx, 1] = P[has, 1]
        if lv <= 5:
            verts[idx, 2] = -1.0 + (lv / 5.0) * (top5[has] + 1.0)
        else:
            verts[idx, 2] = z_edge + ((lv - 5) / 3.0) * (et[has] - z_edge)
    nl = np.where(tin, 5, 8)
    E = int(nl.sum())
    elem_tri = np.repeat(np.arange(T), nl)
    elem_layer = np.concatenate([np.arange(n) for n in nl]).astype(np.int64)
    prisms = np.empty((E, 6), dtype=np.int32)
    tv = tri[elem_tri]
    prisms[:, :3] = voff[:-1][tv] + elem_layer[:, None]
    prisms[:, 3:] = voff[:-1][tv] + elem_layer[:, None] + 1
    face_tag = np.zeros((E, 5), dtype=np.uint8)
    face_tag[:, 0] = np.where(elem_layer == 0, 2, 0)
    top_layer = np.where(tin[elem_tri], 4, 7)
    face_tag[:, 1] = np.where(elem_layer == top_layer, np.where(tin[elem_tri], 2, 1), 0)
    # lateral faces: domain walls (all layers) and hull walls (outer columns, layers 5-7)
    Lbox = (0.0, 0.0, Lx, Ly)
    for f, (i, j) in enumerate([(0, 1), (1, 2), (2, 0)]):
        A, B = P[tri[:, i]], P[tri[:, j]]
        wall = np.zeros(T, dtype=bool)
        for c in (0, 1):
            for val in (Lbox[c], Lbox[c + 2]):
                wall |= (np.abs(A[:, c] - val) < eps) & (np.abs(B[:, c] - val) < eps)
        hull = np.zeros(T, dtype=bool)
        for c, (lo, hi) in enumerate([(x0, x1), (y0, y1)]):
            other = 1 - c
            olo, ohi = (y0, y1) if c == 0 else (x0, x1)
            for val in (lo, hi):
                hull |= (np.abs(A[:, c] - val) < eps) & (np.abs(B[:, c] - val) < eps) & \
                        (A[:, other] >= olo - eps) & (A[:, other] <= ohi + eps) & \
                        (B[:, other] >= olo - eps) & (B[:, other] <= ohi + eps)
        hull &= ~tin
        fw = wall[elem_tri]
        fh = hull[elem_tri] & (elem_layer >= 5)
        face_tag[:, 2 + f] = np.where(fw | fh, 2, 0)
    return HullMesh(name="config5", p=p, vertices=verts, prisms=prisms, face_tag=face_tag, vert2d=P, tri=tri,
                    elem_tri=elem_tri, elem_layer=elem_layer, tri_inside=tin, h=1.0, s_split=z_edge, meta=meta)


def config5_replica(p: int = 3, hf: float = 0.25, seed: int = 5) -> HullMesh:
    """Scaled-down replica for oracle parity: the same hull in a 24 x 12 basin."""
    return config5(p=p, hf=hf, Lx=24.0, Ly=12.0, seed=seed, n_comp=32)
