"""Oracle FNPF time stage (TEST INFRASTRUCTURE; see oracle/__init__.py).

SURVEY §8(f) NEXT-4: the fully nonlinear potential-flow model that re-solves the
Laplace problem at every time stage.  Written in the paper's order and notation:

* state: the free-surface elevation eta and surface potential phi~ at the
  free-surface nodes (eq 2.1: "'~' is used for free surface variables");
* every stage: the fluid volume follows eta through the sigma map
  z = -h + sigma (eta + h) (eq 3.3): each element node keeps its sigma
  and sits on the vertical line of one free-surface node (layered meshes, reading
  O37); the Laplace problem eq 2.2 is solved with phi = phi~ on the free
  surface -- here by the sparse direct solve of the discrete system (sem.py, the
  plain definition the p-multigrid reaches);
* w~ = dphi/dz at the free surface (reading O38), the horizontal gradients of
  eta and phi~ along the surface (reading O39);
* the free-surface conditions eq 2.1a-b:
      d eta / dt  = -grad eta . grad phi~ + w~ (1 + grad eta . grad eta)
      d phi~ / dt = -g eta - 1/2 (grad phi~ . grad phi~ - w~^2 (1 + grad eta . grad eta))
  with g = 9.81; `linear=True` is the small-amplitude version (H/L ~ 0):
  d eta/dt = w~, d phi~/dt = -g eta on the still-water geometry;
* time integration: the classical four-stage explicit Runge-Kutta method (ERK4,
  P:363), one Laplace solve per stage (reading O40).

Readings:
  O37  layered geometry update: sigma of every node from the t = 0 geometry,
       sigma = (z - z_b) / (z_s - z_b) on its vertical line (z_b the line's bottom,
       z_s its free-surface node); the new z = z_b + sigma (eta_s - z_b).
  O38  w~ at a free-surface node: in every top element holding the node, the
       gradient of the element's Lagrange interpolant of phi through the
       isoparametric map, grad phi = J^{-T} grad_ref phi at the node; arithmetic
       mean over those elements (the gradient of a C0 field is two-valued at
       element boundaries; the paper does not state the recovery).
  O39  grad eta, grad phi~: the same recovery for the P_p surface interpolants on
       the top faces (x, y affine per triangle), averaged over the faces.
  O40  ERK4 = classical RK4 (4 stages, 4 solves per step); the paper's count of
       5 solves per step is not reproduced.
"""
from __future__ import annotations

import numpy as np
from scipy.spatial import cKDTree

from . import refelem as R
from . import sem

G_ACC = 9.81


class Surface:
    """Vertical-line structure of a layered mesh at order p (oracle numbering)."""

    def __init__(self, mesh, p: int, tol: float = 1e-9):
        self.mesh, self.p = mesh, p
        self.level = sem.build_level(mesh, p)          # t = 0 geometry: mesh.node_xyz
        xyz = self.level.xyz
        self.snode = np.nonzero(self.level.dirichlet)[0]         # free-surface nodes
        tree = cKDTree(xyz[self.snode, :2])
        d, line = tree.query(xyz[:, :2])
        if d.max() > tol:
            raise ValueError("mesh is not layered: a node is not below a free-surface node")
        self.line = line                                          # surface index of every node
        zb = np.full(len(self.snode), np.inf)
        np.minimum.at(zb, line, xyz[:, 2])
        self.zb = zb
        zs = xyz[self.snode, 2]
        self.sigma = (xyz[:, 2] - zb[line]) / (zs[line] - zb[line])
        self.xy = xyz[:, :2].copy()
        self.eta0 = zs.copy()
        # top elements: top face on the free surface; their top-face local nodes
        self.fn_top = R.face_nodes(p)[1]
        self.top = np.nonzero(mesh.face_tag[:, 1] == 1)[0]

    def xyz(self, eta_s: np.ndarray) -> np.ndarray:
        """Node coordinates for the surface elevation eta_s (reading O37)."""
        z = self.zb[self.line] + self.sigma * (eta_s[self.line] - self.zb[self.line])
        return np.column_stack([self.xy, z])


class StagedMesh:
    """The workload mesh with its nodal map moved to a new free surface (the
    finest-order map, which defines the geometry of every level)."""

    def __init__(self, surf: Surface, eta_s: np.ndarray):
        self.base, self.surf = surf.mesh, surf
        self.p = surf.p
        self.face_tag = surf.mesh.face_tag
        self.n_elem = surf.mesh.n_elem
        self._xyz = surf.xyz(eta_s)

    def node_xyz(self, rst, elems=None):
        rst_p, _ = R.prism_nodes(self.p)
        if rst.shape != rst_p.shape or not np.allclose(rst, rst_p, atol=1e-13):
            raise ValueError("StagedMesh maps the finest-order reference nodes only")
        conn = self.surf.level.conn if elems is None else self.surf.level.conn[np.asarray(elems)]
        return self._xyz[conn]


def laplace_stage(surf: Surface, eta_s, phis_s, geometry: bool = True):
    """phi in the volume for surface data (eta, phi~): the direct solution of eq 2.2
    on the geometry of eta (or the t = 0 geometry when geometry=False, assembled once)."""
    if geometry or getattr(surf, "_lin", None) is None:
        m = StagedMesh(surf, eta_s if geometry else surf.eta0)
        lev = sem.build_system(m, surf.p)
        # the staged level's numbering is re-derived from coordinates: map nodes by position
        d, idx = cKDTree(m._xyz).query(lev.xyz)
        assert d.max() < 1e-9
        if not geometry:
            surf._lin = (m, lev, idx)
    else:
        m, lev, idx = surf._lin
    phiD = np.zeros(lev.n)
    phiD[lev.dirichlet] = phis_s[surf.line[idx[lev.dirichlet]]]
    phi_lev = sem.solve_direct(lev, phiD)
    phi = np.zeros(len(m._xyz))
    phi[idx] = phi_lev
    return phi, m._xyz


def w_tilde(surf: Surface, phi: np.ndarray, xyz: np.ndarray) -> np.ndarray:
    """Reading O38: w~ = dphi/dz at the free-surface nodes, averaged over top elements."""
    p = surf.p
    rst, _ = R.prism_nodes(p)
    _, D = R.prism_basis(p, rst[surf.fn_top])                # [3][Ntop][N]
    acc = np.zeros(len(surf.snode))
    cnt = np.zeros(len(surf.snode))
    for e in surf.top:
        ids = surf.level.conn[e]
        X = xyz[ids]                                        # [N][3]
        for k, n in enumerate(surf.fn_top):
            J = np.array([[D[c][k] @ X[:, i] for c in range(3)] for i in range(3)])   # J[i][c] = dx_i/dxi_c
            gref = np.array([D[c][k] @ phi[ids] for c in range(3)])
            grad = np.linalg.solve(J.T, gref)               # J^T grad = grad_ref
            s = surf.line[ids[n]]
            acc[s] += grad[2]
            cnt[s] += 1.0
    return acc / cnt


def surface_gradient(surf: Surface, f_s: np.ndarray, xyz: np.ndarray) -> np.ndarray:
    """Reading O39: (df/dx, df/dy) of the surface interpolant of f_s [ns] -> [ns][2]."""
    p = surf.p
    r, s = R.tri_nodes(p)
    _, Dr, Ds = R.tri_lagrange(p, r, s)                      # [Nt][Nt]
    acc = np.zeros((len(surf.snode), 2))
    cnt = np.zeros(len(surf.snode))
    for e in surf.top:
        ids = surf.level.conn[e][surf.fn_top]               # top-face nodes, triangle order m
        sidx = surf.line[ids]
        x, y = xyz[ids, 0], xyz[ids, 1]
        f = f_s[sidx]
        for k in range(len(ids)):
            J2 = np.array([[Dr[k] @ x, Ds[k] @ x], [Dr[k] @ y, Ds[k] @ y]])
            g = np.linalg.solve(J2.T, np.array([Dr[k] @ f, Ds[k] @ f]))
            acc[sidx[k]] += g
            cnt[sidx[k]] += 1.0
    return acc / cnt[:, None]


def surface_rhs(surf: Surface, eta_s, phis_s, linear: bool = False, g: float = G_ACC):
    """Eq 2.1a-b at the free-surface nodes: (d eta/dt, d phi~/dt, w~)."""
    phi, xyz = laplace_stage(surf, eta_s, phis_s, geometry=not linear)
    w = w_tilde(surf, phi, xyz)
    if linear:
        return w, -g * eta_s, w
    ge = surface_gradient(surf, eta_s, xyz)
    gp = surface_gradient(surf, phis_s, xyz)
    ge2 = (ge * ge).sum(1)
    deta = -(ge * gp).sum(1) + w * (1.0 + ge2)
    dphi = -g * eta_s - 0.5 * ((gp * gp).sum(1) - w * w * (1.0 + ge2))
    return deta, dphi, w


def erk4_step(surf: Surface, eta_s, phis_s, dt: float, linear: bool = False):
    """Classical RK4 (reading O40): four stages, one Laplace solve each."""
    k1e, k1p, _ = surface_rhs(surf, eta_s, phis_s, linear)
    k2e, k2p, _ = surface_rhs(surf, eta_s + 0.5 * dt * k1e, phis_s + 0.5 * dt * k1p, linear)
    k3e, k3p, _ = surface_rhs(surf, eta_s + 0.5 * dt * k2e, phis_s + 0.5 * dt * k2p, linear)
    k4e, k4p, _ = surface_rhs(surf, eta_s + dt * k3e, phis_s + dt * k3p, linear)
    return (eta_s + dt / 6.0 * (k1e + 2 * k2e + 2 * k3e + k4e),
            phis_s + dt / 6.0 * (k1p + 2 * k2p + 2 * k3p + k4p))
