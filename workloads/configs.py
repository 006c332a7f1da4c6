"""Synthetic workloads of BASELINE.json configs 1-4 (config 5 is NEXT).

Recipe (also in DESIGN.md §"Input recipe"):

* Horizontal mesh: [0,Lx]x[0,Ly] split into nx*ny quads, every quad split along
  the diagonal from its (i+1,j) corner to its (i,j+1) corner (reading O27), both
  triangles counter-clockwise seen from +z.
* Optional jitter (config 3/4): interior vertices move by U(-0.15,0.15)*spacing in
  x and y; non-corner boundary vertices move only along their boundary line.
* Vertical: nz uniform sigma-layers, z = -h + sigma*(eta(x,y)+h) (the
  sigma-map of PAPER.md eq. 3.3), applied to every element node so the
  element map is the degree-p nodal interpolant of that map (curvilinear prisms).
* Element order is column-major: element = triangle*nz + layer (all prisms of a
  vertical column are consecutive).
* Face tags per prism (bot, top, q01, q12, q20): 1 = Dirichlet (free surface,
  P:77), 2 = Neumann (bottom, walls), 0 = interior.
* Random draws use numpy.random.default_rng(seed) (PCG64) in a fixed order:
  jitter (ny+1, nx+1, 2) first, then the wave parameters a, k, theta, psi.

None of this is the method's arithmetic: the generators never evaluate a basis,
a cubature rule or an operator.  The reference node coordinates (r,s,t) that
``node_xyz`` maps are supplied by the caller (each side brings its own).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, Optional

import numpy as np

G_ACC = 9.81


@dataclasses.dataclass
class PrismMesh:
    name: str
    p: int
    vertices: np.ndarray          # [n_vert][3] float64
    prisms: np.ndarray            # [E][6] int32 (bottom v0 v1 v2 CCW, top v3 v4 v5 above)
    face_tag: np.ndarray          # [E][5] uint8 (bot, top, q01, q12, q20)
    # horizontal data of the layered construction
    vert2d: np.ndarray            # [nv2][2]
    tri: np.ndarray               # [T][3] int32
    nz: int
    h: float
    eta: Callable[[np.ndarray, np.ndarray], np.ndarray]
    phi: Callable[[np.ndarray, np.ndarray, np.ndarray], np.ndarray]   # Dirichlet data phi(x,y,z)
    curved: bool = True
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def n_elem(self) -> int:
        return int(self.prisms.shape[0])

    def node_xyz(self, rst: np.ndarray, elems: Optional[np.ndarray] = None) -> np.ndarray:
        """Physical coordinates of element nodes.

        rst: [N][3] reference coordinates (r,s,t) of the caller's local nodes on the
        reference prism {r,s >= -1, r+s <= 0} x [-1,1], with bottom-triangle vertices
        (-1,-1), (1,-1), (-1,1) <-> v0, v1, v2.  Returns [E][N][3] (or [len(elems)][N][3]).
        x,y: affine map of the element's triangle; z: the sigma-map evaluated at the
        node's (x,y) and sigma.  This *defines* the curvilinear geometry of the workload.
        """
        rst = np.asarray(rst, dtype=np.float64)
        if elems is None:
            elems = np.arange(self.n_elem)
        elems = np.asarray(elems)
        tri_id = elems // self.nz
        layer = elems % self.nz
        A = self.vert2d[self.tri[tri_id, 0]]   # [e][2]
        B = self.vert2d[self.tri[tri_id, 1]]
        C = self.vert2d[self.tri[tri_id, 2]]
        l1 = (1.0 + rst[:, 0]) * 0.5           # [N]
        l2 = (1.0 + rst[:, 1]) * 0.5
        l0 = 1.0 - l1 - l2
        x = A[:, None, 0] * l0 + B[:, None, 0] * l1 + C[:, None, 0] * l2
        y = A[:, None, 1] * l0 + B[:, None, 1] * l1 + C[:, None, 1] * l2
        sigma = (layer[:, None] + (1.0 + rst[None, :, 2]) * 0.5) / self.nz
        if self.curved:
            z = -self.h + sigma * (self.eta(x, y) + self.h)
        else:
            z = -self.h + sigma * self.h
        return np.stack([x, y, z], axis=-1)


def _structured_2d(Lx, Ly, nx, ny, jitter, rng):
    xs = np.linspace(0.0, Lx, nx + 1)
    ys = np.linspace(0.0, Ly, ny + 1)
    X, Y = np.meshgrid(xs, ys)            # [ny+1][nx+1]
    if jitter > 0.0:
        d = rng.uniform(-1.0, 1.0, size=(ny + 1, nx + 1, 2))
        dx = d[..., 0] * jitter * (Lx / nx)
        dy = d[..., 1] * jitter * (Ly / ny)
        jj, ii = np.meshgrid(np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
        on_x = (ii == 0) | (ii == nx)     # vertical boundary lines: x fixed
        on_y = (jj == 0) | (jj == ny)     # horizontal boundary lines: y fixed
        dx = np.where(on_x, 0.0, dx)
        dy = np.where(on_y, 0.0, dy)
        X = X + dx
        Y = Y + dy
    vert2d = np.stack([X.ravel(), Y.ravel()], axis=1)
    tris = []
    btag = []  # per triangle, boundary flag of edges (e01, e12, e20)
    vid = lambda i, j: j * (nx + 1) + i
    for j in range(ny):
        for i in range(nx):
            a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
            tris.append((a, b, d))
            btag.append((j == 0, False, i == 0))
            tris.append((b, c, d))
            btag.append((i == nx - 1, j == ny - 1, False))
    return vert2d, np.asarray(tris, dtype=np.int32), np.asarray(btag, dtype=bool)


def structured_basin(name, p, Lx, Ly, nx, ny, nz, h, eta, phi, jitter=0.0, rng=None,
                     curved=True, meta=None) -> PrismMesh:
    vert2d, tri, btag = _structured_2d(Lx, Ly, nx, ny, jitter, rng)
    nv2 = vert2d.shape[0]
    T = tri.shape[0]
    # 3D vertices: sigma level s = 0..nz
    sig = np.arange(nz + 1) / nz
    if curved:
        et = eta(vert2d[:, 0], vert2d[:, 1])
    else:
        et = np.zeros(nv2)
    zv = -h + sig[:, None] * (et[None, :] + h)          # [nz+1][nv2]
    vertices = np.empty(((nz + 1) * nv2, 3))
    vertices[:, 0] = np.tile(vert2d[:, 0], nz + 1)
    vertices[:, 1] = np.tile(vert2d[:, 1], nz + 1)
    vertices[:, 2] = zv.ravel()
    E = T * nz
    t_idx = np.repeat(np.arange(T), nz)
    s_idx = np.tile(np.arange(nz), T)
    prisms = np.empty((E, 6), dtype=np.int32)
    prisms[:, 0:3] = tri[t_idx] + (s_idx * nv2)[:, None]
    prisms[:, 3:6] = tri[t_idx] + ((s_idx + 1) * nv2)[:, None]
    face_tag = np.zeros((E, 5), dtype=np.uint8)
    face_tag[:, 0] = np.where(s_idx == 0, 2, 0)
    face_tag[:, 1] = np.where(s_idx == nz - 1, 1, 0)
    face_tag[:, 2:5] = np.where(btag[t_idx], 2, 0)
    return PrismMesh(name=name, p=p, vertices=vertices, prisms=prisms, face_tag=face_tag,
                     vert2d=vert2d, tri=tri, nz=nz, h=h, eta=eta, phi=phi, curved=curved,
                     meta=dict(meta or {}, Lx=Lx, Ly=Ly, nx=nx, ny=ny, nz=nz))


# ---------------------------------------------------------------- config 1
def config1(p: int = 3, nx: int = 4, ny: int = 4, nz: int = 2) -> PrismMesh:
    """Tiny box [0,2]x[0,1]x[-1,0], straight prisms; phi = cosh(k(z+1))cos(kx), k=pi.

    All non-top fluxes of this phi vanish exactly (sin(0)=sin(2pi)=0, no y
    dependence, sinh(0)=0), so homogeneous Neumann + top Dirichlet is exact.
    """
    k = math.pi
    eta = lambda x, y: np.zeros_like(x)
    phi = lambda x, y, z: np.cosh(k * (z + 1.0)) * np.cos(k * x)
    return structured_basin("config1", p, 2.0, 1.0, nx, ny, nz, 1.0, eta, phi,
                            curved=False, meta=dict(k=k))


# ---------------------------------------------------------------- config 2
def config2(p: int = 4, nx: int = 64, ny: int = 4, nz: int = 4) -> PrismMesh:
    """Curvilinear wave channel [0,16]x[0,1], eta = 0.05 sin(kx), k = 2pi/2.

    Dirichlet phi from linear wave theory (P:83 g=9.81):
    phi = -(g a/omega) cosh(k(z+h))/cosh(kh) cos(kx), omega^2 = g k tanh(kh).
    """
    h, a, k = 1.0, 0.05, math.pi
    om = math.sqrt(G_ACC * k * math.tanh(k * h))
    eta = lambda x, y: a * np.sin(k * x)
    phi = lambda x, y, z: -(G_ACC * a / om) * np.cosh(k * (z + h)) / math.cosh(k * h) * np.cos(k * x)
    return structured_basin("config2", p, 16.0, 1.0, nx, ny, nz, h, eta, phi,
                            meta=dict(a=a, k=k, omega=om))


# ---------------------------------------------------------------- config 3 / 4
def _wave_field(rng, n_waves, h):
    a = rng.uniform(0.0, 0.02, n_waves)
    k = rng.uniform(0.5, 3.0, n_waves)
    th = rng.uniform(0.0, 2 * math.pi, n_waves)
    psi = rng.uniform(0.0, 2 * math.pi, n_waves)
    om = np.sqrt(G_ACC * k * np.tanh(k * h))
    kx, ky = k * np.cos(th), k * np.sin(th)

    def eta(x, y):
        x = np.asarray(x, dtype=np.float64)
        out = np.zeros(np.broadcast(x, y).shape)
        for i in range(n_waves):
            out += a[i] * np.cos(kx[i] * x + ky[i] * y + psi[i])
        return out

    def phi(x, y, z):
        x = np.asarray(x, dtype=np.float64)
        out = np.zeros(np.broadcast(x, y, z).shape)
        for i in range(n_waves):
            out += (G_ACC * a[i] / om[i]) * np.cosh(k[i] * (z + h)) / np.cosh(k[i] * h) \
                * np.sin(kx[i] * x + ky[i] * y + psi[i])
        return out

    return eta, phi, dict(a=a.tolist(), k=k.tolist(), theta=th.tolist(), psi=psi.tolist())


def basin(name, p, L, n, nz, seed, jitter=0.15) -> PrismMesh:
    rng = np.random.default_rng(seed)
    # draw order: jitter first (inside structured_basin), then the waves
    vert_rng_state = rng
    h = 1.0
    # build the 2D mesh with the jitter draw, then the waves from the same stream
    vert2d, tri, btag = _structured_2d(L, L, n, n, jitter, vert_rng_state)
    eta, phi, wmeta = _wave_field(rng, 8, h)
    m = structured_basin(name, p, L, L, n, n, nz, h, eta, phi, jitter=0.0, rng=None,
                         meta=dict(seed=seed, jitter=jitter, waves=wmeta))
    # replace the unjittered horizontal mesh by the jittered one (same topology)
    m.vert2d = vert2d
    nv2 = vert2d.shape[0]
    et = eta(vert2d[:, 0], vert2d[:, 1])
    sig = np.arange(nz + 1) / nz
    zv = -h + sig[:, None] * (et[None, :] + h)
    m.vertices[:, 0] = np.tile(vert2d[:, 0], nz + 1)
    m.vertices[:, 1] = np.tile(vert2d[:, 1], nz + 1)
    m.vertices[:, 2] = zv.ravel()
    assert np.array_equal(m.tri, tri)
    return m


def config3(p: int = 5, n: int = 64, nz: int = 8, L: float = 32.0, seed: int = 3) -> PrismMesh:
    """3D wave basin [0,32]^2, 64x64 quads -> 8192 triangles x 8 layers, p=5."""
    return basin("config3", p, L, n, nz, seed)


# p -> (quads per side n, layers n_z); keeps ~10 M DOF and d_xy/d_z = 4
CONFIG4_SIZES = {1: (424, 53), 2: (216, 27), 3: (144, 18), 4: (104, 13),
                 5: (88, 11), 6: (72, 9), 7: (64, 8), 8: (56, 7)}


def config4(p: int, scale: float = 1.0, seed: int = 4) -> PrismMesh:
    """p-scaling sweep at ~10 M DOF (scale<1 gives the scaled-down replica)."""
    n, nz = CONFIG4_SIZES[p]
    if scale != 1.0:
        n = max(8, int(round(n * scale)) // 8 * 8)
        nz = max(1, n // 8)
    return basin(f"config4_p{p}", p, 32.0, n, nz, seed)


def delaunay_basin(name, p, Lx=2.0, Ly=1.0, n_in=24, n_bx=6, n_by=3, nz=2, seed=0, amp=0.03) -> PrismMesh:
    """Small unstructured layered basin: Delaunay triangulation (scipy.spatial.Delaunay)
    of n_in uniform random interior points plus evenly spaced boundary points, nz
    sigma-layers under eta = amp cos(pi x / Lx) cos(pi y / Ly) (walls: homogeneous
    Neumann, exact for the standing-wave phi below; free surface Dirichlet).  Random
    Delaunay meshes have high-valence vertices, hence larger Schwarz patches than the
    structured configs (used to reach the n_h > 56 FDM kernel on a small mesh).
    Draw order: interior points (n_in, 2)."""
    from scipy.spatial import Delaunay
    rng = np.random.default_rng(seed)
    pin = rng.uniform(0.05, 0.95, size=(n_in, 2)) * np.array([Lx, Ly])
    xs = np.linspace(0.0, Lx, n_bx + 1)
    ys = np.linspace(0.0, Ly, n_by + 1)
    bnd = [(x, 0.0) for x in xs] + [(x, Ly) for x in xs] + [(0.0, y) for y in ys[1:-1]] + [(Lx, y) for y in ys[1:-1]]
    vert2d = np.concatenate([np.asarray(bnd), pin])
    tri = Delaunay(vert2d).simplices.astype(np.int32)
    a = vert2d[tri]
    area = 0.5 * ((a[:, 1, 0] - a[:, 0, 0]) * (a[:, 2, 1] - a[:, 0, 1]) - (a[:, 2, 0] - a[:, 0, 0]) * (a[:, 1, 1] - a[:, 0, 1]))
    tri[area < 0] = tri[area < 0][:, [0, 2, 1]]
    eps = 1e-12
    btag = np.zeros(tri.shape, dtype=bool)
    for f, (i, j) in enumerate([(0, 1), (1, 2), (2, 0)]):
        A, B = vert2d[tri[:, i]], vert2d[tri[:, j]]
        for c, L in ((0, Lx), (1, Ly)):
            for val in (0.0, L):
                btag[:, f] |= (np.abs(A[:, c] - val) < eps) & (np.abs(B[:, c] - val) < eps)
    h = 1.0
    kx, ky = math.pi / Lx, math.pi / Ly
    k = math.hypot(kx, ky)
    om = math.sqrt(G_ACC * k * math.tanh(k * h))
    eta = lambda x, y: amp * np.cos(kx * x) * np.cos(ky * y)
    phi = lambda x, y, z: (G_ACC * amp / om) * np.cosh(k * (z + h)) / math.cosh(k * h) * np.cos(kx * x) * np.cos(ky * y)
    nv2, T = vert2d.shape[0], tri.shape[0]
    sig = np.arange(nz + 1) / nz
    zv = -h + sig[:, None] * (eta(vert2d[:, 0], vert2d[:, 1])[None, :] + h)
    vertices = np.empty(((nz + 1) * nv2, 3))
    vertices[:, 0] = np.tile(vert2d[:, 0], nz + 1)
    vertices[:, 1] = np.tile(vert2d[:, 1], nz + 1)
    vertices[:, 2] = zv.ravel()
    t_idx = np.repeat(np.arange(T), nz)
    s_idx = np.tile(np.arange(nz), T)
    prisms = np.empty((T * nz, 6), dtype=np.int32)
    prisms[:, 0:3] = tri[t_idx] + (s_idx * nv2)[:, None]
    prisms[:, 3:6] = tri[t_idx] + ((s_idx + 1) * nv2)[:, None]
    face_tag = np.zeros((T * nz, 5), dtype=np.uint8)
    face_tag[:, 0] = np.where(s_idx == 0, 2, 0)
    face_tag[:, 1] = np.where(s_idx == nz - 1, 1, 0)
    face_tag[:, 2:5] = np.where(btag[t_idx], 2, 0)
    return PrismMesh(name=name, p=p, vertices=vertices, prisms=prisms, face_tag=face_tag, vert2d=vert2d, tri=tri,
                     nz=nz, h=h, eta=eta, phi=phi, meta=dict(seed=seed, n_in=n_in, Lx=Lx, Ly=Ly, nz=nz))


def random_vector(n: int, seed: int) -> np.ndarray:
    """u ~ U(-1,1) (no cancellation, SURVEY §8(c) parity protocol)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)
