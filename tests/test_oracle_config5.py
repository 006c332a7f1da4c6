"""Pins of the config-5 construction (hull in a graded jittered-Delaunay basin,
readings O29/O31/O34) and of the oracle on it: fluid volume against an
independent quadrature of the free surface and hull bottom, global operator
invariants, face tags, and the hybrid FDM/dense smoother (reading O35) reaching
the direct solution."""
import numpy as np
import pytest

from oracle import pmg, refelem as R, sem
from workloads.config5 import config5


def _volume(m, p):
    pts, w = R.prism_cubature(p)
    rst, _ = R.prism_nodes(p)
    X = m.node_xyz(rst)
    _, dgeo = R.prism_basis(p, pts)
    J = np.einsum("eni,cqn->eqic", X, dgeo)
    det = np.linalg.det(J)
    assert det.min() > 0
    return float((det * w).sum())


def test_config5_volume_converges_to_the_surfaces():
    """sum w detJ = int_outside (eta + 1) + int_footprint (z_h + 1), the surfaces
    integrated independently (midpoint rule, 5 mm); the nodal map interpolates
    eta and the bilge, so the error decreases with p."""
    hx = 0.005
    errs = []
    for p in (2, 3, 4):
        m = config5(p=p, hf=0.5, Lx=16.0, Ly=10.0)
        xs, ys = np.arange(hx / 2, 16, hx), np.arange(hx / 2, 10, hx)
        X, Y = np.meshgrid(xs, ys)
        x0, y0, x1, y1 = m.meta["foot"]
        inside = (X > x0) & (X < x1) & (Y > y0) & (Y < y1)
        ref = float(((np.where(inside, m.z_hull(X, Y), m.eta(X, Y)) + 1.0) * hx * hx).sum())
        errs.append(abs(_volume(m, p) - ref) / ref)
    assert errs[0] > errs[1] > errs[2]
    assert errs[0] < 1e-3 and errs[2] < 2e-4


def test_config5_sizes_and_faces():
    """Default construction: ~61 k triangles (reading O29), 5-layer footprint
    columns and 8-layer outer columns (O31); Dirichlet nodes only on the free
    surface outside the footprint."""
    m = config5(p=6)
    T, Ti = len(m.tri), int(m.tri_inside.sum())
    assert 55_000 < T < 65_000 and Ti == 4608
    assert m.n_elem == 5 * Ti + 8 * (T - Ti)
    r = config5(p=2, hf=0.5, Lx=16.0, Ly=10.0)
    lev = sem.build_level(r, 2)
    x0, y0, x1, y1 = r.meta["foot"]
    d = lev.xyz[lev.dirichlet]
    assert not np.any((d[:, 0] > x0 + 1e-9) & (d[:, 0] < x1 - 1e-9) & (d[:, 1] > y0 + 1e-9) & (d[:, 1] < y1 - 1e-9))
    np.testing.assert_allclose(d[:, 2], r.eta(d[:, 0], d[:, 1]), atol=1e-12)


def test_config5_operator_invariants_and_hybrid_pcg():
    """A = A^T, A 1 = 0 on the hull mesh; PCG with the hybrid FDM/dense smoother
    (O35) and with the exact smoother both reach the sparse-direct solution."""
    m = config5(p=2, hf=0.5, Lx=16.0, Ly=10.0)
    lev = sem.build_system(m, 2)
    assert abs(lev.A - lev.A.T).max() < 1e-12 * abs(lev.A).max()
    assert np.abs(lev.A @ np.ones(lev.n)).max() < 1e-11
    phiD = m.phi(*lev.xyz.T)
    ref = sem.solve_direct(lev, phiD)[lev.free]
    A, b = sem.dirichlet_lift(lev, phiD)
    for ls in ("fdm", "dense"):
        mg = pmg.PMG(m, local_solve=ls)
        u, info = pmg.pcg(mg, b, rtol=1e-12)
        assert np.linalg.norm(u - ref) <= 1e-10 * np.linalg.norm(ref), ls
        assert info["iters"] < 25, (ls, info["iters"])
