"""Pins of the anisotropic element spaces P_p(triangle) x P_q(t) (SURVEY §8(f)
NEXT-2; the paper's (P_xy, P_z) pairs, Table 5.4) and of
semi-coarsening in the oracle: polynomial reproduction, exact stiffness on
polynomials of the space (sympy), node counts, Galerkin consistency of nested
anisotropic levels, a symmetric V-cycle and PCG reaching the direct solution on
the paper's (5,3) -> (3,3) -> (1,1) schedule."""
import numpy as np
import pytest
import sympy as sy

from oracle import pmg, sem
from oracle import refelem as R
from workloads import config1, structured_basin


def _poly_tri(p, rng):
    c = {(a, b): rng.uniform(-1, 1) for a in range(p + 1) for b in range(p + 1 - a)}
    f = lambda r, s: sum(v * r ** a * s ** b for (a, b), v in c.items())
    fr = lambda r, s: sum(v * a * r ** (a - 1) * s ** b for (a, b), v in c.items() if a > 0)
    fs = lambda r, s: sum(v * b * r ** a * s ** (b - 1) for (a, b), v in c.items() if b > 0)
    return f, fr, fs


@pytest.mark.parametrize("p,q", [(3, 1), (4, 2), (2, 3), (5, 3)])
def test_anisotropic_basis_reproduces_polynomials(p, q):
    """Cardinal, and exact for P_p(triangle) x P_q(t) (values and the three
    derivatives at random points); N = Nt(p) (q + 1)."""
    rng = np.random.default_rng(10 * p + q)
    rst, ijl = R.prism_nodes(p, q)
    assert len(rst) == R.n_tri(p) * (q + 1) == R.n_prism(p, q) and ijl[:, 2].max() == q
    val, _ = R.prism_basis(p, rst, q)
    np.testing.assert_allclose(val, np.eye(len(rst)), atol=1e-12)
    f, fr, fs = _poly_tri(p, rng)
    ct = rng.uniform(-1, 1, q + 1)
    g = lambda t: sum(ct[k] * t ** k for k in range(q + 1))
    gt = lambda t: sum(k * ct[k] * t ** (k - 1) for k in range(1, q + 1))
    u = f(rst[:, 0], rst[:, 1]) * g(rst[:, 2])
    pts = np.stack([rng.uniform(-1, 0, 20), rng.uniform(-1, 0, 20), rng.uniform(-1, 1, 20)], 1)
    pts[:, 1] = np.minimum(pts[:, 1], -pts[:, 0])
    v, grad = R.prism_basis(p, pts, q)
    r, s, t = pts.T
    np.testing.assert_allclose(v @ u, f(r, s) * g(t), atol=1e-11)
    np.testing.assert_allclose(grad[0] @ u, fr(r, s) * g(t), atol=1e-10)
    np.testing.assert_allclose(grad[1] @ u, fs(r, s) * g(t), atol=1e-10)
    np.testing.assert_allclose(grad[2] @ u, f(r, s) * gt(t), atol=1e-10)


def _box(p, q, jitter=0.0, nz=2):
    rng = np.random.default_rng(5)
    m = structured_basin("box", p, 2.0, 1.0, 3, 2, nz, 1.0, lambda x, y: 0 * x, lambda x, y, z: 0 * x,
                         jitter=jitter, rng=rng, curved=False)
    m.pz = q
    return m


@pytest.mark.parametrize("p,q,jitter", [(2, 1, 0.0), (3, 2, 0.2), (1, 2, 0.0), (3, 1, 0.2)])
def test_anisotropic_stiffness_exact_on_polynomials(p, q, jitter):
    """u^T A v = int grad u . grad v exactly for u, v in P_p(x, y) x P_q(z) on
    straight prisms (x, y affine per triangle, z affine per layer): the cubature
    (triangle rule of order p, GL(q+1) vertically) integrates these products
    exactly, so a wrong order in any direction fails."""
    m = _box(p, q, jitter)
    lev = sem.build_system(m, p, q=q)
    x, y, z = sy.symbols("x y z")
    rng = np.random.default_rng(7 + p + 3 * q)

    def poly():
        return sum(sy.Rational(int(rng.integers(-9, 10)), 7) * x ** a * y ** b * z ** c
                   for a in range(p + 1) for b in range(p + 1 - a) for c in range(q + 1))
    u, v = poly(), poly()
    exact = float(sy.integrate(sy.expand(sum(sy.diff(u, w) * sy.diff(v, w) for w in (x, y, z))),
                               (x, 0, 2), (y, 0, 1), (z, -1, 0)))
    X = lev.xyz
    fu, fv = sy.lambdify((x, y, z), u, "numpy"), sy.lambdify((x, y, z), v, "numpy")
    U = fu(X[:, 0], X[:, 1], X[:, 2]) * np.ones(lev.n)
    V = fv(X[:, 0], X[:, 1], X[:, 2]) * np.ones(lev.n)
    assert abs(U @ (lev.A @ V) - exact) <= 1e-12 * max(1.0, abs(exact))


def test_anisotropic_node_count():
    """(nx p + 1)(ny p + 1)(nz q + 1) nodes on nx x ny quads (2 triangles each) x nz layers."""
    for p, q, (nx, ny, nz) in [(3, 1, (3, 2, 2)), (2, 4, (2, 2, 3)), (5, 3, (2, 1, 2))]:
        m = config1(p=p, nx=nx, ny=ny, nz=nz)
        lev = sem.build_level(m, p, q)
        assert lev.n == (nx * p + 1) * (ny * p + 1) * (nz * q + 1)
        assert lev.dirichlet.sum() == (nx * p + 1) * (ny * p + 1)


def test_semicoarsening_schedules():
    """Reading O19: coarsen the larger order first until the orders agree, then the
    isotropic rule: (5,3) -> (3,3) -> (2,2) -> (1,1); (4,2) -> (3,2) -> (2,2) -> (1,1);
    (2,4) -> (2,3) -> (2,2) -> (1,1)."""
    assert R.level_schedule_pq(5, 3) == [(5, 3), (3, 3), (2, 2), (1, 1)]
    assert R.level_schedule_pq(4, 2) == [(4, 2), (3, 2), (2, 2), (1, 1)]
    assert R.level_schedule_pq(2, 4) == [(2, 4), (2, 3), (2, 2), (1, 1)]


@pytest.mark.parametrize("chain", [[(5, 3), (3, 3), (1, 1)], [(4, 4), (4, 2), (2, 2), (1, 1)]])
def test_galerkin_consistency_semicoarsened(chain):
    """Nested anisotropic spaces + exact cubature on straight prisms: R A_f P = A_c
    between horizontally (5,3)->(3,3) and vertically (4,4)->(4,2) semi-coarsened
    levels (pins P and A of every pair together)."""
    m = _box(*chain[0])
    levs = [sem.build_system(m, p, q=q) for p, q in chain]
    for f, c in zip(levs[:-1], levs[1:]):
        P = pmg.prolongation(f, c)
        RAP = (P.T @ f.A @ P).toarray()
        np.testing.assert_allclose(RAP, c.A.toarray(), atol=1e-12 * np.abs(c.A).max())


def test_paper_schedule_pcg_on_curved_mesh():
    """Table 5.4's (5,3) -> (3,3) -> (1,1) p-MG on a curved channel (config 2
    construction with a (5,3) nodal map): symmetric V-cycle, PCG to the sparse
    direct solution."""
    from workloads import config2
    m = config2(p=5, nx=8, ny=2, nz=2)
    m.pz = 3
    mg = pmg.PMG(m, schedule=[(5, 3), (3, 3), (1, 1)])
    n = mg.levels[0].A.shape[0]
    rng = np.random.default_rng(2)
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    assert abs(x @ mg.vcycle(y) - y @ mg.vcycle(x)) <= 1e-12 * abs(x @ mg.vcycle(y))
    lev = mg.levels[0].level
    phiD = m.phi(*lev.xyz.T)
    A, b = sem.dirichlet_lift(lev, phiD)
    u, info = pmg.pcg(mg, b, rtol=1e-12)
    ref = sem.solve_direct(lev, phiD)[lev.free]
    assert np.linalg.norm(u - ref) <= 1e-9 * np.linalg.norm(ref) and info["iters"] < 30
