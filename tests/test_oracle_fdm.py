"""Pins of the oracle FDM local solves (reading O33, oracle/fdm.py) against
closed forms, the exact dense smoother where the separable form is exact
(straight prisms with flat layers), and invariants."""
import numpy as np
import pytest

from oracle import fdm, pmg, sem
from workloads import config1, config2
from workloads.configs import basin


def _basin_small(p=3):
    return basin("fdm_small", p, 32.0 * 4 / 64, 4, 3, seed=3)     # jittered, curved, 3 layers


def test_2d_operators_closed_forms():
    """Footprint operators of a jittered mesh: 1^T M 1 = area, K 1 = 0,
    x^T K x = y^T K y = area, x^T K y = 0, 1^T M x = int x (exact: M is exact to
    degree 2p on affine triangles)."""
    m = _basin_small(3)
    lev = sem.build_level(m, 3)
    cols = fdm.Columns(m, lev)
    L = m.meta["Lx"]
    x, y = cols.xy[:, 0], cols.xy[:, 1]
    one = np.ones_like(x)
    area = L * L
    assert abs(one @ cols.M2 @ one - area) < 1e-12 * area
    assert np.abs(cols.K2 @ one).max() < 1e-12
    assert abs(x @ cols.K2 @ x - area) < 1e-12 * area
    assert abs(y @ cols.K2 @ y - area) < 1e-12 * area
    assert abs(x @ cols.K2 @ y) < 1e-12 * area
    assert abs(one @ cols.M2 @ x - L ** 3 / 2) < 1e-12 * L ** 3
    assert abs(x @ cols.M2 @ x - L ** 4 / 3) < 1e-12 * L ** 4


def test_1d_operators_closed_forms():
    """Column operators: 1^T M_v 1 = sum d_j, K_v 1 = 0, z^T K_v z = sum d_j,
    1^T M_v z = (b^2 - a^2)/2 for the column's mapped GLL coordinates z."""
    from oracle import refelem as R
    m = _basin_small(4)
    lev = sem.build_level(m, 4)
    cols = fdm.Columns(m, lev)
    t = R.lgl(4)[0]
    for c in (0, 5, len(cols.col_elems) - 1):
        Kv, Mv = cols.column_line_matrices(c)
        el = cols.col_elems[c]
        d = cols.d[el]
        z = np.zeros(Kv.shape[0])
        z0 = -1.0
        for j, dj in enumerate(d):
            z[4 * j: 4 * j + 5] = z0 + (1 + t) / 2 * dj
            z0 += dj
        one = np.ones_like(z)
        H = d.sum()
        assert abs(one @ Mv @ one - H) < 1e-13
        assert np.abs(Kv @ one).max() < 1e-12
        assert abs(z @ Kv @ z - H) < 1e-12
        assert abs(one @ Mv @ z - (z[-1] ** 2 - z[0] ** 2) / 2) < 1e-13


@pytest.mark.parametrize("overlap", [0, 1, 2])
def test_fdm_sets_equal_dense_sets(overlap):
    """On layered meshes the subdomain of reading O15 is the product H_k x V_k:
    the FDM node sets equal the dense smoother's sets (curved, jittered mesh)."""
    m = _basin_small(3)
    lev = sem.build_level(m, 3)
    dense = pmg.schwarz_sets(lev, overlap)
    for k, (ids, _) in enumerate(fdm.fdm_blocks(m, lev, overlap)):
        np.testing.assert_array_equal(np.sort(ids), dense[k])


@pytest.mark.parametrize("p,overlap", [(3, 1), (2, 2), (3, 0)])
def test_fdm_is_exact_on_straight_flat_prisms(p, overlap):
    """Config 1 (straight prisms, flat layers): A = K_h (x) M_v + M_h (x) K_v, so
    the FDM local inverse equals the exact (R_k A R_k^T)^{-1} of eq 4.4."""
    m = config1(p=p, nx=3, ny=2, nz=3)
    lev = sem.build_system(m, p)
    F = lev.free
    AFF = lev.A[F][:, F].tocsr()
    dense = pmg.build_smoother(lev, AFF, overlap)
    fsm = pmg.build_fdm_smoother(m, lev, overlap)
    np.testing.assert_allclose(fsm.W, dense.W, rtol=0, atol=0)
    for I, Bi, J, Bj in zip(dense.sets, dense.inv, fsm.sets, fsm.inv):
        o = np.argsort(J)
        np.testing.assert_array_equal(J[o], I)
        np.testing.assert_allclose(Bj[np.ix_(o, o)], Bi, atol=1e-12 * np.abs(Bi).max())


@pytest.mark.parametrize("p,q,overlap", [(3, 2, 1), (4, 2, 1), (2, 3, 1), (3, 1, 0)])
def test_fdm_is_exact_on_straight_flat_prisms_anisotropic(p, q, overlap):
    """The same identity on P_p(triangle) x P_q(t) prisms: with straight prisms and
    flat layers A = K_h(p) (x) M_v(q) + M_h(p) (x) K_v(q), so the FDM local inverse built from the
    order-q vertical operators equals the exact inverse of the O15 block of eq 4.4 (a dropped or
    misplaced q -- the order-p vertical rule, layer index z / p -- breaks either the sets or the
    inverses)."""
    m = config1(p=p, nx=3, ny=2, nz=3)
    m.pz = q
    lev = sem.build_system(m, p, q=q)
    F = lev.free
    AFF = lev.A[F][:, F].tocsr()
    dense = pmg.build_smoother(lev, AFF, overlap)
    fsm = pmg.build_fdm_smoother(m, lev, overlap)
    np.testing.assert_allclose(fsm.W, dense.W, rtol=0, atol=0)
    for I, Bi, J, Bj in zip(dense.sets, dense.inv, fsm.sets, fsm.inv):
        o = np.argsort(J)
        np.testing.assert_array_equal(J[o], I)
        np.testing.assert_allclose(Bj[np.ix_(o, o)], Bi, atol=1e-12 * np.abs(Bi).max())


def test_fdm_is_not_exact_on_curved_prisms():
    """Sanity of the pin above: on curved prisms the separable form is only an
    approximation (the pin would be vacuous if the two always agreed)."""
    m = config2(p=3, nx=4, ny=1, nz=2)
    lev = sem.build_system(m, 3)
    F = lev.free
    AFF = lev.A[F][:, F].tocsr()
    dense = pmg.build_smoother(lev, AFF, 1)
    fsm = pmg.build_fdm_smoother(m, lev, 1)
    k = 3
    o = np.argsort(fsm.sets[k])
    d = np.abs(fsm.inv[k][np.ix_(o, o)] - dense.inv[k]).max() / np.abs(dense.inv[k]).max()
    assert 1e-6 < d < 0.5


def test_fdm_vcycle_symmetric_and_pcg_reaches_direct_solution():
    """With FDM local solves the V-cycle stays symmetric positive definite
    (reading O14 post-smoothing), and PCG (Alg 4.3) reaches the direct solution."""
    m = config2(p=4, nx=6, ny=2, nz=2)
    mg = pmg.PMG(m, local_solve="fdm")
    n = mg.levels[0].A.shape[0]
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    vx, vy = mg.vcycle(x), mg.vcycle(y)
    assert abs(x @ vy - vx @ y) < 1e-12 * np.linalg.norm(x) * np.linalg.norm(vy)
    assert x @ vx > 0
    lev = mg.levels[0].level
    phiD = m.phi(*lev.xyz.T)
    A, b = sem.dirichlet_lift(lev, phiD)
    u, info = pmg.pcg(mg, b, rtol=1e-13)
    ref = sem.solve_direct(lev, phiD)[lev.free]
    assert np.linalg.norm(u - ref) <= 1e-10 * np.linalg.norm(ref)
    assert info["iters"] < 30
