"""Pins of the oracle p-multigrid against special cases, closed forms
and invariants (DESIGN.md §"Oracle pins")."""
import numpy as np
import pytest
from scipy.sparse.linalg import spsolve

from oracle import refelem as R
from oracle import pmg, sem
from workloads import config1, config2, structured_basin


def test_prolongation_reproduces_coarse_polynomials():
    """P_{p-1}^p interpolates nested spaces: a degree-p_c polynomial
    sampled at coarse nodes maps to its values at fine nodes; P 1 = 1."""
    m = config2(p=5, nx=3, ny=2, nz=2)
    for pf, pc in [(5, 3), (3, 2), (2, 1)]:
        f, c = sem.build_level(m, pf), sem.build_level(m, pc)
        P = pmg.prolongation(f, c)
        fn = lambda X: 1 + X[:, 0] ** pc - 0.5 * X[:, 1] * X[:, 0] ** (pc - 1) + X[:, 0] * 0.3
        # x,y affine per element, so polynomials in x,y of degree pc are in V^pc
        np.testing.assert_allclose(P @ fn(c.xyz), fn(f.xyz), atol=1e-12)
        np.testing.assert_allclose(P @ np.ones(c.n), 1.0, atol=1e-13)


def test_galerkin_consistency_straight():
    """Nested spaces + exact cubature on straight prisms: R A_f P = A_c with R = P^T
    (eq 4.3).  Pins A on every level and P together (config 1)."""
    m = config1(p=5, nx=2, ny=2, nz=2)
    levs = [sem.build_system(m, q, p_geo=5) for q in (5, 3, 2, 1)]
    for f, c in zip(levs[:-1], levs[1:]):
        P = pmg.prolongation(f, c)
        RAP = (P.T @ f.A @ P).toarray()
        Ac = c.A.toarray()
        np.testing.assert_allclose(RAP, Ac, atol=1e-12 * np.abs(Ac).max())


def test_schwarz_subdomain_size_interior():
    """O15 on an interior element of a valence-6 lattice: n_k = (Nt + 3(p+2))(p+3)
    for overlap 1 and Nt(p+1) for overlap 0."""
    for p in (2, 3):
        m = config1(p=p, nx=4, ny=4, nz=3)
        lev = sem.build_level(m, p)
        # element: lower triangle of quad (1,1), middle layer
        tri_id = 2 * (1 * 4 + 1)
        e = tri_id * 3 + 1
        Nt = (p + 1) * (p + 2) // 2
        s1 = pmg.schwarz_sets(lev, 1)[e]
        s0 = pmg.schwarz_sets(lev, 0)[e]
        assert len(s0) == Nt * (p + 1)
        assert len(s1) == (Nt + 3 * (p + 2)) * (p + 3)


def test_block_jacobi_single_element_is_exact():
    """one element, overlap 0 -> S^{-1} = A_FF^{-1} (W = 1)."""
    m = config2(p=3, nx=1, ny=1, nz=1)
    m.prisms, m.face_tag = m.prisms[:1], m.face_tag[:1]      # a single curved prism
    lev = sem.build_system(m, 3)
    F = lev.free
    AFF = lev.A[F][:, F].tocsr()
    sm = pmg.build_smoother(lev, AFF, overlap=0)
    r = np.random.default_rng(1).uniform(-1, 1, len(F))
    assert len(sm.sets) == 1 and len(sm.sets[0]) == len(F)
    np.testing.assert_allclose(sm.W, 1.0)
    np.testing.assert_allclose(sm.apply(r), spsolve(AFF.tocsc(), r), rtol=1e-10)
    np.testing.assert_allclose(sm.apply(r, transpose=True), spsolve(AFF.tocsc(), r), rtol=1e-10)


def test_weights_count_subdomains():
    """eq 4.6: W = (sum_k R_k R_k^T)^{-1} is the inverse subdomain count."""
    m = config1(p=2, nx=3, ny=2, nz=2)
    lev = sem.build_system(m, 2)
    F = lev.free
    sm = pmg.build_smoother(lev, lev.A[F][:, F].tocsr(), overlap=1)
    cnt = np.zeros(len(F))
    for s in sm.sets:
        for i in s:
            cnt[i] += 1
    np.testing.assert_array_equal(sm.W, 1.0 / cnt)


@pytest.fixture(scope="module")
def mg_c1():
    return config1(), pmg.PMG(config1())


def test_vcycle_symmetric_positive(mg_c1):
    """Reading O14: with post-smoothing S^{-T}, nu1 = nu2, R = P^T and an exact
    coarse solve the V-cycle is a symmetric positive definite operator."""
    _, mg = mg_c1
    n = mg.levels[0].A.shape[0]
    rng = np.random.default_rng(3)
    V = np.stack([mg.vcycle(e) for e in np.eye(n)[:: max(1, n // 60)]], 1)
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    vx, vy = mg.vcycle(x), mg.vcycle(y)
    assert abs(x @ vy - y @ vx) <= 1e-13 * abs(x @ vy)
    assert x @ vx > 0 and y @ vy > 0
    assert V.shape[1] > 0


def test_vcycle_literal_smoother_is_not_symmetric():
    """P:313 literally (W left-applied pre and post) gives a non-symmetric V-cycle
    when W is not constant (why reading O14 exists)."""
    m = config1(p=2, nx=3, ny=2, nz=2)
    mg = pmg.PMG(m, literal=True)
    n = mg.levels[0].A.shape[0]
    rng = np.random.default_rng(4)
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    assert abs(x @ mg.vcycle(y) - y @ mg.vcycle(x)) > 1e-8 * abs(x @ mg.vcycle(y))


def test_single_level_is_direct_solve():
    """S:327 / O26: a hierarchy with only P=1 is the exact coarse solve."""
    m = config1(p=1)
    mg = pmg.PMG(m)
    A = mg.levels[0].A
    f = np.random.default_rng(5).uniform(-1, 1, A.shape[0])
    np.testing.assert_allclose(A @ mg.vcycle(f), f, atol=1e-12)


def test_vcycle_zero_in_zero_out(mg_c1):
    """V(0) = 0; linear: V(2f) = 2 V(f)."""
    _, mg = mg_c1
    n = mg.levels[0].A.shape[0]
    assert np.abs(mg.vcycle(np.zeros(n))).max() == 0.0
    f = np.random.default_rng(6).uniform(-1, 1, n)
    np.testing.assert_allclose(mg.vcycle(2 * f), 2 * mg.vcycle(f), rtol=1e-13)


@pytest.mark.parametrize("method", ["pcg", "pdc"])
def test_solvers_reach_direct_solution(mg_c1, method):
    """Alg 4.2/4.3 solved to rtol 1e-13 agree with the sparse direct solve to
    1e-10 (north_star parity bar) and contract: q < 0.15 per iteration."""
    m, mg = mg_c1
    lev = mg.levels[0].level
    phiD = m.phi(*lev.xyz.T)
    A, b = sem.dirichlet_lift(lev, phiD)
    u_direct = spsolve(A, b)
    fn = pmg.pcg if method == "pcg" else pmg.pdc
    u, info = fn(mg, b, rtol=1e-13)
    assert np.linalg.norm(u - u_direct) <= 1e-10 * np.linalg.norm(u_direct)
    res = np.array(info["res"])
    q = res[1:] / res[:-1]
    assert np.all(q[:-1] < 0.15), q


def test_overlap_improves_contraction():
    """P:320 / S:332-335: one overlapping node improves on block Jacobi (overlap 0)
    and the refined overlap ceil((P+1)/2) improves further: the spectral
    radius of the V-cycle error propagator I - V A decreases with the overlap."""
    m = config2(p=4, nx=6, ny=2, nz=2)
    rho = []
    for ov in (0, 1, -1):
        mg = pmg.PMG(m, overlap=ov)
        A = mg.levels[0].A
        n = A.shape[0]
        rng = np.random.default_rng(0)
        x = rng.standard_normal(n)
        for _ in range(60):          # power iteration on e <- e - V(A e)
            x = x - mg.vcycle(A @ x)
            nx_ = np.linalg.norm(x)
            x /= nx_
        rho.append(nx_)
    assert rho[0] > rho[1] > rho[2], rho
    assert rho[1] < 0.2


def test_smoother_matches_dense_formula_eq44():
    """eq 4.4 written out densely: S^{-1} = W sum_k R_k^T (R_k A R_k^T)^{-1} R_k
    with explicit 0/1 restriction matrices on a two-prism mesh (overlap 0: R_k picks
    element k's free nodes, read off its connectivity), W = (sum_k R_k R_k^T)^{-1}
    non-constant (1/2 on the shared face).  Smoother.apply must be W on the LEFT
    for S^{-1} and on the RIGHT for S^{-T} (reading O14); swapping them fails,
    since the dense S^{-1} is not symmetric here."""
    m = config1(p=2, nx=1, ny=1, nz=1)             # one quad -> 2 triangles x 1 layer = 2 prisms
    lev = sem.build_system(m, 2)
    F = lev.free
    nF = len(F)
    fid = -np.ones(lev.n, dtype=np.int64)
    fid[F] = np.arange(nF)
    AFF = lev.A[F][:, F].toarray()
    Rk = []
    for e in range(lev.conn.shape[0]):
        nodes = sorted({int(fid[g]) for g in lev.conn[e] if fid[g] >= 0})
        R_ = np.zeros((len(nodes), nF))
        R_[np.arange(len(nodes)), nodes] = 1.0
        Rk.append(R_)
    W = np.diag(1.0 / sum(R_.T @ R_ for R_ in Rk).diagonal())
    assert len(set(np.round(W.diagonal(), 12))) == 2     # 1 and 1/2: non-constant
    Ssum = sum(R_.T @ np.linalg.inv(R_ @ AFF @ R_.T) @ R_ for R_ in Rk)
    S_inv = W @ Ssum
    assert np.linalg.norm(S_inv - S_inv.T) > 1e-3 * np.linalg.norm(S_inv)
    sm = pmg.build_smoother(lev, lev.A[F][:, F].tocsr(), overlap=0)
    r = np.random.default_rng(12).uniform(-1, 1, nF)
    np.testing.assert_allclose(sm.apply(r), S_inv @ r, rtol=1e-12, atol=1e-12 * np.abs(S_inv @ r).max())
    np.testing.assert_allclose(sm.apply(r, transpose=True), S_inv.T @ r, rtol=1e-12,
                               atol=1e-12 * np.abs(S_inv.T @ r).max())
