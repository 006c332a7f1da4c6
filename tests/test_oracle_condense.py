"""Pins of the oracle's static condensation (the
supplement's "Static Condensation", eq (laplacecondensed)
P:655-657, interior recovery P:663) against what the mathematics fixes:

* the interior node count of the prism lattice, (p-1)(p-2)/2 (q-1) per element;
* the Schur complement's variational characterisation: u_b^T S u_b is the energy
  of the energy-minimising extension (E(u_i* + d) - E(u_i*) = d^T A_ii d, which
  holds iff the extension is stationary), and S is symmetric;
* eigenvalue interlacing of an SPD Schur complement, lambda_min(A_FF) <=
  lambda(S) <= lambda_max(A_FF) (the supplement's "better conditioned");
* block elimination: the condensed solve is the full system's solution, which
  reproduces the closed-form harmonic phi of config 1 to discretisation error;
* no interior nodes (p = 2): S = A_FF."""
import numpy as np
import pytest

from oracle import condense, sem
from workloads import config1, random_vector


def _level(p, q=None, nx=2, ny=2, nz=2):
    m = config1(p=p, nx=nx, ny=ny, nz=nz)
    if q is not None:
        m.pz = q
    return m, sem.build_system(m, p, q=q)


@pytest.mark.parametrize("p,q", [(3, 3), (4, 4), (5, 3), (4, 2)])
def test_interior_count(p, q):
    m, lev = _level(p, q)
    ni = condense.interior_nodes(lev)
    assert len(ni) == lev.conn.shape[0] * (p - 1) * (p - 2) // 2 * (q - 1)
    assert not lev.dirichlet[ni].any()
    # every interior node belongs to exactly one element
    cnt = np.bincount(lev.conn.ravel(), minlength=lev.n)
    assert np.all(cnt[ni] == 1)


@pytest.mark.parametrize("p,q", [(4, 4), (5, 3)])
def test_schur_complement_is_the_minimal_energy(p, q):
    m, lev = _level(p, q)
    phiD = m.phi(*lev.xyz.T)
    S, g, (B, I, lu, Aib, bF) = condense.condensed_system(lev, phiD)
    AFF, _ = sem.dirichlet_lift(lev, phiD)
    A = AFF.toarray()
    Sd = S.toarray()
    assert np.abs(Sd - Sd.T).max() <= 1e-12 * np.abs(Sd).max()
    rng = np.random.default_rng(3)
    for t in range(3):
        ub = rng.standard_normal(len(B))
        ui = -lu.solve(Aib @ ub)
        x = np.zeros(A.shape[0])
        x[B], x[I] = ub, ui
        e0 = x @ A @ x
        assert abs(ub @ Sd @ ub - e0) <= 1e-11 * abs(e0)
        d = rng.standard_normal(len(I))
        y = x.copy()
        y[I] += d
        dAd = d @ A[np.ix_(I, I)] @ d
        assert abs((y @ A @ y - e0) - dAd) <= 1e-10 * (abs(e0) + dAd)


def test_schur_spectrum_interlaces():
    m, lev = _level(4)
    phiD = m.phi(*lev.xyz.T)
    S, _, _ = condense.condensed_system(lev, phiD)
    AFF, _ = sem.dirichlet_lift(lev, phiD)
    la = np.linalg.eigvalsh(AFF.toarray())
    ls = np.linalg.eigvalsh(S.toarray())
    assert ls[0] > 0
    assert la[0] * (1 - 1e-10) <= ls[0] and ls[-1] <= la[-1] * (1 + 1e-10)
    assert ls[-1] / ls[0] <= la[-1] / la[0]


@pytest.mark.parametrize("p,q", [(4, 4), (5, 3), (6, 6)])
def test_condensed_solve_is_the_full_solution(p, q):
    m, lev = _level(p, q, nx=3, ny=2, nz=2)
    phiD = m.phi(*lev.xyz.T)
    rhs = random_vector(lev.n, seed=p)
    for b in (None, rhs):
        phi_c, _ = condense.solve_condensed(lev, phiD, b)
        phi_f = sem.solve_direct(lev, phiD, b)
        assert np.abs(phi_c - phi_f).max() <= 1e-11 * np.abs(phi_f).max()
    # the closed form of config 1 (harmonic, exact Neumann data) to discretisation error
    phi_c, _ = condense.solve_condensed(lev, phiD)
    assert np.abs(phi_c - phiD).max() <= 5e-2 * np.abs(phiD).max()


def test_no_interior_nodes_leaves_the_system():
    m, lev = _level(2)
    phiD = m.phi(*lev.xyz.T)
    S, g, (B, I, *_ ) = condense.condensed_system(lev, phiD)
    AFF, bF = sem.dirichlet_lift(lev, phiD)
    assert len(I) == 0 and abs(S - AFF).max() == 0 and np.array_equal(g, bF)
