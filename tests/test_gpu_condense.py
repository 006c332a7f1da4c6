"""Static condensation on the GPU (the supplement's
"Static Condensation"; reading O43) through the C ABI
(laplace_solve_condensed), against the oracle (oracle/condense.py, pinned by
tests/test_oracle_condense.py): the condensed solution (skeleton solve + interior
recovery) equals the oracle's, for isotropic and (P_xy, P_z) spaces,
both local solves, PCG and PDC outer iterations, warm starts, a geometry update,
deterministic mode, and the degenerate order without interior nodes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2009_00705_b200 as lib  # noqa: E402
from oracle import condense, sem  # noqa: E402
from tests._mapping import lib_to_oracle  # noqa: E402
from tests.test_gpu_parity import SOLVE_TOL, rel  # noqa: E402
from workloads import config2, random_vector  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def _solver(m, **kw):
    return lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p, m.pz)),
                      pz=m.pz, **kw)


def _case(p, q=None, nx=16, **kw):
    m = config2(p=p, nx=nx, ny=2, nz=3)
    m.pz = p if q is None else q
    s = _solver(m, **kw)
    lev = sem.build_system(m, p, q=q)
    perm = lib_to_oracle(s.node_xyz(0), lev.xyz)
    return m, s, lev, perm


def _to_lib(v, perm):
    return torch.from_numpy(np.ascontiguousarray(v[perm])).cuda()


def _to_orc(t, perm, n):
    out = np.zeros(n)
    out[perm] = t.cpu().numpy()
    return out


@pytest.mark.parametrize("p,q,kw", [
    (4, None, {}),
    (5, None, dict(local_solve=1)),
    (5, 3, {}),
    (6, None, dict(outer=1)),
])
def test_condensed_solve_parity(p, q, kw):
    m, s, lev, perm = _case(p, q, nx=8 if p >= 6 else 16, **kw)
    ni, nb, by = s.condensed_info()
    qq = p if q is None else q
    assert ni == (p - 1) * (p - 2) // 2 * (qq - 1) and ni + nb == lev.conn.shape[1]
    assert by == len(m.prisms) * ni * (ni + nb) * 8
    phiD = m.phi(*lev.xyz.T)
    rhs = random_vector(lev.n, seed=7) * 1e-2
    for b in (None, rhs):
        want, _ = condense.solve_condensed(lev, phiD, b)
        phi, rep = s.solve_condensed(_to_lib(phiD, perm), 1e-13, rhs=None if b is None else _to_lib(b, perm))
        assert rep["converged"]
        assert rel(_to_orc(phi, perm, lev.n), want) <= SOLVE_TOL
    # the residual is the full system's: every free row, interior rows included
    lv = torch.from_numpy(lev.dirichlet[perm].astype(np.uint8)).cuda().bool()
    y = s.apply(phi, masked=False)
    r = (_to_lib(rhs, perm) - y)[~lv]
    assert (r.norm() / _to_lib(rhs, perm)[~lv].norm()).item() <= 1e-8
    s.close()


def test_condensed_iterations_against_the_full_system():
    """The condensed PCG (skeleton block of the same V-cycle, "better conditioned")
    converges in no more outer iterations than the full-system PCG."""
    m, s, lev, perm = _case(5, nx=24)
    phiD = _to_lib(m.phi(*lev.xyz.T), perm)
    _, full = s.solve(phiD, tol=1e-10)
    _, cond = s.solve_condensed(phiD, 1e-10)
    assert cond["converged"] and cond["iters"] <= full["iters"]
    s.close()


def test_condensed_warm_start_and_geometry_update():
    m, s, lev, perm = _case(5)
    phiD = _to_lib(m.phi(*lev.xyz.T), perm)
    phi, rep = s.solve_condensed(phiD, 1e-12)
    phi2, rep2 = s.solve_condensed(phiD, 1e-10, out=phi.clone(), guess=True)
    assert rep2["converged"] and rep2["iters"] == 0
    # next stage: the interior factors follow the new geometry
    m1 = config2(p=5, nx=16, ny=2, nz=3)
    m1.pz = 5
    eta0 = m1.eta
    m1.eta = lambda x, y: 1.1 * eta0(x, y) + 0.004 * np.cos(0.5 * np.asarray(x))
    s.update_geometry(m1.node_xyz(lib.reference_nodes(5)), strategy=2)
    lev1 = sem.build_system(m1, 5)
    perm1 = lib_to_oracle(s.node_xyz(0), lev1.xyz)
    phiD1 = m1.phi(*lev1.xyz.T)
    phi3, rep3 = s.solve_condensed(_to_lib(phiD1, perm1), 1e-13, out=phi.clone(), guess=True)
    assert rep3["converged"] and 0 < rep3["iters"] < rep["iters"] + 2
    assert rel(_to_orc(phi3, perm1, lev1.n), sem.solve_direct(lev1, phiD1)) <= SOLVE_TOL
    s.close()


def test_condensed_deterministic_bit_identical():
    m, s, lev, perm = _case(4, deterministic=1)
    phiD = _to_lib(m.phi(*lev.xyz.T), perm)
    a, ra = s.solve_condensed(phiD, 1e-12)
    b, rb = s.solve_condensed(phiD, 1e-12)
    assert ra["iters"] == rb["iters"] and torch.equal(a, b)
    s.close()


def test_condensed_without_interior_nodes_is_the_plain_solve():
    m, s, lev, perm = _case(2)
    ni, nb, by = s.condensed_info()
    assert ni == 0 and by == 0
    phiD = _to_lib(m.phi(*lev.xyz.T), perm)
    a, ra = s.solve(phiD, tol=1e-12)
    b, rb = s.solve_condensed(phiD, 1e-12)
    assert ra["iters"] == rb["iters"] and rel(b.cpu().numpy(), a.cpu().numpy()) <= 1e-14
    s.close()
