"""SURVEY NEXT-1 (the paper's per-stage solves): a new free surface
for the next time stage through sem_update_geometry (strategy I: only the
finest operator follows it; smoothers and coarse-level operators stay those of
t = 0; strategy 2: every level's operator follows it), then a warm-started
solve (laplace_solve_guess) from the previous stage's solution.  The solution
must be the new geometry's discrete solution (oracle sparse direct), reached in
fewer PCG iterations than a cold solve."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2009_00705_b200 as lib  # noqa: E402
from oracle import sem  # noqa: E402
from tests._mapping import lib_to_oracle  # noqa: E402
from tests.test_gpu_parity import make_solver, rel, SOLVE_TOL  # noqa: E402
from workloads import config2, random_vector  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def _meshes():
    m0 = config2(p=4, nx=32, ny=2, nz=3)
    m1 = config2(p=4, nx=32, ny=2, nz=3)
    eta0 = m0.eta
    m1.eta = lambda x, y: 1.1 * eta0(x, y) + 0.004 * np.cos(0.5 * np.asarray(x))   # the next stage's surface
    return m0, m1


@pytest.mark.parametrize("local_solve", [0, 1])
@pytest.mark.parametrize("strategy", [1, 2])
def test_update_geometry_and_warm_start(strategy, local_solve):
    m0, m1 = _meshes()
    s = make_solver(m0, local_solve=local_solve)
    xyz0 = s.node_xyz(0)
    phi0, rep0 = s.solve(torch.from_numpy(m0.phi(*xyz0.T)).cuda(), tol=1e-13)
    # next stage
    s.update_geometry(m1.node_xyz(lib.reference_nodes(m1.p)), strategy=strategy)
    lev = sem.build_system(m1, m1.p)
    perm = lib_to_oracle(s.node_xyz(0), lev.xyz)              # coordinates follow the new surface
    # the finest operator is the new geometry's
    u = random_vector(lev.n, seed=4)
    y = s.apply(torch.from_numpy(np.ascontiguousarray(u[perm])).cuda())
    yo = np.zeros(lev.n)
    yo[perm] = y.cpu().numpy()
    assert rel(yo, lev.A @ u) <= 1e-12
    phiD = m1.phi(*lev.xyz.T)
    phiD_lib = torch.from_numpy(np.ascontiguousarray(phiD[perm])).cuda()
    cold, rep_c = s.solve(phiD_lib, tol=1e-13)
    phi = phi0.clone()
    phi, rep_w = s.solve_guess(phiD_lib, 1e-13, phi)
    got = np.zeros(lev.n)
    got[perm] = phi.cpu().numpy()
    assert rep_w["converged"] and rel(got, sem.solve_direct(lev, phiD)) <= SOLVE_TOL
    assert rep_w["iters"] < rep_c["iters"]
    s.close()


def test_warm_start_from_the_solution_needs_no_iteration():
    m0, _ = _meshes()
    s = make_solver(m0)
    phiD = torch.from_numpy(m0.phi(*s.node_xyz(0).T)).cuda()
    phi, rep = s.solve(phiD, tol=1e-12)
    phi2, rep2 = s.solve_guess(phiD, 1e-10, phi.clone())
    assert rep2["converged"] and rep2["iters"] == 0
    s.close()


def test_strategy_III_reforms_smoothers_like_a_fresh_setup():
    """Strategy III (4, reading O42): after sem_update_geometry every
    level's operator AND FDM smoother (vertical factors re-formed on the device) and
    the coarse line-Jacobi preconditioner equal those of a ctx set up from scratch
    on the new geometry: the Schwarz correction of every smoothed level and the
    V-cycle agree to 1e-12, and the warm-started solve reaches the new geometry's
    direct solution."""
    m0, m1 = _meshes()
    kw = dict(local_solve=1, coarse_solver=1, coarse_rtol=1e-13)
    s = make_solver(m0, **kw)
    fresh = make_solver(m1, **kw)
    s.update_geometry(m1.node_xyz(lib.reference_nodes(m1.p)), strategy=4)
    for li in range(s.info["n_levels"] - 1):
        r = torch.from_numpy(random_vector(s.n_dof(li), 50 + li)).cuda()
        for tr in (False, True):
            a, b = s.empty(li), fresh.empty(li)
            s.schwarz(li, r, a, transpose=tr)
            fresh.schwarz(li, r, b, transpose=tr)
            assert rel(a.cpu().numpy(), b.cpu().numpy()) <= 1e-12
    dm = torch.from_numpy(s.dirichlet_mask(0)).cuda()
    x = torch.from_numpy(random_vector(s.n_dof(0), 61)).cuda()
    x[dm] = 0
    assert rel(s.vcycle(x).cpu().numpy(), fresh.vcycle(x).cpu().numpy()) <= 1e-10
    lev = sem.build_system(m1, m1.p)
    perm = lib_to_oracle(s.node_xyz(0), lev.xyz)
    phiD = m1.phi(*lev.xyz.T)
    phi, rep = s.solve(torch.from_numpy(np.ascontiguousarray(phiD[perm])).cuda(), tol=1e-13)
    got = np.zeros(lev.n)
    got[perm] = phi.cpu().numpy()
    assert rep["converged"] and rel(got, sem.solve_direct(lev, phiD)) <= SOLVE_TOL
    s.close()
    fresh.close()
