"""Deterministic mode (sem_opts.deterministic; S:240, S:346 require a race-free,
deterministic summation order): repeated solves are bit-identical (solution and
residual history), and the deterministic solve still reaches the oracle's
sparse-direct solution."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import sem  # noqa: E402
from tests._mapping import lib_to_oracle  # noqa: E402
from tests.test_gpu_parity import SOLVE_TOL, make_solver, rel  # noqa: E402
from workloads import config2, random_vector  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def _twice(s, phiD, tol=1e-12):
    a, ra = s.solve(phiD, tol)
    b, rb = s.solve(phiD, tol)
    return a.cpu().numpy(), ra, b.cpu().numpy(), rb


CASES = {
    "dense": dict(),                                        # exact dense Schwarz, dense coarse inverse
    "fdm_iterative_coarse": dict(local_solve=1, coarse_solver=1, coarse_rtol=1e-12),
}


@pytest.mark.parametrize("case", list(CASES))
def test_deterministic_solves_are_bit_identical(case):
    m = config2(p=4, nx=32, ny=2, nz=3)
    s = make_solver(m, deterministic=1, **CASES[case])
    lev = sem.build_system(m, m.p)
    perm = lib_to_oracle(s.node_xyz(0), lev.xyz)
    phiD_o = m.phi(*lev.xyz.T)
    phiD = torch.from_numpy(np.ascontiguousarray(phiD_o[perm])).cuda()
    a, ra, b, rb = _twice(s, phiD)
    assert ra["converged"] and rb["converged"]
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert ra["res_hist"] == rb["res_hist"]
    out = np.zeros(lev.n)
    out[perm] = a
    assert rel(out, sem.solve_direct(lev, phiD_o)) <= SOLVE_TOL
    # the operator and the V-cycle alone
    u = torch.from_numpy(random_vector(s.n_dof(0), 3)).cuda()
    assert torch.equal(s.apply(u), s.apply(u))
    dm = torch.from_numpy(s.dirichlet_mask(0)).cuda()
    u[dm] = 0
    assert torch.equal(s.vcycle(u), s.vcycle(u))
    s.close()


def test_deterministic_hybrid_hull_replica():
    """Config-5 construction (FDM / exact-dense hybrid, reading O35): bit-identical
    repeated solves, equal to the default (atomic) mode's solution to rounding."""
    from workloads.config5 import config5
    m = config5(p=3, hf=0.5, Lx=16.0, Ly=10.0)
    s = make_solver(m, local_solve=1, deterministic=1)
    s0 = make_solver(m, local_solve=1)
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    a, ra, b, rb = _twice(s, phiD)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64)) and ra["res_hist"] == rb["res_hist"]
    c, _ = s0.solve(phiD, 1e-12)
    assert rel(a, c.cpu().numpy()) <= 1e-10
    s.close()
    s0.close()
