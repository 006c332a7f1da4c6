"""Edge cases of the hot path through the C ABI, against the oracle.

* The smallest meshes: one column pair (2 triangles) of 1 or 3 layers, every
  element touching the boundary, at p = 1 (single level, O26), 2, 3 and 5 —
  one ragged tile in every kernel (fewer elements than warps, fewer coarse
  DOF than one 64-row tile).
* Degenerate data: zero Dirichlet data and zero load give phi = 0 after no
  iteration; the apply of 0 is exactly 0 (no stale accumulators).
* The largest order the library takes (p = 8) on a one-column mesh.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import sem  # noqa: E402
from tests.test_gpu_parity import APPLY_TOL, SOLVE_TOL, Case, make_solver, rel  # noqa: E402
from workloads import config1, random_vector  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

TINY = [(1, 1), (2, 1), (3, 3), (5, 1), (5, 3)]   # (p, layers) on nx = ny = 1


@pytest.mark.parametrize("p,nz", TINY)
def test_tiny_mesh_apply_and_solve(p, nz):
    m = config1(p=p, nx=1, ny=1, nz=nz)
    C = Case(m)
    lev, _ = C.levels[0]
    u = random_vector(lev.n, seed=3)
    y = C.s.apply(C.to_lib(0, u), masked=False)
    assert rel(C.to_orc(0, y), lev.A @ u) <= APPLY_TOL
    phiD = m.phi(*lev.xyz.T)
    phi, rep = C.s.solve(C.to_lib(0, phiD), tol=1e-13)
    assert rep["converged"]
    ref = sem.solve_direct(lev, phiD)
    assert rel(C.to_orc(0, phi), ref) <= SOLVE_TOL
    C.s.close()


def test_zero_data_and_zero_apply():
    m = config1(p=3, nx=2, ny=2, nz=2)
    s = make_solver(m)
    n = s.n_dof(0)
    zero = torch.zeros(n, dtype=torch.float64, device="cuda")
    y = s.apply(zero, masked=False)
    assert torch.count_nonzero(y).item() == 0
    phi, rep = s.solve(zero, tol=1e-12, check=False)
    assert rep["converged"] and rep["iters"] == 0
    assert torch.count_nonzero(phi).item() == 0
    s.close()


def test_highest_order_one_column():
    m = config1(p=8, nx=1, ny=1, nz=2)
    C = Case(m, build_mg=False)
    lev, _ = C.levels[0]
    u = random_vector(lev.n, seed=8)
    assert rel(C.to_orc(0, C.s.apply(C.to_lib(0, u), masked=False)), lev.A @ u) <= APPLY_TOL
    phiD = m.phi(*lev.xyz.T)
    phi, rep = C.s.solve(C.to_lib(0, phiD), tol=1e-13)
    assert rep["converged"]
    assert rel(C.to_orc(0, phi), sem.solve_direct(lev, phiD)) <= SOLVE_TOL
    C.s.close()
