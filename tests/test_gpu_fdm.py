"""GPU parity of the FDM local solves (opts.local_solve = 1, reading O33) against
the oracle's FDM smoother (oracle/fdm.py: Kronecker box inverted by
numpy.linalg.inv), element by element through the C ABI; V-cycle and solve
parity; the FDM smoother equals the exact dense one on straight flat prisms."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pmg, sem  # noqa: E402
from tests.test_gpu_parity import Case, SOLVE_TOL, STEP_TOL, rel  # noqa: E402
from workloads import config1, config2, random_vector  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def _c3_small():
    from workloads.configs import basin
    return basin("config3_small", 5, 32.0 * 5 / 64, 5, 3, seed=3)


CASES = {
    "c1": lambda: (config1(), 1),
    "c2": lambda: (config2(p=4, nx=32, ny=2, nz=3), 1),
    "c3s": lambda: (_c3_small(), 1),
    "c3s_refined": lambda: (_c3_small(), -1),       # overlap ceil((P+1)/2) per level
    "c2_o0": lambda: (config2(p=4, nx=32, ny=2, nz=3), 0),
    "c5r": lambda: (_c5_replica(), 1),            # hull: FDM / exact-dense hybrid (reading O35)
    "c2p6": lambda: (config2(p=6, nx=24, ny=2, nz=2), 1),   # n_v = 9: two n-tiles per box
}


def _c5_replica():
    from workloads.config5 import config5
    return config5(p=3, hf=0.5, Lx=16.0, Ly=10.0)


@pytest.fixture(scope="module", params=list(CASES))
def case(request):
    m, ov = CASES[request.param]()
    return Case(m, local_solve=1, overlap=ov)


def test_fdm_smoother_parity(case):
    """u += S^-1 r and u += S^-T r with FDM local inverses, every smoothed level."""
    C = case
    for li in range(C.nl - 1):
        sm = C.mg.levels[li].smoother
        r = random_vector(len(sm.W), seed=31 + li)
        for tr in (False, True):
            u = C.s.empty(li)
            C.s.schwarz(li, C.free_to_lib(li, r), u, transpose=tr)
            assert rel(C.lib_to_free(li, u), sm.apply(r, transpose=tr)) <= STEP_TOL


def test_fdm_vcycle_parity_and_symmetry(case):
    C = case
    nF = C.mg.levels[0].A.shape[0]
    r = random_vector(nF, seed=9)
    z = C.s.vcycle(C.free_to_lib(0, r))
    assert rel(C.lib_to_free(0, z), C.mg.vcycle(r)) <= STEP_TOL
    x = random_vector(nF, seed=10)
    zx = C.lib_to_free(0, C.s.vcycle(C.free_to_lib(0, x)))
    zr = C.lib_to_free(0, z)
    assert abs(x @ zr - r @ zx) <= 1e-12 * abs(x @ zr)


def test_fdm_solve_parity(case):
    C = case
    lev, perm = C.levels[0]
    phiD = C.m.phi(*lev.xyz.T)
    phi, rep = C.s.solve(C.to_lib(0, phiD), tol=1e-13)
    assert rep["converged"] and rep["rel_res"] <= 1e-12
    assert rel(C.to_orc(0, phi), sem.solve_direct(lev, phiD)) <= SOLVE_TOL
    A, b = sem.dirichlet_lift(lev, phiD)
    _, info = pmg.pcg(C.mg, b, rtol=1e-13)
    assert abs(rep["iters"] - info["iters"]) <= 1


def test_fdm_equals_dense_on_straight_prisms():
    """Config 1: the library's FDM and dense smoothers give the same correction."""
    from tests.test_gpu_parity import make_solver
    m = config1()
    sf = make_solver(m, local_solve=1)
    sd = make_solver(m)
    n = sf.info["level_n_dof"][0]
    r = torch.from_numpy(random_vector(n, seed=3)).cuda()
    for tr in (False, True):
        uf, ud = sf.empty(0), sd.empty(0)
        sf.schwarz(0, r, uf, transpose=tr)
        sd.schwarz(0, r, ud, transpose=tr)
        assert rel(uf.cpu().numpy(), ud.cpu().numpy()) <= 1e-12


def test_config5_replica_dense_smoother_solve():
    """The paper's exact smoother on the hull replica: solve parity vs sparse direct."""
    from tests.test_gpu_parity import make_solver
    from tests._mapping import lib_to_oracle
    m = _c5_replica()
    s = make_solver(m)
    lev = sem.build_system(m, m.p)
    perm = lib_to_oracle(s.node_xyz(0), lev.xyz)
    phiD = m.phi(*lev.xyz.T)
    phi, rep = s.solve(torch.from_numpy(np.ascontiguousarray(phiD[perm])).cuda(), tol=1e-13)
    out = np.zeros(lev.n)
    out[perm] = phi.cpu().numpy()
    assert rep["converged"] and rel(out, sem.solve_direct(lev, phiD)) <= SOLVE_TOL
