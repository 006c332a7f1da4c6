"""Anisotropic element spaces P_p(triangle) x P_q(t) and semi-coarsening (SURVEY
§8(f) NEXT-2; the paper's (P_xy, P_z) pairs, Table 5.4) on the GPU
through the C ABI, against the oracle (oracle/ with q-aware refelem / sem / pmg,
pinned by tests/test_oracle_aniso.py): operator on every level, transfers,
Schwarz smoother, V-cycle and solve, for the paper's (5,3) -> (3,3) -> (1,1)
table and the default semi-coarsening of (4,2)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2009_00705_b200 as lib  # noqa: E402
from oracle import pmg, sem  # noqa: E402
from oracle import refelem as R  # noqa: E402
from tests._mapping import lib_to_oracle  # noqa: E402
from tests.test_gpu_parity import SOLVE_TOL, STEP_TOL, APPLY_TOL, rel  # noqa: E402
from workloads import config2, random_vector  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def _fine_map_xyz(m, lev):
    """Positions of a level's oracle nodes on the finest (p, pz) nodal map (the library's
    convention for coarse levels)."""
    rst_c, _ = R.prism_nodes(lev.p, lev.q)
    rst_f, _ = R.prism_nodes(m.p, m.pz)
    X = m.node_xyz(rst_f)
    V, _ = R.prism_basis(m.p, rst_c, m.pz)
    out = np.zeros((lev.n, 3))
    out[lev.conn.ravel()] = np.einsum("cf,efi->eci", V, X).reshape(-1, 3)
    return out


class ACase:
    def __init__(self, m, levels=None, **kw):
        self.m = m
        if levels is not None:
            kw["levels"] = levels
        self.s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p, m.pz)),
                            pz=m.pz, **kw)
        self.sched = list(zip(self.s.info["level_p"], self.s.info["level_pz"]))
        self.mg = pmg.PMG(m, schedule=self.sched, local_solve="fdm" if kw.get("local_solve") == 1 else "dense",
                          overlap=kw.get("overlap", 1))
        self.levels = []
        for li, ml in enumerate(self.mg.levels):
            lev = ml.level
            ref = lev.xyz if li == 0 else _fine_map_xyz(m, lev)
            self.levels.append((lev, lib_to_oracle(self.s.node_xyz(li), ref)))

    def to_lib(self, li, v):
        return torch.from_numpy(np.ascontiguousarray(v[self.levels[li][1]])).cuda()

    def to_orc(self, li, t):
        lev, perm = self.levels[li]
        out = np.zeros(lev.n)
        out[perm] = t.cpu().numpy()
        return out

    def free_to_lib(self, li, f):
        lev, _ = self.levels[li]
        full = np.zeros(lev.n)
        full[lev.free] = f
        return self.to_lib(li, full)

    def lib_to_free(self, li, t):
        return self.to_orc(li, t)[self.levels[li][0].free]


def _mesh(p, q):
    m = config2(p=p, nx=12, ny=2, nz=2)
    m.pz = q
    return m


@pytest.fixture(scope="module", params=["table5.4", "default(4,2)"])
def case(request):
    if request.param == "table5.4":
        return ACase(_mesh(5, 3), levels=[(5, 3), (3, 3), (1, 1)])
    return ACase(_mesh(4, 2))


def test_schedule(case):
    if case.m.p == 5:
        assert case.sched == [(5, 3), (3, 3), (1, 1)]
    else:   # semi-coarsen the larger (horizontal) order first (reading O19), then isotropic
        assert case.sched == [(4, 2), (3, 2), (2, 2), (1, 1)]


def test_aniso_apply_every_level(case):
    C = case
    for li, (lev, perm) in enumerate(C.levels):
        u = random_vector(lev.n, seed=200 + li)
        y = C.s.apply(C.to_lib(li, u), level=li)
        assert rel(C.to_orc(li, y), C.mg.levels[li].level.A @ u) <= APPLY_TOL


def test_aniso_transfers_smoother_vcycle(case):
    C = case
    for li in range(len(C.levels) - 1):
        Pm = C.mg.levels[li].P
        ec = random_vector(len(C.levels[li + 1][0].free), seed=7 + li)
        uf = C.s.empty(li)
        C.s.prolong(li, C.free_to_lib(li + 1, ec), uf)
        assert rel(C.lib_to_free(li, uf), Pm @ ec) <= STEP_TOL
        rf = random_vector(len(C.levels[li][0].free), seed=17 + li)
        assert rel(C.lib_to_free(li + 1, C.s.restrict(li, C.free_to_lib(li, rf))), Pm.T @ rf) <= STEP_TOL
        sm = C.mg.levels[li].smoother
        for tr in (False, True):
            u = C.s.empty(li)
            C.s.schwarz(li, C.free_to_lib(li, rf), u, transpose=tr)
            assert rel(C.lib_to_free(li, u), sm.apply(rf, transpose=tr)) <= STEP_TOL
    nF = C.mg.levels[0].A.shape[0]
    r = random_vector(nF, seed=9)
    z = C.lib_to_free(0, C.s.vcycle(C.free_to_lib(0, r)))
    assert rel(z, C.mg.vcycle(r)) <= STEP_TOL
    x = random_vector(nF, seed=10)
    zx = C.lib_to_free(0, C.s.vcycle(C.free_to_lib(0, x)))
    assert abs(x @ z - r @ zx) <= 1e-12 * abs(x @ z)


def test_aniso_solve(case):
    C = case
    lev, perm = C.levels[0]
    phiD = C.m.phi(*lev.xyz.T)
    phi, rep = C.s.solve(C.to_lib(0, phiD), tol=1e-13)
    assert rep["converged"] and rel(C.to_orc(0, phi), sem.solve_direct(lev, phiD)) <= SOLVE_TOL
    A, b = sem.dirichlet_lift(lev, phiD)
    _, info = pmg.pcg(C.mg, b, rtol=1e-13)
    assert abs(rep["iters"] - info["iters"]) <= 1


ANISO_PAIRS = [(p, q) for p in (3, 4, 5) for q in range(1, 6) if q != p]


@pytest.mark.parametrize("p,q", ANISO_PAIRS)
def test_aniso_tensor_core_kernel_every_pair(p, q):
    """k_apply_qs<p, q> (the default for 3 <= p <= 5, 1 <= q <= 5) and the generic k_apply_pq
    (apply_kernel = 1) on the finest P_p x P_q level against the assembled oracle matrix, raw
    and masked, on 30 prisms (a ragged last quad of four elements)."""
    m = config2(p=p, nx=5, ny=1, nz=3)
    m.pz = q
    lev = sem.build_system(m, p, q=q)
    u = random_vector(lev.n, seed=300 + 10 * p + q)
    F = lev.free
    for kernel in (0, 1):
        s = lib.Solver(m.vertices, m.prisms, m.face_tag, p, node_xyz=m.node_xyz(lib.reference_nodes(p, q)), pz=q,
                       levels=[(p, q), (1, 1)], apply_kernel=kernel)
        perm = lib_to_oracle(s.node_xyz(0), lev.xyz)
        for masked in (False, True):
            y = s.apply(torch.from_numpy(np.ascontiguousarray(u[perm])).cuda(), masked=masked)
            out = np.zeros(lev.n)
            out[perm] = y.cpu().numpy()
            if masked:
                assert rel(out[F], lev.A[F][:, F] @ u[F]) <= APPLY_TOL, (kernel, masked)
            else:
                assert rel(out, lev.A @ u) <= APPLY_TOL, (kernel, masked)
        s.close()


@pytest.mark.parametrize("pq", [(5, 3), (4, 2), (3, 1)])
def test_aniso_fdm_smoother_vcycle_solve(pq):
    """FDM local solves (reading O33) on P_p x P_q levels: the library's separable boxes built
    from the order-q vertical operators (k_fdm_warp) against the oracle's Kronecker inverses on
    every smoothed level (S^-1 and S^-T), the V-cycle and the solve (the oracle's direct
    solution), on the curved wave channel."""
    p, q = pq
    C = ACase(_mesh(p, q), local_solve=1)
    for li in range(len(C.levels) - 1):
        sm = C.mg.levels[li].smoother
        r = random_vector(len(sm.W), seed=400 + li)
        for tr in (False, True):
            u = C.s.empty(li)
            C.s.schwarz(li, C.free_to_lib(li, r), u, transpose=tr)
            assert rel(C.lib_to_free(li, u), sm.apply(r, transpose=tr)) <= STEP_TOL, (li, tr)
    nF = C.mg.levels[0].A.shape[0]
    r = random_vector(nF, seed=41)
    assert rel(C.lib_to_free(0, C.s.vcycle(C.free_to_lib(0, r))), C.mg.vcycle(r)) <= STEP_TOL
    lev = C.levels[0][0]
    phiD = C.m.phi(*lev.xyz.T)
    phi, rep = C.s.solve(C.to_lib(0, phiD), tol=1e-12)
    assert rep["converged"]
    assert rel(C.to_orc(0, phi), sem.solve_direct(lev, phiD)) <= SOLVE_TOL
    C.s.close()
