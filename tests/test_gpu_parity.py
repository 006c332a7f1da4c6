"""GPU parity of every hot-path step against the oracle,
element by element on the same seeded inputs, through the C ABI.

Bars (north_star): apply rel-L2 <= 1e-12; solve rel-L2 <= 1e-10 when solved to
rel. residual <= 1e-12.  Step bars (transfers, smoother, coarse solve, V-cycle)
use the same 1e-12 bound: they are linear maps evaluated in FP64 whose only
difference from the oracle is the summation order (DESIGN.md §"Tolerances").
"""
import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2009_00705_b200 as lib  # noqa: E402
from oracle import pmg, sem  # noqa: E402
from tests._mapping import fine_map_xyz, lib_to_oracle  # noqa: E402
from workloads import config1, config2, config3, config4, random_vector  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

APPLY_TOL = 1e-12
STEP_TOL = 1e-12
SOLVE_TOL = 1e-10


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def make_solver(m, p=None, **kw):
    p = p or m.p
    return lib.Solver(m.vertices, m.prisms, m.face_tag, p, node_xyz=m.node_xyz(lib.reference_nodes(p)), **kw)


class Case:
    """Library solver + oracle hierarchy + numbering maps of one mesh."""

    def __init__(self, m, build_mg=True, **kw):
        self.m = m
        self.s = make_solver(m, **kw)
        self.nl = self.s.info["n_levels"]
        self.levels = []
        for li, pl in enumerate(self.s.info["level_p"]):
            lev = sem.build_system(m, pl, p_geo=m.p)
            ref_xyz = lev.xyz if li == 0 else fine_map_xyz(m, lev, m.p)
            perm = lib_to_oracle(self.s.node_xyz(li), ref_xyz)
            self.levels.append((lev, perm))
        self.mg = pmg.PMG(m, schedule=self.s.info["level_p"], nu1=kw.get("nu1", 3), nu2=kw.get("nu2", 3),
                          overlap=kw.get("overlap", 1), literal=bool(kw.get("literal_smoother", 0)),
                          local_solve="fdm" if kw.get("local_solve", 0) == 1 else "dense") if build_mg else None

    def to_lib(self, li, v_orc_full):
        lev, perm = self.levels[li]
        return torch.from_numpy(np.ascontiguousarray(v_orc_full[perm])).cuda()

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
        lev, _ = self.levels[li]
        return self.to_orc(li, t)[lev.free]


@pytest.fixture(scope="module")
def c1():
    return Case(config1())


@pytest.fixture(scope="module")
def c2():
    return Case(config2())


@pytest.fixture(scope="module")
def c3s():
    # scaled-down config-3 construction (jitter, 8 waves, p=5): 5x3 quads x 3 layers
    # = 90 prisms -> 45 apply CTAs of 2 elements, ragged Schwarz tiles
    return Case(_c3_small())


def _c3_small():
    from workloads.configs import basin
    return basin("config3_small", 5, 32.0 * 5 / 64, 5, 3, seed=3)


ALL = ["c1", "c2", "c3s"]


@pytest.mark.parametrize("case", ALL)
def test_apply_parity_all_levels(case, request):
    """a2/a3: raw Neumann stiffness and masked operator on every level."""
    C = request.getfixturevalue(case)
    for li, (lev, perm) in enumerate(C.levels):
        u = random_vector(lev.n, seed=100 + li)
        y_orc = lev.A @ u
        y = C.s.apply(C.to_lib(li, u), level=li, masked=False)
        assert rel(C.to_orc(li, y), y_orc) <= APPLY_TOL
        # masked: y_F = A_FF u_F, y_D = u_D
        F = lev.free
        um = u.copy()
        ym = C.s.apply(C.to_lib(li, u), level=li, masked=True)
        ymo = C.to_orc(li, ym)
        yF = lev.A[F][:, F] @ u[F]
        assert rel(ymo[F], yF) <= APPLY_TOL
        np.testing.assert_array_equal(ymo[lev.dirichlet], um[lev.dirichlet])


@pytest.mark.parametrize("case", ALL)
def test_transfer_parity(case, request):
    """a7/a9: P and R = P^T (eq 4.3) between every level pair."""
    C = request.getfixturevalue(case)
    for li in range(C.nl - 1):
        Pm = C.mg.levels[li].P
        lf, lc = C.levels[li][0], C.levels[li + 1][0]
        ec = random_vector(len(lc.free), seed=7 + li)
        uf = C.s.empty(li)
        C.s.prolong(li, C.free_to_lib(li + 1, ec), uf)
        assert rel(C.lib_to_free(li, uf), Pm @ ec) <= STEP_TOL
        rf = random_vector(len(lf.free), seed=17 + li)
        rc = C.s.restrict(li, C.free_to_lib(li, rf))
        assert rel(C.lib_to_free(li + 1, rc), Pm.T @ rf) <= STEP_TOL
        assert np.all(C.to_orc(li + 1, rc)[lc.dirichlet] == 0.0)


@pytest.mark.parametrize("case", ALL)
def test_schwarz_parity(case, request):
    """a5: u += S^-1 r and u += S^-T r (eq 4.4-4.6, reading O14)."""
    C = request.getfixturevalue(case)
    for li in range(C.nl - 1):
        sm = C.mg.levels[li].smoother
        r = random_vector(len(sm.W), seed=31 + li)
        for tr in (False, True):
            u = C.s.empty(li)
            C.s.schwarz(li, C.free_to_lib(li, r), u, transpose=tr)
            assert rel(C.lib_to_free(li, u), sm.apply(r, transpose=tr)) <= STEP_TOL


@pytest.mark.parametrize("case", ALL)
def test_coarse_solve_parity(case, request):
    """a8: exact P=1 solve: k_coarse_symv on packed 64x64 tiles of the
    symmetric inverse -- c1's 50 free P=1 nodes fill one ragged diagonal tile, c2's
    1300 span 21 tile rows (ragged tail of 20) with off-diagonal tiles."""
    C = request.getfixturevalue(case)
    last = C.mg.levels[-1]
    r = random_vector(last.A.shape[0], seed=5)
    z = C.s.coarse_solve(C.free_to_lib(C.nl - 1, r))
    assert rel(C.lib_to_free(C.nl - 1, z), last.coarse_lu.solve(r)) <= STEP_TOL


@pytest.mark.parametrize("case", ALL)
def test_vcycle_parity_and_symmetry(case, request):
    """a6/a10: one V-cycle (Alg 4.1) equals the oracle's; it is symmetric."""
    C = request.getfixturevalue(case)
    nF = C.mg.levels[0].A.shape[0]
    r = random_vector(nF, seed=9)
    z = C.s.vcycle(C.free_to_lib(0, r))
    assert rel(C.lib_to_free(0, z), C.mg.vcycle(r)) <= STEP_TOL
    assert np.all(C.to_orc(0, z)[C.levels[0][0].dirichlet] == 0.0)
    x = random_vector(nF, seed=10)
    zx = C.lib_to_free(0, C.s.vcycle(C.free_to_lib(0, x)))
    zr = C.lib_to_free(0, z)
    assert abs(x @ zr - r @ zx) <= 1e-12 * abs(x @ zr)


@pytest.mark.parametrize("case", ALL)
def test_solve_parity(case, request):
    """a1 + a11: lift, PCG (Alg 4.3) to rel. residual <= 1e-13, vs sparse direct."""
    C = request.getfixturevalue(case)
    lev, perm = C.levels[0]
    phiD = C.m.phi(*lev.xyz.T)
    phi_direct = sem.solve_direct(lev, phiD)
    phi, rep = C.s.solve(C.to_lib(0, phiD), tol=1e-13)
    assert rep["converged"] and rep["rel_res"] <= 1e-12
    got = C.to_orc(0, phi)
    assert rel(got, phi_direct) <= SOLVE_TOL
    np.testing.assert_array_equal(got[lev.dirichlet], phiD[lev.dirichlet])
    # iteration count equals the oracle PCG's (same algorithm, same readings)
    A, b = sem.dirichlet_lift(lev, phiD)
    _, info = pmg.pcg(C.mg, b, rtol=1e-13)
    assert abs(rep["iters"] - info["iters"]) <= 1
    assert rep["vcycles"] == rep["iters"]  # final V-cycle skipped


def test_pdc_parity(c1):
    """Alg 4.2 behind the option outer=1."""
    m = c1.m
    s = make_solver(m, outer=1)
    lev, perm = c1.levels[0]
    phiD = m.phi(*lev.xyz.T)
    phi, rep = s.solve(torch.from_numpy(phiD[perm]).cuda(), tol=1e-12)
    out = np.zeros(lev.n)
    out[perm] = phi.cpu().numpy()
    assert rel(out, sem.solve_direct(lev, phiD)) <= SOLVE_TOL
    A, b = sem.dirichlet_lift(lev, phiD)
    _, info = pmg.pdc(c1.mg, b, rtol=1e-12)
    assert abs(rep["iters"] - info["iters"]) <= 1


def test_literal_smoother_option(c1):
    """literal_smoother=1 reproduces the oracle's literal (non-symmetric) V-cycle."""
    m = c1.m
    s = make_solver(m, literal_smoother=1)
    mg = pmg.PMG(m, literal=True)
    lev, perm = c1.levels[0]
    r = random_vector(mg.levels[0].A.shape[0], seed=2)
    full = np.zeros(lev.n)
    full[lev.free] = r
    z = s.vcycle(torch.from_numpy(full[perm]).cuda())
    out = np.zeros(lev.n)
    out[perm] = z.cpu().numpy()
    assert rel(out[lev.free], mg.vcycle(r)) <= STEP_TOL


@pytest.mark.parametrize("apply_kernel", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("p", range(1, 9))
def test_config4_construction_every_order(p, apply_kernel):
    """Config-4 construction (scaled replica) at every order p = 1..8, both operator
    kernels (0 = default, 1 = FMA, 2 = batched DMMA, 3 = four elements per warp, 4 = four elements per
    group of warps): apply and solve parity; p = 1 is the
    single-level coarse solve (O26).  3x3 (p <= 5) or 2x2 quads x 2 layers = 36 / 16
    prisms: several element batches with a ragged last batch for every p."""
    m, lev, phiD, phi_direct = _c4_oracle(p)      # the oracle side, shared by the four kernel variants
    s = make_solver(m, apply_kernel=apply_kernel)
    perm = lib_to_oracle(s.node_xyz(0), lev.xyz)
    u = random_vector(lev.n, seed=p)
    y = s.apply(torch.from_numpy(u[perm]).cuda())
    out = np.zeros(lev.n)
    out[perm] = y.cpu().numpy()
    assert rel(out, lev.A @ u) <= APPLY_TOL
    phi, rep = s.solve(torch.from_numpy(phiD[perm]).cuda(), tol=1e-13)
    out[perm] = phi.cpu().numpy()
    assert rel(out, phi_direct) <= SOLVE_TOL


@pytest.mark.parametrize("apply_kernel", [3, 4])
@pytest.mark.parametrize("p", [3, 4, 5, 6])
@pytest.mark.parametrize("nx,ny,nz", [(1, 1, 3), (5, 3, 3)])
def test_quad_kernels_ragged(p, apply_kernel, nx, ny, nz):
    """The four-element kernels on element counts that are not a multiple of four (6 and 90
    prisms: a ragged last quad, one or several CTAs), masked and raw operator, against the
    assembled oracle matrix (eq 3.8)."""
    m = config1(p=p, nx=nx, ny=ny, nz=nz)
    lev = sem.build_system(m, p)
    s = make_solver(m, apply_kernel=apply_kernel)
    perm = lib_to_oracle(s.node_xyz(0), lev.xyz)
    u = random_vector(lev.n, seed=11 + p)
    for masked in (False, True):
        y = s.apply(torch.from_numpy(u[perm]).cuda(), masked=masked)
        out = np.zeros(lev.n)
        out[perm] = y.cpu().numpy()
        if masked:   # y_F = A_FF u_F, y_D = u_D
            F = lev.free
            assert rel(out[F], lev.A[F][:, F] @ u[F]) <= APPLY_TOL
            np.testing.assert_array_equal(out[lev.dirichlet], u[lev.dirichlet])
        else:
            assert rel(out, lev.A @ u) <= APPLY_TOL
    s.close()


@functools.lru_cache(maxsize=None)
def _c4_oracle(p):
    from workloads.configs import basin
    n = 2 if p >= 6 else 3
    m = basin(f"c4r_p{p}", p, 32.0 * n / 56, n, 2, seed=4)
    lev = sem.build_system(m, p)
    phiD = m.phi(*lev.xyz.T)
    return m, lev, phiD, sem.solve_direct(lev, phiD)


def test_solve_host_matches_device(c2):
    """laplace_solve_host (H2D + solve + D2H in one call) = laplace_solve (to the
    rounding of the atomic scatter order, which differs run to run)."""
    lev, perm = c2.levels[0]
    phiD = np.ascontiguousarray(c2.m.phi(*lev.xyz.T)[perm])
    phi_d, _ = c2.s.solve(torch.from_numpy(phiD).cuda(), tol=1e-10)
    out = np.zeros_like(phiD)
    rep = c2.s.solve_host(phiD, 1e-10, out)
    assert rep["converged"]
    ref = phi_d.cpu().numpy()
    assert rel(out, ref) <= 1e-12


def test_error_paths():
    m = config1(p=2)
    tags = m.face_tag.copy()
    tags[0, 1] = 9
    with pytest.raises(lib.SemError) as ei:
        lib.Solver(m.vertices, m.prisms, tags, 2)
    assert ei.value.code == -1
    # an inverted prism (top below bottom): detJ <= 0
    bad = m.prisms.copy()
    bad[0] = bad[0][[3, 4, 5, 0, 1, 2]]
    with pytest.raises(lib.SemError) as ei:
        lib.Solver(m.vertices, bad, m.face_tag, 2)
    assert ei.value.code == -2
    with pytest.raises(lib.SemError):
        lib.Solver(m.vertices, m.prisms, m.face_tag, 9)


def test_not_converged_flag(c1):
    """imax reached -> SEM_ENOTCONV with the last iterate and converged=0."""
    m = c1.m
    s = make_solver(m, imax=1)
    lev, perm = c1.levels[0]
    phiD = torch.from_numpy(m.phi(*lev.xyz.T)[perm]).cuda()
    phi, rep = s.solve(phiD, tol=1e-14, check=False)
    assert not rep["converged"] and rep["iters"] == 1


@pytest.mark.parametrize("agg", [0, 16])
def test_iterative_coarse_solver(c2, agg):
    """Reading O9 for large P=1 problems: line-Jacobi PCG coarse solve (coarse_solver=1),
    with and without the two-level aggregate correction (reading O44, coarse_agg
    aggregates), agrees with the exact coarse solve to its tolerance, and the flexible
    outer PCG still reaches the sparse-direct solution to 1e-10."""
    m = c2.m
    s = make_solver(m, coarse_solver=1, coarse_rtol=1e-12, coarse_agg=agg)
    assert s.info["coarse_agg"] == agg
    last = c2.mg.levels[-1]
    li = c2.nl - 1
    r = random_vector(last.A.shape[0], seed=12)
    z = s.coarse_solve(c2.free_to_lib(li, r))
    assert rel(c2.lib_to_free(li, z), last.coarse_lu.solve(r)) <= 1e-9
    lev, perm = c2.levels[0]
    phiD = m.phi(*lev.xyz.T)
    phi, rep = s.solve(c2.to_lib(0, phiD), tol=1e-13)
    assert rep["converged"] and rep["coarse_iters"] > 0
    assert rel(c2.to_orc(0, phi), sem.solve_direct(lev, phiD)) <= SOLVE_TOL
    s.close()


def test_mixed_precision_storage(c2):
    """mixed_precision=1: FP32 storage of the exact Schwarz and coarse
    inverses, FP64 arithmetic.  Each step stays within FP32 rounding of the FP64
    step; the solve still reaches the sparse-direct solution (the preconditioner is
    a fixed symmetric linear operator)."""
    m = c2.m
    s = make_solver(m, mixed_precision=1)
    assert s.info["schwarz_bytes"][0] * 2 == c2.s.info["schwarz_bytes"][0]
    sm = c2.mg.levels[0].smoother
    r = random_vector(len(sm.W), seed=41)
    u = s.empty(0)
    s.schwarz(0, c2.free_to_lib(0, r), u)
    assert 1e-12 < rel(c2.lib_to_free(0, u), sm.apply(r)) <= 1e-5
    nF = c2.mg.levels[0].A.shape[0]
    x = random_vector(nF, seed=42)
    y = random_vector(nF, seed=43)
    vx = c2.lib_to_free(0, s.vcycle(c2.free_to_lib(0, x)))
    vy = c2.lib_to_free(0, s.vcycle(c2.free_to_lib(0, y)))
    assert rel(vx, c2.mg.vcycle(x)) <= 1e-5
    assert abs(x @ vy - y @ vx) <= 1e-12 * abs(x @ vy)      # still symmetric
    lev, perm = c2.levels[0]
    phiD = m.phi(*lev.xyz.T)
    phi, rep = s.solve(c2.to_lib(0, phiD), tol=1e-13)
    assert rep["converged"]
    assert rel(c2.to_orc(0, phi), sem.solve_direct(lev, phiD)) <= SOLVE_TOL


@pytest.mark.parametrize("levels", [(6, 3, 1), (5, 3, 1)])
def test_explicit_level_tables(levels):
    """Explicit coarsening tables through opts.levels: 6 -> 3 -> 1 (Table 5.1,
    P:391) and 5 -> 3 -> 1 (Table 5.4 with P_xy = P_z): the library's
    hierarchy is the requested one; V-cycle, solve and iteration count match the
    oracle built on the same schedule."""
    p = levels[0]
    m = config2(p=6, nx=12, ny=2, nz=2) if p == 6 else _c3_small()
    C = Case(m, levels=list(levels))
    assert C.s.info["level_p"] == list(levels)
    nF = C.mg.levels[0].A.shape[0]
    r = random_vector(nF, seed=19)
    assert rel(C.lib_to_free(0, C.s.vcycle(C.free_to_lib(0, r))), C.mg.vcycle(r)) <= STEP_TOL
    lev, perm = C.levels[0]
    phiD = m.phi(*lev.xyz.T)
    phi, rep = C.s.solve(C.to_lib(0, phiD), tol=1e-13)
    assert rep["converged"] and rel(C.to_orc(0, phi), sem.solve_direct(lev, phiD)) <= SOLVE_TOL
    A, b = sem.dirichlet_lift(lev, phiD)
    _, info = pmg.pcg(C.mg, b, rtol=1e-13)
    assert abs(rep["iters"] - info["iters"]) <= 1


def test_standalone_mg_outer2(c1):
    """outer = 2: the V-cycle of Alg 4.1 iterated as the solver, u <- u + V(b - A u)
    (the same stationary iteration as PDC with the MG preconditioner, Alg 4.2):
    reaches the sparse-direct solution; iteration count = the oracle's PDC's."""
    m = c1.m
    s = make_solver(m, outer=2)
    lev, perm = c1.levels[0]
    phiD = m.phi(*lev.xyz.T)
    phi, rep = s.solve(torch.from_numpy(phiD[perm]).cuda(), tol=1e-12)
    out = np.zeros(lev.n)
    out[perm] = phi.cpu().numpy()
    assert rep["converged"] and rel(out, sem.solve_direct(lev, phiD)) <= SOLVE_TOL
    A, b = sem.dirichlet_lift(lev, phiD)
    _, info = pmg.pdc(c1.mg, b, rtol=1e-12)
    assert abs(rep["iters"] - info["iters"]) <= 1 and rep["vcycles"] == rep["iters"]
    assert rep["wu"] > 0
