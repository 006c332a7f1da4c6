"""Parity at BASELINE.json's full sizes, in the configuration bench.py times.

The oracle cannot assemble config 3 (4.2 M DOF) or config 5 (52.8 M DOF), so it
computes sampled outputs one by one from its own geometry and element matrices
(oracle/sem.py): at element-interior nodes (one element each) and at mesh
vertices (every prism holding the vertex), with the element vectors gathered
from the library's vector by node coordinates.  Properties that hold at any
size are checked on the whole vectors: A 1 = 0, <x, A y> = <A x, y>,
<x, V y> = <V x, y>, R = P^T.  The full-size solve is checked row by row:
its oracle residual at sampled free rows vanishes against the row's scale.

Whole vectors (SURVEY §8(c) parity protocol, steps 5(a)-(b)): the oracle's
streamed element apply (oracle/sem.py apply_streamed: y_e = D^T (G (.) D u_e)
with the oracle's own geometry, element matrices never formed) over EVERY
element, in a process pool over the host cores, gives A u at every row -- the
library's apply must match it to rel-L2 <= 1e-12 -- and the oracle residual
of the library's full-size solution: ||(A phi)_F|| / ||(A phi_D0)_F|| (phi_D0 =
the Dirichlet data, 0 elsewhere; rhs = 0, so b_F = -(A phi_D0)_F) <= 1e-11 for
a solve to 1e-12."""
import numpy as np
import pytest
from scipy.spatial import cKDTree

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2009_00705_b200 as lib  # noqa: E402
from oracle import refelem as R, sem  # noqa: E402
from tests._mapping import streamed_apply_lib  # noqa: E402
from tests.test_gpu_parity import make_solver  # noqa: E402
from workloads import config3, random_vector  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


class Full:
    def __init__(self, m, **kw):
        self.m = m
        self.s = make_solver(m, **kw)
        self.xyz = self.s.node_xyz(0)
        self.tree = cKDTree(self.xyz)
        self.p = m.p

    def elem_ids(self, elems):
        """library node ids of the oracle's element nodes (by coordinates)."""
        rst, _ = R.prism_nodes(self.p)
        X = self.m.node_xyz(rst, elems)                       # [k][N][3]
        d, idx = self.tree.query(X.reshape(-1, 3))
        assert d.max() < 1e-9
        return idx.reshape(X.shape[0], X.shape[1])

    def elem_mats(self, elems):
        G = sem.geometry(self.m, self.p, self.p, elems)
        return sem.element_matrices(G, self.p)


def _interior_locals(p):
    _, ijl = R.prism_nodes(p)
    i, j, l = ijl[:, 0], ijl[:, 1], ijl[:, 2]
    k = p - i - j
    return np.nonzero((i > 0) & (j > 0) & (k > 0) & (l > 0) & (l < p))[0]


@pytest.fixture(scope="module")
def c3full():
    F = Full(config3())              # bench.py's headline configuration (exact dense Schwarz)
    yield F
    F.s.close()
    torch.cuda.empty_cache()


def test_full_config3_apply_sampled_rows(c3full):
    """y = A u (raw Neumann stiffness) at 200 sampled elements' interior nodes and
    at 100 sampled mesh vertices, against the oracle's element matrices."""
    F = c3full
    n = F.s.n_dof(0)
    u = random_vector(n, seed=11)
    y = F.s.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    rng = np.random.default_rng(0)
    E = F.m.n_elem
    el = np.sort(rng.choice(E, 200, replace=False))
    ids = F.elem_ids(el)
    Ae = F.elem_mats(el)
    inner = _interior_locals(F.p)
    yo = np.einsum("eij,ej->ei", Ae, u[ids])[:, inner].ravel()
    yl = y[ids[:, inner]].ravel()
    assert np.linalg.norm(yl - yo) <= 1e-12 * np.linalg.norm(yo)
    # mesh vertices: sum over every prism holding the vertex (corner local nodes)
    p, Nt = F.p, R.n_tri(F.p)
    corner_local = [0, p, Nt - 1, Nt * p, Nt * p + p, Nt * p + Nt - 1]
    verts = rng.choice(F.m.vertices.shape[0], 100, replace=False)
    errs, refs = [], []
    for v in verts:
        hold = np.nonzero((F.m.prisms == v).any(axis=1))[0]
        ids_h = F.elem_ids(hold)
        A_h = F.elem_mats(hold)
        tot = 0.0
        for k, e in enumerate(hold):
            c = corner_local[int(np.nonzero(F.m.prisms[e] == v)[0][0])]
            tot += A_h[k, c] @ u[ids_h[k]]
        g = ids_h[0, corner_local[int(np.nonzero(F.m.prisms[hold[0]] == v)[0][0])]]
        errs.append(y[g] - tot)
        refs.append(tot)
    assert np.linalg.norm(errs) <= 1e-12 * np.linalg.norm(refs)


def test_full_config3_properties(c3full):
    """A 1 = 0, A symmetric, V-cycle symmetric, R = P^T on the whole vectors."""
    F = c3full
    s = F.s
    n = s.n_dof(0)
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    a1 = s.apply(one).abs().max().item()
    x = torch.from_numpy(random_vector(n, 1)).cuda()
    yv = torch.from_numpy(random_vector(n, 2)).cuda()
    Ax, Ay = s.apply(x), s.apply(yv)
    scale = Ax.abs().max().item()
    assert a1 <= 1e-11 * scale
    nrm = lambda a: a.norm().item()
    assert abs((x @ Ay).item() - (Ax @ yv).item()) <= 1e-12 * nrm(x) * nrm(Ay)
    dm = torch.from_numpy(s.dirichlet_mask(0)).cuda()
    xf, yf = x.clone(), yv.clone()
    xf[dm] = 0
    yf[dm] = 0
    vx, vy = s.vcycle(xf), s.vcycle(yf)
    assert abs((xf @ vy).item() - (vx @ yf).item()) <= 1e-12 * nrm(xf) * nrm(vy)
    # R = P^T between levels 0 and 1 on free-node vectors
    nc = s.n_dof(1)
    dmc = torch.from_numpy(s.dirichlet_mask(1)).cuda()
    ec = torch.from_numpy(random_vector(nc, 3)).cuda()
    ec[dmc] = 0
    pe = s.empty(0)
    s.prolong(0, ec, pe)
    rx = s.restrict(0, xf)
    assert abs((xf @ pe).item() - (rx @ ec).item()) <= 1e-12 * nrm(xf) * nrm(pe)


def test_full_config3_solution_rows(c3full):
    """Full-size solve (bench.py's configuration) to rel. residual 1e-12: the
    oracle's residual (A phi)_i at sampled free interior rows vanishes against the
    row scale sum_j |A_ij phi_j|."""
    F = c3full
    s = F.s
    phiD = F.m.phi(F.xyz[:, 0], F.xyz[:, 1], F.xyz[:, 2])
    phi, rep = s.solve(torch.from_numpy(phiD).cuda(), tol=1e-12)
    assert rep["converged"] and rep["rel_res"] <= 1e-12
    ph = phi.cpu().numpy()
    dm = s.dirichlet_mask(0)
    np.testing.assert_array_equal(ph[dm], phiD[dm])
    rng = np.random.default_rng(5)
    el = np.sort(rng.choice(F.m.n_elem, 200, replace=False))
    ids = F.elem_ids(el)
    Ae = F.elem_mats(el)
    inner = _interior_locals(F.p)
    res = np.einsum("eij,ej->ei", Ae, ph[ids])[:, inner]
    scale = np.einsum("eij,ej->ei", np.abs(Ae), np.abs(ph[ids]))[:, inner]
    assert np.max(np.abs(res) / scale) <= 1e-9


def _whole_vector_checks(F, u, seed_sol_tol=1e-12):
    """Library apply of u vs the oracle's streamed apply at every row; library
    solve to rel. residual 1e-12 and the oracle residual of its solution."""
    s = F.s
    n = s.n_dof(0)
    y = s.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    phiD = F.m.phi(F.xyz[:, 0], F.xyz[:, 1], F.xyz[:, 2])
    phi, rep = s.solve(torch.from_numpy(phiD).cuda(), tol=seed_sol_tol, check=False)
    assert rep["converged"] and rep["rel_res"] <= seed_sol_tol, (rep["iters"], rep["res_hist"][-12:])
    ph = phi.cpu().numpy()
    dm = s.dirichlet_mask(0)
    np.testing.assert_array_equal(ph[dm], phiD[dm])
    phiD0 = np.where(dm, phiD, 0.0)
    Y = streamed_apply_lib(F.m, F.p, F.xyz, np.stack([u, ph, phiD0], axis=1), tree=F.tree)
    err = np.linalg.norm(y - Y[:, 0]) / np.linalg.norm(Y[:, 0])
    assert err <= 1e-12, err
    free = ~dm
    res = np.linalg.norm(Y[free, 1]) / np.linalg.norm(Y[free, 2])
    assert res <= 1e-11, res
    return err, res


def test_full_config3_whole_vector_apply_and_solution_residual(c3full):
    """Config 3 at full size (4.2 M DOF, bench.py's headline configuration): the
    library's A u equals the oracle's streamed apply at all 4,224,681 rows, and
    the oracle residual of the library's solution (solved to 1e-12) is <= 1e-11."""
    _whole_vector_checks(c3full, random_vector(c3full.s.n_dof(0), seed=13))


def test_full_config5_whole_vector_apply_and_solution_residual():
    """Config 5 at full size (52.8 M DOF, 477,600 prisms, p = 6; FDM / exact-dense
    hybrid smoother as bench.py runs it): A u vs the oracle's streamed apply at
    every row; the oracle residual of the library's solution; A 1 = 0; V-cycle
    symmetry (its P=1 problem is solved iteratively to 1e-10, reading O9)."""
    from workloads.config5 import config5
    F = Full(config5(), local_solve=1)
    s = F.s
    n = s.n_dof(0)
    assert s.info["smoother_kernel"][0] == "k_fdm_cta<MT>"
    u = random_vector(n, seed=21)
    _whole_vector_checks(F, u)
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    ymax = s.apply(torch.from_numpy(u).cuda()).abs().max().item()
    assert s.apply(one).abs().max().item() <= 1e-11 * ymax
    x = torch.from_numpy(random_vector(n, 7)).cuda()
    dm = torch.from_numpy(s.dirichlet_mask(0)).cuda()
    x[dm] = 0
    z = torch.from_numpy(random_vector(n, 8)).cuda()
    z[dm] = 0
    vx, vz = s.vcycle(x), s.vcycle(z)
    assert abs((x @ vz).item() - (vx @ z).item()) <= 1e-9 * x.norm().item() * vz.norm().item()
    s.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("p", [8])
def test_full_config4_whole_vector(p):
    """Config 4 at full size (~11.5 M DOF, p = 8: the CTA-batched DMMA kernel) with
    the FDM smoother of the sweep: A u vs the oracle's streamed apply at every
    row, the oracle residual of the solution, sampled element rows, A 1 = 0."""
    from workloads import config4
    F = Full(config4(p), local_solve=1)
    s = F.s
    n = s.n_dof(0)
    u = random_vector(n, seed=31)
    _whole_vector_checks(F, u)
    y = s.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    rng = np.random.default_rng(2)
    el = np.sort(rng.choice(F.m.n_elem, 60, replace=False))
    ids = F.elem_ids(el)
    Ae = F.elem_mats(el)
    inner = _interior_locals(F.p)
    yo = np.einsum("eij,ej->ei", Ae, u[ids])[:, inner].ravel()
    assert np.linalg.norm(y[ids[:, inner]].ravel() - yo) <= 1e-12 * np.linalg.norm(yo)
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    assert s.apply(one).abs().max().item() <= 1e-11 * np.abs(y).max()
    s.close()
