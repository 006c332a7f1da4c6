"""GPU parity of the FNPF stage (eq 2.1-2.2) against
oracle/fnpf.py on the same seeded surface state, through the C ABI: the stage
rates (geometry update O37, Laplace solve, w~ O38, surface gradients O39, eq 2.1)
and one ERK4 step (O40); the linear standing wave returns after one period of
the dispersion relation (the pin of tests/test_oracle_fnpf.py, on the GPU path)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from scipy.spatial import cKDTree  # noqa: E402

from oracle import fnpf  # noqa: E402
from tests.test_gpu_parity import make_solver, rel  # noqa: E402
from workloads import config1, config2  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2009_00705_b200 as lib  # noqa: E402


def _setup(m, strategy=1, **kw):
    s = make_solver(m, **kw)
    ids = s.fnpf_init(m.node_xyz(lib.reference_nodes(m.p)), strategy=strategy)
    S = fnpf.Surface(m, m.p)
    lib_xy = s.node_xyz(0)[ids]
    d, perm = cKDTree(S.level.xyz[S.snode]).query(lib_xy)     # library surface k <-> oracle surface perm[k]
    assert d.max() < 1e-9 and len(np.unique(perm)) == len(perm) == len(S.snode)
    return s, S, perm, lib_xy


def _state(S, seed):
    xs = S.level.xyz[S.snode]
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.01, 0.03, 3)
    eta = S.eta0 + a[0] * np.cos(math.pi * xs[:, 0] / 2) * np.cos(math.pi * xs[:, 1]) + a[1] * np.sin(0.5 * xs[:, 0])
    phis = a[2] * np.cosh(1.0) * np.cos(math.pi * xs[:, 0] / 4) + 0.1 * xs[:, 1] ** 2
    return eta, phis


@pytest.mark.parametrize("strategy", [1, 2, 3, 4])
def test_fnpf_rates_parity(strategy):
    """Rates of eq 2.1 at a curved, moving surface (config 2 construction, p = 4):
    GPU (PCG-p-MG to 1e-13) vs oracle (sparse direct) at every surface node, for the
    paper's strategies I (1), II (3), III (4) and operators-only (2): the strategy
    changes the preconditioner, never the solution."""
    m = config2(p=4, nx=16, ny=2, nz=2)
    kw = dict(local_solve=1, coarse_solver=1, coarse_rtol=1e-13) if strategy >= 3 else {}
    s, S, perm, _ = _setup(m, strategy, **kw)
    eta, phis = _state(S, 1)
    de_o, dp_o, w_o = fnpf.surface_rhs(S, eta, phis)
    t = lambda v: torch.from_numpy(np.ascontiguousarray(v[perm])).cuda()
    de, dp, w, rep = s.fnpf_rhs(t(eta), t(phis), 1e-13)
    assert rep["converged"]
    assert rel(w.cpu().numpy(), w_o[perm]) <= 1e-10
    assert rel(de.cpu().numpy(), de_o[perm]) <= 1e-10
    assert rel(dp.cpu().numpy(), dp_o[perm]) <= 1e-10
    # a second stage at another state: warm start, same parity
    eta2, phis2 = _state(S, 2)
    de_o, dp_o, _ = fnpf.surface_rhs(S, eta2, phis2)
    de, dp, _, rep2 = s.fnpf_rhs(t(eta2), t(phis2), 1e-13)
    assert rel(de.cpu().numpy(), de_o[perm]) <= 1e-10 and rel(dp.cpu().numpy(), dp_o[perm]) <= 1e-10
    s.close()


def test_fnpf_erk4_step_parity():
    """One classical RK4 step (four stage solves) from the same state."""
    m = config2(p=3, nx=16, ny=2, nz=2)
    s, S, perm, _ = _setup(m)
    eta, phis = _state(S, 3)
    e_o, p_o = fnpf.erk4_step(S, eta, phis, 0.01)
    te = torch.from_numpy(np.ascontiguousarray(eta[perm])).cuda()
    tp = torch.from_numpy(np.ascontiguousarray(phis[perm])).cuda()
    its = s.fnpf_erk4_step(te, tp, 0.01, 1e-13)
    assert its > 0
    assert rel(te.cpu().numpy(), e_o[perm]) <= 1e-10
    assert rel(tp.cpu().numpy(), p_o[perm]) <= 1e-10
    s.close()


@pytest.mark.parametrize("linear", [True, False])
def test_fnpf_standing_wave_period(linear):
    """eta0 = A cos(k x), phi~0 = 0 in the closed box (k = pi, h = 1): after one
    period T = 2 pi / omega, omega^2 = g k tanh(k h), eta is back to eta0 within
    1e-3 (linear version) / 3e-2 (fully nonlinear at A = 0.005: the nonlinear
    standing wave departs from the linear one at relative order k A = 0.016)."""
    p = 4
    m = config1(p=p, nx=4, ny=2, nz=2)
    s, S, perm, xy = _setup(m)
    k, A = math.pi, 0.005
    om = math.sqrt(9.81 * k * math.tanh(k))
    T = 2 * math.pi / om
    eta0 = A * np.cos(k * xy[:, 0])
    te = torch.from_numpy(eta0.copy()).cuda()
    tp = torch.zeros_like(te)
    for _ in range(32):
        s.fnpf_erk4_step(te, tp, T / 32, 1e-12, linear=linear)
    assert np.linalg.norm(te.cpu().numpy() - eta0) <= (1e-3 if linear else 3e-2) * np.linalg.norm(eta0)
    s.close()


def test_fnpf_strategy_III_smoother_equals_fresh_setup():
    """Strategy III after one stage: the FDM smoothers re-formed on the device equal a
    fresh setup on the staged geometry (the oracle's sigma-map nodal map of O37)."""
    m = config2(p=4, nx=16, ny=2, nz=2)
    kw = dict(local_solve=1, coarse_solver=1, coarse_rtol=1e-13)
    s, S, perm, _ = _setup(m, 4, **kw)
    eta, phis = _state(S, 4)
    t = lambda v: torch.from_numpy(np.ascontiguousarray(v[perm])).cuda()
    s.fnpf_rhs(t(eta), t(phis), 1e-10)
    staged = fnpf.StagedMesh(S, eta)
    fresh = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=_lib_order_nodes(staged, m.p), **kw)
    from workloads import random_vector
    for li in range(s.info["n_levels"] - 1):
        r = torch.from_numpy(random_vector(s.n_dof(li), 70 + li)).cuda()
        a, b = s.empty(li), fresh.empty(li)
        s.schwarz(li, r, a)
        fresh.schwarz(li, r, b)
        assert rel(a.cpu().numpy(), b.cpu().numpy()) <= 1e-12
    s.close()
    fresh.close()


def _lib_order_nodes(staged, p):
    """The staged nodal map at the LIBRARY's reference nodes (its local order): the
    oracle's nodes matched by reference coordinates."""
    rst_lib = lib.reference_nodes(p)
    rst_orc, _ = fnpf.R.prism_nodes(p)
    d, idx = cKDTree(rst_orc).query(rst_lib)
    assert d.max() < 1e-12
    return staged.node_xyz(rst_orc)[:, idx, :]
