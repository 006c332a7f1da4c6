"""Partitioned solve validated on one GPU: nranks column
partitions emulated in one process (exchanges as device copies, the same code
path as the NCCL transport).  Results must equal the single-domain solver's
(same arithmetic up to summation order) and the oracle's."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2009_00705_b200 as lib  # noqa: E402
from oracle import sem  # noqa: E402
from tests._mapping import lib_to_oracle  # noqa: E402
from workloads import config2, random_vector  # noqa: E402
from workloads.configs import basin  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def mk(m, **kw):
    return lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)), **kw)


MESHES = {
    "c3s": lambda: basin("c3s", 5, 32.0 * 6 / 64, 6, 3, seed=3),
    "c2": lambda: config2(),
}


@pytest.fixture(scope="module", params=list(MESHES))
def pair(request):
    m = MESHES[request.param]()
    return m, mk(m)


@pytest.fixture(autouse=True)
def _overlap_forced(monkeypatch):
    """Every partitioned ctx of this module splits its applies and sweeps into interface /
    interior parts with the exchange in flight (the NCCL default; emulated ranks default to the
    serial path, which has no transfer to hide).  SEM_DIST_OVERLAP is read at setup."""
    monkeypatch.setenv("SEM_DIST_OVERLAP", "2")


@pytest.mark.parametrize("overlap", ["2", "0"])
@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_partitioned_matches_single_domain(pair, nranks, overlap, monkeypatch):
    m, s1 = pair
    monkeypatch.setenv("SEM_DIST_OVERLAP", overlap)
    sd = mk(m, nranks=nranks)
    assert sd.info["n_dof"] == s1.info["n_dof"] and sd.info["level_p"] == s1.info["level_p"]
    np.testing.assert_array_equal(sd.node_xyz(0), s1.node_xyz(0))
    n = s1.info["n_dof"]
    mask = torch.from_numpy(s1.dirichlet_mask(0)).cuda()
    # operator, every level, raw and masked
    for li, nl in enumerate(s1.info["level_n_dof"]):
        u = torch.from_numpy(random_vector(nl, seed=40 + li)).cuda()
        for masked in (False, True):
            y1 = s1.apply(u, level=li, masked=masked).cpu().numpy()
            yd = sd.apply(u, level=li, masked=masked).cpu().numpy()
            assert rel(yd, y1) <= 1e-13, (li, masked)
    # one V-cycle
    r = torch.from_numpy(random_vector(n, seed=3)).cuda().masked_fill(mask, 0.0)
    z1 = s1.vcycle(r).cpu().numpy()
    zd = sd.vcycle(r).cpu().numpy()
    assert rel(zd, z1) <= 1e-12
    # full solve
    xyz = s1.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    p1, r1 = s1.solve(phiD, 1e-12)
    pd, rd = sd.solve(phiD, 1e-12)
    assert rd["converged"] and abs(rd["iters"] - r1["iters"]) <= 1
    assert rel(pd.cpu().numpy(), p1.cpu().numpy()) <= 1e-10
    sd.close()


def test_partitioned_solve_matches_oracle():
    m = MESHES["c3s"]()
    sd = mk(m, nranks=4)
    lev = sem.build_system(m, m.p)
    perm = lib_to_oracle(sd.node_xyz(0), lev.xyz)
    phiD = m.phi(*lev.xyz.T)
    phi, rep = sd.solve(torch.from_numpy(np.ascontiguousarray(phiD[perm])).cuda(), tol=1e-13)
    got = np.zeros(lev.n)
    got[perm] = phi.cpu().numpy()
    assert rep["converged"] and rel(got, sem.solve_direct(lev, phiD)) <= 1e-10
    sd.close()


FDM_MESHES = {
    "c3s": lambda: basin("c3s", 5, 32.0 * 6 / 64, 6, 3, seed=3),
    "c5r": lambda: __import__("workloads.config5", fromlist=["config5"]).config5(p=3, hf=0.5, Lx=16.0, Ly=10.0),
}


@pytest.mark.parametrize("name", list(FDM_MESHES))
@pytest.mark.parametrize("nranks", [2, 3])
def test_partitioned_fdm_matches_single_domain(name, nranks, monkeypatch):
    """Partitioned FDM / exact-dense hybrid (O33, O35): smoother sweep, V-cycle and
    solve equal the single-domain FDM solver (hull replica included).  Every FDM sweep
    split into interface / interior column units (SEM_DIST_OVERLAP=2)."""
    monkeypatch.setenv("SEM_DIST_OVERLAP", "2")
    m = FDM_MESHES[name]()
    s1 = mk(m, local_solve=1)
    sd = mk(m, local_solve=1, nranks=nranks)
    n = s1.info["n_dof"]
    mask = torch.from_numpy(s1.dirichlet_mask(0)).cuda()
    r = torch.from_numpy(random_vector(n, seed=5)).cuda().masked_fill(mask, 0.0)
    z1 = s1.vcycle(r).cpu().numpy()
    zd = sd.vcycle(r).cpu().numpy()
    assert rel(zd, z1) <= 1e-12
    xyz = s1.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    p1, r1 = s1.solve(phiD, 1e-12)
    pd, rd = sd.solve(phiD, 1e-12)
    assert rd["converged"] and abs(rd["iters"] - r1["iters"]) <= 1
    assert rel(pd.cpu().numpy(), p1.cpu().numpy()) <= 1e-10
    sd.close()
    s1.close()


@pytest.mark.parametrize("nranks", [2, 3])
def test_partitioned_fdm_cta_overlap(nranks, monkeypatch):
    """p = 6 Delaunay basin whose level-0 sweep runs k_fdm_cta<8>: the partitioned sweep
    (interface column units, exchange in flight, interior units; FDM unit lists) and the
    V-cycle equal the single domain."""
    from workloads.configs import delaunay_basin
    monkeypatch.setenv("SEM_DIST_OVERLAP", "2")
    m = delaunay_basin("fdm_cta8", 6, n_in=16, nz=3, seed=1)
    s1 = mk(m, local_solve=1)
    assert s1.info["smoother_kernel"][0] == "k_fdm_cta<MT>"
    sd = mk(m, local_solve=1, nranks=nranks)
    n = s1.info["n_dof"]
    mask = torch.from_numpy(s1.dirichlet_mask(0)).cuda()
    r = torch.from_numpy(random_vector(n, seed=7)).cuda().masked_fill(mask, 0.0)
    assert rel(sd.vcycle(r).cpu().numpy(), s1.vcycle(r).cpu().numpy()) <= 1e-12
    sd.close()
    s1.close()


@pytest.mark.parametrize("local_solve", [0, 1])
def test_user_partition_sem_mesh_part(local_solve):
    """sem_mesh.part: a caller-given partition -- here three strips of
    whole columns by the x of the column's triangle, a different cut from the
    library's recursive bisection -- gives the single-domain solution."""
    m = basin("c3s_part", 5, 32.0 * 6 / 64, 6, 3, seed=3)
    cx = m.vert2d[m.tri].mean(axis=1)[:, 0]                   # per triangle (column)
    col = np.arange(m.n_elem) // m.nz                           # element -> column (column-major order)
    part = np.minimum(2, (3 * cx[col] / cx.max()).astype(np.int32))
    s1 = mk(m, local_solve=local_solve)
    sd = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)),
                    nranks=3, part=part, local_solve=local_solve)
    xyz = s1.node_xyz(0)
    phiD = torch.from_numpy(m.phi(*xyz.T)).cuda()
    a, _ = s1.solve(phiD, 1e-12)
    b, _ = sd.solve(phiD, 1e-12)
    assert rel(b.cpu().numpy(), a.cpu().numpy()) <= 1e-10
    u = torch.from_numpy(random_vector(s1.n_dof(0), 9)).cuda()
    assert rel(sd.apply(u).cpu().numpy(), s1.apply(u).cpu().numpy()) <= 1e-13
