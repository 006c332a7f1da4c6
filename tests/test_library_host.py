"""CPU tier of the C-ABI library: it loads, exports every symbol the header
declares, and its host logic (reference element, numbering of V^p, Dirichlet
set, Schwarz subdomains and weights) agrees with the independent oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2009_00705_b200 as lib
from paper_2009_00705_b200 import _capi
from oracle import pmg, refelem as R, sem
from workloads import config1, config2, config3
from tests._mapping import lib_node_xyz, lib_to_oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    hdr = open(os.path.join(ROOT, "include", "sem_pmg.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(\w+)\s*\([^;{]*\)\s*;", hdr)) - {"if", "while"}
    assert len(names) >= 20, names
    so = ctypes.CDLL(lib.LIB_PATH)
    for nme in names:
        assert hasattr(so, nme), f"missing export {nme}"
    assert set(_capi.EXPORTS) <= names


@pytest.mark.parametrize("p", range(1, 9))
def test_reference_element_matches_oracle(p):
    rst = lib.reference_nodes(p)
    orst, _ = R.prism_nodes(p)
    np.testing.assert_allclose(rst, orst, atol=1e-15)
    ref = lib.host_reference(p)
    r, s, wt = R.tri_cubature(p)
    Lt, Lr, Ls = R.tri_lagrange(p, r, s)
    np.testing.assert_allclose(ref["B0"], Lt, atol=1e-12)
    np.testing.assert_allclose(ref["Br"], Lr, atol=1e-11)
    np.testing.assert_allclose(ref["Bs"], Ls, atol=1e-11)
    t, _ = R.gauss_legendre(p + 1)
    h, dh = R.lagrange1d(R.lgl(p)[0], t)
    np.testing.assert_allclose(ref["Bt"], h, atol=1e-13)
    np.testing.assert_allclose(ref["Dt"], dh, atol=1e-11)
    _, w = R.prism_cubature(p)
    np.testing.assert_allclose(ref["w"], w, atol=1e-15)


@pytest.mark.parametrize("mk,p", [(lambda: config1(p=3), 3), (lambda: config2(p=4, nx=8, ny=2, nz=2), 4),
                                  (lambda: config3(p=2, n=4, nz=2), 2), (lambda: config3(p=5, n=2, nz=2), 5),
                                  (lambda: config3(p=1, n=4, nz=3), 1)])
def test_numbering_matches_oracle(mk, p):
    """Same node set (by coordinates), same element connectivity, same Dirichlet
    set, owners = first element holding the node."""
    m = mk()
    conn, dirm, own = lib.host_numbering(m.vertices, m.prisms, m.face_tag, p)
    lev = sem.build_level(m, p)
    xyz = lib_node_xyz(m, conn, lib.reference_nodes(p))
    perm = lib_to_oracle(xyz, lev.xyz)
    np.testing.assert_array_equal(perm[conn], lev.conn)
    np.testing.assert_array_equal(dirm, lev.dirichlet[perm])
    # owner = first occurrence in element order
    seen = np.zeros(conn.max() + 1, dtype=bool)
    for e in range(conn.shape[0]):
        for n in range(conn.shape[1]):
            g = conn[e, n]
            assert own[e, n] == (not seen[g])
            seen[g] = True


@pytest.mark.parametrize("overlap", [0, 1, 2])
def test_schwarz_sets_match_oracle(overlap):
    m = config3(p=3, n=4, nz=3)
    p = 3
    conn, dirm, _ = lib.host_numbering(m.vertices, m.prisms, m.face_tag, p)
    lev = sem.build_level(m, p)
    perm = lib_to_oracle(lib_node_xyz(m, conn, lib.reference_nodes(p)), lev.xyz)
    sets, W = lib.host_schwarz(m.vertices, m.prisms, m.face_tag, p, overlap)
    osets = pmg.schwarz_sets(lev, overlap)
    for k in range(m.n_elem):
        np.testing.assert_array_equal(np.sort(perm[sets[k]]), osets[k])
    cnt = np.zeros(lev.n)
    for s in osets:
        cnt[s] += 1
    Wo = np.where(lev.dirichlet, 0.0, 1.0 / np.maximum(cnt, 1))
    np.testing.assert_allclose(W, Wo[perm], rtol=0, atol=0)


def test_host_numbering_rejects_bad_input():
    m = config1(p=2)
    bad = m.prisms.copy()
    bad[0, 0] = 10 ** 6
    with pytest.raises(lib.SemError):
        lib.host_numbering(m.vertices, bad, m.face_tag, 2)
    tags = m.face_tag.copy()
    tags[0, 0] = 7
    with pytest.raises(lib.SemError):
        lib.host_numbering(m.vertices, m.prisms, tags, 2)


@pytest.mark.parametrize("p,overlap", [(3, 0), (3, 1), (2, 2), (4, 3)])
def test_fdm_sets_match_oracle(p, overlap):
    """FDM product subdomains H_k x V_k (reading O33): the library (prism stacking)
    and the oracle (lines found by coordinates) build the same node sets and W."""
    from oracle import fdm
    m = config3(p=p, n=4, nz=3)
    conn, dirm, _ = lib.host_numbering(m.vertices, m.prisms, m.face_tag, p)
    lev = sem.build_level(m, p)
    perm = lib_to_oracle(lib_node_xyz(m, conn, lib.reference_nodes(p)), lev.xyz)
    sets, W = lib.host_fdm(m.vertices, m.prisms, m.face_tag, p, overlap,
                           node_xyz=m.node_xyz(lib.reference_nodes(m.p)))
    osets, reg = pmg.hybrid_sets(m, lev, overlap)
    assert reg.all()
    cnt = np.zeros(lev.n)
    for k, ids in enumerate(osets):
        np.testing.assert_array_equal(np.sort(perm[sets[k]]), ids)
        cnt[ids] += 1
    Wo = np.where(lev.dirichlet, 0.0, 1.0 / np.maximum(cnt, 1))
    np.testing.assert_allclose(W, Wo[perm], rtol=0, atol=0)


def test_fdm_rejects_unlayered_mesh():
    """Two prisms on the same bottom triangle: not a stack of layers."""
    m = config1(p=2, nx=1, ny=1, nz=2)
    prisms = m.prisms.copy()
    prisms[1, :3] = prisms[0, :3]
    with pytest.raises(lib.SemError):
        lib.host_fdm(m.vertices, prisms, m.face_tag, 2, 1)


@pytest.mark.parametrize("p", [2, 3])
def test_hybrid_sets_match_oracle_on_hull_mesh(p):
    """Config-5 construction (hull, graded jittered Delaunay, 5/8-layer columns):
    the library's FDM/dense split (reading O35), node sets and W equal the oracle's."""
    from workloads.config5 import config5
    m = config5(p=p, hf=0.5, Lx=16.0, Ly=10.0)
    conn, dirm, _ = lib.host_numbering(m.vertices, m.prisms, m.face_tag, p)
    lev = sem.build_level(m, p)
    perm = lib_to_oracle(lib_node_xyz(m, conn, lib.reference_nodes(p)), lev.xyz)
    sets, W = lib.host_fdm(m.vertices, m.prisms, m.face_tag, p, 1, node_xyz=m.node_xyz(lib.reference_nodes(p)))
    osets, reg = pmg.hybrid_sets(m, lev, 1)
    assert 0 < (~reg).sum() < len(reg)
    cnt = np.zeros(lev.n)
    for k, ids in enumerate(osets):
        np.testing.assert_array_equal(np.sort(perm[sets[k]]), ids)
        cnt[ids] += 1
    Wo = np.where(lev.dirichlet, 0.0, 1.0 / np.maximum(cnt, 1))
    np.testing.assert_allclose(W, Wo[perm], rtol=0, atol=0)
