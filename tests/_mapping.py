"""Test helpers: map the library's node numbering onto the oracle's by
coordinates (SURVEY §8(c) parity protocol step 1)."""
import numpy as np
from scipy.spatial import cKDTree


def lib_to_oracle(xyz_lib: np.ndarray, xyz_orc: np.ndarray, tol: float = 1e-5) -> np.ndarray:
    """perm with xyz_orc[perm[i]] == xyz_lib[i]; asserts a bijection.

    On coarse levels of curved meshes the library reports node positions on the
    finest-order nodal map while the oracle labels them with the exact
    sigma-map, so positions differ by the map's interpolation error (~1e-6);
    node spacing is >= 1e-3, so 1e-5 is unambiguous and the bijection is checked."""
    tree = cKDTree(xyz_orc)
    d, perm = tree.query(xyz_lib)
    assert d.max() < tol, f"unmatched node (distance {d.max():.3g})"
    assert len(np.unique(perm)) == len(perm) == len(xyz_orc), "numberings are not in bijection"
    return perm


def lib_node_xyz(mesh, conn: np.ndarray, rst: np.ndarray) -> np.ndarray:
    pts = mesh.node_xyz(rst)
    n = int(conn.max()) + 1
    xyz = np.zeros((n, 3))
    xyz[conn.ravel()] = pts.reshape(-1, 3)
    return xyz


def fine_map_xyz(mesh, level, p_fine: int) -> np.ndarray:
    """Positions of a (coarse) level's oracle nodes on the FINEST-order nodal map
    (the library's convention) instead of the exact workload map: the
    order-p_fine interpolant of each element's nodes, evaluated at the level's
    reference nodes (oracle basis; test-side helper)."""
    from oracle import refelem as R
    rst_c, _ = R.prism_nodes(level.p)
    rst_f, _ = R.prism_nodes(p_fine)
    X = mesh.node_xyz(rst_f)                               # [E][Nf][3]
    V, _ = R.prism_basis(p_fine, rst_c)                    # [Nc][Nf]
    pts = np.einsum("cf,efi->eci", V, X)
    out = np.zeros((level.n, 3))
    out[level.conn.ravel()] = pts.reshape(-1, 3)
    return out


# ---------------------------------------------------------------- whole-vector streamed oracle apply
_POOL_STATE = {}


def _streamed_chunk(el):
    """Oracle y_e = D^T (G (.) D u_e) of the elements `el` (oracle/sem.py apply_streamed),
    the element nodes identified in the library numbering by coordinates."""
    from oracle import sem, refelem as R
    st = _POOL_STATE
    mesh, p, tree, U = st["mesh"], st["p"], st["tree"], st["U"]
    rst, _ = R.prism_nodes(p)
    X = mesh.node_xyz(rst, el)                            # [e][N][3] the workload's nodal map
    d, ids = tree.query(X.reshape(-1, 3))
    assert d.max() < 1e-9, f"element node not found in the library numbering ({d.max():.3g})"
    uniq, loc = np.unique(ids, return_inverse=True)
    lev = sem.Level(p=p, conn=loc.reshape(len(el), -1), xyz=np.empty((len(uniq), 3)),
                    dirichlet=np.zeros(len(uniq), dtype=bool))
    y = sem.apply_streamed(mesh, lev, U[uniq], elems=el, chunk=len(el))
    return uniq, y


def streamed_apply_lib(mesh, p, xyz_lib, U, chunk=2048, procs=None, tree=None):
    """y = A U (raw Neumann stiffness, every row) by the oracle's streamed element
    apply, in the LIBRARY's node numbering (nodes matched by coordinates): U [n] or
    [n][k].  Element chunks run in a process pool (fork) over the host cores."""
    import multiprocessing as mp
    import os
    _POOL_STATE.update(mesh=mesh, p=p, tree=tree if tree is not None else cKDTree(xyz_lib), U=U)
    E = mesh.n_elem
    chunks = [np.arange(e0, min(E, e0 + chunk)) for e0 in range(0, E, chunk)]
    y = np.zeros(U.shape)
    procs = procs or max(1, min(32, len(os.sched_getaffinity(0))))
    try:
        if procs > 1:
            ctx = mp.get_context("fork")
            with ctx.Pool(procs) as pool:
                for uniq, yl in pool.imap_unordered(_streamed_chunk, chunks):
                    y[uniq] += yl
        else:
            for c in chunks:
                uniq, yl = _streamed_chunk(c)
                y[uniq] += yl
    finally:
        _POOL_STATE.clear()
    return y
