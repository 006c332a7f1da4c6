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
