"""ctypes marshalling for include/sem_pmg.h (names follow the C ABI)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

# SEM_PMG_LIB: an alternative build of the same library (A/B timing tools only)
LIB_PATH = os.environ.get("SEM_PMG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsem_pmg.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build the CUDA library first "
                      "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)

_dp = C.POINTER(C.c_double)


class SemMesh(C.Structure):
    _fields_ = [("n_vert", C.c_int32), ("xyz", _dp), ("n_prism", C.c_int32),
                ("prism", C.POINTER(C.c_int32)), ("face_tag", C.POINTER(C.c_uint8)),
                ("node_xyz", _dp), ("part", C.POINTER(C.c_int32))]


class SemOpts(C.Structure):
    _fields_ = [("nu1", C.c_int), ("nu2", C.c_int), ("overlap", C.c_int), ("literal_smoother", C.c_int),
                ("outer", C.c_int), ("levels", C.POINTER(C.c_int)), ("n_levels", C.c_int),
                ("atol", C.c_double), ("imax", C.c_int), ("stream", C.c_void_p), ("device", C.c_int),
                ("verbose", C.c_int), ("apply_kernel", C.c_int), ("coarse_solver", C.c_int),
                ("coarse_rtol", C.c_double), ("coarse_maxit", C.c_int), ("nranks", C.c_int), ("rank", C.c_int),
                ("nccl_id", C.c_void_p), ("local_solve", C.c_int),
                ("mixed_precision", C.c_int), ("deterministic", C.c_int), ("pz", C.c_int),
                ("levels_z", C.POINTER(C.c_int)), ("coarse_agg", C.c_int)]


class SemReport(C.Structure):
    _fields_ = [("iters", C.c_int), ("vcycles", C.c_int), ("converged", C.c_int), ("rel_res", C.c_double),
                ("q_mean", C.c_double), ("t_ms", C.c_double), ("norm_f", C.c_double), ("wu", C.c_double),
                ("coarse_iters", C.c_int),
                ("n_hist", C.c_int),
                ("res_hist", C.c_double * 256)]

    def as_dict(self):
        return dict(iters=self.iters, vcycles=self.vcycles, converged=bool(self.converged),
                    rel_res=self.rel_res, q_mean=self.q_mean, t_ms=self.t_ms, norm_f=self.norm_f, wu=self.wu,
                    coarse_iters=self.coarse_iters,
                    res_hist=list(self.res_hist[: self.n_hist]))


class SemInfo(C.Structure):
    _fields_ = [("n_dof", C.c_int64), ("n_free", C.c_int64), ("n_elem", C.c_int64), ("n_levels", C.c_int),
                ("level_p", C.c_int * 16), ("level_n_dof", C.c_int64 * 16), ("level_n_free", C.c_int64 * 16),
                ("schwarz_bytes", C.c_int64 * 16), ("schwarz_nk_sum", C.c_int64 * 16),
                ("schwarz_packed", C.c_int64 * 16), ("coarse_n", C.c_int64), ("device_bytes", C.c_int64),
                ("setup_ms", C.c_double), ("smoother_kernel", C.c_int * 16), ("smoother_mt", C.c_int * 16),
                ("level_pz", C.c_int * 16), ("coarse_agg", C.c_int)]


SMOOTHER_KERNELS = {0: "coarse", 1: "k_schwarz", 2: "k_fdm_warp<MT,1>", 3: "k_fdm_warp<MT,2>", 4: "k_fdm_cta<MT>",
                    5: "k_fdm_col", 6: "k_fdm"}


_vp = C.c_void_p
_lib.sem_default_opts.argtypes = [C.POINTER(SemOpts)]
_lib.sem_reference_nodes.argtypes = [C.c_int, _dp]
_lib.sem_reference_nodes_pq.argtypes = [C.c_int, C.c_int, _dp]
_lib.sem_setup.argtypes = [C.POINTER(SemMesh), C.c_int, C.POINTER(SemOpts), C.POINTER(_vp)]
_lib.sem_get_info.argtypes = [_vp, C.POINTER(SemInfo)]
_lib.sem_node_xyz.argtypes = [_vp, C.c_int, _vp, C.c_int]
_lib.sem_dirichlet_mask.argtypes = [_vp, C.c_int, _vp, C.c_int]
_lib.sem_apply_laplace.argtypes = [_vp, _vp, _vp, C.c_int, C.c_int]
_lib.pmg_vcycle.argtypes = [_vp, _vp, _vp]
_lib.laplace_solve.argtypes = [_vp, _vp, _vp, C.c_double, _vp, C.POINTER(SemReport)]
_lib.laplace_solve_host.argtypes = [_vp, _vp, _vp, C.c_double, _vp, C.POINTER(SemReport)]
_lib.laplace_solve_guess.argtypes = [_vp, _vp, _vp, C.c_double, _vp, C.POINTER(SemReport)]
_lib.laplace_solve_condensed.argtypes = [_vp, _vp, _vp, C.c_double, _vp, C.c_int, C.POINTER(SemReport)]
_lib.sem_condensed_info.argtypes = [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int64)]
_lib.sem_update_geometry.argtypes = [_vp, _dp, C.c_int]
_lib.sem_prolong.argtypes = [_vp, C.c_int, _vp, _vp]
_lib.sem_restrict.argtypes = [_vp, C.c_int, _vp, _vp]
_lib.sem_schwarz.argtypes = [_vp, C.c_int, _vp, _vp, C.c_int]
_lib.sem_coarse_solve.argtypes = [_vp, _vp, _vp]
_lib.sem_nccl_unique_id.argtypes = [_vp]
_lib.sem_fnpf_init.argtypes = [_vp, _dp, C.c_int, C.POINTER(C.c_int64)]
_lib.sem_fnpf_surface_nodes.argtypes = [_vp, _vp]
_lib.fnpf_rhs.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, C.c_double, C.c_int, C.POINTER(SemReport)]
_lib.fnpf_erk4_step.argtypes = [_vp, _vp, _vp, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_int)]
_lib.sem_bench_kernel.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
_lib.sem_launch_count.argtypes = [_vp, C.c_int]
_lib.sem_launch_count.restype = C.c_int64
_lib.sem_destroy.argtypes = [_vp]
_lib.sem_strerror.argtypes = [C.c_int]
_lib.sem_strerror.restype = C.c_char_p
_lib.sem_last_error.restype = C.c_char_p

_lib.sem_host_numbering.argtypes = [C.POINTER(SemMesh), C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                    _vp, _vp, _vp]
_lib.sem_host_schwarz.argtypes = [C.POINTER(SemMesh), C.c_int, C.c_int, C.POINTER(C.c_int64), _vp, _vp, _vp]
_lib.sem_host_fdm.argtypes = [C.POINTER(SemMesh), C.c_int, C.c_int, C.POINTER(C.c_int64), _vp, _vp, _vp]
_lib.sem_host_reference.argtypes = [C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.sem_host_partition.argtypes = [C.POINTER(SemMesh), C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp,
                                    _vp, _vp, _vp]

EXPORTS = ["laplace_solve_condensed", "sem_condensed_info", "sem_reference_nodes_pq", "sem_fnpf_init", "sem_fnpf_surface_nodes", "fnpf_rhs", "fnpf_erk4_step", "laplace_solve_guess", "sem_update_geometry", "sem_host_fdm", "sem_bench_kernel", "sem_host_partition", "sem_nccl_unique_id", "sem_host_numbering", "sem_host_schwarz", "sem_host_reference", "sem_default_opts", "sem_reference_nodes", "sem_setup", "sem_get_info", "sem_node_xyz",
           "sem_dirichlet_mask", "sem_apply_laplace", "pmg_vcycle", "laplace_solve", "laplace_solve_host",
           "sem_prolong", "sem_restrict", "sem_schwarz", "sem_coarse_solve", "sem_launch_count",
           "sem_destroy", "sem_strerror", "sem_last_error"]

SEM_ENOTCONV = -5


class SemError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        super().__init__(f"{where}: {_lib.sem_strerror(code).decode()} ({_lib.sem_last_error().decode()})")


def _check(code, where):
    if code != 0:
        raise SemError(code, where)


def default_opts() -> dict:
    o = SemOpts()
    _lib.sem_default_opts(C.byref(o))
    return {k: getattr(o, k) for k, _ in SemOpts._fields_ if k not in ("levels", "stream", "levels_z")}


def reference_nodes(p: int, pz: int | None = None) -> np.ndarray:
    """Reference coordinates of the library's local nodes of P_p(triangle) x P_pz(t)."""
    q = p if pz is None else pz
    n = (p + 1) * (p + 2) // 2 * (q + 1)
    out = np.zeros((n, 3))
    if q == p:
        _check(_lib.sem_reference_nodes(p, out.ctypes.data_as(_dp)), "sem_reference_nodes")
    else:
        _check(_lib.sem_reference_nodes_pq(p, q, out.ctypes.data_as(_dp)), "sem_reference_nodes_pq")
    return out


def _mesh_struct(vertices, prisms, face_tag, node_xyz=None):
    keep = [np.ascontiguousarray(vertices, dtype=np.float64), np.ascontiguousarray(prisms, dtype=np.int32),
            np.ascontiguousarray(face_tag, dtype=np.uint8)]
    m = SemMesh()
    m.n_vert = keep[0].shape[0]
    m.xyz = keep[0].ctypes.data_as(_dp)
    m.n_prism = keep[1].shape[0]
    m.prism = keep[1].ctypes.data_as(C.POINTER(C.c_int32))
    m.face_tag = keep[2].ctypes.data_as(C.POINTER(C.c_uint8))
    if node_xyz is not None:
        keep.append(np.ascontiguousarray(node_xyz, dtype=np.float64))
        m.node_xyz = keep[3].ctypes.data_as(_dp)
    return m, keep


def host_numbering(vertices, prisms, face_tag, p):
    """sem_host_numbering: (conn [E][N], dirichlet [n] bool, owner [E][N] bool)."""
    m, keep = _mesh_struct(vertices, prisms, face_tag)
    n, nf = C.c_int64(), C.c_int64()
    _check(_lib.sem_host_numbering(C.byref(m), p, C.byref(n), C.byref(nf), None, None, None), "sem_host_numbering")
    E = keep[1].shape[0]
    N = (p + 1) ** 2 * (p + 2) // 2
    conn = np.zeros((E, N), dtype=np.int32)
    dirm = np.zeros(n.value, dtype=np.uint8)
    own = np.zeros((E, N), dtype=np.uint8)
    _check(_lib.sem_host_numbering(C.byref(m), p, None, None, C.c_void_p(conn.ctypes.data),
                                   C.c_void_p(dirm.ctypes.data), C.c_void_p(own.ctypes.data)), "sem_host_numbering")
    return conn, dirm.astype(bool), own.astype(bool)


def host_schwarz(vertices, prisms, face_tag, p, overlap):
    """sem_host_schwarz: (list of subdomain node arrays, W)."""
    m, keep = _mesh_struct(vertices, prisms, face_tag)
    tot = C.c_int64()
    _check(_lib.sem_host_schwarz(C.byref(m), p, overlap, C.byref(tot), None, None, None), "sem_host_schwarz")
    E = keep[1].shape[0]
    conn, dirm, _ = host_numbering(vertices, prisms, face_tag, p)
    off = np.zeros(E + 1, dtype=np.int64)
    idx = np.zeros(tot.value, dtype=np.int32)
    W = np.zeros(dirm.size)
    _check(_lib.sem_host_schwarz(C.byref(m), p, overlap, None, C.c_void_p(off.ctypes.data),
                                 C.c_void_p(idx.ctypes.data), C.c_void_p(W.ctypes.data)), "sem_host_schwarz")
    return [idx[off[k]:off[k + 1]] for k in range(E)], W


def host_fdm(vertices, prisms, face_tag, p, overlap, node_xyz=None):
    """sem_host_fdm: (list of FDM subdomain node arrays, W)."""
    m, keep = _mesh_struct(vertices, prisms, face_tag, node_xyz)
    tot = C.c_int64()
    _check(_lib.sem_host_fdm(C.byref(m), p, overlap, C.byref(tot), None, None, None), "sem_host_fdm")
    E = keep[1].shape[0]
    _, dirm, _ = host_numbering(vertices, prisms, face_tag, p)
    off = np.zeros(E + 1, dtype=np.int64)
    idx = np.zeros(max(1, tot.value), dtype=np.int32)
    W = np.zeros(dirm.size)
    _check(_lib.sem_host_fdm(C.byref(m), p, overlap, None, C.c_void_p(off.ctypes.data),
                             C.c_void_p(idx.ctypes.data), C.c_void_p(W.ctypes.data)), "sem_host_fdm")
    return [idx[off[k]:off[k + 1]] for k in range(E)], W


def host_partition(vertices, prisms, face_tag, p, nranks, rank, level=0):
    """sem_host_partition: dict(elems, E_own, gid, owned, nbr, xidx=[per neighbour local ids])."""
    m, keep = _mesh_struct(vertices, prisms, face_tag)
    sizes = np.zeros(5, dtype=np.int64)
    vp = lambda a: C.c_void_p(a.ctypes.data)
    _check(_lib.sem_host_partition(C.byref(m), p, nranks, rank, level, vp(sizes), None, None, None, None, None, None),
           "sem_host_partition")
    elems = np.zeros(sizes[0], dtype=np.int32)
    gid = np.zeros(sizes[2], dtype=np.int32)
    owned = np.zeros(sizes[2], dtype=np.uint8)
    nbr = np.zeros(sizes[3], dtype=np.int32)
    xoff = np.zeros(sizes[3] + 1, dtype=np.int64)
    xidx = np.zeros(max(1, sizes[4]), dtype=np.int32)
    _check(_lib.sem_host_partition(C.byref(m), p, nranks, rank, level, vp(sizes), vp(elems), vp(gid), vp(owned),
                                   vp(nbr), vp(xoff), vp(xidx)), "sem_host_partition")
    return dict(elems=elems, E_own=int(sizes[1]), gid=gid, owned=owned.astype(bool), nbr=nbr.tolist(),
                xidx=[xidx[xoff[j]:xoff[j + 1]] for j in range(len(nbr))])


def host_reference(p):
    """sem_host_reference: dict of B0, Br, Bs [(p+1)^2][Nt], Bt, Dt [p+1][p+1], w [(p+1)^3]."""
    nt, qt, n1 = (p + 1) * (p + 2) // 2, (p + 1) ** 2, p + 1
    out = dict(B0=np.zeros((qt, nt)), Br=np.zeros((qt, nt)), Bs=np.zeros((qt, nt)), Bt=np.zeros((n1, n1)),
               Dt=np.zeros((n1, n1)), w=np.zeros(qt * n1))
    _check(_lib.sem_host_reference(p, *[C.c_void_p(out[k].ctypes.data) for k in ("B0", "Br", "Bs", "Bt", "Dt", "w")]),
           "sem_host_reference")
    return out


def nccl_unique_id() -> bytes:
    """sem_nccl_unique_id: 128 opaque bytes to broadcast to every rank."""
    buf = C.create_string_buffer(128)
    _check(_lib.sem_nccl_unique_id(C.cast(buf, C.c_void_p)), "sem_nccl_unique_id")
    return buf.raw


def _ptr(t):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError("expected a contiguous CUDA float64 tensor")
    return C.c_void_p(t.data_ptr())


class Solver:
    """sem_setup(mesh, p) + the compute calls of include/sem_pmg.h."""

    def __init__(self, vertices, prisms, face_tag, p: int, node_xyz=None, *, levels=None, stream=None,
                 nccl_id: bytes | None = None, part=None, **opts):
        import torch
        self._torch = torch
        o = SemOpts()
        _lib.sem_default_opts(C.byref(o))
        for k, v in opts.items():
            if not hasattr(o, k):
                raise TypeError(f"unknown option {k}")
            setattr(o, k, v)
        self._levels = None
        if levels is not None:
            # orders, or (P_xy, P_z) pairs
            pairs = [tuple(x) if not np.isscalar(x) else (int(x), int(x)) for x in levels]
            self._levels = (C.c_int * len(pairs))(*[a for a, _ in pairs])
            o.levels = self._levels
            o.n_levels = len(pairs)
            if any(not np.isscalar(x) for x in levels):
                self._levels_z = (C.c_int * len(pairs))(*[b for _, b in pairs])
                o.levels_z = self._levels_z
        self._nccl = None
        if nccl_id is not None:
            self._nccl = C.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = C.cast(self._nccl, C.c_void_p)
        if stream is None:
            stream = torch.cuda.current_stream()
        self.stream = stream
        o.stream = C.c_void_p(stream.cuda_stream)
        o.device = torch.cuda.current_device() if o.device < 0 else o.device
        self._keep = [np.ascontiguousarray(vertices, dtype=np.float64),
                      np.ascontiguousarray(prisms, dtype=np.int32),
                      np.ascontiguousarray(face_tag, dtype=np.uint8)]
        m = SemMesh()
        m.n_vert = self._keep[0].shape[0]
        m.xyz = self._keep[0].ctypes.data_as(_dp)
        m.n_prism = self._keep[1].shape[0]
        m.prism = self._keep[1].ctypes.data_as(C.POINTER(C.c_int32))
        m.face_tag = self._keep[2].ctypes.data_as(C.POINTER(C.c_uint8))
        if node_xyz is not None:
            nx = np.ascontiguousarray(node_xyz, dtype=np.float64)
            self._keep.append(nx)
            m.node_xyz = nx.ctypes.data_as(_dp)
        if part is not None:
            pa = np.ascontiguousarray(part, dtype=np.int32)
            self._keep.append(pa)
            m.part = pa.ctypes.data_as(C.POINTER(C.c_int32))
        self._ctx = C.c_void_p()
        _check(_lib.sem_setup(C.byref(m), p, C.byref(o), C.byref(self._ctx)), "sem_setup")
        self._keep = None
        self.p = p
        inf = SemInfo()
        _check(_lib.sem_get_info(self._ctx, C.byref(inf)), "sem_get_info")
        self.info = dict(n_dof=inf.n_dof, n_free=inf.n_free, n_elem=inf.n_elem, n_levels=inf.n_levels,
                         level_p=list(inf.level_p[: inf.n_levels]),
                         level_pz=list(inf.level_pz[: inf.n_levels]), coarse_agg=inf.coarse_agg,
                         level_n_dof=list(inf.level_n_dof[: inf.n_levels]),
                         level_n_free=list(inf.level_n_free[: inf.n_levels]),
                         schwarz_bytes=list(inf.schwarz_bytes[: inf.n_levels]),
                         schwarz_nk_sum=list(inf.schwarz_nk_sum[: inf.n_levels]),
                         schwarz_packed=list(inf.schwarz_packed[: inf.n_levels]),
                         coarse_n=inf.coarse_n, device_bytes=inf.device_bytes, setup_ms=inf.setup_ms,
                         smoother_kernel=[SMOOTHER_KERNELS[k] for k in inf.smoother_kernel[: inf.n_levels]],
                         smoother_mt=list(inf.smoother_mt[: inf.n_levels]))

    # ---------------------------------------------------------------- helpers
    def n_dof(self, level=0):
        return self.info["level_n_dof"][level]

    def empty(self, level=0):
        return self._torch.zeros(self.n_dof(level), dtype=self._torch.float64, device="cuda")

    def node_xyz(self, level=0) -> np.ndarray:
        out = np.zeros((self.n_dof(level), 3))
        _check(_lib.sem_node_xyz(self._ctx, level, C.c_void_p(out.ctypes.data), 0), "sem_node_xyz")
        return out

    def dirichlet_mask(self, level=0) -> np.ndarray:
        out = np.zeros(self.n_dof(level), dtype=np.uint8)
        _check(_lib.sem_dirichlet_mask(self._ctx, level, C.c_void_p(out.ctypes.data), 0), "sem_dirichlet_mask")
        return out.astype(bool)

    # ---------------------------------------------------------------- compute
    def apply(self, u, level=0, masked=False, out=None):
        y = self.empty(level) if out is None else out
        _check(_lib.sem_apply_laplace(self._ctx, _ptr(u), _ptr(y), level, int(masked)), "sem_apply_laplace")
        return y

    def vcycle(self, r, out=None):
        z = self.empty(0) if out is None else out
        _check(_lib.pmg_vcycle(self._ctx, _ptr(r), _ptr(z)), "pmg_vcycle")
        return z

    def solve(self, dirichlet_phi, tol, rhs=None, out=None, check=True):
        phi = self.empty(0) if out is None else out
        rep = SemReport()
        code = _lib.laplace_solve(self._ctx, None if rhs is None else _ptr(rhs), _ptr(dirichlet_phi), tol,
                                  _ptr(phi), C.byref(rep))
        if check and code not in (0,):
            raise SemError(code, "laplace_solve")
        return phi, rep.as_dict()

    def solve_guess(self, dirichlet_phi, tol, phi, rhs=None, check=True):
        """laplace_solve_guess: phi (CUDA tensor) is the initial guess and the output."""
        rep = SemReport()
        code = _lib.laplace_solve_guess(self._ctx, None if rhs is None else _ptr(rhs), _ptr(dirichlet_phi), tol,
                                        _ptr(phi), C.byref(rep))
        if check and code != 0:
            raise SemError(code, "laplace_solve_guess")
        return phi, rep.as_dict()

    def solve_condensed(self, dirichlet_phi, tol, rhs=None, out=None, guess=False, check=True):
        """laplace_solve_condensed (static condensation, NEXT-3): with guess=True `out` holds the
        initial guess (read on free skeleton nodes)."""
        phi = self.empty(0) if out is None else out
        rep = SemReport()
        code = _lib.laplace_solve_condensed(self._ctx, None if rhs is None else _ptr(rhs), _ptr(dirichlet_phi), tol,
                                            _ptr(phi), int(bool(guess)), C.byref(rep))
        if check and code != 0:
            raise SemError(code, "laplace_solve_condensed")
        return phi, rep.as_dict()

    def condensed_info(self):
        """sem_condensed_info: (interior, skeleton) nodes per element and the factor bytes."""
        ni, nb, by = C.c_int(), C.c_int(), C.c_int64()
        _check(_lib.sem_condensed_info(self._ctx, C.byref(ni), C.byref(nb), C.byref(by)), "sem_condensed_info")
        return ni.value, nb.value, by.value

    def update_geometry(self, node_xyz, strategy=1):
        """sem_update_geometry: new nodal map [n_prism][N(p)][3] (same topology)."""
        nx = np.ascontiguousarray(node_xyz, dtype=np.float64)
        _check(_lib.sem_update_geometry(self._ctx, nx.ctypes.data_as(_dp), int(strategy)), "sem_update_geometry")

    # ---------------------------------------------------------------- FNPF stages (NEXT-4)
    def fnpf_init(self, node_xyz, strategy=1):
        """sem_fnpf_init: returns the library node ids of the free-surface nodes."""
        nx = np.ascontiguousarray(node_xyz, dtype=np.float64)
        ns = C.c_int64()
        _check(_lib.sem_fnpf_init(self._ctx, nx.ctypes.data_as(_dp), int(strategy), C.byref(ns)), "sem_fnpf_init")
        ids = np.zeros(ns.value, dtype=np.int32)
        _check(_lib.sem_fnpf_surface_nodes(self._ctx, C.c_void_p(ids.ctypes.data)), "sem_fnpf_surface_nodes")
        return ids

    def fnpf_rhs(self, eta, phis, tol, linear=False):
        """fnpf_rhs: (deta, dphis, w, report) for the surface state (CUDA tensors)."""
        de, dp, w = (self._torch.empty_like(eta) for _ in range(3))
        rep = SemReport()
        code = _lib.fnpf_rhs(self._ctx, _ptr(eta), _ptr(phis), _ptr(de), _ptr(dp), _ptr(w), tol, int(linear),
                             C.byref(rep))
        if code not in (0, SEM_ENOTCONV):
            raise SemError(code, "fnpf_rhs")
        return de, dp, w, rep.as_dict()

    def fnpf_erk4_step(self, eta, phis, dt, tol, linear=False):
        """fnpf_erk4_step: eta, phis (CUDA tensors) advanced in place; returns the PCG iterations."""
        it = C.c_int()
        _check(_lib.fnpf_erk4_step(self._ctx, _ptr(eta), _ptr(phis), dt, tol, int(linear), C.byref(it)),
               "fnpf_erk4_step")
        return it.value

    def solve_host(self, dirichlet_phi_host, tol, out_host, rhs_host=None):
        """Host buffers (numpy arrays or pinned CPU tensors), copies inside the call."""
        def hp(a):
            if a is None:
                return None
            if isinstance(a, np.ndarray):
                return C.c_void_p(a.ctypes.data)
            return C.c_void_p(a.data_ptr())
        rep = SemReport()
        code = _lib.laplace_solve_host(self._ctx, hp(rhs_host), hp(dirichlet_phi_host), tol, hp(out_host),
                                       C.byref(rep))
        if code != 0:
            raise SemError(code, "laplace_solve_host")
        return rep.as_dict()

    def prolong(self, level, uc, uf):
        _check(_lib.sem_prolong(self._ctx, level, _ptr(uc), _ptr(uf)), "sem_prolong")
        return uf

    def restrict(self, level, rf, out=None):
        rc = self.empty(level + 1) if out is None else out
        _check(_lib.sem_restrict(self._ctx, level, _ptr(rf), _ptr(rc)), "sem_restrict")
        return rc

    def schwarz(self, level, r, u, transpose=False):
        _check(_lib.sem_schwarz(self._ctx, level, _ptr(r), _ptr(u), int(transpose)), "sem_schwarz")
        return u

    def coarse_solve(self, r, out=None):
        z = self.empty(self.info["n_levels"] - 1) if out is None else out
        _check(_lib.sem_coarse_solve(self._ctx, _ptr(r), _ptr(z)), "sem_coarse_solve")
        return z

    def bench_kernel(self, kernel: str, level=0, reps=20):
        """sem_bench_kernel: (mean microseconds, algorithmic bytes) of 'schwarz', 'apply' or 'coarse'."""
        us, b = C.c_double(), C.c_double()
        _check(_lib.sem_bench_kernel(self._ctx, {"schwarz": 0, "apply": 1, "coarse": 2}[kernel], level, reps, C.byref(us),
                                     C.byref(b)), "sem_bench_kernel")
        return us.value, b.value

    def launches(self, reset=False) -> int:
        return int(_lib.sem_launch_count(self._ctx, int(reset)))

    def close(self):
        if getattr(self, "_ctx", None) is not None and self._ctx.value:
            _lib.sem_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
