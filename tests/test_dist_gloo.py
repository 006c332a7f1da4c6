"""World-size-2 gloo test (CPU) of the partitioned solve's host logic: the
library's column partition, local numberings, owned sets and exchange lists
(sem_host_partition) reproduce the global operator when every rank applies
only its owned elements and the partial sums are exchanged exactly as the GPU
transport does (pack -> send/recv -> add); owned-node dot products all-reduce
to the global ones.  Element matrices come from the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2009_00705_b200 as lib
        from oracle import refelem as R, sem
        from tests._mapping import lib_node_xyz, lib_to_oracle
        from workloads.configs import basin
        m = basin("gloo", 3, 32.0 * 6 / 64, 6, 2, seed=3)
        p = m.p
        lev = sem.build_system(m, p)
        Ae = sem.element_matrices(lev.G, p)
        conn_lib, _, _ = lib.host_numbering(m.vertices, m.prisms, m.face_tag, p)
        perm = lib_to_oracle(lib_node_xyz(m, conn_lib, lib.reference_nodes(p)), lev.xyz)  # lib id -> oracle id
        part = lib.host_partition(m.vertices, m.prisms, m.face_tag, p, world, rank)
        u = np.random.default_rng(7).uniform(-1, 1, lev.n)       # oracle numbering, identical on all ranks
        y_full = lev.A @ u
        # local partial sums of the owned elements, in the rank's local numbering
        gid = part["gid"]
        loc_of = {int(g): i for i, g in enumerate(gid)}
        y_loc = np.zeros(len(gid))
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(perm))                           # oracle id -> lib id
        for e in part["elems"][: part["E_own"]]:
            ye = Ae[e] @ u[lev.conn[e]]
            for a, oid in enumerate(lev.conn[e]):
                y_loc[loc_of[int(inv[oid])]] += ye[a]
        # exchange: pack shared entries per neighbour, send/recv, add
        reqs, recv = [], []
        for q, idx in zip(part["nbr"], part["xidx"]):
            buf = torch.from_numpy(y_loc[idx].copy())
            rb = torch.empty_like(buf)
            reqs.append(dist.isend(buf, q))
            reqs.append(dist.irecv(rb, q))
            recv.append((idx, rb))
        for r in reqs:
            r.wait()
        for idx, rb in recv:
            np.add.at(y_loc, idx, rb.numpy())
        err = np.abs(y_loc - y_full[perm[gid]]).max() / np.abs(y_full).max()
        # owned-node dot all-reduced == global dot
        own = part["owned"]
        d = torch.tensor([float(np.sum(y_loc[own] * u[perm[gid]][own]))], dtype=torch.float64)
        dist.all_reduce(d)
        derr = abs(d.item() - float(y_full @ u)) / abs(float(y_full @ u))
        cnt = torch.tensor([int(own.sum())])
        dist.all_reduce(cnt)
        results[rank] = (float(err), float(derr), int(cnt.item()), lev.n, part["E_own"], len(part["elems"]))
    finally:
        dist.destroy_process_group()


def test_partitioned_apply_and_dots_gloo():
    port = _free_port()
    # spawn, not fork: the parent may already hold OpenMP / CUDA-runtime threads
    # (libsem_pmg loaded by earlier tests), and a forked manager deadlocks on them
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(WORLD, port, results), nprocs=WORLD, join=True)
    assert len(results) == WORLD
    for r in range(WORLD):
        err, derr, cnt, n, e_own, e_held = results[r]
        assert err <= 1e-13, (r, err)
        assert derr <= 1e-13, (r, derr)
        assert cnt == n            # every global node owned exactly once
        assert e_held > e_own > 0  # halo elements present
    assert sum(results[r][4] for r in range(WORLD)) == 144  # 6x6 quads x 2 triangles x 2 layers


def _worker_smoother(rank, world, port, results):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2009_00705_b200 as lib
        from oracle import pmg, sem
        from tests._mapping import lib_node_xyz, lib_to_oracle
        from workloads.configs import basin
        m = basin("gloo_s", 3, 32.0 * 6 / 64, 6, 2, seed=3)
        p = m.p
        lev = sem.build_system(m, p)
        F = lev.free
        sm = pmg.build_smoother(lev, lev.A[F][:, F].tocsr(), overlap=1)
        conn_lib, _, _ = lib.host_numbering(m.vertices, m.prisms, m.face_tag, p)
        perm = lib_to_oracle(lib_node_xyz(m, conn_lib, lib.reference_nodes(p)), lev.xyz)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(perm))                          # oracle id -> lib id
        part = lib.host_partition(m.vertices, m.prisms, m.face_tag, p, world, rank)
        gid = part["gid"]
        loc_of = {int(g): i for i, g in enumerate(gid)}
        fid = np.full(lev.n, -1)
        fid[F] = np.arange(len(F))
        r = np.random.default_rng(9).uniform(-1, 1, len(F))       # free-node residual, all ranks
        z_full = sm.apply(r)                                      # S^-1 r = W sum_k R_k^T B_k^-1 R_k r
        # this rank: partial sums of its owned subdomains (element k's subdomain), local numbering
        z_loc = np.zeros(len(gid))
        for e in part["elems"][: part["E_own"]]:
            I = sm.sets[e]
            zk = sm.inv[e] @ r[I]
            for a, f in enumerate(I):
                z_loc[loc_of[int(inv[F[f]])]] += zk[a]
        reqs, recv = [], []
        for q, idx in zip(part["nbr"], part["xidx"]):
            buf = torch.from_numpy(z_loc[idx].copy())
            rb = torch.empty_like(buf)
            reqs.append(dist.isend(buf, q))
            reqs.append(dist.irecv(rb, q))
            recv.append((idx, rb))
        for rq in reqs:
            rq.wait()
        for idx, rb in recv:
            np.add.at(z_loc, idx, rb.numpy())
        # x W on every held free node, compare with the global smoother
        oid = perm[gid]
        free = fid[oid] >= 0
        got = z_loc[free] * sm.W[fid[oid[free]]]
        ref = z_full[fid[oid[free]]]
        results[rank] = float(np.abs(got - ref).max() / np.abs(z_full).max())
    finally:
        dist.destroy_process_group()


def test_partitioned_schwarz_sweep_gloo():
    """The partitioned additive-Schwarz sweep (eq 4.4): each rank solves only its
    owned subdomains on its held nodes; one neighbour sum-exchange of the shared
    entries (the GPU transport's pack / send-recv / add) then W reproduces the
    global S^-1 r on every held node -- the halo covers every subdomain."""
    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.spawn(_worker_smoother, args=(WORLD, port, results), nprocs=WORLD, join=True)
    assert len(results) == WORLD
    for r in range(WORLD):
        assert results[r] <= 1e-13, (r, results[r])
