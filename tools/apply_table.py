"""BASELINE.md §4 apply columns: the library's operator apply (level 0, sem_bench_kernel,
CUDA events, 30 launches) on configs 1-5 (config 4 at p = 2..8), and the oracle's apply on
the box's host cores: SciPy CSR SpMV (configs 1-2, assembled) and the streamed element
apply (oracle/sem.py apply_streamed, NumPy/BLAS) on a bounded element sample (configs 3-5).
One JSON line per row."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2009_00705_b200 as lib
from workloads import config1, config2, config3, config4
from workloads.config5 import config5

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6470.8
cores = len(os.sched_getaffinity(0))
rows = [("config1", config1), ("config2", config2), ("config3", config3)] + \
       [(f"config4_p{p}", (lambda p=p: config4(p))) for p in range(2, 9)] + [("config5", config5)]
only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
for name, mk in rows:
    if only and name not in only:
        continue
    m = mk()
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)), local_solve=1)
    us, b = s.bench_kernel("apply", 0, 30)
    n = s.info["n_dof"]
    out = dict(config=name, p=m.p, n_dof=n, apply_us=us, apply_MDOF_s=n / us, apply_GBs=b / us / 1e3,
               frac_measured=b / us / 1e3 / peak, frac_8TBs=b / us / 1e3 / 8000.0)
    s.close()
    del s
    torch.cuda.empty_cache()
    # oracle on the host
    from oracle import sem
    if name in ("config1", "config2"):
        lev = sem.build_system(m, m.p)
        u = np.random.default_rng(0).uniform(-1, 1, lev.n)
        t0 = time.perf_counter(); k = 0
        while time.perf_counter() - t0 < 2.0:
            lev.A @ u; k += 1
        t = (time.perf_counter() - t0) / k
        out.update(oracle_apply="SciPy CSR SpMV (single thread)", oracle_apply_MDOF_s=lev.n / t / 1e6)
    else:
        ne = min(m.n_elem, 2048)
        el = np.arange(ne)
        from oracle import refelem as R
        rst, _ = R.prism_nodes(m.p)
        X = m.node_xyz(rst, el)
        conn = np.arange(ne * X.shape[1]).reshape(ne, -1)       # element-local numbering of the sample
        L = sem.Level(p=m.p, conn=conn, xyz=X.reshape(-1, 3), dirichlet=np.zeros(conn.size, dtype=bool))
        u = np.random.default_rng(0).uniform(-1, 1, conn.size)
        t0 = time.perf_counter()
        sem.apply_streamed(m, L, u, elems=el, chunk=ne)
        t = time.perf_counter() - t0
        dof_per_elem = n / m.n_elem
        out.update(oracle_apply=f"streamed element apply (NumPy/BLAS) on {ne} elements",
                   oracle_apply_MDOF_s=ne * dof_per_elem / t / 1e6)
    out["host_cores"] = cores
    print(json.dumps(out), flush=True)
