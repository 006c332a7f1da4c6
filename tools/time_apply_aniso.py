"""Operator apply of anisotropic (P_xy, P_z) levels (k_apply_pq) next to the
isotropic kernels on the config-3 construction: mean us per apply (CUDA events) and the
algorithmic-byte fraction of HBM.  Prints one JSON line per (p, pz)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_00705_b200 as lib  # noqa: E402
from workloads import config3  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
for p, pz in [(5, 5), (5, 3), (5, 2), (4, 2), (3, 3), (3, 1)]:
    m = config3(p=p)
    m.pz = pz
    # anisotropic levels take exact dense local solves only (FDM stays isotropic)
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, p, node_xyz=m.node_xyz(lib.reference_nodes(p, pz)), pz=pz,
                   local_solve=0 if pz != p else 1)
    us, b = s.bench_kernel("apply", 0, 20)
    print(json.dumps({"p": p, "pz": pz, "n_dof": s.info["n_dof"], "us": us, "alg_bytes": b,
                      "frac_hbm": b / us / 1e3 / peak, "MDOF_s": s.info["n_dof"] / us}), flush=True)
    s.close()
