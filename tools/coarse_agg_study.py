"""Two-level aggregate correction of the iterative P=1 solve (reading O44): inner iterations
and solve time vs the aggregate count, on config 5 (FDM hybrid, the bench variant) and
config 4 at p = 2, 3 (FDM refined, the sweep's fastest).  One JSON line per case.
Usage: python tools/coarse_agg_study.py [counts, default 0,256,1024,2048]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2009_00705_b200 as lib
from workloads import config4
from workloads.config5 import config5

counts = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,256,1024,2048").split(",")]
for name, mk, p, kw in [("config5", config5, 6, dict(local_solve=1)),
                        ("config4", lambda: config4(2), 2, dict(local_solve=1, overlap=-1)),
                        ("config4", lambda: config4(3), 3, dict(local_solve=1, overlap=-1))]:
    m = mk()
    nodes = m.node_xyz(lib.reference_nodes(p))
    for na in counts:
        t0 = time.time()
        s = lib.Solver(m.vertices, m.prisms, m.face_tag, p, node_xyz=nodes, coarse_agg=na, **kw)
        st = time.time() - t0
        xyz = s.node_xyz(0)
        phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
        s.solve(phiD, 1e-8, check=False)
        best = None
        for _ in range(3):
            _, rep = s.solve(phiD, 1e-8, check=False)
            if best is None or rep["t_ms"] < best["t_ms"]:
                best = rep
        print(json.dumps(dict(config=name, p=p, coarse_agg=s.info["coarse_agg"], coarse_n=s.info["coarse_n"],
                              iters=best["iters"], coarse_iters=best["coarse_iters"], ms=round(best["t_ms"], 2),
                              MDOF_s=round(s.info["n_free"] / best["t_ms"] / 1e3, 2), setup_s=round(st, 1),
                              converged=best["converged"])), flush=True)
        s.close()
        del s
        torch.cuda.empty_cache()
