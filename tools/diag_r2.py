"""Round-2 diagnostics on the GPU box: residual history of the p=6 hull replica
solve; inner coarse iterations (line-Jacobi PCG) on config 4 p=2 and config 5."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2009_00705_b200 as lib
from workloads.config5 import config5
from workloads import config4


def run(m, tol, **kw):
    t0 = time.time()
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)), **kw)
    st = time.time() - t0
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    s.solve(phiD, tol, check=False)
    torch.cuda.synchronize()
    t0 = time.time()
    phi, rep = s.solve(phiD, tol, check=False)
    torch.cuda.synchronize()
    out = dict(name=m.name, setup_s=st, wall_s=time.time() - t0, t_ms=rep["t_ms"], iters=rep["iters"],
               coarse_iters=rep["coarse_iters"], rel_res=rep["rel_res"], converged=rep["converged"],
               hist=rep["res_hist"], coarse_n=s.info["coarse_n"], launches=s.launches())
    s.close()
    del s
    torch.cuda.empty_cache()
    return out


which = sys.argv[1:] or ["hull6", "c4p2", "c5"]
for w in which:
    if w == "hull6":
        r = run(config5(p=6, hf=0.5, Lx=10.0, Ly=4.0), 1e-13, local_solve=1)
    elif w == "c4p2":
        r = run(config4(2), 1e-8, local_solve=1)
    elif w == "c5":
        r = run(config5(), 1e-8, local_solve=1)
    print(json.dumps(r), flush=True)
