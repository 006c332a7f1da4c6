"""Config 4 at p = 4 (the o = 1 outlier: 16 V-cycles on d_xy/d_z = 4 elements)
with semi-coarsened schedules: the default 4 -> 3 -> 2 -> 1, vertical-first
(4,4) -> (4,2) -> (2,2) -> (1,1), horizontal-first (4,4) -> (2,4) -> (2,2) -> (1,1); exact dense
Schwarz o = 1, rtol 1e-8.  One JSON line per schedule."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2009_00705_b200 as lib
from workloads import config4

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
m = config4(4, scale=scale)
nodes = m.node_xyz(lib.reference_nodes(4))
for name, levels in [("default", None), ("vertical-first", [(4, 4), (4, 2), (2, 2), (1, 1)]),
                     ("horizontal-first", [(4, 4), (2, 4), (2, 2), (1, 1)])]:
    kw = {} if levels is None else dict(levels=levels)
    t0 = time.time()
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, 4, node_xyz=nodes, **kw)
    st = time.time() - t0
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(*xyz.T)).cuda()
    s.solve(phiD, 1e-8, check=False)
    torch.cuda.synchronize()
    phi, rep = s.solve(phiD, 1e-8, check=False)
    print(json.dumps(dict(schedule=name, levels=list(zip(s.info["level_p"], s.info["level_pz"])),
                          vcycles=rep["vcycles"], q_mean=rep["q_mean"], ms=rep["t_ms"], setup_s=st,
                          converged=rep["converged"], n_dof=s.info["n_dof"],
                          MDOF_s=s.info["n_free"] / rep["t_ms"] / 1e3)), flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
