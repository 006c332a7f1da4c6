"""FDM vs exact local solves: V-cycles per solve on config-3/4 constructions at several orders."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_00705_b200 as lib
from workloads import config3, config4

cases = [("config3 n=32 p=6", lambda: config3(p=6, n=32, nz=4)),
         ("config3 n=32 p=4", lambda: config3(p=4, n=32, nz=4)),
         ("config3 n=32 flat p=6", lambda: config3(p=6, n=32, nz=4, seed=3)),
         ("config4 p=6 scale .5", lambda: config4(6, scale=0.5)),
         ("config4 p=8 scale .5", lambda: config4(8, scale=0.5))]
for name, mk in cases:
    m = mk()
    if "flat" in name:
        m.eta = lambda x, y: 0.0 * x
        m.curved = False
    for v in (dict(local_solve=1), dict(local_solve=0)):
        s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)), **v)
        xyz = s.node_xyz(0)
        phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
        phi, rep = s.solve(phiD, 1e-8, check=False)
        print(f"{name}: {v} n_free {s.info['n_free']} iters {rep['iters']} q {rep['q_mean']:.3f} t {rep['t_ms']:.0f} ms",
              flush=True)
        s.close()
        del s
        torch.cuda.empty_cache()
