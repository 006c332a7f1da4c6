"""Diagnostics of the FDM smoother: per-level sweep on a small refined-overlap case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_00705_b200 as lib
from workloads.configs import basin

m = basin("c3s", 5, 32.0 * 5 / 64, 5, 3, seed=3)
ov = int(sys.argv[1]) if len(sys.argv) > 1 else -1
s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)),
               local_solve=1, overlap=ov, verbose=1)
for li in range(s.info["n_levels"] - 1):
    n = s.n_dof(li)
    r = torch.from_numpy(np.random.default_rng(li).uniform(-1, 1, n)).cuda()
    u = s.empty(li)
    try:
        s.schwarz(li, r, u)
        torch.cuda.synchronize()
        print("level", li, "ok", float(u.norm()))
    except Exception as e:
        print("level", li, "FAILED", e)
