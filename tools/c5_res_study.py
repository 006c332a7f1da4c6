"""Config-5 construction at the full near-hull resolution (hf = 1/12) on a 24 x 12
basin: exact dense vs FDM-hybrid PCG iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_00705_b200 as lib
from workloads.config5 import config5

P = int(os.environ.get("P", "4"))
m = config5(p=P, hf=1.0 / 12.0, Lx=24.0, Ly=12.0)
for v in [dict(local_solve=1)] + ([dict(local_solve=0)] if P < 6 else []):
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)), **v)
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    phi, rep = s.solve(phiD, 1e-8, check=False)
    print(f"p={P} hf=1/12 24x12: {v} elems {s.info['n_elem']} n_free {s.info['n_free']} iters {rep['iters']} "
          f"q {rep['q_mean']:.3f} t {rep['t_ms']:.0f} ms res {[round(x / rep['res_hist'][0], 9) for x in rep['res_hist'][:8]]}",
          flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
