"""Config 5 full: PCG iterations vs the inner coarse-solve tolerance (reading O9)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_00705_b200 as lib
from workloads.config5 import config5

m = config5()
for crt in [float(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1e-10,1e-6,1e-4,1e-2").split(",")]:
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)),
                   local_solve=1, coarse_rtol=crt)
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    phi, rep = s.solve(phiD, 1e-8, check=False)
    phi, rep = s.solve(phiD, 1e-8, check=False)
    print(f"coarse_rtol {crt:g}: iters {rep['iters']} coarse_iters {rep['coarse_iters']} t {rep['t_ms']:.0f} ms "
          f"q {rep['q_mean']:.3f} res {[round(x / rep['res_hist'][0], 8) for x in rep['res_hist'][:12]]}", flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
