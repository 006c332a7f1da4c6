"""Diagnose V-cycle counts vs mesh size / kernel / coarse solver for a config-4 order."""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2009_00705_b200 as lib  # noqa: E402
from workloads.configs import basin  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sizes = [(16, 4), (32, 4), (64, 8), (104, 13)]
for (n, nz), ak, cs in itertools.product(sizes, (0, 1), (0, 1)):
    m = basin("d", p, 32.0 * n / 104, n, nz, seed=4)
    try:
        s = lib.Solver(m.vertices, m.prisms, m.face_tag, p, node_xyz=m.node_xyz(lib.reference_nodes(p)),
                       apply_kernel=ak, coarse_solver=cs)
    except Exception as e:
        print(json.dumps(dict(n=n, nz=nz, ak=ak, cs=cs, err=str(e)[:200])), flush=True)
        continue
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    phi, rep = s.solve(phiD, 1e-8, check=False)
    print(json.dumps(dict(n=n, nz=nz, E=m.n_elem, ak=ak, cs=cs, coarse_n=s.info["coarse_n"], iters=rep["iters"],
                          q=rep["q_mean"], cit=rep["coarse_iters"], hist=[f"{x:.2e}" for x in rep["res_hist"][:8]])),
          flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
