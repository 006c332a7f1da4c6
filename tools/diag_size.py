"""Probe size dependence of PCG-p-MG convergence (diagnostic)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2009_00705_b200 as lib  # noqa: E402
from workloads.configs import basin  # noqa: E402


def run(p, n, nz, **kw):
    m = basin("d", p, 32.0 * n / 104, n, nz, seed=4)
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, p, node_xyz=m.node_xyz(lib.reference_nodes(p)), **kw)
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    phi, rep = s.solve(phiD, 1e-8, check=False)
    # V-cycle symmetry on random free vectors
    mask = torch.from_numpy(s.dirichlet_mask(0)).cuda()
    x = torch.randn(s.info["n_dof"], dtype=torch.float64, device="cuda").masked_fill(mask, 0)
    y = torch.randn(s.info["n_dof"], dtype=torch.float64, device="cuda").masked_fill(mask, 0)
    vx, vy = s.vcycle(x), s.vcycle(y)
    sym = float((x @ vy - y @ vx).abs() / (x @ vy).abs())
    pos = float(x @ vx)
    out = dict(p=p, n=n, nz=nz, E=m.n_elem, kw={k: v for k, v in kw.items()}, iters=rep["iters"], q=rep["q_mean"],
               cit=rep["coarse_iters"], sym=sym, xVx=pos)
    print(json.dumps(out), flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()


for args in [(4, 104, 13, {}), (4, 104, 13, dict(coarse_rtol=1e-13)), (4, 96, 12, {}), (4, 88, 11, {}),
             (4, 104, 13, dict(overlap=0)), (5, 104, 13, {}), (3, 104, 13, {})]:
    try:
        run(*args[:3], **args[3])
    except Exception as e:
        print(json.dumps(dict(args=str(args), err=str(e)[:300])), flush=True)
