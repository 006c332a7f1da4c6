"""Diagnose the p=6 hull-replica solve: smoother variants, V-cycle symmetry, levels."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2009_00705_b200 as lib
from workloads.config5 import config5
from workloads import random_vector

m = config5(p=int(os.environ.get("P", "6")), hf=0.5, Lx=float(os.environ.get("LX", "10")), Ly=float(os.environ.get("LY", "4")))
nodes = m.node_xyz(lib.reference_nodes(m.p))
variant = sys.argv[1]
kw = dict(local_solve=1)
if variant == "dense":
    kw = dict(local_solve=0)
elif variant == "levels2":
    kw = dict(local_solve=1, levels=[m.p, 1])
elif variant == "o0":
    kw = dict(local_solve=1, overlap=0)
s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=nodes, **kw)
xyz = s.node_xyz(0)
phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
phi, rep = s.solve(phiD, 1e-10, check=False)
n = s.n_dof(0)
dm = torch.from_numpy(s.dirichlet_mask(0)).cuda()
x = torch.from_numpy(random_vector(n, 1)).cuda(); x[dm] = 0
y = torch.from_numpy(random_vector(n, 2)).cuda(); y[dm] = 0
vx, vy = s.vcycle(x), s.vcycle(y)
sym = abs((x @ vy).item() - (y @ vx).item()) / abs((x @ vy).item())
pos = [(x @ vx).item(), (y @ vy).item()]
# smoother symmetry per level
lev = []
for li in range(s.info["n_levels"] - 1):
    nl = s.n_dof(li)
    dml = torch.from_numpy(s.dirichlet_mask(li)).cuda()
    a = torch.from_numpy(random_vector(nl, 3)).cuda(); a[dml] = 0
    b = torch.from_numpy(random_vector(nl, 4)).cuda(); b[dml] = 0
    sa, sb = s.empty(li), s.empty(li)
    s.schwarz(li, a, sa, transpose=False); s.schwarz(li, b, sb, transpose=True)
    # <S^-1 a, b> vs <a, S^-T b>
    l1 = (sa @ b).item(); l2 = (a @ sb).item()
    nan = bool(torch.isnan(sa).any().item())
    lev.append(dict(level=li, p=s.info["level_p"][li], kernel=s.info["smoother_kernel"][li], mt=s.info["smoother_mt"][li],
                    adjoint_err=abs(l1 - l2) / abs(l1), aSa=(a @ sa).item(), nan=nan, maxabs=sa.abs().max().item()))
print(json.dumps(dict(variant=variant, env=os.environ.get("SEM_FDM_CTA", "") + os.environ.get("SEM_FDM_SIMPLE", ""),
                      iters=rep["iters"], rel_res=rep["rel_res"], hist=rep["res_hist"][:8], vsym=sym, vpos=pos,
                      levels=lev, coarse_n=s.info["coarse_n"])), flush=True)
