"""Run one measured region under cudaProfilerStart/Stop for ncu
(--profile-from-start off): a full solve step, or one Schwarz sweep, or one
operator apply, after setup and a warm-up solve."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2009_00705_b200 as lib  # noqa: E402
from workloads import config1, config2, config3  # noqa: E402
from workloads.config5 import config5  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="config3")
ap.add_argument("--mode", default="step", choices=["step", "schwarz", "apply", "vcycle"])
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--smoother", default="dense", choices=["dense", "fdm"])
ap.add_argument("--overlap", type=int, default=1)
a = ap.parse_args()
m = {"config1": config1, "config2": config2, "config3": config3, "config5": config5}[a.config]()
s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)),
               local_solve=1 if a.smoother == "fdm" else 0, overlap=a.overlap)
xyz = s.node_xyz(0)
phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
phi, rep = s.solve(phiD, a.tol)
r = torch.randn(s.info["n_dof"], dtype=torch.float64, device="cuda")
u = s.empty(0)
torch.cuda.synchronize()
torch.cuda.profiler.start()
if a.mode == "step":
    phi, rep = s.solve(phiD, a.tol, out=phi)
elif a.mode == "schwarz":
    s.schwarz(0, r, u)
elif a.mode == "apply":
    s.apply(r, out=u)
else:
    s.vcycle(r, out=u)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profile region done", a.mode, rep["iters"], "launches", s.launches())
