"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck), SURVEY §5:
configs 1-2 with the dense and FDM smoothers, the iterative coarse solve, the
deterministic mode, one FNPF stage and the four-elements-per-warp apply."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2009_00705_b200 as lib
from workloads import config1, config2

for name, m, kw in [("c1 dense", config1(), {}),
                    ("c1 fdm", config1(), dict(local_solve=1)),
                    ("c2 fdm + iterative coarse", config2(p=4, nx=16, ny=2, nz=2), dict(local_solve=1, coarse_solver=1)),
                    ("c2 dense deterministic", config2(p=3, nx=16, ny=2, nz=2), dict(deterministic=1)),
                    ("c2 quad apply", config2(p=3, nx=16, ny=2, nz=2), dict(apply_kernel=3))]:
    nodes = m.node_xyz(lib.reference_nodes(m.p))
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=nodes, **kw)
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(*xyz.T)).cuda()
    phi, rep = s.solve(phiD, 1e-10)
    phi, rep = s.solve(phiD, 1e-10)      # graph replay
    y = s.apply(phi)
    if name.startswith("c2 fdm"):
        ids = s.fnpf_init(nodes, strategy=4)
        eta = torch.from_numpy(xyz[ids, 2].copy()).cuda()
        ph = phiD[torch.from_numpy(ids).long().cuda()].clone()
        s.fnpf_erk4_step(eta, ph, 0.01, 1e-10)
    torch.cuda.synchronize()
    print(name, "ok", rep["iters"], flush=True)
    s.close()
