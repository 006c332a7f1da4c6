"""torchrun worker: the partitioned solve over NCCL (one process per GPU) equals
the single-domain solve on every rank (tests/test_gpu_nccl.py launches it)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_2009_00705_b200 as lib
from workloads import config2

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
obj = [lib.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
m = config2(p=4, nx=32, ny=2, nz=3)
nodes = m.node_xyz(lib.reference_nodes(m.p))
s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=nodes, nranks=world, rank=rank, nccl_id=obj[0])
xyz = s.node_xyz(0)
phiD = torch.from_numpy(m.phi(*xyz.T)).cuda()
phi, rep = s.solve(phiD, 1e-13)
u = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, s.n_dof(0))).cuda()
y = s.apply(u)
s1 = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=nodes)
phi1, rep1 = s1.solve(phiD, 1e-13)
y1 = s1.apply(u)
rel = lambda a, b: float((a - b).norm() / b.norm())
out = dict(rank=rank, solve_rel=rel(phi, phi1), apply_rel=rel(y, y1), iters=rep["iters"], iters1=rep1["iters"])
print("NCCLCHECK " + json.dumps(out), flush=True)
dist.destroy_process_group()
