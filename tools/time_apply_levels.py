"""Apply time per kernel variant (0 warp-DMMA, 1 FMA, 2 batched DMMA) on config-4 meshes of low order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_00705_b200 as lib
from workloads import config4

for p in (2, 3, 4):
    m = config4(p)
    for v in (0, 1, 2):
        s = lib.Solver(m.vertices, m.prisms, m.face_tag, p, node_xyz=m.node_xyz(lib.reference_nodes(p)),
                       local_solve=1, apply_kernel=v)
        us, b = s.bench_kernel("apply", 0, 10)
        print(f"config4 p={p} apply_kernel={v}: {us:.1f} us  {b / us / 1e3:.0f} GB/s", flush=True)
        s.close()
        del s
        torch.cuda.empty_cache()
