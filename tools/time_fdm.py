"""Time one FDM sweep per level (config 3, or config 5 with CONFIG=config5) with
sem_bench_kernel: mean us, algorithmic bytes, GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_00705_b200 as lib
from workloads import config3

ov = int(os.environ.get("OV", "1"))
if os.environ.get("CONFIG") == "config5":
    from workloads.config5 import config5
    m = config5()
else:
    m = config3()
s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)),
               local_solve=1, overlap=ov, verbose=1)
for li in range(s.info["n_levels"] - 1):
    us, b = s.bench_kernel("schwarz", li, int(os.environ.get("REPS", "20")))
    print(f"level {li} p={s.info['level_p'][li]} fdm sweep {us:.1f} us  alg {b/1e6:.1f} MB  {b/us/1e3:.0f} GB/s")
