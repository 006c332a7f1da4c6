"""Convergence study on config-5 constructions: V-cycles per solve for the
smoother variants (GPU, through the C ABI)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_00705_b200 as lib
from workloads.config5 import config5

P = int(os.environ.get("P", "4"))
cases = [
    ("hull", dict(p=P, hf=0.25, Lx=16.0, Ly=10.0)),
    ("no hull", dict(p=P, hf=0.25, Lx=16.0, Ly=10.0, hull=False)),
    ("hull, small waves", dict(p=P, hf=0.25, Lx=16.0, Ly=10.0, amp=0.003)),
    ("no hull, small waves", dict(p=P, hf=0.25, Lx=16.0, Ly=10.0, hull=False, amp=0.003)),
]
for name, mk in cases:
    m = config5(**mk)
    for v in (dict(local_solve=1), dict(local_solve=0)):
        s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)), **v)
        xyz = s.node_xyz(0)
        phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
        phi, rep = s.solve(phiD, 1e-8, check=False)
        print(f"p={P} {name}: {v} n_free {s.info['n_free']} iters {rep['iters']} q {rep['q_mean']:.3f} "
              f"t {rep['t_ms']:.0f} ms", flush=True)
        s.close()
        del s
        torch.cuda.empty_cache()
