"""Solve time of the small configs (launch-bound): median of 20 solves to 1e-8."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import statistics

import torch

import paper_2009_00705_b200 as lib
from workloads import config1, config2

for name, mk in (("config1", config1), ("config2", config2)):
    m = mk()
    for ls in (0, 1):
        s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)),
                       local_solve=ls)
        xyz = s.node_xyz(0)
        phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
        phi = s.empty(0)
        for _ in range(3):
            s.solve(phiD, 1e-8, out=phi)
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s.stream)
            _, rep = s.solve(phiD, 1e-8, out=phi)
            e1.record(s.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        s.launches(reset=True)
        s.solve(phiD, 1e-8, out=phi)
        print(f"{name} local_solve={ls}: n_free {s.info['n_free']} iters {rep['iters']} solve {t:.3f} ms "
              f"{s.info['n_free'] / t / 1e3:.2f} MDOF/s launches/solve {s.launches()}", flush=True)
        s.close()
