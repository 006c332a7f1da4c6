"""Per-level timing of one operator apply and one smoother sweep (sem_bench_kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_00705_b200 as lib
from workloads import config3, config4

cfg = os.environ.get("CFG", "config3")
m = config3() if cfg == "config3" else config4(int(cfg[len("config4_p"):]))
s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)),
               local_solve=int(os.environ.get("FDM", "1")), overlap=int(os.environ.get("OV", "1")))
for li in range(s.info["n_levels"]):
    ua, ba = s.bench_kernel("apply", li, 20)
    line = f"{cfg} level {li} p={s.info['level_p'][li]}: apply {ua:.1f} us ({ba / ua / 1e3:.0f} GB/s)"
    if li + 1 < s.info["n_levels"]:
        us, bs = s.bench_kernel("schwarz", li, 20)
        line += f", smoother {us:.1f} us ({bs / us / 1e3:.0f} GB/s)"
    print(line, flush=True)
