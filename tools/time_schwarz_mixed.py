"""One dense Schwarz sweep on config 3 level 0 (FP64 or FP32-stored inverses)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_00705_b200 as lib
from workloads import config3

m = config3()
mixed = int(os.environ.get("MIXED", "1"))
s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)),
               mixed_precision=mixed)
us, b = s.bench_kernel("schwarz", 0, int(os.environ.get("REPS", "10")))
print(f"mixed={mixed} schwarz level 0: {us:.1f} us, {b / us / 1e3:.0f} GB/s algorithmic")
