"""Time the exact coarse solve (k_coarse_symv on the packed FP64 inverse, or the
FP32 GEMV with --mixed) on config 3 via sem_bench_kernel: mean us, algorithmic
bytes, achieved GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_00705_b200 as lib  # noqa: E402
from workloads import config3  # noqa: E402

mixed = int("--mixed" in sys.argv)
m = config3()
s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)), mixed_precision=mixed)
us, b = s.bench_kernel("coarse", reps=20)
print(f"coarse n={s.info['coarse_n']} mixed={mixed}: {us:.1f} us, {b / 1e9:.3f} GB, {b / us / 1e3:.0f} GB/s")
