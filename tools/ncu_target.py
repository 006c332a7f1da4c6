"""Single-kernel targets for ncu (run under `ncu -k regex:<kernel> -c 1 ...`):
  schwarz3        one level-0 k_schwarz<double> sweep of config 3 (exact dense ASM)
  apply3 <v>      one level-0 operator apply of config 3 with apply_kernel v
  apply <cfg> <v> one level-0 apply of config2/config3/config4p<P> with apply_kernel v
  fdm3            one level-0 FDM sweep of config 3
  fdm5            one level-0 FDM sweep of config 5
Prints the library's algorithmic bytes per launch (sem_bench_kernel) as JSON."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa
import paper_2009_00705_b200 as lib  # noqa
from workloads import config2, config3, config4  # noqa

what = sys.argv[1]
if what == "schwarz3":
    m, kw, kern = config3(), {}, "schwarz"
elif what == "fdm3":
    m, kw, kern = config3(), dict(local_solve=1), "schwarz"
elif what == "fdm5":
    from workloads.config5 import config5
    m, kw, kern = config5(), dict(local_solve=1), "schwarz"
else:
    cfg = "config3" if what == "apply3" else sys.argv[2]
    v = int(sys.argv[-1])
    m = config4(int(cfg[-1])) if cfg.startswith("config4") else {"config2": config2, "config3": config3}[cfg]()
    kw, kern = dict(apply_kernel=v, local_solve=1), "apply"
s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)), **kw)
torch.cuda.synchronize()
us, b = s.bench_kernel(kern, 0, 1)   # 3 warm-up launches + 1 timed (ncu -c selects which)
print(json.dumps({"target": what, "alg_bytes_per_launch": b, "us_unprofiled_is_meaningless_under_ncu": us}))
