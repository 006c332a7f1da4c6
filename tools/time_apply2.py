"""Operator apply per level and kernel variant (sem_bench_kernel: CUDA events on the
ctx stream, algorithmic bytes from the library's byte model).  One JSON line per
(config, variant, level)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa
import paper_2009_00705_b200 as lib  # noqa
from workloads import config2, config3, config4  # noqa

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6470.8
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["config3"]
variants = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "3"])]
for cfg in cfgs:
    m = config4(int(cfg[-1])) if cfg.startswith("config4") else {"config2": config2, "config3": config3}[cfg]()
    nodes = m.node_xyz(lib.reference_nodes(m.p))
    for v in variants:
        s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=nodes, apply_kernel=v, local_solve=1)
        for li, pl in enumerate(s.info["level_p"]):
            us, b = s.bench_kernel("apply", li, 30)
            print(json.dumps({"config": cfg, "variant": v, "level": li, "p": pl, "us": us, "GBs": b / us / 1e3,
                              "frac": b / us / 1e3 / peak, "n_dof": s.info["level_n_dof"][li]}), flush=True)
        s.close()
        del s
        torch.cuda.empty_cache()
