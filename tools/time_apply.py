"""Time the operator apply (both kernel variants) and one Schwarz sweep on a
config with CUDA events; prints one JSON line per variant."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2009_00705_b200 as lib  # noqa: E402
from paper_2009_00705_b200.metrics import apply_bytes_model, apply_flops_model  # noqa: E402
from workloads import config1, config2, config3, config4  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="config3")
ap.add_argument("--p", type=int, default=0, help="config4 order")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--levels", default="")
a = ap.parse_args()
if a.config == "config4":
    m = config4(a.p)
else:
    m = {"config1": config1, "config2": config2, "config3": config3}[a.config]()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
nodes = m.node_xyz(lib.reference_nodes(m.p))
VARIANTS = {0: "default", 1: "fma", 2: "batched-dmma", 3: "quad", 4: "quad-split"}
for variant in [int(v) for v in os.environ.get("VARIANTS", "0,2").split(",")]:
    kw = dict(apply_kernel=variant, local_solve=1)
    if a.levels:
        kw["levels"] = [int(x) for x in a.levels.split(",")]
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=nodes, overlap=0, **kw) if a.config == "config4" \
        else lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=nodes, **kw)
    x = torch.randn(s.info["n_dof"], dtype=torch.float64, device="cuda")
    y = s.empty(0)
    for _ in range(3):
        s.apply(x, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream)
    for _ in range(a.reps):
        s.apply(x, out=y)
    e1.record(s.stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / a.reps * 1e-3
    b = apply_bytes_model(s, m)
    f = apply_flops_model(m.p, s.info["n_elem"])
    print(json.dumps({"config": a.config, "p": m.p, "variant": VARIANTS[variant], "us": t * 1e6,
                      "MDOF_s": s.info["n_dof"] / t / 1e6, "GBs": b / t / 1e9, "frac_hbm": b / t / 1e9 / peak,
                      "TFLOPs": f / t / 1e12, "n_dof": s.info["n_dof"]}))
    s.close()
    del s
    torch.cuda.empty_cache()
