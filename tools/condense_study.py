"""Static condensation against the full-system solve at the
bench workloads: config 3 (p = 5, exact dense Schwarz and FDM) and config 4 at p = 4..8,
rtol 1e-8 (the bench's).  One JSON line per case: outer iterations, device time, WU
and the factor bytes.  Usage: python tools/condense_study.py [config3|config4|all]."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2009_00705_b200 as lib
from workloads import config3, config4

which = sys.argv[1] if len(sys.argv) > 1 else "all"
cases = []
if which in ("config3", "all"):
    cases += [("config3", 5, {}), ("config3", 5, dict(local_solve=1))]
if which in ("config4", "all"):
    cases += [("config4", p, dict(overlap=2) if p <= 3 else {}) for p in (4, 5, 6, 7, 8)]
for name, p, kw in cases:
    m = config3() if name == "config3" else config4(p)
    t0 = time.time()
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, p, node_xyz=m.node_xyz(lib.reference_nodes(p)), **kw)
    st = time.time() - t0
    phiD = torch.from_numpy(m.phi(*s.node_xyz(0).T)).cuda()
    out = dict(config=name, p=p, opts=kw, n_dof=s.info["n_dof"], setup_s=round(st, 2))
    t0 = time.time()
    ni, nb, by = s.condensed_info()
    out.update(cond_setup_s=round(time.time() - t0, 2), ni=ni, nb=nb, cond_MiB=by >> 20)
    for mode in ("full", "condensed"):
        f = s.solve if mode == "full" else (lambda d, t, **k: s.solve_condensed(d, t, **k))
        f(phiD, 1e-8, check=False)
        torch.cuda.synchronize()
        best = None
        for _ in range(3):
            _, rep = f(phiD, 1e-8, check=False)
            if best is None or rep["t_ms"] < best["t_ms"]:
                best = rep
        out[mode] = dict(iters=best["iters"], vcycles=best["vcycles"], ms=round(best["t_ms"], 3),
                         wu=round(best["wu"], 2), q_mean=round(best["q_mean"], 4), converged=best["converged"],
                         MDOF_s=round(s.info["n_free"] / best["t_ms"] / 1e3, 2))
    print(json.dumps(out), flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
