"""Config-4 p-sweep at ~10 M DOF (BASELINE config 4): for each p, set up the
solver, solve to rtol 1e-8 from zero and report V-cycles, iterations, q,
MDOF/s, setup time and device memory.  Each p runs in its own process."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


LS = int(os.environ.get("LOCAL_SOLVE", "0"))
OV = int(os.environ.get("OVERLAP", "1"))


def one(p, scale, steps):
    import torch
    import paper_2009_00705_b200 as lib
    from workloads import config4
    t0 = time.perf_counter()
    m = config4(p, scale=scale)
    nodes = m.node_xyz(lib.reference_nodes(p))
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, p, node_xyz=nodes, verbose=1, local_solve=LS, overlap=OV)
    t_setup = time.perf_counter() - t0
    del nodes
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    phi, rep = s.solve(phiD, 1e-8, check=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s.stream)
        phi, rep = s.solve(phiD, 1e-8, out=phi, check=False)
        e1.record(s.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[len(ts) // 2] * 1e-3
    i = s.info
    print(json.dumps(dict(config="config4", p=p, scale=scale, local_solve=LS, overlap=OV, n_elem=i["n_elem"], n_dof=i["n_dof"], n_free=i["n_free"],
                          levels=i["level_p"], coarse_n=i["coarse_n"], vcycles=rep["vcycles"], iters=rep["iters"],
                          q_mean=rep["q_mean"], rel_res=rep["rel_res"], coarse_iters=rep["coarse_iters"],
                          solve_ms=t * 1e3, MDOF_s=i["n_free"] / t / 1e6, setup_s=t_setup, gen_s=t_gen,
                          device_GB=i["device_bytes"] / 1e9, schwarz_GB=sum(i["schwarz_bytes"]) / 1e9)), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]))
        sys.exit(0)
    ps = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,7,6,5,4,3,2,1").split(",")]
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    for p in ps:
        r = subprocess.run([sys.executable, __file__, "--one", str(p), str(scale), str(steps)], capture_output=True,
                           text=True, timeout=1500)
        out = [l for l in r.stdout.splitlines() if l.startswith("{")]
        if out:
            print(out[-1], flush=True)
        else:
            print(json.dumps(dict(config="config4", p=p, scale=scale, error=(r.stderr or "")[-600:])), flush=True)
        sys.stderr.write(r.stderr[-2000:])
