#!/usr/bin/env python
"""Benchmark: FP64 Laplace solve by PCG + geometric p-multigrid on B200.

One step = one full Laplace solve (all SURVEY §8(a) rows: lift, PCG with one
V-cycle per iteration -- Schwarz smoothing, transfers, P=1 coarse solve -- to
rtol 1e-8 from phi_F = 0) of BASELINE.json config 3 (65,536 curvilinear
prisms, p = 5, 4.2 M DOF), inputs resident in HBM.  Metric: Laplace solve
MDOF/s (free DOF / solve time).  See DESIGN.md §"Measurement".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
N > 1 runs under torchrun: the same config-3 problem is partitioned by columns
over the N ranks (one GPU each; NCCL halo exchange), strong scaling.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Laplace solve MDOF/s (p-MG, tol 1e-8) at 1/2/4/8 B200; % of HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config3", choices=["config1", "config2", "config3", "config5"])
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--smoother", default="dense", choices=["dense", "fdm"],
                    help="Schwarz local solves: exact dense inverses (eq 4.4) or FDM (reading O33)")
    ap.add_argument("--overlap", type=int, default=1, help="Schwarz overlap (-1 = refined ceil((P+1)/2), P:536)")
    ap.add_argument("--mixed", type=int, default=0,
                    help="1: FP32 storage of the exact Schwarz / coarse inverses, FP64 arithmetic (P:35)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the variant solves (FDM local solves, mixed-precision storage) reported beside the headline")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-4 p-sweep block")
    ap.add_argument("--sweep-one", default="", help=argparse.SUPPRESS)
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="validation only: run the partitioned solve with R emulated ranks on one GPU")
    return ap.parse_args()


def make_mesh(name):
    from workloads import config1, config2, config3
    from workloads.config5 import config5
    return {"config1": config1, "config2": config2, "config3": config3, "config5": config5}[name]()


WORKLOAD = {
    "config1": "config1: box [0,2]x[0,1]x[-1,0], 64 straight prisms, p=3",
    "config2": "config2: wave channel [0,16]x[0,1], 2048 curved prisms, p=4",
    "config3": "config3: 3D wave basin [0,32]^2, 8192 jittered triangles x 8 layers = 65,536 curved prisms, p=5",
    "config5": "config5: basin [0,64]x[0,32] with a box hull 8x2x0.6 (bilge r=0.2), graded jittered Delaunay "
               "61,428 triangles x 5/8 layers = 477,600 curved prisms, p=6",
}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ CPU oracle
def oracle_sample(tol, budget_s=20.0):
    """The oracle as it stands (PCG + p-MG of Alg 4.1/4.3 on the assembled
    matrices, hierarchy setup excluded like the GPU's) on a bounded sample of
    the config-3 workload: the same construction (jitter, 8 waves, p = 5,
    same element size) on an 8x8-quad x 2-layer patch."""
    import numpy as np
    from oracle import pmg, sem
    from workloads.configs import basin
    m = basin("config3_sample", 5, 32.0 * 8 / 64, 8, 2, seed=3)
    mg = pmg.PMG(m)
    lev = mg.levels[0].level
    phiD = m.phi(*lev.xyz.T)
    A, b = sem.dirichlet_lift(lev, phiD)
    times, info = [], None
    t_end = time.perf_counter() + budget_s
    while True:
        t0 = time.perf_counter()
        _, info = pmg.pcg(mg, b, rtol=tol)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end or len(times) >= 50:
            break
    t = statistics.median(times)
    nfree = len(lev.free)
    # one fine-level SpMV of the assembled operator (the paper's work unit), single thread
    import numpy as np
    u = np.random.default_rng(0).uniform(-1, 1, lev.n)
    t0, k = time.perf_counter(), 0
    while time.perf_counter() - t0 < 1.0:
        lev.A @ u
        k += 1
    t_spmv = (time.perf_counter() - t0) / k
    try:
        from threadpoolctl import threadpool_info
        thr = max([d.get("num_threads", 1) for d in threadpool_info()] or [1])
    except Exception:
        thr = 1
    return dict(value=nfree / t / 1e6, unit="MDOF/s", cores=int(thr), kind="oracle",
                sample=f"oracle PCG-p-MG solve (tol {tol:g}, levels {mg.schedule}) of a config-3-construction "
                       f"patch: 8x8 quads x 2 layers = {m.n_elem} prisms, p=5, {nfree} free DOF; median of "
                       f"{len(times)} solves ({info['iters']} iterations); host cores available "
                       f"{len(os.sched_getaffinity(0))}",
                t_solve_s=t, n_free=nfree, iters=info["iters"], apply_spmv_MDOF_s=lev.n / t_spmv / 1e6)


def run_reference(args, rank, world):
    if rank != 0:
        return
    samples = []
    for i in range(args.warmup + args.steps):
        s = oracle_sample(args.tol, budget_s=0.0)
        if i >= args.warmup:
            samples.append(s)
    v = statistics.median([s["value"] for s in samples])
    ms = statistics.median([s["t_solve_s"] for s in samples]) * 1e3
    cb = dict(samples[0])
    cb["value"] = v
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "MDOF/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD["config3"] + " (CPU oracle on a bounded sample, see cpu_baseline.sample)",
                   "tol": args.tol},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": v, "unit": "MDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ------------------------------------------------------------------ variants
VARIANTS = [
    ("fdm", "FDM local solves (reading O33) of the same Schwarz subdomains, overlap 1",
     dict(local_solve=1, overlap=1)),
    ("mixed", "exact dense local inverses and coarse inverse STORED in FP32, FP64 arithmetic (P:35)",
     dict(local_solve=0, overlap=1, mixed_precision=1)),
    ("condensed", "statically condensed system (element-interior nodes eliminated, P:630-663, reading O43), "
     "exact dense local inverses, overlap 1", dict(local_solve=0, overlap=1, condensed=True)),
    ("fdm_condensed", "statically condensed system (P:630-663, O43), FDM local solves, overlap 1",
     dict(local_solve=1, overlap=1, condensed=True)),
]


def run_variants(args, lib, m, phiD_h, peak, base_kw):
    """The same workload and stop test with the other smoother implementations
    (not the headline: the headline is the paper's exact local inverses)."""
    import torch
    out = []
    for name, desc, extra in VARIANTS:
        kw = dict(base_kw)
        extra = dict(extra)
        cond = extra.pop("condensed", False)
        kw.update(extra)
        if kw == base_kw and not cond:
            continue
        t0 = time.perf_counter()
        s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)), **kw)
        if cond:
            s.condensed_info()   # forms the interior factors (setup)
        setup_s = time.perf_counter() - t0
        phiD = torch.from_numpy(phiD_h).cuda()
        phi = s.empty(0)
        solve = (lambda: s.solve_condensed(phiD, args.tol, out=phi)) if cond else (
            lambda: s.solve(phiD, args.tol, out=phi))
        for _ in range(args.warmup):
            solve()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s.stream)
        for _ in range(args.steps):
            _, rep = solve()
        e1.record(s.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        us, b = s.bench_kernel("schwarz", 0, 20)
        ach = b / (us * 1e-6) / 1e9
        out.append({"name": name, "smoother": desc, "solve": "laplace_solve_condensed" if cond else "laplace_solve",
                    "value": s.info["n_free"] / (ms * 1e-3) / 1e6,
                    "unit": "MDOF/s", "ms_per_step": ms, "iters": rep["iters"], "vcycles": rep["vcycles"],
                    "rel_res": rep["rel_res"], "setup_s": setup_s,
                    "smoother_kernel": {"kernel": "k_fdm_warp" if extra.get("local_solve") else (
                                        "k_schwarz<float>" if extra.get("mixed_precision") else "k_schwarz<double>"),
                                        "us": us, "alg_bytes_per_launch": b, "achieved_GBs": ach,
                                        "frac_hbm": ach / peak}})
        s.close()
        del s
        torch.cuda.empty_cache()
    return out


def run_aniso(args, lib, peak):
    """SURVEY NEXT-2 at full config-3 size: the same basin with (P_xy, P_z) = (5, 3) elements and the
    paper's Table 5.4 schedule (5,3) -> (3,3) -> (1,1), exact dense local inverses, the
    headline's stop test; a different discretisation (fewer vertical nodes), so not the headline."""
    import torch
    from workloads import config3
    m = config3()
    m.pz = 3
    t0 = time.perf_counter()
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p, 3)), pz=3,
                   levels=[(5, 3), (3, 3), (1, 1)])
    setup_s = time.perf_counter() - t0
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    phi = s.empty(0)
    for _ in range(args.warmup):
        s.solve(phiD, args.tol, out=phi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream)
    for _ in range(args.steps):
        _, rep = s.solve(phiD, args.tol, out=phi)
    e1.record(s.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    us_a, b_a = s.bench_kernel("apply", 0, 20)
    out = {"name": "aniso_table5.4", "workload": "config3 basin, P_5(triangle) x P_3(t) prisms (NEXT-2)",
           "smoother": "exact dense local inverses, levels (5,3) -> (3,3) -> (1,1) (Table 5.4)",
           "value": s.info["n_free"] / (ms * 1e-3) / 1e6, "unit": "MDOF/s", "ms_per_step": ms,
           "iters": rep["iters"], "vcycles": rep["vcycles"], "rel_res": rep["rel_res"], "n_dof": s.info["n_dof"],
           "setup_s": setup_s,
           "apply": {"kernel": "k_apply_qs<5, 3>", "us": us_a, "alg_bytes_per_launch": b_a,
                     "achieved_GBs": b_a / (us_a * 1e-6) / 1e9, "frac": b_a / (us_a * 1e-6) / 1e9 / peak}}
    s.close()
    del s
    torch.cuda.empty_cache()
    return out


def run_config5(args, lib, peak):
    """BASELINE.json config 5 (52.8 M DOF, hull) on one GPU: its exact dense
    Schwarz inverses would need ~400 GB, so it runs with the FDM / exact-dense
    hybrid (readings O33, O35); same stop test."""
    import torch
    from workloads.config5 import config5
    m = config5()
    t0 = time.perf_counter()
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)),
                   local_solve=1)
    setup_s = time.perf_counter() - t0
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    phi = s.empty(0)
    for _ in range(args.warmup):
        s.solve(phiD, args.tol, out=phi)
    torch.cuda.synchronize()
    steps = args.steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream)
    for _ in range(steps):
        _, rep = s.solve(phiD, args.tol, out=phi)
    e1.record(s.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    us, b = s.bench_kernel("schwarz", 0, 5)
    ua, ba = s.bench_kernel("apply", 0, 5)
    i = s.info
    sroof = solve_roofline(s, rep, ms, peak)
    out = {"name": "config5", "workload": WORKLOAD["config5"], "smoother": "FDM / exact-dense hybrid (O33, O35)",
           "value": i["n_free"] / (ms * 1e-3) / 1e6, "unit": "MDOF/s", "ms_per_step": ms, "steps": steps,
           "iters": rep["iters"], "vcycles": rep["vcycles"], "rel_res": rep["rel_res"], "n_dof": i["n_dof"],
           "n_free": i["n_free"], "coarse": f"P=1, {i['coarse_n']} free DOF (line-Jacobi PCG, "
           f"{rep['coarse_iters']} inner iterations per solve)", "setup_s": setup_s, "warmup": args.warmup,
           "solve_roofline": sroof, "smoother_kernels": i["smoother_kernel"],
           "device_GB": i["device_bytes"] / 1e9,
           "smoother_kernel": {"kernel": "k_fdm_cta<8> + k_schwarz<double> (O35 subset)", "us": us,
                               "alg_bytes_per_launch": b, "achieved_GBs": b / us / 1e3, "frac_hbm": b / us / 1e3 / peak},
           "apply": {"kernel": "k_apply_warp<6>", "us": ua, "achieved_GBs": ba / ua / 1e3, "frac": ba / ua / 1e3 / peak}}
    try:  # the same solve on the statically condensed system (NEXT-3), same ctx and stop test
        out["condensed"] = timed_condensed(args, s, phiD, phi)
    except lib.SemError as e:
        out["condensed"] = {"error": str(e)}
    s.close()
    del s
    torch.cuda.empty_cache()
    return out


def solve_roofline(s, rep, ms, peak, nu=(3, 3)):
    """Algorithmic HBM bytes of one whole solve (DESIGN.md §7 byte model) / solve time.
    Per level: the library's own per-launch algorithmic bytes of one smoother sweep and
    one operator apply (sem_bench_kernel); a V-cycle does nu1 + nu2 sweeps and nu1 + nu2
    applies per smoothed level (Alg 4.1 with the first pre-sweep from u = 0), residual
    inits (17 B/node), restriction + prolongation (~16 B per fine + coarse node each)
    and the coarse solve (the stored inverse's bytes, or per inner iteration one P=1
    apply + 10 vector passes); PCG adds per iteration one finest apply and 10 vector
    passes (8 B/node each), the lift one apply."""
    i = s.info
    L = i["n_levels"]
    nd = i["level_n_dof"]
    vc = 0.0
    for li in range(L - 1):
        _, bs = s.bench_kernel("schwarz", li, 1)
        _, ba = s.bench_kernel("apply", li, 1)
        vc += (nu[0] + nu[1]) * (bs + ba) + (nu[0] + nu[1]) * 17.0 * nd[li] + 2 * 16.0 * (nd[li] + nd[li + 1])
    _, ba0 = s.bench_kernel("apply", 0, 1)
    _, bac = s.bench_kernel("apply", L - 1, 1)
    vcycles, iters = max(rep["vcycles"], 1), rep["iters"]
    try:
        _, bc = s.bench_kernel("coarse", 0, 1)
        coarse = vcycles * bc
    except Exception:
        coarse = rep["coarse_iters"] * (bac + 80.0 * nd[-1])
    total = vcycles * vc + coarse + iters * (ba0 + 80.0 * nd[0]) + ba0 + 32.0 * nd[0]
    ach = total / (ms * 1e-3) / 1e9
    return {"model_bytes": total, "achieved_GBs": ach, "peak": peak, "frac": ach / peak,
            "note": "algorithmic bytes of every kernel of the solve (byte model of DESIGN.md §7) / solve time"}


FNPF_VARIANTS = [("strategy I, exact dense ASM", dict(), 1),
                 ("strategy III, FDM ASM + line-Jacobi coarse PCG", dict(local_solve=1, coarse_solver=1), 4)]


def run_fnpf(args, lib, m, dt=0.05, steps=3):
    """NEXT-4 / NEXT-1: FNPF time stepping on the headline mesh (eq 2.1, ERK4 with one
    warm-started Laplace solve per stage to the metric's tol), per-stage PCG iterations
    (the paper reports ~2 per stage at rtol 1e-7; context only)."""
    import torch
    out = []
    nodes = m.node_xyz(lib.reference_nodes(m.p))
    for name, kw, strategy in FNPF_VARIANTS:
        s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=nodes, **kw)
        ids = s.fnpf_init(nodes, strategy=strategy)
        xyz = s.node_xyz(0)[ids]
        eta = torch.from_numpy(xyz[:, 2].copy()).cuda()
        phis = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
        s.fnpf_erk4_step(eta, phis, dt, args.tol)            # warm-up step
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its = 0
        e0.record(s.stream)
        for _ in range(steps):
            its += s.fnpf_erk4_step(eta, phis, dt, args.tol)
        e1.record(s.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        out.append({"variant": name, "strategy": strategy, "dt": dt, "steps": steps, "ms_per_step": ms,
                    "stage_solves_per_s": 4.0 / (ms * 1e-3), "pcg_iters_per_stage": its / (4.0 * steps),
                    "MDOF_s": s.info["n_free"] * 4.0 / (ms * 1e-3) / 1e6, "tol": args.tol,
                    "eta_max": float(eta.abs().max().item())})
        s.close()
        del s
        torch.cuda.empty_cache()
    return out


SWEEP = [("dense_o1", "exact dense local inverses, overlap 1 (the paper's smoother, eq 4.4, P:320)",
          dict(local_solve=0, overlap=1)),
         ("fdm_refined", "FDM local solves (O33), refined overlap ceil((P+1)/2) (P:536)",
          dict(local_solve=1, overlap=-1))]


def sweep_one(args, p, variant):
    """One config-4 point (subprocess: frees the device between points)."""
    import torch
    import paper_2009_00705_b200 as lib
    from workloads import config4
    extra = [v for v in SWEEP if v[0] == variant][0][2]
    t0 = time.perf_counter()
    m = config4(p)
    nodes = m.node_xyz(lib.reference_nodes(p))
    t0 = time.perf_counter()
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, p, node_xyz=nodes, **(extra if p > 1 else {}))
    setup_s = time.perf_counter() - t0
    del nodes
    apply = None
    if variant == SWEEP[0][0]:  # the finest operator apply of this p (the same kernel for every variant)
        us_a, b_a = s.bench_kernel("apply", 0, 20)
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        pk = json.load(open(peaks_path))["hbm_gbs"] if os.path.exists(peaks_path) else 6470.8
        kern = ("k_apply_em<%d>" % (6 if p == 1 else 18)) if p <= 2 else (
            "k_apply_qs<%d>" % p if p <= 5 else ("k_apply_warp<6>" if p == 6 else "k_apply_dmma<%d>" % p))
        apply = {"kernel": kern, "us": us_a, "alg_bytes_per_launch": b_a,
                 "achieved_GBs": b_a / (us_a * 1e-6) / 1e9, "frac": b_a / (us_a * 1e-6) / 1e9 / pk}
    xyz = s.node_xyz(0)
    phiD = torch.from_numpy(m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])).cuda()
    phi = s.empty(0)
    for _ in range(args.warmup):
        s.solve(phiD, args.tol, out=phi, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream)
    for _ in range(args.steps):
        _, rep = s.solve(phiD, args.tol, out=phi, check=False)
    e1.record(s.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak = json.load(open(peaks_path))["hbm_gbs"] if os.path.exists(peaks_path) else 6470.8
    i = s.info
    out = {"p": p, "variant": variant if p > 1 else "coarse solver only (single level, O26)",
           "n_elem": i["n_elem"], "n_dof": i["n_dof"], "n_free": i["n_free"], "levels": i["level_p"],
           "coarse_n": i["coarse_n"], "vcycles": rep["vcycles"], "iters": rep["iters"], "q_mean": rep["q_mean"],
           "converged": rep["converged"], "coarse_iters": rep["coarse_iters"], "ms_per_step": ms,
           "MDOF_s": i["n_free"] / (ms * 1e-3) / 1e6, "setup_s": setup_s, "device_GB": i["device_bytes"] / 1e9,
           "smoother_kernels": i["smoother_kernel"],
           "solve_roofline": solve_roofline(s, rep, ms, peak) if p > 1 else None}
    if apply:
        out["apply"] = apply
    if p >= 3:  # the same solve on the statically condensed system (NEXT-3): same ctx, same stop test
        out["condensed"] = timed_condensed(args, s, phiD, phi)
    print("SWEEP " + json.dumps(out), flush=True)


def timed_condensed(args, s, phiD, phi):
    """laplace_solve_condensed timed like the plain solve (warm-ups, then args.steps solves
    between CUDA events on the ctx's stream); the one-off interior factorisation is setup."""
    import torch
    t0 = time.perf_counter()
    ni, nb, by = s.condensed_info()
    cond_setup_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        s.solve_condensed(phiD, args.tol, out=phi, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream)
    for _ in range(args.steps):
        _, rep = s.solve_condensed(phiD, args.tol, out=phi, check=False)
    e1.record(s.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    return {"MDOF_s": s.info["n_free"] / (ms * 1e-3) / 1e6, "ms_per_step": ms, "iters": rep["iters"],
            "vcycles": rep["vcycles"], "q_mean": rep["q_mean"], "rel_res": rep["rel_res"],
            "converged": rep["converged"], "interior_per_elem": ni, "skeleton_per_elem": nb,
            "factor_GB": by / 1e9, "factor_setup_s": cond_setup_s}


def run_sweep(args):
    """BASELINE.json config 4: ~10 M DOF per p, p = 1..8, each point in its own process."""
    out = []
    for p in range(1, 9):
        for variant, desc, _ in (SWEEP if p > 1 else SWEEP[:1]):
            cmd = [sys.executable, os.path.abspath(__file__), "--sweep-one", f"{p}:{variant}", "--steps",
                   str(args.steps), "--warmup", str(args.warmup), "--tol", str(args.tol)]
            try:
                r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
                lines = [l[6:] for l in r.stdout.splitlines() if l.startswith("SWEEP ")]
                out.append(json.loads(lines[-1]) if lines else {"p": p, "variant": variant,
                                                                 "error": (r.stderr or "")[-400:]})
            except subprocess.TimeoutExpired:
                out.append({"p": p, "variant": variant, "error": "timeout"})
    return out


# ------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.sweep_one:
        import torch
        torch.cuda.set_device(local)
        p, variant = args.sweep_one.split(":")
        sweep_one(args, int(p), variant)
        return
    import torch
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    import paper_2009_00705_b200 as lib
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [lib.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    m = make_mesh(args.config)
    t0 = time.perf_counter()
    kw = dict(verbose=int(os.environ.get("SEM_VERBOSE", "0")), overlap=args.overlap,
              local_solve=1 if args.smoother == "fdm" else 0, mixed_precision=args.mixed)
    if world > 1:
        kw.update(nranks=world, rank=rank, nccl_id=nccl_id)
    elif args.emulate_ranks > 1:
        kw.update(nranks=args.emulate_ranks)
    s = lib.Solver(m.vertices, m.prisms, m.face_tag, m.p, node_xyz=m.node_xyz(lib.reference_nodes(m.p)), **kw)
    setup_s = time.perf_counter() - t0
    info = s.info
    xyz = s.node_xyz(0)
    phiD_h = m.phi(xyz[:, 0], xyz[:, 1], xyz[:, 2])
    phiD = torch.from_numpy(phiD_h).cuda()
    phi = s.empty(0)
    stream = s.stream

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # the finest operator apply alone, before the solves (the long Schwarz stream of the timed solves
    # draws the power cap; the same kernel is timed again after them, below)
    us_a0, b_a0 = s.bench_kernel("apply", 0, 20)
    for _ in range(args.warmup):
        _, rep = s.solve(phiD, args.tol, out=phi)
    barrier()
    clk = ClockSampler(local)
    clk.start()
    s.launches(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    ev0.record(stream)
    for _ in range(args.steps):
        _, rep = s.solve(phiD, args.tol, out=phi)
        reps.append(rep)
    ev1.record(stream)
    barrier()
    launches = s.launches()
    clocks = clk.stop()
    ms_step = max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
    n_free = info["n_free"]
    value = n_free / (ms_step * 1e-3) / 1e6          # one problem solved by all ranks together

    # ---- dominant kernel (Schwarz sweep, finest level) and the operator, timed alone on the solve's stream
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {"hbm_gbs": 6650.0}
    peak = peaks["hbm_gbs"]
    us_s, b_s = s.bench_kernel("schwarz", 0, 20)
    us_a, b_a = s.bench_kernel("apply", 0, 20)
    ach = b_s / (us_s * 1e-6) / 1e9
    roof = {"kernel": ("k_fdm" if args.smoother == "fdm" else "k_schwarz") + " (level 0, one sweep" + (", this rank's partition)" if world > 1 else ")"),
            "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": None,
            "alg_bytes_per_launch": b_s, "launch_us": us_s,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if "when" in peaks else "fallback 6650 GB/s"}
    tpath = os.path.join(ROOT, "profiles", "r2_schwarz_traffic.json")
    if world == 1 and args.emulate_ranks <= 1 and args.config == "config3" and args.smoother == "dense" \
            and not args.mixed and os.path.exists(tpath):
        tr = json.load(open(tpath))       # one ncu --set full capture of this kernel on this workload
        if abs(tr.get("alg_bytes_per_launch", 0) - b_s) < 1e-6 * b_s:
            roof["traffic"] = tr["dram_bytes_per_launch"]
            roof["traffic_note"] = tr["source"]
    ach_a = b_a0 / (us_a0 * 1e-6) / 1e9
    apply = {"kernel": ("k_apply_qs<%d> (FP64 tensor cores, four elements per group of warps)" if m.p <= 5 else
                        "k_apply_warp<%d> (FP64 tensor cores, warp per element)") % m.p, "us": us_a0,
             "alg_bytes_per_launch": b_a0,
             "achieved_GBs": ach_a, "frac": ach_a / peak,
             "MDOF_s": info["n_dof"] / us_a0 if world == 1 else None,
             "note": "timed alone before the solves; after the timed solves (power-capped clock): "
                     "us_after_solves / frac_after_solves",
             "us_after_solves": us_a, "frac_after_solves": b_a / (us_a * 1e-6) / 1e9 / peak}
    # ---- end to end through the public host API (pinned host buffers, H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        ph = torch.from_numpy(phiD_h).pin_memory()
        out_h = torch.empty(info["n_dof"], dtype=torch.float64).pin_memory()
        s.solve_host(ph, args.tol, out_h)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s.solve_host(ph, args.tol, out_h)
        barrier()
        t_e2e = max_over_ranks((time.perf_counter() - t0) / args.steps)
        e2e = {"value": n_free / t_e2e / 1e6, "unit": "MDOF/s",
               "h2d_bytes_per_step": info["n_dof"] * 8, "d2h_bytes_per_step": info["n_dof"] * 8,
               "ms_per_step": t_e2e * 1e3, "api": "laplace_solve_host (pinned host buffers)"}
    sroof = solve_roofline(s, reps[-1], ms_step, peak) if world == 1 and args.emulate_ranks <= 1 else None
    variants = None
    sweep = None
    if world == 1 and args.emulate_ranks <= 1 and not args.no_variants:
        variants = run_variants(args, lib, m, phiD_h, peak, kw)
        if args.config == "config3":
            s.close()
            del s
            torch.cuda.empty_cache()
            variants.append(run_aniso(args, lib, peak))
            variants.append(run_config5(args, lib, peak))
    fnpf_block = None
    if world == 1 and args.emulate_ranks <= 1 and not args.no_variants and args.config == "config3":
        fnpf_block = run_fnpf(args, lib, m)
    if world == 1 and args.emulate_ranks <= 1 and not args.no_sweep and args.config == "config3":
        sweep = run_sweep(args)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = oracle_sample(args.tol)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "apply_spmv_MDOF_s")}
    rep = reps[-1]
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "MDOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config], "p": m.p, "n_dof": info["n_dof"], "n_free": n_free,
                       "n_elem": info["n_elem"], "levels": info["level_p"], "tol": args.tol, "nu": [3, 3],
                       "smoother": f"additive Schwarz, overlap {args.overlap}, " + (
                           "exact dense local inverses (eq 4.4-4.6)" if args.smoother == "dense" else
                           "FDM local solves of K_h(x)M_v + M_h(x)K_v (reading O33)"),
                       "outer": "PCG (Alg 4.3)", "coarse": f"P=1, {info['coarse_n']} free DOF "
                       + ("(dense inverse)" if info["coarse_n"] <= 46000 else "(Jacobi-PCG)"),
                       "l2": "inputs larger than L2: each V-cycle streams "
                             f"{sum(info['schwarz_bytes']) / 1e9:.1f} GB of Schwarz inverses",
                       "parallelism": f"column partition x{world} (NCCL halo exchange)" if world > 1
                       else (f"{args.emulate_ranks} emulated ranks on 1 GPU (validation, not a scaling number)"
                             if args.emulate_ranks > 1 else "single GPU"), "setup_s": setup_s},
            "iters": rep["iters"], "vcycles": rep["vcycles"], "rel_res": rep["rel_res"], "q_mean": rep["q_mean"],
            "work_units": ms_step * 1e3 / us_a,    # solve time / one finest operator apply (O25)
            "roofline": roof, "solve_roofline": sroof, "apply": apply, "variants": variants,
            "config4_sweep": sweep, "fnpf": fnpf_block, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
