#!/usr/bin/env python
"""Benchmark: hPLMM-preconditioned GMRES time-to-1e-8 on one B200 (per rank).

A *step* is one full hplmm_solve: GMRES(50) to relative residual 1e-8 with
every iteration applying M^-1 = M_G^-1 + M_CG^-1 (I - A M_G^-1) (all of
SURVEY §8(a) a1-a11 plus the per-RHS correction columns s6).  The one-time
setup (T_ML + T_MG, §8(a) s1-s5, s7) is timed separately, as the paper's
Table 3 and north_star (6) do, and reported in the JSON line.

Inputs (A, b, all factors) are resident in HBM when the timed region starts;
the working set (tens of GB of packed local inverses) is far larger than the
126 MB L2, so no explicit flush is needed (stated in config.l2).

Multi-GPU (torchrun, N>1): replicas only -- each rank
solves its own copy; the time is the max over ranks.
``--impl reference`` times the CPU oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hPLMM-GMRES time-to-1e-8 residual (s), iterations/s, SpMV HBM GB/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.lines = []

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(2)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def symv_algorithmic_bytes(sizes):
    """Bytes a symmetric packed apply of each SPD inverse must move: the lower
    triangle n(n+1)/2 doubles, plus reading x and writing y (8n each)."""
    return sum(8 * (n * (n + 1) // 2) + 16 * n for n in sizes)


# ---------------------------------------------------------------------------
class OracleSample:
    """CPU-oracle per-iteration cost on a bounded sample of the same workload.

    Prepared once (untimed: oracle assembly, decomposition, SuperLU factors of
    the sampled subdomains -- the factorisations are the paper's T_ML); each
    measure() times one GMRES iteration's worth of oracle work: 3 full SpMVs,
    SuperLU solves on the sampled grains / contact grids scaled by their
    counts, the coarse Cholesky solve (two triangular solves of size N_m), and
    CGS2 at j = 11 basis vectors.  A full solve = per-iteration x iterations."""

    def __init__(self, prob, kg=24, kc=48):
        import numpy as np
        import scipy.sparse.linalg as spla
        from oracle import decomp, fem
        from oracle.decomp import node_dofs
        t0 = time.time()
        s = fem.build_system(prob)
        d = decomp.Decomposition(s, prob.contact_h)
        self.A = s.A.tocsr()
        self.n = s.n_dof
        rng = np.random.default_rng(0)
        self.rng = rng
        grains = [g for g in d.grain_nodes if g.size]
        contacts = [c for c in d.contact_nodes if c.size]

        def pick(sets, k):
            idx = np.unique(np.linspace(0, len(sets) - 1, min(k, len(sets))).astype(int))
            out = []
            for i in idx:
                dofs = node_dofs(sets[i])
                out.append((spla.splu(self.A[dofs][:, dofs].tocsc()), rng.standard_normal(dofs.size)))
            return out, len(sets)

        self.g, self.G = pick(grains, kg)
        self.c, self.C = pick(contacts, kc)
        nm = 3 * sum(min(prob.n_mortar, F.size) for F in d.interfaces)
        self.nm = nm
        L = np.tril(rng.standard_normal((nm, nm)) * 1e-3)
        L[np.diag_indices(nm)] = 1.0 + np.abs(L.diagonal())
        self.L = L
        self.rm = rng.standard_normal(nm)
        self.V = rng.standard_normal((11, self.n))
        self.v = rng.standard_normal(self.n)
        self.prep_s = time.time() - t0

    def measure(self):
        import scipy.linalg as sla
        t0 = time.perf_counter()
        for _ in range(3):
            self.A @ self.v
        t_spmv = time.perf_counter() - t0
        t0 = time.perf_counter()
        for lu, r in self.g:
            lu.solve(r)
        t_g = (time.perf_counter() - t0) * self.G / len(self.g)
        t0 = time.perf_counter()
        for lu, r in self.c:
            lu.solve(r)
        t_c = (time.perf_counter() - t0) * self.C / len(self.c)
        t0 = time.perf_counter()
        y = sla.solve_triangular(self.L, self.rm, lower=True)
        sla.solve_triangular(self.L, y, lower=True, trans="T")
        t_coarse = time.perf_counter() - t0
        t0 = time.perf_counter()
        v = self.v
        for _ in range(2):
            h = self.V @ v
            v = v - self.V.T @ h
        t_cgs = time.perf_counter() - t0
        return t_spmv + t_g + t_c + t_coarse + t_cgs

    def describe(self, iterations, per_it):
        return (f"per-iteration oracle cost on the same workload: 3 full SpMVs, SuperLU solves on "
                f"{len(self.g)}/{self.G} grains and {len(self.c)}/{self.C} contact grids (scaled by "
                f"count), coarse Cholesky solve N_m={self.nm}, CGS2 at j=11; x {iterations} "
                f"iterations; per-iteration {per_it:.3f}s")


def cpu_oracle_sample(prob, iterations):
    o = OracleSample(prob)
    o.measure()
    per_it = min(o.measure() for _ in range(2))
    return {"value": per_it * iterations, "unit": "s", "cores": len(os.sched_getaffinity(0)),
            "kind": "oracle", "sample": o.describe(iterations, per_it), "per_iteration_s": per_it}


# GMRES iterations to 1e-8 per workload (GPU path == oracle within +-1 where
# the oracle runs in full); used only by the reference arm to scale its sample
REF_ITERATIONS = {"cube8": 24, "cfg1": 28, "porous20": 25, "cfg2": 38, "cfg3": 38}


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    from workloads import make_problem
    prob = make_problem(args.config)
    its = args.ref_iterations or REF_ITERATIONS.get(args.config, 40)
    o = OracleSample(prob)
    for _ in range(args.warmup):
        o.measure()
    ts = [o.measure() * its for _ in range(max(1, args.steps))]
    v = sum(ts) / len(ts)
    cores = len(os.sched_getaffinity(0))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s",
            "higher_is_better": False, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "iterations_assumed": its},
            "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "oracle",
                             "sample": o.describe(its, v / its)},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def reduce_max(vals, dist=None):
    """Element-wise max over ranks (device timing: the slowest rank counts)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(v) for v in vals]
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=os.environ.get("HPLMM_BENCH_CONFIG", "cfg3"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-iterations", type=int, default=0,
                    help="GMRES iterations assumed by the reference arm")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    import numpy as np
    import __graft_entry__
    __graft_entry__.build()
    from paper_2509_19777_b200 import Solver
    from workloads import make_problem

    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream()
    prob = make_problem(args.config)
    lf = os.environ.get("HPLMM_LOCAL_FACTOR")
    smoother = os.environ.get("HPLMM_SMOOTHER", "cg")       # cg (default) | ilu0 (NEXT #4)
    n_st = int(os.environ.get("HPLMM_NST", "6" if smoother == "ilu0" else "1"))
    sv = Solver(prob, local_factor=int(lf) if lf else None, smoother=smoother,
                n_st=n_st).assemble(local).setup()
    rep0 = sv.report()
    b_host = sv.export("RHS")
    b = torch.from_numpy(b_host).cuda()
    x = torch.zeros_like(b)

    for _ in range(args.warmup):
        sv.solve(b, tol=prob.tol, x=x)
    torch.cuda.synchronize()
    sv.profile(True, True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    with Clocks(local) as clk:
        torch.cuda.profiler.start()   # ncu --profile-from-start off: the timed steps only
        e0.record(stream)
        for _ in range(args.steps):
            _, rep, hist = sv.solve(b, tol=prob.tol, x=x)
            reps.append(rep)
        e1.record(stream)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    sv.profile(False, False)
    sparse = int(sv.options.local_factor) == 1
    # kernel classes: 0/1/2 packed SYMV (grain/contact/coarse inverse tiles),
    # 3/4 supernodal solve (grain/contact factors)
    stats = [sv.kernel_stats(k) for k in range(6)]
    p = prob
    iters = reps[-1]["iterations"]

    # e2e: pinned host buffers through the same public call (the H2D of b and
    # the D2H of x happen inside hplmm_solve, inside the timed region)
    bh_t = torch.from_numpy(np.ascontiguousarray(b_host)).pin_memory()
    xh_t = torch.zeros_like(bh_t).pin_memory()
    bh, xh = bh_t.numpy(), xh_t.numpy()
    torch.cuda.synchronize()
    k2 = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(k2):
        sv.solve(bh, tol=prob.tol, x=xh)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / k2

    # SpMV HBM GB/s (the metric's third part): the solve's fine operator from
    # the timed region (class 6, plain and residual forms mixed), and the
    # stored-block BSR SpMV y = A^ x timed alone (class 7, 20 applies, CUDA
    # events on the library stream around each launch)
    fo_ms, fo_n, fo_bytes = sv.kernel_stats(6)
    vd = torch.from_numpy(np.random.default_rng(5).standard_normal(sv.n_dof)).cuda()
    od = torch.empty_like(vd)
    for _ in range(3):
        sv.apply("SPMV_BSR", vd, od)
    sv.profile(True, True)
    for _ in range(20):
        sv.apply("SPMV_BSR", vd, od)
    sv.profile(False, False)
    bs_ms, bs_n, bs_bytes = sv.kernel_stats(7)
    spmv = {"solve_operator": "element-by-element" if rep0.get("fine_operator", 1) == 0 else "bsr",
            "solve_operator_ms_per_apply": (fo_ms / fo_n) if fo_n else None,
            "solve_operator_applies_per_step": fo_n / args.steps,
            "bsr_spmv_ms": (bs_ms / bs_n) if bs_n else None,
            "bsr_spmv_algorithmic_bytes": bs_bytes,
            "bsr_spmv_gbs": (bs_bytes / (bs_ms / bs_n / 1e3) / 1e9) if bs_n else None}
    if rep0.get("fine_operator", 1) == 0 and fo_n:
        spmv["solve_operator_algorithmic_bytes"] = fo_bytes

    t_s, e2e_s = reduce_max([ms / 1e3, e2e_s], dist)

    # algorithmic bytes per launch, per kernel class
    sizes = {0: [], 1: [], 2: []}
    iface_ptr = sv.export("CONTACT_PTR")
    sizes[1] = [int(v) for v in 3 * np.diff(iface_ptr)]
    cls = sv.export("NODE_CLASS")
    own = sv.export("NODE_OWNER")
    gsz = np.bincount(own[cls != 1], minlength=prob.n_grains)
    sizes[0] = [int(v) for v in 3 * gsz]
    sizes[2] = [rep0["n_mortar_dofs"]]
    alg = {k: symv_algorithmic_bytes(sizes[k]) for k in sizes}
    ilu = smoother == "ilu0"
    if ilu:
        # ILU(0) apply: every stored 3x3 block once (L forward, U and A~_II^-1
        # backward) + r read, y written and read, x written, sentinel fill
        alg[5] = stats[5][2] + 24 * 5 * rep0["n_nodes"]
        alg[3] = stats[3][2] + 16 * sum(sizes[0])
        alg[4] = 0
        dom = 5
        dom_name = ("k_ilu_fwd + k_ilu_bwd (ILU(0) apply, level-ordered sync-free sweeps; "
                    "bound by the dependency chain, not by HBM)")
        local_classes = (5, 4)
    elif sparse:
        # block-LDL^T solve: W_S read twice, F_SS^-1 once, row lists twice
        # (library-reported stream bytes), plus x gathered and y written (16 B/DOF)
        alg[3] = stats[3][2] + 16 * sum(sizes[0])
        alg[4] = stats[4][2] + 16 * sum(sizes[1])
        dom = 4 if stats[4][1] else 3
        dom_name = ("k_sn_solve, contact-grid batch (supernodal block-LDL^T forward+backward sweep)"
                    if dom == 4 else "k_sn_solve, grain batch (supernodal block-LDL^T sweeps)")
        local_classes = (3, 4)
    else:
        dom = 0
        dom_name = "k_symv_tma, grain batch (packed SPD-inverse apply)"
        local_classes = (0, 1)
    d_ms, d_n, _ = stats[dom]
    achieved = alg[dom] / (d_ms / d_n / 1e3) / 1e9 if d_n else None
    tot_ms = sum(stats[k][0] for k in local_classes + (2,))
    tot_bytes = sum(alg[k] * stats[k][1] for k in local_classes + (2,))
    agg_achieved = tot_bytes / (tot_ms / 1e3) / 1e9 if tot_ms > 0 else None
    peak, peak_kind = _peaks()
    launches_per_step = reps[-1]["kernel_launches"]
    iters_per_s = iters / t_s
    # per-iteration algorithmic bytes (whole hot path)
    nnzb = rep0["nnzb"]
    n = 3 * rep0["n_nodes"]
    ebe = rep0.get("fine_operator", 1) == 0
    if ebe:   # element-by-element A^: x, v, y + node coordinates and Dirichlet flag,
        # lattice map (4 B / lattice point) and voxel moduli (8 B / voxel)
        nxyz = (p.nx, p.ny, p.nz)
        spmv_bytes = (24 * n + 13 * rep0["n_nodes"]
                      + 4 * (nxyz[0] + 1) * (nxyz[1] + 1) * (nxyz[2] + 1)
                      + 8 * nxyz[0] * nxyz[1] * nxyz[2])
    else:     # stored BSR blocks: 72 B values + 4 B column per block, row pointers
        spmv_bytes = 76 * nnzb + 4 * rep0["n_nodes"] + 24 * n
    # P^ values only: the per-grain blocks are dense over their column sets,
    # so no column indices stream (SURVEY §8(d)'s 12 B/entry assumes CSR)
    pb = 8 * rep0["prolong_nnz"]
    if ilu:   # n_st ILU applies + their n_st - 1 stage residuals; y and w SpMVs
        per_iter_bytes = (n_st * alg[5] + alg[2] + (2 + n_st - 1) * spmv_bytes + 2 * pb
                          + (4 * 11 + 6) * 8 * n)
    else:
        local_bytes = alg[local_classes[0]] + alg[local_classes[1]]
        per_iter_bytes = (local_bytes + alg[2] + 3 * spmv_bytes + 2 * pb + (4 * 11 + 6) * 8 * n)
    per_iter_frac = (per_iter_bytes / (t_s / max(iters, 1)) / 1e9) / peak

    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_{'sn' if sparse else 'symv'}_{args.config}.json")
    if os.path.exists(tp) and not ilu:
        try:
            traffic = json.load(open(tp))["dram_bytes_per_launch"]["contact" if dom == 4 else "grain"]
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": t_s, "unit": "s", "higher_is_better": False,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_s * 1e3, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "n_dof": n, "nnzb": nnzb,
                   "grains": rep0["n_grains"], "interfaces": rep0["n_interfaces"],
                   "mortar_dofs": rep0["n_mortar_dofs"], "n_mortar": p.n_mortar,
                   "contact_h": p.contact_h, "restart": p.restart, "tol": p.tol,
                   "parallelism": f"replicas{world}",
                   "local_factor": "supernodal" if sparse else "dense-inverse",
                   "smoother": smoother, "n_st": n_st,
                   "fine_operator": "element-by-element" if ebe else "bsr",
                   "l2": "no flush: working set (local factors) >> 126 MB L2"},
        "iterations": iters, "iterations_per_s": iters_per_s * world,
        "solves_per_s_aggregate": world / t_s,
        "setup_s": {"host_integer": rep0["t_host_setup_s"], "assemble": rep0["t_assemble_s"],
                    "local_T_ML": rep0["t_setup_local_s"],
                    "coarse_T_MG": rep0["t_setup_coarse_s"], "rhs": reps[-1]["t_rhs_s"]},
        "final_true_relres": reps[-1]["final_true_relres"],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": dom_name,
                     "algorithmic_bytes_per_launch": alg[dom], "launch_ms": d_ms / max(d_n, 1),
                     "peak_kind": peak_kind,
                     "local_and_coarse_solves": {
                         "achieved_gbs": agg_achieved,
                         "bytes_per_step": tot_bytes / args.steps,
                         "share_of_step": (tot_ms / args.steps) / (t_s * 1e3)}},
        "per_iteration": {"algorithmic_bytes": per_iter_bytes, "ms": t_s * 1e3 / max(iters, 1),
                          "roofline_frac": per_iter_frac},
        "spmv": spmv,
        "gpu_launches": int(launches_per_step * args.steps),
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = {k: v for k, v in cpu_oracle_sample(prob, iters).items()
                                if k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
