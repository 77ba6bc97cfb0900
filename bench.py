#!/usr/bin/env python
"""Benchmark: hPLMM-preconditioned GMRES time-to-1e-8 on one B200 (per rank).

A *step* is one full hplmm_solve: GMRES(50) to relative residual 1e-8 with
every iteration applying M^-1 = M_G^-1 + M_CG^-1 (I - A M_G^-1) (all of
SURVEY §8(a) a1-a11 plus the per-RHS correction columns s6).  The one-time
setup (T_ML + T_MG, §8(a) s1-s5, s7) is timed separately, as the paper's
Table 3 and north_star (6) do, and reported in the JSON line.

Timing: inputs (A, b, all factors) are resident in HBM when
the timed region starts; the working set (~20 GB of local factors streamed
per iteration at cfg3) is far larger than the 126 MB L2, so no explicit flush
(stated in config.l2).  The K timed steps run with profiling OFF (the solve is
then one CUDA-graph launch per step); each step is bracketed by CUDA events on
the library's stream; `value` is the MEDIAN step time, `ms_per_step` the mean
over the bracketed region.  Kernel statistics for the roofline come from a
separate pass afterwards (profiling on: CUDA events around every local-solve
and fine-operator launch, the host-driven loop).

Multi-GPU (torchrun, N>1): replicas only -- each rank solves
its own copy; times are the max over ranks.

``--impl reference`` times the CPU oracle (this tier's reference arm) on a
bounded sample of the same workload (one oracle GMRES iteration per step);
its `value` is a MODEL of the oracle's time to solution built from those
measurements and the oracle's own iteration count, labelled as such.
"""
from __future__ import annotations

import argparse
import json
import math
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
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _median(v):
    v = sorted(v)
    k = len(v)
    return 0.5 * (v[(k - 1) // 2] + v[k // 2])


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


def _golden(config):
    p = os.path.join(ROOT, "tests", "golden", f"{config}_oracle.json")
    return json.load(open(p)) if os.path.exists(p) else None


def arnoldi_j_sequence(iterations, restart):
    """Step index j of every Arnoldi step of a run of `iterations` total steps
    with restart m (cycles of m steps; the last one shorter), and the cycle count."""
    js = [t % restart for t in range(iterations)]
    return js, max(1, -(-iterations // restart))


def config_of(prob, sizes, world):
    """The workload description shared by both arms (same dict => same_config)."""
    return {"workload": prob.name, "n_dof": sizes["n_dof"], "nnzb": sizes["nnzb"],
            "grains": sizes["grains"], "interfaces": sizes["interfaces"],
            "mortar_dofs": sizes["mortar_dofs"], "n_mortar": prob.n_mortar,
            "contact_h": prob.contact_h, "restart": prob.restart, "tol": prob.tol,
            "parallelism": f"replicas{world}",
            "l2": "no flush: working set (local factors, ~20 GB per iteration at cfg3) >> 126 MB L2"}


# ---------------------------------------------------------------------------
# CPU oracle: measured full run (small configs) and a bounded per-iteration
# sample of a large one (the model)
# ---------------------------------------------------------------------------
def oracle_full_run(prob):
    """The oracle as it stands, end to end: setup (T_ML-like: local SuperLU
    factorisations; T_MG-like: decomposition, mortars, shape vectors, S and its
    Cholesky -- oracle/hplmm.py timings), per-RHS correction columns, GMRES."""
    from oracle import gmres, hplmm
    t0 = time.perf_counter()
    s, h = hplmm.setup(prob)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    h.set_rhs(s.b)
    x, it, hist, rr, conv = gmres.gmres(s.A, s.b, h.apply_M, tol=prob.tol, restart=prob.restart,
                                         maxit=prob.maxit)
    t_sol = time.perf_counter() - t0
    return {"config": prob.name, "T_setup_s": t_setup, "T_ML_s": h.timings["T_ML"],
            "T_MG_s": h.timings["T_MG"], "T_sol_s": t_sol, "iterations": int(it),
            "s_per_iteration": t_sol / max(it, 1), "converged": bool(conv)}


class OracleModel:
    """Per-iteration cost of the oracle's GMRES on a workload, measured on the
    oracle's own operations at full size wherever that is bounded:

      * fine operator A^ x (scipy CSR, the oracle's A^): 3 per step, full size;
      * local solves (SuperLU, the oracle's exact local solve of eq:Mg_Mz) on
        kg grains and kc contact grids of the workload, scaled by count;
      * restriction / prolongation: CSR mat-vecs with nnz(P^)/8 entries, x 8
        (nnz(P^) from the decomposition: per grain |I_g| x its R14 columns,
        plus the interface mortar entries);
      * coarse solve: cho_solve of order N_m on a synthetic SPD matrix (the
        cost of two dense triangular solves does not depend on the values);
      * CGS2 at the Arnoldi step j actually run (numpy V[:j+1] @ w, twice).

    A solve = sum over the steps of the oracle's own iteration sequence + one
    M^-1, A^ x and norm per cycle.  This is a MODEL (labelled in the JSON);
    its error is measured at cfg2 against the full oracle run."""

    def __init__(self, prob, kg=32, kc=64):
        import numpy as np
        import scipy.linalg as sla
        import scipy.sparse as sp
        import scipy.sparse.linalg as spla
        from oracle import decomp, fem
        from oracle.decomp import CLASS_G, node_dofs
        t0 = time.perf_counter()
        s = fem.build_system(prob)
        d = decomp.Decomposition(s, prob.contact_h)
        self.A = s.A.tocsr()
        self.n = s.n_dof
        rng = np.random.default_rng(0)
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
        nu = [min(prob.n_mortar, F.size) for F in d.interfaces]
        self.nm = 3 * sum(nu)
        # nnz(P^_B): per grain |I_g| x (mortar columns of the interfaces coupled
        # to its class-G nodes, R14) + the interface entries of Q^o
        rp, ci = s.row_ptr, s.col_idx
        nnz = sum(3 * F.size * 3 * v for F, v in zip(d.interfaces, nu)) // 3
        for nodes in d.grain_nodes:
            ifs = set()
            for p in nodes:
                if d.node_class[p] == CLASS_G:
                    ifs.update(int(d.node_iface[q]) for q in ci[rp[p]:rp[p + 1]] if d.node_iface[q] >= 0)
            nnz += 3 * nodes.size * 3 * sum(nu[c] for c in ifs)
        self.prolong_nnz = int(nnz)
        k = max(1, self.prolong_nnz // 8)
        rows = rng.integers(0, max(self.nm, 1), k)
        cols = rng.integers(0, self.n, k)
        self.PT8 = sp.csr_matrix((rng.standard_normal(k), (rows, cols)), shape=(max(self.nm, 1), self.n))
        self.P8 = self.PT8.T.tocsc()
        M = rng.standard_normal((self.nm, self.nm)) * 1e-3
        self.Sc = sla.cho_factor(M @ M.T + np.eye(self.nm), lower=True) if self.nm else None
        self.rm = rng.standard_normal(self.nm)
        self.v = rng.standard_normal(self.n)
        self.V = rng.standard_normal((prob.restart + 1, self.n))
        self.prep_s = time.perf_counter() - t0

    def parts(self):
        """Seconds of one M^-1 apply and of one A^ x (measured once)."""
        import scipy.linalg as sla
        t0 = time.perf_counter()
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
        if self.Sc is not None:
            sla.cho_solve(self.Sc, self.rm)
        t_coarse = time.perf_counter() - t0
        t0 = time.perf_counter()
        self.PT8 @ self.v
        if self.nm:
            self.P8 @ self.rm
        t_rp = 8 * (time.perf_counter() - t0)
        # M^-1 = M_G (restrict, coarse, prolong) + A y + M_zeta + A z1 + M_g
        t_minv = t_rp + t_coarse + 2 * t_spmv + t_g + t_c
        return t_minv, t_spmv

    def cgs2(self, j):
        t0 = time.perf_counter()
        w = self.v
        for _ in range(2):
            h = self.V[:j + 1] @ w
            w = w - self.V[:j + 1].T @ h
        return time.perf_counter() - t0

    def step(self, j):
        """One oracle GMRES iteration at Arnoldi index j: (seconds, parts)."""
        t_minv, t_spmv = self.parts()
        t_cgs = self.cgs2(j)
        return t_minv + t_spmv + t_cgs, (t_minv, t_spmv)

    def solve_model(self, iterations, restart, reps=1):
        js, cycles = arnoldi_j_sequence(iterations, restart)
        parts = [self.parts() for _ in range(max(1, reps))]
        t_minv = _median([p[0] for p in parts])
        t_spmv = _median([p[1] for p in parts])
        t_cgs = sum(self.cgs2(j) for j in js)
        return iterations * (t_minv + t_spmv) + t_cgs + cycles * (t_minv + t_spmv)

    def describe(self):
        return (f"oracle operations at full size: 3 A^x (scipy CSR) per step, SuperLU solves on "
                f"{len(self.g)}/{self.G} grains and {len(self.c)}/{self.C} contact grids (scaled "
                f"by count), restriction+prolongation CSR mat-vecs with nnz(P^)/8 = "
                f"{self.prolong_nnz // 8} entries (x8), coarse cho_solve N_m = {self.nm}, CGS2 at "
                f"the actual Arnoldi index j")


def oracle_iterations(prob):
    """The oracle's OWN iteration count on this workload: from its stored full
    run (tests/golden, written by a script that calls only oracle/) or, for
    the small configs, by running it."""
    g = _golden(prob.name)
    if g is not None:
        return int(g["iterations"]), "tests/golden/%s_oracle.json" % prob.name
    if prob.name in ("cube8", "cfg1", "porous20", "cfg2"):
        return oracle_full_run(prob)["iterations"], "full oracle run"
    raise RuntimeError(f"no oracle iteration count for {prob.name}: run tests/golden/make_golden.py")


def cpu_baseline(prob):
    """cpu_baseline of the GPU line: the full oracle at cfg2 (measured) and the
    per-iteration model at the bench workload, with its error at cfg2."""
    from workloads import make_problem
    cores = len(os.sched_getaffinity(0))
    out = {"unit": "s", "cores": cores, "kind": "oracle"}
    c2 = make_problem("cfg2")
    full2 = oracle_full_run(c2)
    m2 = OracleModel(c2)
    model2 = m2.solve_model(full2["iterations"], c2.restart, reps=2)
    out["measured_full_cfg2"] = full2
    out["model_error_cfg2"] = model2 / full2["T_sol_s"] - 1.0
    if prob.name == "cfg2":
        out["value"] = full2["T_sol_s"]
        out["sample"] = "full oracle solve (cfg2, measured)"
        return out
    its, src = oracle_iterations(prob)
    m = OracleModel(prob)
    out["value"] = m.solve_model(its, prob.restart, reps=2)
    out["value_kind"] = "model (measured oracle operations x the oracle's own iteration count)"
    out["oracle_iterations"] = its
    out["oracle_iterations_source"] = src
    out["sample"] = m.describe() + f"; x {its} oracle iterations ({src}); model error at cfg2 " \
                                   f"{100 * out['model_error_cfg2']:+.1f}% vs the measured full run"
    g = _golden(prob.name)
    if g is not None:
        out["full_run_on_build_box"] = {k: g[k] for k in ("t_setup_s", "t_ML_s", "t_MG_s", "t_solve_s",
                                                          "iterations", "cores") if k in g}
    return out


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    """Reference arm = the CPU oracle (this tier has no reference program)."""
    if rank != 0:
        return
    import numpy as np
    from workloads import make_problem
    prob = make_problem(args.config)
    its, src = oracle_iterations(prob)
    t0 = time.perf_counter()
    m = OracleModel(prob)
    prep = time.perf_counter() - t0
    js, cycles = arnoldi_j_sequence(its, prob.restart)
    for w in range(args.warmup):
        m.step(js[w % len(js)])
    steps = []
    parts = []
    t_start = time.perf_counter()
    for k in range(args.steps):
        t, p = m.step(js[k % len(js)])
        steps.append(t)
        parts.append(p)
    wall = time.perf_counter() - t_start
    t_minv = _median([p[0] for p in parts])
    t_spmv = _median([p[1] for p in parts])
    t_cgs = sum(m.cgs2(j) for j in js)
    est = its * (t_minv + t_spmv) + t_cgs + cycles * (t_minv + t_spmv)
    cores = len(os.sched_getaffinity(0))
    sizes = {"n_dof": int(m.n), "nnzb": int(m.A.nnz // 9), "grains": int(prob.n_grains),
             "interfaces": None, "mortar_dofs": int(m.nm)}
    line = {"impl": "reference", "metric": METRIC, "value": est, "unit": "s",
            "higher_is_better": False, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(args.steps, 1),
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "value_kind": "model: the oracle's time to 1e-8 = (measured per-iteration oracle "
                          "operations) x (the oracle's own iteration count); ms_per_step is the "
                          "measured wall time of one sampled oracle iteration",
            "estimated_s": est, "oracle_iterations": its, "oracle_iterations_source": src,
            "sample_prep_s": prep,
            "config": None,
            "cpu_baseline": {"value": est, "unit": "s", "cores": cores, "kind": "oracle",
                             "sample": m.describe() + f"; one sampled iteration per step, "
                                                      f"x {its} oracle iterations ({src})"},
            "e2e": {"value": est, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    g = _golden(prob.name)
    if g is not None:
        sizes["interfaces"] = int(g["n_interfaces"])
        line["full_run_on_build_box"] = {k: g[k] for k in ("t_setup_s", "t_ML_s", "t_MG_s",
                                                           "t_solve_s", "iterations", "cores")}
    line["config"] = config_of(prob, sizes, world)
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


def timed_solves(sv, b, x, tol, steps, stream, clocks=None):
    """K solves, each bracketed by CUDA events on the library's stream; returns
    (per-step ms list, bracketed total ms, last report)."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rep = None
    torch.cuda.synchronize()
    e0.record(stream)
    for k in range(steps):
        ev[k][0].record(stream)
        _, rep, _ = sv.solve(b, tol=tol, x=x)
        ev[k][1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(c) for a, c in ev], e0.elapsed_time(e1), rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=os.environ.get("HPLMM_BENCH_CONFIG", "cfg3"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bsr", action="store_true", help="skip the stored-block operator line")
    ap.add_argument("--no-multi", action="store_true", help="skip the multi-RHS block line")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    dist = None
    if args.impl == "reference":
        # rank 0 alone runs the oracle and prints; the other ranks exit 0
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

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
    if dist:
        dist.barrier()
    # ---- timed region: profiling off, K bracketed steps ---------------------
    with Clocks(local) as clk:
        torch.cuda.profiler.start()   # ncu --profile-from-start off: the timed steps only
        step_ms, total_ms, rep_t = timed_solves(sv, b, x, prob.tol, args.steps, stream)
        torch.cuda.profiler.stop()
    if dist:
        dist.barrier()
    med_s, mean_s = reduce_max([_median(step_ms) / 1e3, total_ms / args.steps / 1e3], dist)
    iters = rep_t["iterations"]
    launches_per_step = rep_t["kernel_launches"]

    # ---- kernel statistics pass (separate; CUDA events around each launch) --
    prof_steps = 3
    sv.profile(True, True)
    prof_ms = []
    for _ in range(prof_steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, rep_p, _ = sv.solve(b, tol=prob.tol, x=x)
        e1.record(stream)
        torch.cuda.synchronize()
        prof_ms.append(e0.elapsed_time(e1))
    sv.profile(False, False)
    sparse = int(sv.options.local_factor) == 1
    # kernel classes: 0/1/2 packed SYMV (grain/contact/coarse inverse tiles),
    # 3/4 supernodal solve (grain/contact factors), 5 ILU(0), 6 fine operator
    stats = [sv.kernel_stats(k) for k in range(8)]
    fo_ms, fo_n, fo_bytes = stats[6]

    # ---- e2e: pinned host buffers through the same public call --------------
    bh_t = torch.from_numpy(np.ascontiguousarray(b_host)).pin_memory()
    xh_t = torch.zeros_like(bh_t).pin_memory()
    bh, xh = bh_t.numpy(), xh_t.numpy()
    e2e = []
    for _ in range(max(3, min(args.steps, 5))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sv.solve(bh, tol=prob.tol, x=xh)
        e2e.append(time.perf_counter() - t0)
    e2e_s = _median(e2e)

    # ---- the metric's SpMV GB/s: stored-block BSR SpMV y = A^ x alone -------
    vd = torch.from_numpy(np.random.default_rng(5).standard_normal(sv.n_dof)).cuda()
    od = torch.empty_like(vd)
    for _ in range(3):
        sv.apply("SPMV_BSR", vd, od)
    sv.profile(True, True)
    for _ in range(20):
        sv.apply("SPMV_BSR", vd, od)
    sv.profile(False, False)
    bs_ms, bs_n, bs_bytes = sv.kernel_stats(7)
    ebe = rep0.get("fine_operator", 1) == 0
    spmv = {"solve_operator": "element-by-element (matrix-free, from the voxel moduli)" if ebe
            else "bsr (stored 3x3 blocks)",
            "solve_operator_ms_per_apply": (fo_ms / fo_n) if fo_n else None,
            "solve_operator_applies_per_step": fo_n / prof_steps,
            "bsr_spmv_ms": (bs_ms / bs_n) if bs_n else None,
            "bsr_spmv_algorithmic_bytes": bs_bytes,
            "bsr_spmv_gbs": (bs_bytes / (bs_ms / bs_n / 1e3) / 1e9) if bs_n else None}
    if ebe and fo_n:
        spmv["solve_operator_algorithmic_bytes"] = fo_bytes

    # ---- algorithmic bytes per launch, per kernel class ------
    p = prob
    n = 3 * rep0["n_nodes"]
    sizes = {0: [], 1: [], 2: []}
    cptr = sv.export("CONTACT_PTR")
    sizes[1] = [int(v) for v in 3 * np.diff(cptr)]
    cls = sv.export("NODE_CLASS")
    own = sv.export("NODE_OWNER")
    gsz = np.bincount(own[cls != 1], minlength=prob.n_grains)
    sizes[0] = [int(v) for v in 3 * gsz]
    sizes[2] = [rep0["n_mortar_dofs"]]
    Lc, Lg = sum(sizes[1]), sum(sizes[0])
    alg = {k: symv_algorithmic_bytes(sizes[k]) for k in sizes}
    ilu = smoother == "ilu0"
    if ilu:
        # ILU(0) apply: every stored 3x3 block once (L forward, U and A~_II^-1
        # backward) + r read, y written and read, x written, sentinel fill
        alg[5] = stats[5][2] + 24 * 5 * rep0["n_nodes"]
        alg[3] = stats[3][2] + 16 * Lg
        alg[4] = 0
        dom = 5
        dom_name = ("k_ilu_fwd + k_ilu_bwd (ILU(0) apply, level-ordered sync-free sweeps; "
                    "bound by the dependency chain, not by HBM)")
        local_classes = (5, 4)
    elif sparse:
        # block-LDL^T solve: W_S read twice, F_SS^-1 once, row lists twice
        # (library-reported stream bytes), plus x gathered and y written (16 B/DOF)
        alg[3] = stats[3][2] + 16 * Lg
        alg[4] = stats[4][2] + 16 * Lc
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

    # ---- per-iteration algorithmic bytes (whole hot path) -----
    def op_bytes(kind):
        if kind == "ebe":   # x, v, y + node coords / Dirichlet flag, lattice map, voxel moduli
            nxyz = (p.nx, p.ny, p.nz)
            return (24 * n + 13 * rep0["n_nodes"] + 4 * (nxyz[0] + 1) * (nxyz[1] + 1) * (nxyz[2] + 1)
                    + 8 * nxyz[0] * nxyz[1] * nxyz[2])
        return 76 * rep0["nnzb"] + 4 * rep0["n_nodes"] + 24 * n   # 72 B values + 4 B col / block

    def per_iteration_bytes(kind, iterations):
        spmv_b = op_bytes(kind)
        pb = 8 * rep0["prolong_nnz"]          # P^ values (dense per-grain blocks: no indices)
        # restrict (P^ + in) and prolong (P^ + out); M_zeta scatter-sum (cptr, cidx,
        # yloc, out) and the M_g combine (gpos, yloc, a, b, out)
        small = (pb + 8 * n) + (pb + 8 * n) + (4 * n + 12 * Lc + 8 * n) + (28 * n + 8 * Lg)
        if ilu:
            minv = n_st * alg[5] + alg[2] + (n_st - 1) * spmv_b + 2 * pb + 16 * n + 16 * n * n_st
            minv_spmv = 1
        else:
            minv = alg[local_classes[0]] + alg[local_classes[1]] + alg[2] + small
            minv_spmv = 2                      # r1 = v - A y, r'' = r1 - A z1
        step = minv + (minv_spmv + 1) * spmv_b + 24 * n   # + w = A u, + scale (w -> V, vj)
        js, cycles = arnoldi_j_sequence(iterations, p.restart)
        cgs = sum((4 * (j + 1) + 6) * 8 * n for j in js)
        # per cycle of k steps: V y (k vectors read, x written), x += M^-1 (.)
        # (axpy 24 B/DOF), r = b - A^ x, ||r|| (8 B/DOF)
        ks = [min(p.restart, iterations - c * p.restart) for c in range(cycles)]
        cycle = sum(minv + (minv_spmv + 1) * spmv_b + 8 * n * (k + 1) + 24 * n + 8 * n for k in ks)
        return (iterations * step + cgs + cycle) / max(iterations, 1)

    kind = "ebe" if ebe else "bsr"
    per_iter_bytes = per_iteration_bytes(kind, iters)
    per_iter_frac = (per_iter_bytes / (med_s / max(iters, 1)) / 1e9) / peak

    # ---- the stored-block operator (operator_kind = 1) in the same line -----
    bsr_line = None
    if not args.no_bsr and not ilu:
        sb = Solver(prob, local_factor=int(lf) if lf else None, operator="bsr").assemble(local).setup()
        for _ in range(2):
            sb.solve(b, tol=prob.tol, x=x)
        sm, _, rb = timed_solves(sb, b, x, prob.tol, max(3, min(args.steps, 5)), stream)
        tb = _median(sm) / 1e3
        pib = per_iteration_bytes("bsr", rb["iterations"])
        bsr_line = {"value": tb, "unit": "s", "iterations": rb["iterations"],
                    "per_iteration": {"algorithmic_bytes": pib, "ms": tb * 1e3 / rb["iterations"],
                                      "roofline_frac": (pib / (tb / rb["iterations"]) / 1e9) / peak}}
        del sb

    # ---- multi-RHS reuse (NEXT #2): 4 load cases, one block -----
    multi = None
    if not args.no_multi and not ilu and sparse:
        from paper_2509_19777_b200 import assemble_bsr
        from workloads import load_cases
        cases = load_cases(prob, 4)
        Bh = np.stack([b_host] + [assemble_bsr(q, local)["b"] for q in cases[1:]])
        Bd = torch.from_numpy(Bh).cuda()
        Xd = torch.zeros_like(Bd)
        sv.solve_many(Bd, tol=prob.tol, X=Xd)      # warm-up (work lists of the block solves)
        ms_block = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, mreps = sv.solve_many(Bd, tol=prob.tol, X=Xd)
            e1.record(stream)
            torch.cuda.synchronize()
            ms_block.append(e0.elapsed_time(e1))
        ms_single = []
        its_single = []
        for c in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, r1, _ = sv.solve(Bd[c], tol=prob.tol, x=Xd[c])
            e1.record(stream)
            torch.cuda.synchronize()
            ms_single.append(e0.elapsed_time(e1))
            its_single.append(r1["iterations"])
        multi = {"rhs": 4, "load_cases": "workloads.load_cases (shifted prescribed displacements + "
                                         "seeded nodal forces)",
                 "block_s": _median(ms_block) / 1e3, "single_solves_s": sum(ms_single) / 1e3,
                 "one_solve_s": med_s,
                 "block_over_one_solve": _median(ms_block) / 1e3 / med_s,
                 "iterations_block": [r["iterations"] for r in mreps],
                 "iterations_single": its_single,
                 "converged": [r["converged"] for r in mreps]}

    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_{'sn' if sparse else 'symv'}_{args.config}.json")
    if os.path.exists(tp) and not ilu:
        try:
            traffic = json.load(open(tp))["dram_bytes_per_launch"]["contact" if dom == 4 else "grain"]
        except Exception:
            traffic = None

    sizes_cfg = {"n_dof": n, "nnzb": rep0["nnzb"], "grains": rep0["n_grains"],
                 "interfaces": rep0["n_interfaces"], "mortar_dofs": rep0["n_mortar_dofs"]}
    line = {
        "metric": METRIC, "value": med_s, "unit": "s", "higher_is_better": False,
        "value_stat": f"median of {args.steps} CUDA-event-bracketed solves (profiling off)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean_s * 1e3, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_of(prob, sizes_cfg, world),
        "impl_options": {"local_factor": "supernodal" if sparse else "dense-inverse",
                         "smoother": smoother, "n_st": n_st,
                         "fine_operator": "element-by-element" if ebe else "bsr",
                         "sn_shape": [rep0.get("sn_shape_grain"), rep0.get("sn_shape_contact")],
                         "sn_teams": {"grain": rep0.get("sn_teams_grain"),
                                      "contact": rep0.get("sn_teams_contact"),
                                      "max_ctas": rep0.get("sn_team_max")},
                         "sn_x_in_global": [rep0.get("sn_xg_grain"), rep0.get("sn_xg_contact")],
                         "solve_driver": "device-resident CUDA graph (one launch per solve)"
                         if (not ilu) else "host loop"},
        "iterations": iters, "iterations_per_s": iters / med_s * world,
        "solves_per_s_aggregate": world / med_s,
        "step_ms": {"min": min(step_ms), "median": _median(step_ms), "max": max(step_ms)},
        "setup_s": {"host_integer": rep0["t_host_setup_s"], "assemble": rep0["t_assemble_s"],
                    "local_T_ML": rep0["t_setup_local_s"],
                    "coarse_T_MG": rep0["t_setup_coarse_s"], "rhs": rep_t["t_rhs_s"]},
        "final_true_relres": rep_t["final_true_relres"],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": dom_name,
                     "algorithmic_bytes_per_launch": alg[dom], "launch_ms": d_ms / max(d_n, 1),
                     "launches_measured": d_n,
                     "measured_in": f"kernel-statistics pass: {prof_steps} solves after the timed "
                                    f"region, CUDA events on the library stream around each launch",
                     "peak_kind": peak_kind,
                     "local_and_coarse_solves": {
                         "achieved_gbs": agg_achieved,
                         "bytes_per_step": tot_bytes / prof_steps,
                         "share_of_step": (tot_ms / prof_steps) / _median(prof_ms)}},
        "per_iteration": {"algorithmic_bytes": per_iter_bytes, "ms": med_s * 1e3 / max(iters, 1),
                          "roofline_frac": per_iter_frac,
                          "bytes_model": "local solves + coarse S^-1 + 3 fine-operator applies + "
                                         "P^ twice + scatter/combine vectors + CGS2 at the actual "
                                         "Arnoldi index j of every step + per-cycle update"},
        "bsr_operator": bsr_line,
        "multi_rhs": multi,
        "spmv": spmv,
        "gpu_launches": int(launches_per_step * args.steps),
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n,
                "how": "hplmm_solve with pinned host b and x (H2D of b and D2H of x inside the call), "
                       "wall clock, median"},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(prob)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
