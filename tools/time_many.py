"""Time block applications hplmm_apply_many(op, k columns) against k single
applies (CUDA events), on a named workload.
usage: python tools/time_many.py cfg3 [k] [OP ...]   (PROFILE=1: one block apply
between cudaProfilerStart/Stop after the timing, for ncu --profile-from-start off)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ops = sys.argv[3:] or ["MZETA", "MGRAIN"]
p = make_problem(cfg)
sv = Solver(p).assemble(0).setup()
V = torch.from_numpy(np.random.default_rng(1).standard_normal((k, sv.n_dof))).cuda()
out = torch.empty_like(V)


def timed(f, n=10):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for op in ops:
    tb = timed(lambda: sv.apply_many(op, V, out))
    ts = timed(lambda: [sv.apply(op, V[c], out[c]) for c in range(k)])
    print(f"{cfg} {op}: block of {k} {tb:.3f} ms, {k} single applies {ts:.3f} ms "
          f"(block / one single {tb / (ts / k):.2f})", flush=True)
if os.environ.get("PROFILE"):
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    sv.apply_many(ops[0], V, out)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
