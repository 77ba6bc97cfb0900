"""Time single operator applications (device vectors) on a named workload.

usage: python tools/time_ops.py cfg3 smoother=1 n_st=6 -- MILU ML MINV SPMV
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem

args = sys.argv[1:]
cfg = args[0]
sep = args.index("--") if "--" in args else len(args)
kw = {k: int(v) for k, v in (a.split("=") for a in args[1:sep])}
ops = args[sep + 1:] or ["SPMV"]
p = make_problem(cfg)
sv = Solver(p, **kw).assemble(0).setup()
r = sv.report()
print(cfg, kw, "T_ML", round(r["t_setup_local_s"], 3), "T_MG", round(r["t_setup_coarse_s"], 3),
      flush=True)
b = torch.from_numpy(sv.export("RHS")).cuda()
sv.set_rhs(b)
v = torch.from_numpy(np.random.default_rng(1).standard_normal(sv.n_dof)).cuda()
out = torch.empty_like(v)
for op in ops:
    for _ in range(3):
        sv.apply(op, v, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        sv.apply(op, v, out)
    e1.record()
    torch.cuda.synchronize()
    print(op, "ms per apply", round(e0.elapsed_time(e1) / n, 3), flush=True)
if os.environ.get("NOSOLVE"):
    sys.exit(0)
x, rep, _ = sv.solve(b, tol=p.tol)
print("solve iterations", rep["iterations"], "t_solve", round(rep["t_solve_s"], 4), "relres",
      rep["final_true_relres"], flush=True)
