"""Profiling driver: setup, one warm-up hplmm_solve_many of K load cases, then
ONE more between cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver, assemble_bsr
from workloads import load_cases, make_problem

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = make_problem(cfg)
sv = Solver(p).assemble(0).setup()
B = np.stack([sv.export("RHS")] + [assemble_bsr(q, 0)["b"] for q in load_cases(p, K)[1:]])
Bd = torch.from_numpy(B).cuda()
X, reps = sv.solve_many(Bd, tol=p.tol)
torch.cuda.synchronize()
torch.cuda.profiler.start()
X, reps = sv.solve_many(Bd, tol=p.tol)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(cfg, K, [r["iterations"] for r in reps], reps[0]["t_solve_s"])
