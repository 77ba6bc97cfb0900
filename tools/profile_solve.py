"""Profiling driver: setup, one warm-up solve, then ONE solve bracketed by
cudaProfilerStart/Stop (use with ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
p = make_problem(cfg)
sv = Solver(p).assemble(0).setup()
b = torch.from_numpy(sv.export("RHS")).cuda()
sv.solve(b, tol=p.tol)
torch.cuda.synchronize()
torch.cuda.profiler.start()
x, rep, hist = sv.solve(b, tol=p.tol)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(cfg, "iterations", rep["iterations"], "t_solve", rep["t_solve_s"])
