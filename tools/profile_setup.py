"""Profiling driver: hplmm_setup bracketed by cudaProfilerStart/Stop
(use with ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
lf = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = make_problem(cfg)
sv = Solver(p, local_factor=lf).assemble(0)
torch.cuda.synchronize()
torch.cuda.profiler.start()
sv.setup()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(cfg, sv.report()["t_setup_local_s"], sv.report()["t_setup_coarse_s"])
