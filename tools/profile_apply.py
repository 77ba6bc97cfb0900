"""Profiling driver: setup, then ONE apply(<op>) bracketed by
cudaProfilerStart/Stop (use with ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem, random_vector

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
op = sys.argv[2] if len(sys.argv) > 2 else "MGRAIN"
lf = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = make_problem(cfg)
sv = Solver(p, local_factor=lf).assemble(0).setup()
b = torch.from_numpy(sv.export("RHS")).cuda()
sv.set_rhs(b)
v = torch.from_numpy(random_vector(sv.n_dof)).cuda()
sv.apply(op, v)
torch.cuda.synchronize()
torch.cuda.profiler.start()
sv.apply(op, v)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(cfg, op, "local_bytes", sv.report()["local_bytes"])
