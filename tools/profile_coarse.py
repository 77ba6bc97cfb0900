"""One COARSE apply under cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem, random_vector
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = make_problem(cfg)
sv = Solver(p, coarse_solver=cs).assemble(0).setup()
r = torch.from_numpy(random_vector(sv.report()["n_mortar_dofs"])).cuda()
sv.apply("COARSE", r)
torch.cuda.synchronize()
torch.cuda.profiler.start()
sv.apply("COARSE", r)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
