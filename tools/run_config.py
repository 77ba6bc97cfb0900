"""Setup + one solve of a named workload on cuda:0 (sizes, timings, memory)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem

cfg = sys.argv[1]
kw = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = int(v)
t = time.time()
p = make_problem(cfg)
print(cfg, "generated", round(time.time() - t, 1), "s", flush=True)
t = time.time()
sv = Solver(p, **kw)
print("host setup", round(time.time() - t, 1), "s", sv.report()["n_nodes"] * 3, "DOF", flush=True)
sv.assemble(0).setup()
r = sv.report()
print({k: r[k] for k in ("n_grains", "n_interfaces", "n_mortar_dofs", "local_bytes", "coarse_bytes",
                         "prolong_nnz", "t_host_setup_s", "t_assemble_s", "t_setup_local_s",
                         "t_setup_coarse_s")}, flush=True)
print("device memory allocated GB", torch.cuda.mem_get_info(), flush=True)
b = torch.from_numpy(sv.export("RHS")).cuda()
for i in range(2):
    x, rep, hist = sv.solve(b, tol=p.tol)
    print("solve", i, "iterations", rep["iterations"], "t_solve", round(rep["t_solve_s"], 4),
          "relres", rep["final_true_relres"], "converged", rep["converged"], flush=True)
