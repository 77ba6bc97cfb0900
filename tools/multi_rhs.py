"""NEXT #2 (multi-RHS reuse, P:743 / P:819): one setup, K right-hand sides.

Reports T_setup (T_ML + T_MG), the per-RHS cost of solve_many (correction
columns + GMRES) and the amortised time per RHS against setup + solve each time.
usage: python tools/multi_rhs.py [cfg] [K]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = make_problem(cfg)
sv = Solver(p).assemble(0)
torch.cuda.synchronize()
t0 = time.perf_counter()
sv.setup()
torch.cuda.synchronize()
t_setup = time.perf_counter() - t0
r = sv.report()
b = sv.export("RHS")
# K load cases: the configured load scaled, plus smooth random body loads
rng = np.random.default_rng(5)
B = np.stack([b * (1.0 + 0.25 * k) + (0.0 if k == 0 else 1e-3) * np.linalg.norm(b) /
              np.sqrt(b.size) * rng.standard_normal(b.size) for k in range(K)])
Bd = torch.from_numpy(B).cuda()
sv.solve_many(Bd[:1])            # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
X, reps = sv.solve_many(Bd)
torch.cuda.synchronize()
t_many = time.perf_counter() - t0
its = [q["iterations"] for q in reps]
print(f"{cfg}: setup {t_setup:.3f} s (T_ML {r['t_setup_local_s']:.3f}, T_MG {r['t_setup_coarse_s']:.3f}); "
      f"{K} RHS in {t_many:.3f} s = {t_many / K:.3f} s per RHS (iterations {its}, "
      f"relres max {max(q['final_true_relres'] for q in reps):.2e}); "
      f"amortised (setup + solves) / K = {(t_setup + t_many) / K:.3f} s vs setup + solve "
      f"= {t_setup + t_many / K:.3f} s per RHS")
