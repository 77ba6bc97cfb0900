"""NEXT #3: the paper's n trade-off (T_MG grows with n, T_sol falls then
rises, Figs) on a synthetic workload: T_ML, T_MG, T_sol and
iterations for n in {1, 2, 4, 8} (n = 1 is PLMM), Gaussian and Algebraic mortars.
usage: python tools/n_sweep.py [cfg]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
p = make_problem(cfg)
print(f"{cfg}: mortar n | N_m | iterations | T_ML s | T_MG s | T_sol s | T_tot s")
for mortar in ("gaussian", "algebraic", "surface"):
    for n in (1, 2, 4, 8):
        if mortar != "gaussian" and n == 1:
            continue
        sv = Solver(p, n_mortar=n, mortar=mortar).assemble(0).setup()
        b = torch.from_numpy(sv.export("RHS")).cuda()
        sv.solve(b, tol=p.tol)
        x, rep, _ = sv.solve(b, tol=p.tol)
        r = sv.report()
        tot = r["t_setup_local_s"] + r["t_setup_coarse_s"] + rep["t_solve_s"]
        print(f"{mortar:9s} {n} | {r['n_mortar_dofs']:6d} | {rep['iterations']:3d} | "
              f"{r['t_setup_local_s']:.3f} | {r['t_setup_coarse_s']:.3f} | {rep['t_solve_s']:.4f} | "
              f"{tot:.3f}", flush=True)
        del sv
        torch.cuda.empty_cache()
