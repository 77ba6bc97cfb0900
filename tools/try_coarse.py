"""coarse_solver 0 (explicit S^-1) vs 1 (Cholesky + triangular solves)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem, random_vector

for cfg in sys.argv[1:] or ["cube8", "porous20"]:
    p = make_problem(cfg)
    out = {}
    for cs in (0, 1):
        sv = Solver(p, coarse_solver=cs).assemble(0).setup()
        rep = sv.report()
        b = torch.from_numpy(sv.export("RHS")).cuda()
        sv.set_rhs(b)
        r = random_vector(rep["n_mortar_dofs"])
        y = sv.apply("COARSE", r)
        v = torch.from_numpy(random_vector(sv.n_dof)).cuda()
        m = sv.apply("MINV", v).cpu().numpy()
        sv.solve(b, tol=p.tol)
        x, rr, h = sv.solve(b, tol=p.tol)
        out[cs] = (y, m, x.cpu().numpy())
        print(f"{cfg} coarse_solver={cs}: T_MG {rep['t_setup_coarse_s']:.3f}s iters {rr['iterations']} "
              f"t_solve {rr['t_solve_s']*1e3:.2f} ms relres {rr['final_true_relres']:.2e}", flush=True)
        del sv
    for i, nm in enumerate(("COARSE", "MINV", "x")):
        a, c = out[0][i], out[1][i]
        print(f"  {nm}: rel diff {np.linalg.norm(a - c) / np.linalg.norm(a):.3e}")
