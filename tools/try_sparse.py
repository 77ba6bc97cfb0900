"""Dense-inverse vs supernodal local factors: operator agreement + solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem, random_vector

for cfg in sys.argv[1:] or ["cube8", "cfg1", "porous20"]:
    p = make_problem(cfg)
    out = {}
    for lf in (0, 1):
        t = time.time()
        sv = Solver(p, local_factor=lf).assemble(0).setup()
        rep = sv.report()
        b = torch.from_numpy(sv.export("RHS")).cuda()
        sv.set_rhs(b)
        v = torch.from_numpy(random_vector(sv.n_dof)).cuda()
        ops = {op: sv.apply(op, v).cpu().numpy() for op in ("MGRAIN", "MZETA", "MINV")}
        x, r, h = sv.solve(b, tol=1e-8)
        torch.cuda.synchronize()
        x2, r2, h2 = sv.solve(b, tol=1e-8)
        out[lf] = (ops, x.cpu().numpy(), r2)
        print(f"{cfg} lf={lf}: setup local {rep['t_setup_local_s']:.3f}s coarse {rep['t_setup_coarse_s']:.3f}s "
              f"local_bytes {rep['local_bytes']/1e9:.3f} GB; iters {r2['iterations']} t_solve {r2['t_solve_s']*1e3:.2f} ms "
              f"relres {r2['final_true_relres']:.2e} wall {time.time()-t:.1f}s", flush=True)
        del sv
    for op in out[0][0]:
        a, c = out[0][0][op], out[1][0][op]
        print(f"  {op}: rel diff {np.linalg.norm(a-c)/np.linalg.norm(a):.3e}")
    a, c = out[0][1], out[1][1]
    print(f"  x: rel diff {np.linalg.norm(a-c)/np.linalg.norm(a):.3e}")
