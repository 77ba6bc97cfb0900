"""Reuse of M_G across perturbed moduli (hplmm_update_moduli):
update time vs a fresh setup, and GMRES iterations with the reused vs a fresh
coarse space.   usage: python tools/update_reuse.py cfg3"""
import copy, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem, perturbed_moduli

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
p = make_problem(cfg)
sv = Solver(p).assemble(0).setup()
r = sv.report()
setup_s = r["t_assemble_s"] + r["t_setup_local_s"] + r["t_setup_coarse_s"]
b = torch.from_numpy(sv.export("RHS")).cuda()
x, rep, _ = sv.solve(b, tol=p.tol)
x, rep, _ = sv.solve(b, tol=p.tol)
print(f"{cfg} original: setup {setup_s:.3f} s (assemble {r['t_assemble_s']:.3f}, T_ML {r['t_setup_local_s']:.3f}, "
      f"T_MG {r['t_setup_coarse_s']:.3f}); solve {rep['iterations']} iterations {rep['t_solve_s']:.4f} s", flush=True)
for kind in ("crack", "smooth", "global"):
    E2 = perturbed_moduli(p, kind)
    sv.update_moduli(E2)
    sv.update_moduli(E2)
    tu = sv.report()["t_update_s"]
    b2 = torch.from_numpy(sv.export("RHS")).cuda()
    x2, rep2, _ = sv.solve(b2, tol=p.tol)
    x2, rep2, _ = sv.solve(b2, tol=p.tol)
    p2 = copy.copy(p)
    p2.E = E2
    sf = Solver(p2).assemble(0).setup()
    rf = sf.report()
    x3, rep3, _ = sf.solve(b2, tol=p.tol)
    x3, rep3, _ = sf.solve(b2, tol=p.tol)
    dx = float(torch.linalg.norm(x2 - x3) / torch.linalg.norm(x3))
    print(f"{cfg} {kind}: update {tu:.3f} s, reused M_G {rep2['iterations']} iterations {rep2['t_solve_s']:.4f} s "
          f"(relres {rep2['final_true_relres']:.2e}); fresh setup "
          f"{rf['t_assemble_s'] + rf['t_setup_local_s'] + rf['t_setup_coarse_s']:.3f} s, "
          f"{rep3['iterations']} iterations {rep3['t_solve_s']:.4f} s; |x_reused - x_fresh| / |x| = {dx:.1e}",
          flush=True)
    del sf
    sv.refresh_coarse()
    tr = sv.report()["t_setup_coarse_s"]
    x4, rep4, _ = sv.solve(b2, tol=p.tol)
    x4, rep4, _ = sv.solve(b2, tol=p.tol)
    print(f"{cfg} {kind}: + refresh_coarse {tr:.3f} s -> {rep4['iterations']} iterations {rep4['t_solve_s']:.4f} s "
          f"(update + refresh {tu + tr:.3f} s)", flush=True)
    sv.update_moduli(p.E)
    sv.refresh_coarse()
