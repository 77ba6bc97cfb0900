"""Stress of the subtree-parallel team solves (exchange flags, one-shot reset): 300 random
vectors through M_zeta / M_g with teams against the one-CTA-per-subdomain solves of the same
factors (cfg2), then 40 graph solves.  usage: python tools/stress_teams.py"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem
p = make_problem("cfg2")
a = Solver(p).assemble(0).setup()
b = Solver(p, sn_split=-1).assemble(0).setup()
print(a.report()["sn_teams_grain"], a.report()["sn_teams_contact"], b.report()["sn_teams_grain"])
rng = np.random.default_rng(0)
worst = 0.0
for it in range(300):
    v = torch.from_numpy(rng.standard_normal(a.n_dof)).cuda()
    for op in ("MZETA", "MGRAIN"):
        ya = a.apply(op, v); yb = b.apply(op, v)
        d = float(torch.linalg.norm(ya - yb) / torch.linalg.norm(yb))
        worst = max(worst, d)
        assert d < 1e-12, (it, op, d)
print("300 x 2 applies, worst rel diff", worst)
rhs = torch.from_numpy(a.export("RHS")).cuda()
its = set()
for it in range(40):
    x, rep, _ = a.solve(rhs, tol=1e-8)
    its.add((rep["iterations"], rep["converged"]))
print("40 graph solves:", its)
