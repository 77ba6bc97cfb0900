"""Measured GPU-vs-oracle errors (not pass/fail) at the full-size golden runs
(tests/golden/<cfg>_oracle.*) in the bench launch configuration: iterations,
history, x at the sampled DOFs, and every operator with its gate.
usage: python tools/parity_report.py cfg2 cfg3"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2509_19777_b200 import Solver
from workloads import make_problem, random_vector

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
for name in sys.argv[1:] or ["cfg2", "cfg3"]:
    g = json.load(open(os.path.join(G, f"{name}_oracle.json")))
    a = dict(np.load(os.path.join(G, f"{name}_oracle.npz")))
    p = make_problem(name)
    sv = Solver(p).assemble(0).setup()
    r = sv.report()
    b = torch.from_numpy(sv.export("RHS")).cuda()
    x, rep, hist = sv.solve(b, tol=p.tol)
    x = x.cpu().numpy()
    idx = a["idx"]
    k = min(len(hist), len(g["hist"]))
    out = {"config": name, "sn_shape": [r["sn_shape_grain"], r["sn_shape_contact"]],
           "iterations": [rep["iterations"], g["iterations"]],
           "hist_max_rel_dev": float(np.max(np.abs(np.asarray(hist[:k]) / np.asarray(g["hist"][:k]) - 1))),
           "x_rel_err_sampled": rel(x[idx], a["x"]), "kappa_S": g.get("kappa_S")}
    v = torch.from_numpy(random_vector(g["n_dof"])).cuda()
    sv.set_rhs(b)
    for op in ("MZETA", "MGRAIN", "MCG", "MG", "MINV"):
        y = sv.apply(op, v).cpu().numpy()[idx]
        e = {"err": rel(y, a[op])}
        if op in ("MG", "MINV"):
            e["oracle_spread_chol_vs_lu"] = rel(a[op + "_inv"], a[op])
            e["gate"] = max(1e-12, 10 * e["oracle_spread_chol_vs_lu"], 3 * g.get("kappa_S", 0) * 2.0 ** -53)
        else:
            e["gate"] = 1e-12
        out[op] = e
    print(json.dumps(out), flush=True)
