"""Writes tests/golden/cfg2_update_oracle.json: the ORACLE's GMRES runs on cfg2
after HPLMM.update_matrix (M_G reused for perturbed moduli, P:743, P:819,
reading R30).  Calls only oracle/ and workloads/ (never the CUDA path).
usage: python tests/golden/make_update_golden.py      (~6 min on 8 cores)"""
import copy
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import fem, gmres, hplmm            # noqa: E402
from workloads import make_problem, perturbed_moduli   # noqa: E402

p = make_problem("cfg2")
t = time.time()
s, h = hplmm.setup(p)
out = {"config": "cfg2", "t_setup_s": time.time() - t, "cases": {}}
for kind in ("crack", "smooth", "global"):
    p2 = copy.copy(p)
    p2.E = perturbed_moduli(p, kind)
    s2 = fem.build_system(p2)
    h2 = copy.copy(h)
    h2.update_matrix(s2)
    h2.set_rhs(s2.b)
    t = time.time()
    x, it, hist, rr, conv = gmres.gmres(s2.A, s2.b, h2.apply_M, tol=1e-8, maxit=300)
    out["cases"][kind] = {"iterations": int(it), "converged": bool(conv), "final_true_relres": float(rr),
                          "hist": [float(v) for v in hist], "norm_x": float((x @ x) ** 0.5),
                          "t_solve_s": time.time() - t}
    print(kind, it, conv, rr, flush=True)
json.dump(out, open(os.path.join(HERE, "cfg2_update_oracle.json"), "w"), indent=1)
