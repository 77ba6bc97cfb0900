"""Write the oracle's golden results for a full-size workload (cfg2 / cfg3).

Calls ONLY ``oracle/`` (and the seeded generators in ``workloads``): every
stored value is the oracle's.  Run from the repo root on a CPU box:

    python tests/golden/make_golden.py cfg3        # ~10-20 min, ~25 GB RAM

Writes tests/golden/<cfg>_oracle.json (iterations, residual history, norms,
setup/solve wall times of the oracle on this box, SHA-256 of every integer
artifact) and tests/golden/<cfg>_oracle.npz (values at 4096 sampled DOFs:
the GMRES solution x (R22) and, for the parity input v =
workloads.random_vector(n_dof) (seed 12345), M_zeta^-1 v, M_g^-1 v, M_CG^-1 v
(eq:Mg_Mz, eq:local_smoother_CG), M_G^-1 v and M^-1 v (eq:mg_struct,
eq:multi_precond) with the oracle's Cholesky coarse solve (R17), plus the same
two with an explicit S^-1 -- the spread of two correct fp64 coarse solves).
tests/test_gpu_golden.py compares the GPU path with these.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import gmres, hplmm  # noqa: E402
from workloads import make_problem, random_vector  # noqa: E402

N_SAMPLE = 4096
SAMPLE_SEED = 2024


def sample_dofs(n_dof):
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(n_dof, N_SAMPLE, replace=False))


def rss_gb():
    with open("/proc/self/statm") as f:
        return int(f.read().split()[1]) * os.sysconf("SC_PAGE_SIZE") / 1e9


def int_hash(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, np.int64)).tobytes()).hexdigest()


def csr(lists):
    ptr = np.zeros(len(lists) + 1, np.int64)
    ptr[1:] = np.cumsum([len(x) for x in lists])
    val = np.concatenate([np.asarray(x, np.int64) for x in lists]) if lists else np.zeros(0, np.int64)
    return ptr, val


def main(name):
    out = {"config": name, "n_sample": N_SAMPLE, "sample_seed": SAMPLE_SEED,
           "cores": len(os.sched_getaffinity(0))}
    p = make_problem(name)
    from oracle import fem
    t0 = time.perf_counter()
    s = fem.build_system(p)
    s.full = None        # the unconstrained matrix is only for pins (frees ~2 GB at cfg3)
    h = hplmm.HPLMM(s, n_mortar=p.n_mortar, beta=p.beta, contact_h=p.contact_h, mortar=p.mortar)
    out["t_setup_s"] = time.perf_counter() - t0
    out["t_ML_s"], out["t_MG_s"] = h.timings["T_ML"], h.timings["T_MG"]
    h.B = None           # dense per-grain shape-vector blocks: folded into h.PB already
    import gc
    gc.collect()
    print(f"setup {out['t_setup_s']:.1f} s, rss {rss_gb():.1f} GB", flush=True)
    d = h.dec
    out["n_dof"], out["nnzb"], out["Nm"] = int(s.n_dof), int(s.nnzb), int(h.Nm)
    out["n_interfaces"] = int(d.n_interfaces)
    hashes = {"NODE_KEY": int_hash(s.mesh.node_key), "ROW_PTR": int_hash(s.row_ptr),
              "COL_IDX": int_hash(s.col_idx), "NODE_CLASS": int_hash(d.node_class),
              "NODE_IFACE": int_hash(d.node_iface), "NODE_OWNER": int_hash(d.owner)}
    for key, lists in (("IFACE", d.interfaces), ("CONTACT", d.contact_nodes),
                       ("MORTAR", h.mor.nodes), ("GRAIN_COLS", h.grain_cols)):
        ptr, val = csr(lists)
        hashes[key + "_PTR"] = int_hash(ptr)
        hashes[(key + "_NODES") if key != "GRAIN_COLS" else "GRAIN_COLS"] = int_hash(val)
    out["int_sha256"] = hashes

    t0 = time.perf_counter()
    h.set_rhs(s.b)
    out["t_rhs_s"] = time.perf_counter() - t0
    out["n_coarse"] = int(h.n_coarse)
    idx = sample_dofs(s.n_dof)
    arrays = {"idx": idx}
    v = random_vector(s.n_dof)
    t0 = time.perf_counter()
    for op, f in (("MZETA", h.apply_Mzeta), ("MGRAIN", h.apply_Mg), ("MCG", h.apply_MCG),
                  ("MG", h.apply_MG), ("MINV", h.apply_M)):
        y = f(v)
        arrays[op] = y[idx]
        out["norm_" + op] = float(np.linalg.norm(y))
        print(op, flush=True)
    out["t_apply_ops_s"] = time.perf_counter() - t0
    # the same two operators with a second correct fp64 coarse solve (LU with
    # partial pivoting of S instead of its Cholesky factor): the spread any
    # correct implementation may show.  M^-1 v = y + M_L^-1 (v - A^ y) with the
    # same y = M_G^-1 v (eq:multi_precond), so one alternative coarse solve serves both.
    import scipy.linalg as sla
    rm, _ = h.restrict(v)
    lu = sla.lu_factor(h.S)
    ym_alt = sla.lu_solve(lu, rm)
    del lu
    gc.collect()
    orig = sla.cho_solve
    try:
        sla.cho_solve = lambda c, r: ym_alt if r is rm or np.array_equal(r, rm) else orig(c, r)
        y_alt = h.apply_MG(v)
        arrays["MG_inv"] = y_alt[idx]
        arrays["MINV_inv"] = (y_alt + h.apply_ML(v - h.A @ y_alt))[idx]
    finally:
        sla.cho_solve = orig
    print(f"spread done, rss {rss_gb():.1f} GB", flush=True)
    # kappa_2(S) by Lanczos on S and on S^-1 (the oracle's Cholesky solve)
    import scipy.sparse.linalg as spla
    Sop = spla.LinearOperator(h.S.shape, matvec=lambda x: h.S @ x, dtype=np.float64)
    Siop = spla.LinearOperator(h.S.shape, matvec=lambda x: sla.cho_solve(h.S_chol, x),
                               dtype=np.float64)
    lmax = float(spla.eigsh(Sop, k=1, which="LA", return_eigenvectors=False, tol=1e-6)[0])
    imax = float(spla.eigsh(Siop, k=1, which="LA", return_eigenvectors=False, tol=1e-6)[0])
    out["kappa_S"] = lmax * imax
    t0 = time.perf_counter()
    x, it, hist, rr, conv = gmres.gmres(s.A, s.b, h.apply_M, tol=p.tol, restart=p.restart,
                                         maxit=p.maxit)
    out["t_solve_s"] = time.perf_counter() - t0
    out["iterations"] = int(it)
    out["converged"] = bool(conv)
    out["final_true_relres"] = float(rr)
    out["hist"] = [float(e) for e in hist]
    out["norm_x"] = float(np.linalg.norm(x))
    out["norm_b"] = float(np.linalg.norm(s.b))
    arrays["x"] = x[idx]
    print(f"gmres {it} iterations, {out['t_solve_s']:.1f} s", flush=True)
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, f"{name}_oracle.json"), "w") as f:
        json.dump(out, f, indent=1)
    np.savez_compressed(os.path.join(here, f"{name}_oracle.npz"), **arrays)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
