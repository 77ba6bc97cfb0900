"""Multi-RHS blocks (the paper's reuse of one setup for
several load cases): hplmm_solve_many solves up to 4 right-hand
sides in lockstep GMRES(50) with every operator application batched (the
supernodal factors and P^_B streamed once per block).  Each column must be
exactly its own GMRES run (R22) with its own correction columns (eq:col_cg,
R15): compared column by column with the ORACLE's GMRES on that right-hand side
-- iterations +-1, x rel-L2 <= 1e-8, true residual < tol -- and with the
per-column path (rhs_block = 1).
"""
import numpy as np
import pytest

from tests.conftest import oracle_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _rhs(name, k):
    """k right-hand sides of the oracle's system: the load cases of
    workloads.load_cases (assembled by the oracle), one of them zero if k == 4."""
    from oracle import fem
    from workloads import load_cases
    p, s, h = oracle_case(name)
    bs = [fem.build_system(q).b for q in load_cases(p, k)]
    if k == 4:
        bs[2] = np.zeros_like(bs[2])          # b = 0 => x = 0, 0 iterations
    return p, s, h, np.stack(bs)


@pytest.mark.parametrize("case", ["cube8", "cfg1", "porous20"])
@pytest.mark.parametrize("k", [2, 3, 4])
def test_solve_many_block_vs_oracle(case, k):
    from oracle import gmres
    from paper_2509_19777_b200 import Solver
    p, s, h, B = _rhs(case, k)
    sv = Solver(p, rhs_block=4).assemble(0).setup()   # blocks (automatic would pick team solves here)
    X, reps = sv.solve_many(torch.from_numpy(B).cuda(), tol=1e-8)
    X = X.cpu().numpy()
    for c in range(k):
        b = B[c]
        if not np.any(b):
            assert reps[c]["iterations"] == 0 and not np.any(X[c])
            continue
        h.set_rhs(b)
        xo, ito, _, _, convo = gmres.gmres(s.A, b, h.apply_M, tol=1e-8)
        assert convo and reps[c]["converged"] == 1
        assert abs(reps[c]["iterations"] - ito) <= 1, (c, reps[c]["iterations"], ito)
        assert rel(X[c], xo) <= 1e-8, (c, rel(X[c], xo))
        assert np.linalg.norm(b - s.A @ X[c]) / np.linalg.norm(b) < 1e-8


@pytest.mark.parametrize("case", ["cfg1", "porous20"])
def test_solve_many_block_matches_per_column(case):
    from paper_2509_19777_b200 import Solver
    p, s, h, B = _rhs(case, 3)
    a = Solver(p, rhs_block=4).assemble(0).setup()
    b = Solver(p, rhs_block=1).assemble(0).setup()
    Xa, ra = a.solve_many(B.copy(), tol=1e-8)          # host buffers
    Xb, rb = b.solve_many(B.copy(), tol=1e-8)
    for c in range(3):
        assert ra[c]["iterations"] == rb[c]["iterations"]
        assert rel(Xa[c], Xb[c]) <= 1e-9


def test_solve_many_restart_and_cap():
    """Restart cycles (m = 5) and the iteration cap inside a block: every column
    follows its own cycle sequence, as the single-RHS path does."""
    from paper_2509_19777_b200 import Solver
    p, s, h, B = _rhs("cfg1", 3)
    a = Solver(p, restart=5, rhs_block=4).assemble(0).setup()
    b = Solver(p, restart=5, rhs_block=1).assemble(0).setup()
    Xa, ra = a.solve_many(B.copy(), tol=1e-8)
    Xb, rb = b.solve_many(B.copy(), tol=1e-8)
    for c in range(3):
        assert ra[c]["iterations"] == rb[c]["iterations"] and ra[c]["converged"] == 1
        assert rel(Xa[c], Xb[c]) <= 1e-9
    capped = Solver(p, max_iter=7, restart=5, rhs_block=4).assemble(0).setup()
    Xc, rc = capped.solve_many(B.copy(), tol=1e-8)
    assert all(r["iterations"] == 7 and r["converged"] == 0 for r in rc)


_mr_solvers = {}


@pytest.mark.parametrize("shape", [8, 16])
@pytest.mark.parametrize("case", ["cube8", "cfg1", "porous20"])
@pytest.mark.parametrize("op", ["SPMV", "MZETA", "MGRAIN", "MCG"])
@pytest.mark.parametrize("k", [2, 3, 4])
def test_apply_many_vs_oracle(case, op, k, shape):
    """The block local solves (k_sn_solve with NRHS = 2 / 4 columns, x in
    global memory with x_S / x_R staged per supernode) in both launch shapes --
    8 consumer warps x 2 CTAs per SM, what cfg3's multi-RHS block runs, and
    16 x 1 -- column by column against the oracle's M_zeta^-1, M_g^-1 and
    M_CG^-1 (eq:Mg_Mz, eq:local_smoother_CG) at north_star's 1e-12; SPMV: the
    block element-by-element operator (k_ebe_k) against the oracle's A^."""
    from paper_2509_19777_b200 import Solver
    if (case, shape) not in _mr_solvers:
        p, s, h = oracle_case(case)
        _mr_solvers[(case, shape)] = Solver(p, sn_shape=shape).assemble(0).setup()
    sv = _mr_solvers[(case, shape)]
    p, s, h = oracle_case(case)
    V = np.random.default_rng(12345 + k).standard_normal((k, s.n_dof))
    out = sv.apply_many(op, torch.from_numpy(V).cuda()).cpu().numpy()
    ref = {"MZETA": h.apply_Mzeta, "MGRAIN": h.apply_Mg, "MCG": h.apply_MCG,
           "SPMV": lambda v: s.A @ v}[op]
    for c in range(k):
        r = ref(V[c])
        assert rel(out[c], r) <= 1e-12, (c, rel(out[c], r))


def test_apply_many_errors():
    """hplmm_apply_many's argument and state checks (include/hplmm.h): bad op,
    ncols outside 1..4, ld < n_dof -> ERR_ARG; the dense local solver -> ERR_STATE."""
    from paper_2509_19777_b200 import Solver
    from paper_2509_19777_b200.hplmm import HPLMMError
    p, s, h = oracle_case("cube8")
    sv = Solver(p).assemble(0).setup()
    V = torch.zeros((5, s.n_dof), dtype=torch.float64, device="cuda")
    for op, cols in (("MG", 2), ("MZETA", 5)):
        with pytest.raises(HPLMMError, match="ERR_ARG"):
            sv.apply_many(op, V[:cols])
    with pytest.raises(HPLMMError, match="ERR_ARG"):
        sv.apply_many("MZETA", V[:2, :-1].contiguous())   # ld = n_dof - 1
    dense = Solver(p, local_factor=0).assemble(0).setup()
    with pytest.raises(HPLMMError, match="ERR_STATE"):
        dense.apply_many("MZETA", V[:2])


def test_solve_many_automatic_block_choice():
    """rhs_block = 0 (default): a batch that forms CTA teams (these small cases)
    solves column by column, one without teams in blocks -- same results."""
    from paper_2509_19777_b200 import Solver
    p, s, h, B = _rhs("cfg1", 3)
    auto = Solver(p).assemble(0).setup()
    assert auto.report()["sn_teams_grain"] > 0
    blk = Solver(p, sn_split=-1).assemble(0).setup()          # no teams: automatic = blocks
    Xa, ra = auto.solve_many(B.copy(), tol=1e-8)
    Xb, rb = blk.solve_many(B.copy(), tol=1e-8)
    for c in range(3):
        assert ra[c]["converged"] == 1 and rb[c]["converged"] == 1
        assert abs(ra[c]["iterations"] - rb[c]["iterations"]) <= 1
        assert rel(Xa[c], Xb[c]) <= 1e-8
