"""GPU parity of the ILU(0) base smoother and the n_st-stage local smoother
(eq:local_smoother; readings R26-R28) against the oracle.

* MILU (one U^-1 L^-1 apply), ML (n_st stages) and MINV vs oracle/ilu.py +
  oracle/hplmm.py, rel-L2 <= 1e-12 (MINV: max(1e-12, the coarse kappa floor)).
* The exported block factor satisfies ILU(0)'s defining equations
  (L U)_IJ = A_IJ on every stored block (checked at every row here, on sampled
  rows at full size in test_gpu_fullsize.py).
* GMRES with M_G + ILU(0), n_st = 6 (the paper's pairing): iterations within
  +-1 of the oracle, x rel-L2 <= 1e-8.
* n_st > 1 with the contact-grain base smoother (apply parity only: the
  stationary M_CG iteration is not convergent, rho(I - M_CG^-1 A) ~ 11 on
  cube8, so its multi-stage M_L is not a useful preconditioner -- the paper's
  n_st = 1 for M_CG).
"""
import numpy as np
import pytest

from tests.test_gpu_parity import coarse_floor, coarse_spread_gate, dev, rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = ["cube8", "cfg1", "porous20"]
_cache = {}


def ilu_case(name, smoother="ilu0", n_st=6, lf=1):
    key = (name, smoother, n_st, lf)
    if key not in _cache:
        import __graft_entry__
        __graft_entry__.build()
        from oracle import hplmm
        from paper_2509_19777_b200 import Solver
        from workloads import make_problem
        p = make_problem(name)
        s, h = hplmm.setup(p, smoother=smoother, n_st=n_st)
        sv = Solver(p, local_factor=lf, smoother=smoother, n_st=n_st).assemble(0).setup()
        _cache[key] = (p, s, h, sv)
    return _cache[key]


def block_factors(sv, s):
    """(L_B, U_B) as scipy BSR from the exported factor: L_IK below the
    diagonal with identity diagonal blocks, A~_IJ above it, A~_II = inv(stored)."""
    import scipy.sparse as sp
    F = sv.export("ILU").reshape(-1, 3, 3)
    rp, ci = s.row_ptr, s.col_idx
    rows = np.repeat(np.arange(rp.size - 1), np.diff(rp))
    lo, dg, up = ci < rows, ci == rows, ci > rows
    n = 3 * (rp.size - 1)

    def bsr(mask, blocks):
        r, c = rows[mask], ci[mask]
        ptr = np.zeros(rp.size, dtype=np.int64)
        np.add.at(ptr, r + 1, 1)
        return sp.bsr_matrix((blocks, c, np.cumsum(ptr)), shape=(n, n))

    eye = np.broadcast_to(np.eye(3), (int(dg.sum()), 3, 3))
    L = (bsr(lo, F[lo]) + bsr(dg, eye)).tocsr()
    U = (bsr(up, F[up]) + bsr(dg, np.linalg.inv(F[dg]))).tocsr()
    return L, U


@pytest.mark.parametrize("case", CASES)
def test_ilu_apply(case):
    p, s, h, sv = ilu_case(case)
    v = np.random.default_rng(12345).standard_normal(s.n_dof)
    assert rel(sv.apply("MILU", dev(v)).cpu().numpy(), h.ilu.solve(v)) <= 1e-12
    assert rel(sv.apply("ML", v), h.apply_ML(v)) <= 1e-12
    h.set_rhs(s.b)
    sv.set_rhs(s.b)
    ref = h.apply_M(v)
    assert rel(sv.apply("MINV", v), ref) <= coarse_spread_gate(h, "MINV", v, ref)


@pytest.mark.parametrize("case", CASES)
def test_ilu_factor_equations(case):
    p, s, h, sv = ilu_case(case)
    L, U = block_factors(sv, s)
    LU = (L @ U).tocsr()
    A = s.A.tocsr()
    # on every stored entry of A^ (block pattern incl. explicit zeros)
    from oracle.ilu import block_pattern_csr
    P = block_pattern_csr(s.row_ptr, s.col_idx, s.val, s.mesh.n_nodes)
    r, c = P.nonzero()
    d = np.asarray(LU[r, c]).ravel() - np.asarray(A[r, c]).ravel()
    assert np.abs(d).max() <= 1e-12 * np.abs(s.val).max()
    # and the apply is U^-1 L^-1: L (U z) = v
    v = np.random.default_rng(1).standard_normal(s.n_dof)
    z = sv.apply("MILU", v)
    assert rel(L @ (U @ z), v) <= 1e-13


@pytest.mark.parametrize("case", CASES)
def test_ilu_solve(case):
    from oracle import gmres
    p, s, h, sv = ilu_case(case)
    h.set_rhs(s.b)
    xo, ito, _, _, convo = gmres.gmres(s.A, s.b, h.apply_M, tol=1e-8)
    x, rep, hist = sv.solve(dev(s.b), tol=1e-8)
    x = x.cpu().numpy()
    assert convo and rep["converged"] == 1
    assert abs(rep["iterations"] - ito) <= 1, (rep["iterations"], ito)
    assert rel(x, xo) <= 1e-8
    assert np.linalg.norm(s.b - s.A @ x) / np.linalg.norm(s.b) < 1e-8


def test_ilu_dense_local_factor():
    """local_factor = 0 (dense grain inverses) with the ILU smoother."""
    from oracle import gmres
    p, s, h, sv = ilu_case("porous20", lf=0)
    h.set_rhs(s.b)
    xo, ito, _, _, _ = gmres.gmres(s.A, s.b, h.apply_M, tol=1e-8)
    x, rep, _ = sv.solve(s.b.copy(), tol=1e-8)
    assert rep["converged"] == 1 and abs(rep["iterations"] - ito) <= 1
    assert rel(x, xo) <= 1e-8


@pytest.mark.parametrize("n_st", [1, 2, 3])
def test_ilu_stage_count(n_st):
    p, s, h, sv = ilu_case("cfg1", n_st=n_st)
    v = np.random.default_rng(12345).standard_normal(s.n_dof)
    assert rel(sv.apply("ML", v), h.apply_ML(v)) <= 1e-12


@pytest.mark.parametrize("case", ["cube8", "porous20"])
def test_cg_two_stages(case):
    p, s, h, sv = ilu_case(case, smoother="cg", n_st=2)
    v = np.random.default_rng(12345).standard_normal(s.n_dof)
    assert rel(sv.apply("ML", v), h.apply_ML(v)) <= 1e-12
    h.set_rhs(s.b)
    sv.set_rhs(s.b)
    ref = h.apply_M(v)
    assert rel(sv.apply("MINV", v), ref) <= coarse_spread_gate(h, "MINV", v, ref)


def test_ilu_state_errors():
    from paper_2509_19777_b200 import HPLMMError as HplmmError
    p, s, h, sv = ilu_case("cube8")
    v = np.ones(s.n_dof)
    for op in ("MZETA", "MCG"):
        with pytest.raises(HplmmError):
            sv.apply(op, v)
    p2, s2, h2, sv2 = ilu_case("cube8", smoother="cg", n_st=1)
    with pytest.raises(HplmmError):
        sv2.apply("MILU", v)
    with pytest.raises(HplmmError):
        sv2.export("ILU")
