"""Pins for oracle.hplmm.HPLMM.update_matrix (reuse of M_G across a perturbed
A^; reading R30).

What the paper and the algebra fix, independently of the oracle's own code:
 * the local solves follow the NEW matrix: A_new[I_g, I_g] (M_g^-1 r)[I_g] = r[I_g]
   and the same on every contact grid with a single-grid right-hand side
   (eq:Mg_Mz written out with the new blocks);
 * M_G is the ORIGINAL one: its mortar part P^_B S^-1 P^_B^T (eq:mg_struct) is
   unchanged, and it is no longer a projection for the new matrix
   (M_G A_new P_B != P_B) while it still is for the old one;
 * GMRES on the new system converges to the NEW system's solution (a sparse
   direct solve of A_new x = b_new), whatever the preconditioner's age;
 * an update with unchanged moduli is the identity on M^-1.
"""
import copy

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import fem, gmres, hplmm
from workloads import make_problem, perturbed_moduli, random_vector


def _updated(name, kind):
    p = make_problem(name)
    s, h = hplmm.setup(p)
    p2 = copy.copy(p)
    p2.E = perturbed_moduli(p, kind)
    s2 = fem.build_system(p2)
    h0 = copy.copy(h)          # shallow: keeps the original solves for comparison
    h.update_matrix(s2)
    return p, s, h0, p2, s2, h


@pytest.mark.parametrize("kind", ["crack", "global"])
def test_update_changes_the_matrix(kind):
    p, s, h0, p2, s2, h = _updated("porous20", kind)
    assert np.array_equal(s.col_idx, s2.col_idx) and np.array_equal(s.row_ptr, s2.row_ptr)
    d = abs(s2.A - s.A).max()
    assert d > 1e-3 * abs(s.A).max()


@pytest.mark.parametrize("kind", ["crack", "global"])
def test_local_solves_follow_the_new_matrix(kind):
    p, s, h0, p2, s2, h = _updated("porous20", kind)
    r = random_vector(s.n_dof)
    A2 = s2.A.tocsr()
    z = h.apply_Mg(r)
    for dg in h.grain_dofs:
        if dg.size:
            res = A2[dg][:, dg] @ z[dg] - r[dg]
            assert np.linalg.norm(res) <= 1e-10 * np.linalg.norm(r[dg])
    # one contact grid at a time (their DOF sets overlap, R19)
    for c in (0, len(h.contact_dofs) // 2, len(h.contact_dofs) - 1):
        dc = h.contact_dofs[c]
        rc = np.zeros_like(r)
        rc[dc] = r[dc]
        zc = np.zeros_like(r)
        zc[dc] = h.contact_solve[c].solve(rc[dc])
        assert np.linalg.norm(A2[dc][:, dc] @ zc[dc] - rc[dc]) <= 1e-10 * np.linalg.norm(rc[dc])
    # and differ from the old ones
    assert np.linalg.norm(z - h0.apply_Mg(r)) > 1e-6 * np.linalg.norm(z)


def test_coarse_space_is_the_original_one():
    p, s, h0, p2, s2, h = _updated("porous20", "crack")
    assert h.PB is h0.PB and h.S is h0.S
    r = random_vector(s.n_dof)
    h.corr, h0.corr = [], []
    assert np.array_equal(h.apply_MG(r), h0.apply_MG(r))
    # projection for the old matrix (eq:mg_struct), not for the new one
    e = np.zeros(h.Nm)
    e[::7] = 1.0
    v = h.PB @ e
    assert np.linalg.norm(h.apply_MG(s.A @ v) - v) <= 1e-9 * np.linalg.norm(v)
    assert np.linalg.norm(h.apply_MG(s2.A @ v) - v) >= 1e-4 * np.linalg.norm(v)


@pytest.mark.parametrize("name,kind", [("cube8", "global"), ("porous20", "crack"), ("porous20", "global")])
def test_gmres_converges_to_the_new_solution(name, kind):
    p, s, h0, p2, s2, h = _updated(name, kind)
    h.set_rhs(s2.b)
    x, it, hist, rr, conv = gmres.gmres(s2.A, s2.b, h.apply_M, tol=1e-10)
    assert conv
    xd = spla.spsolve(s2.A.tocsc(), s2.b)
    assert np.linalg.norm(x - xd) <= 1e-7 * np.linalg.norm(xd)
    # and it is NOT the old system's solution
    xo = spla.spsolve(s.A.tocsc(), s.b)
    assert np.linalg.norm(xd - xo) >= 1e-3 * np.linalg.norm(xo)
    # the fresh preconditioner needs no more iterations than the reused one + slack
    s3, h3 = hplmm.setup(p2)
    h3.set_rhs(s3.b)
    _, it3, *_ = gmres.gmres(s3.A, s3.b, h3.apply_M, tol=1e-10)
    assert it3 <= it + 2, (it3, it)


def test_identity_update_is_identity():
    p = make_problem("cube8")
    s, h = hplmm.setup(p)
    r = random_vector(s.n_dof)
    h.set_rhs(s.b)
    before = h.apply_M(r)
    h.update_matrix(fem.build_system(p))
    h.set_rhs(s.b)
    assert np.linalg.norm(h.apply_M(r) - before) <= 1e-13 * np.linalg.norm(before)


def test_residual_operator_is_the_new_matrix():
    """eq:local_smoother_CG / eq:multi_precond written out with the NEW A^
    between the stages (a stale residual operator would only cost iterations,
    which the GMRES pin cannot see)."""
    p, s, h0, p2, s2, h = _updated("cube8", "global")
    r = random_vector(s.n_dof)
    z1 = h.apply_Mzeta(r)
    assert np.linalg.norm(h.apply_MCG(r) - (z1 + h.apply_Mg(r - s2.A @ z1))) <= 1e-13 * np.linalg.norm(r)
    h.set_rhs(s2.b)
    y = h.apply_MG(r)
    want = y + h.apply_MCG(r - s2.A @ y)
    assert np.linalg.norm(h.apply_M(r) - want) <= 1e-13 * np.linalg.norm(want)
    stale = y + h.apply_MCG(r - s.A @ y)
    assert np.linalg.norm(stale - want) >= 1e-6 * np.linalg.norm(want)


def test_refresh_coarse_restores_the_projection():
    """After update_matrix + refresh_coarse M_G is again the A-orthogonal
    projection onto range(P_B) for the NEW matrix (eq:mg_struct), the shape
    vectors are A_new-harmonic in the grain interiors (eq:col_pk), and GMRES
    needs the fresh count again."""
    p, s, h0, p2, s2, h = _updated("porous20", "global")
    h.refresh_coarse()
    h.corr = []
    e = np.zeros(h.Nm)
    e[::5] = 1.0
    v = h.PB @ e
    assert np.linalg.norm(h.apply_MG(s2.A @ v) - v) <= 1e-9 * np.linalg.norm(v)
    AP = (s2.A @ h.PB).tocsr()
    scale = abs(s2.A).max() * abs(h.PB).max()
    for dg in h.grain_dofs:
        if dg.size:
            assert abs(AP[dg]).max() <= 1e-12 * scale
    h.set_rhs(s2.b)
    _, it, _, _, conv = gmres.gmres(s2.A, s2.b, h.apply_M, tol=1e-8)
    s3, h3 = hplmm.setup(p2)
    h3.set_rhs(s3.b)
    _, it3, _, _, conv3 = gmres.gmres(s3.A, s3.b, h3.apply_M, tol=1e-8)
    assert conv and conv3 and it == it3
