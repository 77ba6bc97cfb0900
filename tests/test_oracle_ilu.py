"""Pins for oracle/ilu.py (ILU(0) base smoother, eq:local_smoother).

What pins it (none of these retypes the oracle's loop):
* exactness where ILU(0) drops nothing: a tridiagonal matrix (Thomas
  algorithm = exact LU) and the FEM matrix of a 1 x 1 x n voxel column, whose
  block pattern is closed under fill (its rows' envelopes lie inside NZ), so
  M_ILU^-1 = A^-1 (numpy.linalg.solve);
* the defining equations of ILU(0): L unit lower, U upper, both inside NZ,
  (L U)_ij = a_ij on NZ (Saad, Def. of ILU(0)) -- they determine L, U uniquely;
* an independent loop order: the right-looking KIJ elimination with dropping,
  on a small random sparse matrix and a tiny FEM matrix;
* symmetry: for symmetric A, U = diag(U) L^T;
* eq:local_smoother's error propagation (I - M_L^-1 A) = (I - M_l^-1 A)^n_st
  (eq:error_prop's smoother factor), for both base smoothers;
* GMRES with M_G + M_ILU(0), n_st = 6 converges to the direct solution.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import gmres, hplmm
from oracle.fem import build_system
from oracle.ilu import ILU0, block_pattern_csr, local_smoother
from workloads import Problem, make_problem, random_vector


def _pattern(A):
    A = A.tocsr()
    return sp.csr_matrix((np.ones(A.nnz), A.indices, A.indptr), shape=A.shape).toarray() != 0


def _system_pattern(s):
    return block_pattern_csr(s.row_ptr, s.col_idx, s.val, s.mesh.n_nodes)


def _kij(Ad, mask):
    """Right-looking (KIJ) incomplete elimination on a dense copy: entries
    outside the mask are never created."""
    a = np.where(mask, Ad, 0.0).astype(np.float64)
    n = a.shape[0]
    for k in range(n - 1):
        rows = np.nonzero(mask[k + 1:, k])[0] + k + 1
        for i in rows:
            a[i, k] /= a[k, k]
            cols = np.nonzero(mask[i, k + 1:] & mask[k, k + 1:])[0] + k + 1
            a[i, cols] -= a[i, k] * a[k, cols]
    return np.tril(a, -1) + np.eye(n), np.triu(a)


def test_tridiagonal_is_exact():
    n = 40
    rng = np.random.default_rng(3)
    d = 4.0 + rng.random(n)
    off = rng.standard_normal(n - 1)
    A = sp.diags([off, d, off], [-1, 0, 1], format="csr")
    r = rng.standard_normal(n)
    z = ILU0(A).solve(r)
    x = np.linalg.solve(A.toarray(), r)
    assert np.linalg.norm(z - x) <= 1e-13 * np.linalg.norm(x)


def _box_problem(nz, ny=1, nx=1):
    """nx x ny x nz solid box (one grain), bottom clamped, top corners loaded."""
    solid = np.ones((nz, ny, nx), dtype=np.uint8)
    q = Problem(name="box", nx=nx, ny=ny, nz=nz, solid=solid, E=np.ones(solid.shape), nu=0.3,
                grain=np.zeros(solid.shape, dtype=np.int32), n_grains=1,
                node_dirichlet=np.zeros((nz + 1, ny + 1, nx + 1), dtype=np.uint8),
                node_u=np.zeros((nz + 1, ny + 1, nx + 1, 3)),
                node_f=np.zeros((nz + 1, ny + 1, nx + 1, 3)), block=max(nx, ny, nz))
    q.node_dirichlet[0] = 1
    q.node_f[nz, :, :, 2] = -0.25
    return q


def test_fill_closed_pattern_is_exact():
    s = build_system(_box_problem(6))
    A = _system_pattern(s)
    r = random_vector(A.shape[0])
    z = ILU0(A).solve(r)
    x = np.linalg.solve(s.A.toarray(), r)
    assert np.linalg.norm(z - x) <= 1e-12 * np.linalg.norm(x)


def test_defining_equations_cube8():
    s = build_system(make_problem("cube8"))
    A = _system_pattern(s)
    il = ILU0(A)
    NZ = _pattern(A)
    L, U = il.L.toarray(), il.U.toarray()
    assert np.all(np.diag(L) == 1.0) and not np.any(np.triu(L, 1))
    assert not np.any(np.tril(U, -1))
    assert not np.any((L != 0) & ~NZ & ~np.eye(L.shape[0], dtype=bool))
    assert not np.any((U != 0) & ~NZ)
    Ad = A.toarray()
    LU = L @ U
    scale = np.abs(Ad).max()
    assert np.abs((LU - Ad)[NZ]).max() <= 1e-12 * scale
    # something is dropped (otherwise this would be an exact LU)
    assert np.abs((LU - Ad)[~NZ]).max() > 1e-6 * scale
    # symmetric A: U = diag(U) L^T
    assert np.abs(U - np.diag(np.diag(U)) @ L.T).max() <= 1e-12 * scale


def test_kij_agrees_random_sparse():
    rng = np.random.default_rng(11)
    n = 60
    M = sp.random(n, n, density=0.08, random_state=rng, format="csr")
    A = (M + M.T + sp.identity(n) * 6.0).tocsr()
    A.sort_indices()
    il = ILU0(A)
    L, U = _kij(A.toarray(), _pattern(A))
    assert np.abs(il.L.toarray() - L).max() <= 1e-13
    assert np.abs(il.U.toarray() - U).max() <= 1e-13 * np.abs(U).max()


def test_kij_agrees_tiny_fem():
    s = build_system(_box_problem(3, 2, 2))
    A = _system_pattern(s)
    il = ILU0(A)
    L, U = _kij(A.toarray(), _pattern(A))
    assert np.abs(il.L.toarray() - L).max() <= 1e-12
    assert np.abs(il.U.toarray() - U).max() <= 1e-12 * np.abs(U).max()


@pytest.mark.parametrize("smoother,n_st", [("ilu0", 1), ("ilu0", 3), ("ilu0", 6), ("cg", 2)])
def test_error_propagation(smoother, n_st):
    p = make_problem("cube8")
    s, h = hplmm.setup(p, smoother=smoother, n_st=n_st)
    A = s.A
    e = random_vector(s.n_dof, seed=5)
    lhs = e - h.apply_ML(A @ e)
    v = e.copy()
    for _ in range(n_st):
        v = v - h.apply_Ml(A @ v)
    assert np.linalg.norm(lhs - v) <= 1e-12 * max(np.linalg.norm(v), np.linalg.norm(e))
    if n_st == 1:   # M_L = M_l
        r = random_vector(s.n_dof, seed=6)
        assert np.array_equal(h.apply_ML(r), h.apply_Ml(r))


def test_local_smoother_order():
    """local_smoother with a scalar 'smoother' m: M_L = m sum_i (1 - a m)^(i-1)."""
    a, m, n_st = 3.0, 0.2, 5
    A = sp.identity(1, format="csr") * a
    got = local_smoother(A, lambda t: m * t, np.array([1.0]), n_st)[0]
    want = m * sum((1 - a * m) ** i for i in range(n_st))
    assert abs(got - want) <= 1e-15


@pytest.mark.parametrize("case", ["cube8", "porous20"])
def test_gmres_ilu_converges(case):
    p = make_problem(case)
    s, h = hplmm.setup(p, smoother="ilu0", n_st=6)
    h.set_rhs(s.b)
    x, it, hist, rr, conv = gmres.gmres(s.A, s.b, h.apply_M, tol=1e-8)
    assert conv and rr < 1e-8 and it < 50
    xd = np.linalg.solve(s.A.toarray(), s.b) if s.n_dof < 5000 else None
    if xd is not None:
        assert np.linalg.norm(x - xd) <= 1e-6 * np.linalg.norm(xd)
