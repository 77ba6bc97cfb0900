"""ILU(0) base smoother and the n_st-stage local smoother M_L (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §4:
  eq:local_smoother
      M_L^-1 = sum_{i=1}^{n_st} M_l^-1 prod_{j=1}^{i-1} (I - A^ M_l^-1)
  P:245   "Any black-box base smoother, like ... incomplete LU-factorization
          (M_ILU(k)), can be used"
  P:484   the paper's second smoother: M_ILU(k) with n_st = 6, k = 0.

Readings (R26-R28):
  R26  ILU(0) is the scalar incomplete LU of A^ in the natural DOF order
       (node-major, R3) with the zero-fill pattern NZ = every entry of every
       stored 3x3 block (explicit zeros inside a block belong to NZ); no
       pivoting; L unit lower, U upper (Saad, Iterative Methods, Alg. 10.4,
       the IKJ variant).
  R27  M_ILU^-1 r = U^-1 (L^-1 r).
  R28  eq:local_smoother is evaluated in its written order: t_1 = r,
       u_i = M_l^-1 t_i, t_{i+1} = (I - A^ M_l^-1) t_i = t_i - A^ u_i,
       M_L^-1 r = sum_i u_i (summed in ascending i).

The factorisation below is the textbook loop, one scalar row at a time (slow,
obviously correct): for i, for k < i with (i,k) in NZ (ascending):
a_ik /= a_kk; for j > k with (i,j) in NZ: a_ij -= a_ik a_kj.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular


def block_pattern_csr(row_ptr, col_idx, val, n_nodes) -> sp.csr_matrix:
    """Scalar CSR of a 3x3-block matrix that keeps all 9 entries of every
    stored block (explicit zeros included): the ILU(0) pattern NZ (R26)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col_idx = np.asarray(col_idx, dtype=np.int64)
    val = np.asarray(val, dtype=np.float64).reshape(-1, 3, 3)
    nb = np.diff(row_ptr)
    indptr = np.zeros(3 * n_nodes + 1, dtype=np.int64)
    indptr[1:] = np.repeat(3 * nb, 3)
    indptr = np.cumsum(indptr)
    indices = np.empty(int(indptr[-1]), dtype=np.int64)
    data = np.empty(int(indptr[-1]))
    for p in range(n_nodes):
        blocks = slice(row_ptr[p], row_ptr[p + 1])
        cols = (3 * col_idx[blocks][:, None] + np.arange(3)[None, :]).ravel()
        for a in range(3):
            s = indptr[3 * p + a]
            indices[s:s + cols.size] = cols
            data[s:s + cols.size] = val[blocks, a, :].ravel()
    m = sp.csr_matrix((data, indices, indptr), shape=(3 * n_nodes, 3 * n_nodes))
    m.has_sorted_indices = True
    return m


class ILU0:
    """Scalar ILU(0) of a CSR matrix on its stored pattern (R26)."""

    def __init__(self, A: sp.csr_matrix):
        A = A.tocsr()
        A.sort_indices()
        n = A.shape[0]
        indptr, indices = A.indptr, A.indices
        a = A.data.astype(np.float64).copy()
        diag = np.full(n, -1, dtype=np.int64)
        for i in range(n):
            cols = indices[indptr[i]:indptr[i + 1]]
            d = np.searchsorted(cols, i)
            if d >= cols.size or cols[d] != i:
                raise ValueError(f"ILU(0): row {i} has no diagonal entry")
            diag[i] = indptr[i] + d
        for i in range(1, n):
            s, e = indptr[i], indptr[i + 1]
            cols = indices[s:e]
            for kp in range(s, diag[i]):            # k < i, ascending
                k = indices[kp]
                a[kp] /= a[diag[k]]                  # a_ik = a_ik / a_kk
                ks, ke = diag[k] + 1, indptr[k + 1]  # a_kj, j > k
                kc = indices[ks:ke]
                pos = np.searchsorted(cols, kc)
                hit = pos < cols.size
                hit[hit] = cols[pos[hit]] == kc[hit]
                a[s + pos[hit]] -= a[kp] * a[ks:ke][hit]   # a_ij -= a_ik a_kj
            if a[diag[i]] == 0.0:
                raise ZeroDivisionError(f"ILU(0): zero pivot in row {i}")
        F = sp.csr_matrix((a, indices.copy(), indptr.copy()), shape=A.shape)
        self.n = n
        self.L = (sp.tril(F, -1) + sp.identity(n)).tocsr()   # unit lower
        self.U = sp.triu(F).tocsr()                           # upper, pivots on diag

    def solve(self, r):
        """M_ILU^-1 r = U^-1 (L^-1 r) (R27)."""
        y = spsolve_triangular(self.L, r, lower=True, unit_diagonal=True)
        return spsolve_triangular(self.U, y, lower=False)


def local_smoother(A, base_solve, r, n_st: int):
    """eq:local_smoother applied to r, in the written order (R28)."""
    t = np.array(r, dtype=np.float64, copy=True)
    out = np.zeros_like(t)
    for i in range(n_st):
        u = base_solve(t)          # M_l^-1 prod_{j<i} (I - A^ M_l^-1) r
        out += u
        if i + 1 < n_st:
            t = t - A @ u          # (I - A^ M_l^-1) t
    return out
