"""Pins for oracle/gmres.py (reading R22: right-preconditioned GMRES(m), x0 = 0,
CGS2 Arnoldi, Givens rotations) against the DEFINITION of GMRES rather than
against its own Arnoldi/Givens arithmetic:

* step j of a cycle started at x_s minimises the residual over the shifted
  Krylov space: x_j = x_s + M^-1 K_j(A M^-1, r_s), ||b - A x_j|| minimal
  (Saad & Schultz; right preconditioning), so the per-step estimate
  |g_{j+1}| / ||b|| must equal min_c ||r_s - A M^-1 K c|| / ||b|| computed by
  a least-squares solve on an independently built Krylov basis (QR of
  [r, B r, B^2 r, ...]); the returned x equals that minimiser;
* a restart begins the next cycle at the true residual of the last iterate;
* on a matrix with k distinct eigenvalues GMRES terminates at step k (the
  degree of the minimal polynomial of A with respect to b) and not before.
"""
import numpy as np
import scipy.sparse as sp

from oracle import gmres


def _krylov_min(B, r, j):
    """min_c ||r - B Q c|| and the minimiser's Q c, Q = orth basis of K_j(B, r)."""
    K = np.empty((r.size, j))
    K[:, 0] = r / np.linalg.norm(r)
    for i in range(1, j):
        v = B @ K[:, i - 1]
        K[:, i] = v / np.linalg.norm(v)
    Q, _ = np.linalg.qr(K)
    c, *_ = np.linalg.lstsq(B @ Q, r, rcond=None)
    return float(np.linalg.norm(r - B @ Q @ c)), Q @ c


def _problem(n=40, seed=7):
    rng = np.random.default_rng(seed)
    A = 3.0 * np.eye(n) + rng.standard_normal((n, n)) / np.sqrt(n)   # non-symmetric
    d = 0.5 + rng.random(n)                                          # M^-1 = diag(d)
    b = rng.standard_normal(n)
    return A, d, b


def test_history_is_the_minimal_residual():
    A, d, b = _problem()
    B = A * d[None, :]                                   # A M^-1
    m = 8
    x, it, hist, rr, conv = gmres.gmres(sp.csr_matrix(A), b, lambda v: d * v,
                                        tol=1e-300, restart=m, maxit=m)
    assert it == m and len(hist) == m and not conv
    bn = np.linalg.norm(b)
    for j in range(1, m + 1):
        res, _ = _krylov_min(B, b, j)
        assert abs(hist[j - 1] * bn - res) <= 1e-10 * bn, j
    _, y = _krylov_min(B, b, m)
    assert np.linalg.norm(x - d * y) <= 1e-10 * np.linalg.norm(x)
    assert abs(rr - np.linalg.norm(b - A @ x) / bn) <= 1e-12


def test_restart_starts_from_the_true_residual():
    A, d, b = _problem(seed=11)
    B = A * d[None, :]
    m = 3
    x, it, hist, rr, conv = gmres.gmres(sp.csr_matrix(A), b, lambda v: d * v,
                                        tol=1e-300, restart=m, maxit=2 * m)
    assert it == 2 * m and len(hist) == 2 * m
    bn = np.linalg.norm(b)
    _, y1 = _krylov_min(B, b, m)
    x1 = d * y1
    r1 = b - A @ x1
    for j in range(1, m + 1):
        res, _ = _krylov_min(B, r1, j)
        assert abs(hist[m + j - 1] * bn - res) <= 1e-10 * bn, j
    _, y2 = _krylov_min(B, r1, m)
    assert np.linalg.norm(x - (x1 + d * y2)) <= 1e-10 * np.linalg.norm(x)


def test_terminates_at_the_number_of_distinct_eigenvalues():
    rng = np.random.default_rng(3)
    k = 5
    lam = np.repeat(np.array([1.0, 2.0, 3.5, 5.0, 8.0]), 12)
    A = sp.diags(lam).tocsr()
    b = rng.standard_normal(lam.size)
    x, it, hist, rr, conv = gmres.gmres(A, b, lambda v: v.copy(), tol=1e-10)
    assert conv and it == k
    assert hist[k - 2] > 1e-6                        # not before step k
    assert np.linalg.norm(x - b / lam) <= 1e-10 * np.linalg.norm(b / lam)
