"""Right-preconditioned restarted GMRES (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:482: "right-preconditioned GMRES ... converged if
||A^ x^ - b^|| / ||b^|| < 1e-9 or the number of iterations reaches 300".
Reading R22 (BASELINE.json + north_star): GMRES(m=50), x0 = 0, Arnoldi with
CGS2 (two classical Gram-Schmidt passes, h = h1 + h2), Givens rotations, stop
when the Arnoldi estimate |g_{j+1}|/||b|| < tol or 300 total Arnoldi steps; at
each cycle end x += M^-1 (V_j y) and the true residual b - A^ x is formed; a
new cycle starts if it is still >= tol.  Iterations = total Arnoldi steps;
history = the per-step estimates.  Happy breakdown (h_{j+1,j} == 0) ends the
cycle as converged.
"""
from __future__ import annotations

import math

import numpy as np


def gmres(A, b, Minv, tol=1e-8, restart=50, maxit=300):
    """Returns (x, iterations, history, final_true_relres, converged)."""
    n = b.size
    bnorm = float(np.linalg.norm(b))
    x = np.zeros(n)
    hist = []
    if bnorm == 0.0:
        return x, 0, hist, 0.0, True
    r = b.copy()
    total = 0
    relres = 1.0
    while True:
        beta = float(np.linalg.norm(r))
        V = np.zeros((restart + 1, n))
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(restart):
            w = A @ Minv(V[j])
            h1 = V[:j + 1] @ w                       # CGS pass 1
            w = w - V[:j + 1].T @ h1
            h2 = V[:j + 1] @ w                       # CGS pass 2
            w = w - V[:j + 1].T @ h2
            h = h1 + h2
            hn = float(np.linalg.norm(w))
            col = np.zeros(j + 2)
            col[:j + 1] = h
            col[j + 1] = hn
            for i in range(j):                       # previous rotations
                t = cs[i] * col[i] + sn[i] * col[i + 1]
                col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
                col[i] = t
            den = math.hypot(col[j], col[j + 1])
            cs[j] = col[j] / den
            sn[j] = col[j + 1] / den
            col[j] = den
            col[j + 1] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            H[:j + 1, j] = col[:j + 1]
            total += 1
            k = j + 1
            est = abs(g[j + 1]) / bnorm
            hist.append(est)
            if hn == 0.0 or est < tol or total >= maxit:
                break
            V[j + 1] = w / hn
        # y = H[:k,:k]^-1 g[:k]  (back substitution)
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        x = x + Minv(V[:k].T @ y)
        r = b - A @ x
        relres = float(np.linalg.norm(r)) / bnorm
        if relres < tol or total >= maxit:
            break
    return x, total, hist, relres, relres < tol
