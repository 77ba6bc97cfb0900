"""Pins for the surface reading of eq:algebra (oracle/mortar.py, reading R29).

* the face element matrix: symmetric, exactly four zero-energy modes -- the
  three translations and the in-plane rotation (tangential strain only) --
  and the textbook patch test: a linear in-plane field and a linear normal
  field leave no residual at the interior nodes of a flat patch;
* the mortar blocks: exact 0/1 constraints at the mortar nodes, partition of
  unity sum_i eta_{m_i gamma} = e_gamma (by superposition: the operator
  annihilates translations), the full cap (every node a mortar) is the
  identity;
* GMRES with the resulting M^-1 reaches the direct solution.
"""
import numpy as np
import pytest

from oracle import gmres, hplmm
from oracle.mortar import surface_block, surface_face_matrix
from workloads import make_problem

CORNERS = [(0, 0), (1, 0), (0, 1), (1, 1)]


def test_face_matrix_null_space():
    K = surface_face_matrix(2.0, 0.3)
    assert np.abs(K - K.T).max() <= 1e-15 * np.abs(K).max()
    ev = np.linalg.eigvalsh(K)
    assert np.sum(np.abs(ev) < 1e-12 * ev.max()) == 4 and ev.min() > -1e-12 * ev.max()
    for c in range(3):                                    # translations
        u = np.zeros(12)
        u[c::3] = 1.0
        assert np.abs(K @ u).max() <= 1e-13
    u = np.zeros(12)                                      # in-plane rotation
    for k, (a, b) in enumerate(CORNERS):
        u[3 * k], u[3 * k + 1] = -b, a
    assert np.abs(K @ u).max() <= 1e-13


def test_face_patch_test():
    """4 x 4 nodes of a flat patch (3 x 3 faces): linear fields are exact."""
    m = 4
    node = lambda a, b: a + m * b
    K = np.zeros((3 * m * m, 3 * m * m))
    Kf = surface_face_matrix(1.0, 0.25)
    for b in range(m - 1):
        for a in range(m - 1):
            ids = [node(a + da, b + db) for da, db in CORNERS]
            idx = np.array([3 * q + c for q in ids for c in range(3)])
            K[np.ix_(idx, idx)] += Kf
    interior = [node(a, b) for b in range(1, m - 1) for a in range(1, m - 1)]
    rows = np.array([3 * q + c for q in interior for c in range(3)])
    rng = np.random.default_rng(2)
    G = rng.standard_normal((3, 2))        # u = G [a, b]^T (in-plane and normal parts)
    u = np.zeros(3 * m * m)
    for b in range(m):
        for a in range(m):
            u[3 * node(a, b):3 * node(a, b) + 3] = G @ np.array([a, b])
    assert np.abs((K @ u)[rows]).max() <= 1e-12 * np.abs(K).max()


@pytest.mark.parametrize("case", ["cube8", "porous20"])
def test_surface_blocks(case):
    p = make_problem(case)
    s, h = hplmm.setup(p, mortar="surface")
    for F, X, M in zip(h.dec.interfaces, h.mor.nodes, h.mor.blocks):
        nf, nu = len(F), len(X)
        pos = {int(y): f for f, y in enumerate(F)}
        # constraints: identity on the mortar-node rows
        con = [3 * pos[int(x)] + g for x in X for g in range(3)]
        assert np.array_equal(M[con], np.eye(3 * nu))
        # partition of unity
        S = M.reshape(nf, 3, nu, 3).sum(axis=2)
        assert np.abs(S - np.eye(3)[None]).max() <= 1e-12


def test_full_cap_identity():
    F = np.arange(4)
    faces = [([0, 1, 2, 3], (0, 1, 2), 1.0)]
    M = surface_block(F, faces, [(0, 1), (1, 3)], 0.3, 0.4, list(F))
    assert np.array_equal(M, np.eye(12))


def test_gmres_surface_mortars():
    p = make_problem("cube8")
    s, h = hplmm.setup(p, mortar="surface")
    h.set_rhs(s.b)
    x, it, hist, rr, conv = gmres.gmres(s.A, s.b, h.apply_M, tol=1e-8)
    assert conv and rr < 1e-8 and it <= 35
    xd = np.linalg.solve(s.A.toarray(), s.b)
    assert np.linalg.norm(x - xd) <= 1e-7 * np.linalg.norm(xd)
