"""Pins for oracle/hplmm.py and oracle/gmres.py.

SURVEY §8(c) pins O10 (harmonicity, translation reproduction; eq:col_pk),
O12 (A^o = R^A^P^ brute force; eq:mg_struct), O13 (projection, coarse residual
orthogonality, full-cap exactness = App. B), O14-O16 (dense brute force of
eq:Mg_Mz, eq:local_smoother_CG, eq:multi_precond and eq:error_prop), O17
(GMRES: A = I, monotone history, dense direct solve).
"""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import decomp, gmres, hplmm
from workloads import make_problem, random_vector


def _P(h):
    return sp.hstack([h.PB, h.P_C()]).tocsc()


@pytest.mark.parametrize("case", ["cube8", "porous20"])
def test_harmonic_and_translation(case, request):
    p, s, h = request.getfixturevalue(case)
    AP = (s.A @ h.PB).tocsr()
    scale = abs(s.A).max() * abs(h.PB).max()
    for g, dg in enumerate(h.grain_dofs):
        if dg.size:
            assert abs(AP[dg]).max() <= 1e-12 * scale          # (A^ P_B)[I_g] = 0
    # translation reproduction on grains whose rows never touch a Dirichlet node
    D = s.mesh.dirichlet
    rp, ci = s.row_ptr, s.col_idx
    full_rows = s.full.indptr
    checked = 0
    for g, nodes in enumerate(h.dec.grain_nodes):
        if nodes.size == 0:
            continue
        touches = any(D[q] for pnode in nodes
                      for q in s.full.indices[full_rows[pnode]:full_rows[pnode + 1]])
        if touches or D[nodes].any():
            continue
        for gam in range(3):
            e = np.zeros(h.Nm); e[gam::3] = 1.0
            v = (h.PB @ e)[h.grain_dofs[g]].reshape(-1, 3)
            want = np.zeros(3); want[gam] = 1.0
            assert np.abs(v - want).max() <= 1e-12
        checked += 1
    assert checked > 0


def test_coarse_matrix_brute_force(cube8):
    p, s, h = cube8
    h.set_rhs(s.b)
    Ao = h.coarse_matrix_literal()
    n = h.Nm
    nc = len(h.corr)
    scale = np.abs(Ao).max()
    assert np.abs(Ao - Ao.T).max() <= 1e-12 * scale
    assert np.abs(Ao[:n, n:]).max() <= 1e-12 * scale              # R16 off-diagonal
    assert np.abs(Ao[:n, :n] - h.S).max() <= 1e-12 * scale
    Dc = np.array([Dc for _, _, Dc in h.corr])
    assert np.abs(Ao[n:, n:] - np.diag(Dc)).max() <= 1e-12 * scale
    # dense brute force P^T A P with a dense A and a dense P
    Ad = s.A.toarray(); Pd = _P(h).toarray()
    assert np.abs(Pd.T @ Ad @ Pd - Ao).max() <= 1e-12 * scale


@pytest.mark.parametrize("case", ["cube8", "porous20"])
def test_MG_projection_and_orthogonality(case, request):
    p, s, h = request.getfixturevalue(case)
    h.set_rhs(s.b)
    P = _P(h)
    z = random_vector(P.shape[1], 1)
    Pz = P @ z
    assert np.linalg.norm(h.apply_MG(s.A @ Pz) - Pz) <= 1e-12 * np.linalg.norm(Pz)
    r = s.b - s.A @ h.apply_MG(s.b)
    assert np.linalg.norm(P.T @ r) <= 1e-12 * np.linalg.norm(P.T @ s.b)


def test_full_cap_is_direct_solve():
    """App. B: with every interface node a mortar node the first pass
    equals the direct solve and GMRES converges in one iteration."""
    p = make_problem("cube8")
    s, h = hplmm.setup(p, n_mortar=10 ** 6)
    h.set_rhs(s.b)
    xs = spla.spsolve(s.A.tocsc(), s.b)
    x1 = h.apply_MG(s.b)
    assert np.linalg.norm(x1 - xs) <= 1e-10 * np.linalg.norm(xs)
    x, it, hist, rr, conv = gmres.gmres(s.A, s.b, h.apply_M)
    assert it == 1 and conv


def _dense_schwarz(Ad, sets):
    n = Ad.shape[0]
    M = np.zeros((n, n))
    for d in sets:
        if d.size:
            M[np.ix_(d, d)] += np.linalg.inv(Ad[np.ix_(d, d)])
    return M


def test_dense_brute_force_composition(cube8):
    p, s, h = cube8
    h.set_rhs(s.b)
    Ad = s.A.toarray()
    n = Ad.shape[0]
    I = np.eye(n)
    P = _P(h).toarray()
    MG = P @ np.linalg.inv(P.T @ Ad @ P) @ P.T               # eq:mg_struct literally
    Mz = _dense_schwarz(Ad, h.contact_dofs)                   # eq:Mg_Mz
    Mg = _dense_schwarz(Ad, h.grain_dofs)
    MCG = Mz + Mg @ (I - Ad @ Mz)                             # eq:local_smoother_CG
    M = MG + MCG @ (I - Ad @ MG)                              # eq:multi_precond
    r = random_vector(n)
    for f, Md in [(h.apply_MG, MG), (h.apply_Mzeta, Mz), (h.apply_Mg, Mg),
                  (h.apply_MCG, MCG), (h.apply_M, M)]:
        want = Md @ r
        assert np.linalg.norm(f(r) - want) <= 1e-12 * np.linalg.norm(want)
    # eq:error_prop: I - M^-1 A = (I - M_L^-1 A)(I - M_G^-1 A)
    E = (I - MCG @ Ad) @ (I - MG @ Ad)
    assert np.abs((I - M @ Ad) - E).max() <= 1e-10
    # M_g^-1 A e = e for e on grain-interior DOFs (O14)
    e = np.zeros(n); allg = np.concatenate(h.grain_dofs); e[allg] = random_vector(allg.size, 3)
    assert np.linalg.norm(h.apply_Mg(s.A @ e) - e) <= 1e-13 * np.linalg.norm(e) * 10


def test_gmres_identity_one_iteration():
    n = 50
    A = sp.identity(n, format="csr")
    b = random_vector(n)
    x, it, hist, rr, conv = gmres.gmres(A, b, lambda v: v.copy())
    assert it == 1 and conv and np.allclose(x, b, rtol=1e-15, atol=0)


@pytest.mark.parametrize("case", ["cube8", "cfg1"])
def test_gmres_vs_dense_direct(case, request):
    p, s, h = request.getfixturevalue(case)
    h.set_rhs(s.b)
    x, it, hist, rr, conv = gmres.gmres(s.A, s.b, h.apply_M, tol=1e-8)
    assert conv and rr < 1e-8
    assert all(b <= a * (1 + 1e-12) for a, b in zip(hist, hist[1:]))    # monotone
    xd = np.linalg.solve(s.A.toarray(), s.b)
    assert np.linalg.norm(x - xd) <= 1e-7 * np.linalg.norm(xd)
    # restarted variant reaches the same answer (exercises the restart path)
    x2, it2, _, rr2, conv2 = gmres.gmres(s.A, s.b, h.apply_M, tol=1e-8, restart=5)
    assert conv2 and np.linalg.norm(x2 - xd) <= 1e-7 * np.linalg.norm(xd)
