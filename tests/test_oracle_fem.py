"""Pins for oracle/fem.py against closed forms / invariants (not against itself).

SURVEY §8(c) pin table rows O1, O2, O3.
"""
import itertools

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import fem
from workloads import Problem, make_problem


def test_cfg1_counts():
    # BASELINE.json configs[0]: 14,739 DOF = 17^3 * 3; nnzb closed form
    # (3*17-2)^3 = 117,649 before and 110,735 after Dirichlet removal
    # (tests/golden/cfg1_counts.json).
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg1_counts.json")))
    s = fem.build_system(make_problem("cfg1"))
    assert s.n_dof == g["n_dof"] == 17 ** 3 * 3
    assert s.full.nnz // 9 == g["nnzb_full"] == (3 * 17 - 2) ** 3
    assert s.nnzb == g["nnzb_constrained"]
    assert int(s.mesh.dirichlet.sum()) == g["dirichlet_nodes"] == 17 * 17


@pytest.mark.parametrize("nu", [0.25, 0.3, 0.45])
def test_K0_kernel_and_exactness(nu):
    K = fem.element_K0(nu)
    assert np.abs(K - K.T).max() <= 1e-15 * np.abs(K).max()
    ev = np.linalg.eigvalsh(0.5 * (K + K.T))
    tol = 1e-12 * ev.max()
    assert np.sum(np.abs(ev) < tol) == 6          # 3 translations + 3 rotations
    assert np.sum(ev > tol) == 18
    # 2x2x2 Gauss is exact for constant-coefficient Q1 (equals 3x3x3)
    assert np.abs(fem.element_K0(nu, 3) - K).max() <= 1e-14 * np.abs(K).max()


def test_K0_constant_strain_closed_form():
    """u = eps x (eps symmetric)  =>  K0 u = boundary integral of sigma.n N_a:
    each corner gets, from each of its 3 faces, sigma.n * (1/4)."""
    rng = np.random.default_rng(0)
    nu = 0.3
    e = rng.standard_normal((3, 3)); e = 0.5 * (e + e.T)
    lam, mu = fem.lame(1.0, nu)
    sig = lam * np.trace(e) * np.eye(3) + 2 * mu * e
    u = np.zeros(24)
    f = np.zeros(24)
    for a in range(8):
        x = np.array([a & 1, (a >> 1) & 1, (a >> 2) & 1], float)
        u[3 * a:3 * a + 3] = e @ x
        for d in range(3):
            n = np.zeros(3); n[d] = 1.0 if x[d] == 1 else -1.0
            f[3 * a:3 * a + 3] += sig @ n / 4.0
    assert np.abs(fem.element_K0(nu) @ u - f).max() <= 1e-14 * np.abs(f).max()


@pytest.mark.parametrize("name", ["cfg1", "porous20"])
def test_rigid_body_modes_and_symmetry(name):
    s = fem.build_system(make_problem(name))
    R = fem.rigid_body_modes(s.mesh.node_ijk)
    assert np.linalg.norm(s.full @ R) <= 1e-14 * np.linalg.norm(R) * abs(s.full).max()
    d = abs(s.A - s.A.T).max()
    assert d <= 1e-15 * abs(s.A).max()


def _patch_problem(L=4):
    solid = np.ones((L, L, L), np.uint8)
    lat = (L + 1,) * 3
    k, j, i = np.meshgrid(*[np.arange(L + 1)] * 3, indexing="ij")
    bnd = (i == 0) | (i == L) | (j == 0) | (j == L) | (k == 0) | (k == L)
    a = np.array([0.1, -0.2, 0.3])
    G = np.array([[0.01, 0.02, -0.03], [0.04, -0.05, 0.06], [0.07, 0.08, 0.02]])
    X = np.stack([i, j, k], -1).astype(float)
    u = a + X @ G.T
    return Problem(name="patch", nx=L, ny=L, nz=L, solid=solid, E=np.ones((L, L, L)),
                   nu=0.3, grain=np.zeros((L, L, L), np.int32), n_grains=1,
                   node_dirichlet=bnd.astype(np.uint8), node_u=u, node_f=np.zeros(lat + (3,)),
                   block=L), u


def test_patch_test():
    """Linear u prescribed on the whole boundary, f = 0 => the interior
    reproduces u (Q1 exactness for linear fields)."""
    p, u = _patch_problem()
    s = fem.build_system(p)
    x = spla.spsolve(s.A.tocsc(), s.b)
    ue = u.reshape(-1, 3)[s.mesh.node_key].ravel()
    assert np.abs(x - ue).max() <= 1e-12 * np.abs(ue).max()


def test_cfg1_load_equilibrium():
    s = fem.build_system(make_problem("cfg1"))
    assert s.mesh.f[:, 2].sum() == -256.0
    x = spla.spsolve(s.A.tocsc(), s.b)
    reac = (s.full @ x).reshape(-1, 3)[s.mesh.dirichlet]
    assert abs(reac[:, 2].sum() - 256.0) <= 1e-10 * 256.0
    assert np.abs(reac[:, :2].sum(0)).max() <= 1e-9


@pytest.mark.parametrize("case", ["porous20", "cfg1"])
def test_assemble_rows_matches_system(case):
    """The per-node row assembly (used for sampled checks at cfg4/cfg5 sizes)
    reproduces the full constrained assembly, pattern exactly and values to
    roundoff (different summation order)."""
    from oracle.fem import assemble_rows, build_system
    from workloads import make_problem
    s = build_system(make_problem(case))
    nodes = np.arange(s.mesh.n_nodes)
    if nodes.size > 2000:
        nodes = np.sort(np.random.default_rng(3).choice(nodes, 2000, replace=False))
    scale = np.abs(s.val).max()
    for p, (cols, blocks, bp) in zip(nodes, assemble_rows(s.mesh, nodes)):
        lo, hi = s.row_ptr[p], s.row_ptr[p + 1]
        assert np.array_equal(cols, s.col_idx[lo:hi])
        assert np.abs(blocks - s.val[lo:hi]).max() <= 1e-14 * scale
        assert np.abs(bp - s.b[3 * p:3 * p + 3]).max() <= 1e-13 * max(1.0, np.abs(s.b).max())


def _uniaxial_problem(E, nu, sigma, L=3, M=4):
    """L x L x M solid box (x, y, z), uniform (E, nu); top face z = M loaded by
    a normal traction sigma (consistent nodal loads: sigma/4 per corner of each
    top voxel face); sides traction-free; the bottom face z = 0 prescribed to
    the exact uniaxial-stress field u = (-nu sigma x / E, -nu sigma y / E, 0)."""
    solid = np.ones((M, L, L), np.uint8)
    lat = (M + 1, L + 1, L + 1)
    k, j, i = np.meshgrid(np.arange(M + 1), np.arange(L + 1), np.arange(L + 1), indexing="ij")
    X = np.stack([i, j, k], -1).astype(float)
    u_exact = np.stack([-nu * sigma * X[..., 0] / E, -nu * sigma * X[..., 1] / E,
                        sigma * X[..., 2] / E], -1)
    node_u = u_exact.copy()
    node_u[..., 2] = np.where(k == 0, 0.0, node_u[..., 2])
    f = np.zeros(lat + (3,))
    for vj in range(L):
        for vi in range(L):
            for dy in (0, 1):
                for dx in (0, 1):
                    f[M, vj + dy, vi + dx, 2] += sigma / 4.0
    p = Problem(name="uniaxial", nx=L, ny=L, nz=M, solid=solid, E=np.full((M, L, L), E),
                nu=nu, grain=np.zeros((M, L, L), np.int32), n_grains=1,
                node_dirichlet=(k == 0).astype(np.uint8), node_u=node_u, node_f=f, block=L)
    return p, u_exact


@pytest.mark.parametrize("E,nu", [(1.0, 0.3), (2.5, 0.25), (0.7, 0.45)])
def test_uniaxial_stress_closed_form(E, nu):
    """Pins (E, nu) -> (lambda, mu) (eq:stiff_iso P:69-71, reading R2) without
    calling the oracle's own formula: under a uniform top traction sigma with
    free sides, linear elasticity has the exact linear solution
    eps_zz = sigma/E, eps_xx = eps_yy = -nu sigma/E (Hooke's law for uniaxial
    stress, any textbook), which Q1 reproduces exactly.  The FEM solution must
    equal it to 1e-12.  Any other (lambda, mu) pair -- e.g. plane-stress lambda
    or mu = E/(1+nu) -- changes both strains."""
    sigma = 0.3
    p, u = _uniaxial_problem(E, nu, sigma)
    s = fem.build_system(p)
    x = spla.spsolve(s.A.tocsc(), s.b)
    ue = u.reshape(-1, 3)[s.mesh.node_key].ravel()
    assert np.abs(x - ue).max() <= 1e-12 * np.abs(ue).max()
