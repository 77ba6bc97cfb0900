"""Pins for oracle/decomp.py and oracle/mortar.py.

SURVEY §8(c) pins O4 (closed-form cfg1 decomposition), O5 (brute-force contact
grids), O6 (brute-force global minimum of the Coulomb energy, eq:node_init),
O7 (partition of unity, nu=1 reduction, two-node closed form; eq:gauss).
"""
import functools
import itertools
import math

import numpy as np
import pytest

from oracle import decomp, mortar


def _golden(name):
    import json, os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", name)))


def test_cfg1_decomposition_closed_form(cfg1):
    _, s, h = cfg1
    d = h.dec
    g = _golden("cfg1_counts.json")
    assert d.n_grains == g["grains"]
    assert d.n_interfaces == g["interfaces"]
    sizes = sorted(F.size for F in d.interfaces)
    assert sizes == g["interface_sizes_sorted"]
    big = [list(map(int, d.iface_pair[c])) for c, F in enumerate(d.interfaces) if F.size == 72]
    assert big == g["big_interface_pairs"]
    assert sum(F.size for F in d.interfaces) == g["interface_nodes"]
    assert int((d.node_class == decomp.CLASS_D).sum()) == g["dirichlet_nodes"]
    assert max(gn.size for gn in d.grain_nodes) == g["max_grain_interior_nodes"]
    # every node is in exactly one of: some I_g, some interface
    cover = np.zeros(s.mesh.n_nodes, int)
    for g in d.grain_nodes:
        cover[g] += 1
    for F in d.interfaces:
        cover[F] += 1
    assert np.all(cover == 1)


def _brute_components(nodes, adj):
    """Union-find over an explicit adjacency (plain Python)."""
    parent = {p: p for p in nodes}

    def find(p):
        while parent[p] != p:
            parent[p] = parent[parent[p]]
            p = parent[p]
        return p
    for p in nodes:
        for q in adj(p):
            if q in parent:
                a, b = find(p), find(q)
                if a != b:
                    parent[max(a, b)] = min(a, b)
    comps = {}
    for p in nodes:
        comps.setdefault(find(p), []).append(p)
    return comps


def test_porous_interfaces_and_contact_grids_brute_force(porous20):
    p, s, h = porous20
    d = h.dec
    mesh = s.mesh
    ijk = mesh.node_ijk
    # R6: interface nodes = non-D nodes touching >= 2 grains, pair = 2 smallest
    vox_of = {}
    for v, nodes in enumerate(mesh.vox_nodes):
        for q in nodes:
            vox_of.setdefault(int(q), set()).add(int(mesh.vox_grain[v]))
    for q in range(mesh.n_nodes):
        gs = sorted(vox_of[q])
        if mesh.dirichlet[q]:
            assert d.node_class[q] == decomp.CLASS_D and d.owner[q] == gs[0]
        elif len(gs) >= 2:
            assert d.node_class[q] == decomp.CLASS_I and tuple(d.pair[q]) == tuple(gs[:2])
        else:
            assert d.node_class[q] == decomp.CLASS_G and d.owner[q] == gs[0]
    # R7: components under "share a solid voxel", brute force
    share = {}
    for nodes in mesh.vox_nodes:
        for a in nodes:
            share.setdefault(int(a), set()).update(int(b) for b in nodes)
    want = []
    pairs = sorted({tuple(d.pair[q]) for q in range(mesh.n_nodes) if d.node_class[q] == decomp.CLASS_I})
    for pr in pairs:
        nodes = [q for q in range(mesh.n_nodes)
                 if d.node_class[q] == decomp.CLASS_I and tuple(d.pair[q]) == pr]
        comps = _brute_components(nodes, lambda q: share[q])
        want += sorted((pr, min(c), sorted(c)) for c in comps.values())
    got = [(tuple(d.iface_pair[c]), int(F[0]), list(map(int, F))) for c, F in enumerate(d.interfaces)]
    assert got == [(pr, m, c) for pr, m, c in want]
    # R8: contact grid = all non-D nodes within Chebyshev distance h (no bbox)
    hh = d.contact_h
    nonD = np.flatnonzero(~mesh.dirichlet)
    for F, Z in zip(d.interfaces, d.contact_nodes):
        dist = np.abs(ijk[nonD][:, None, :] - ijk[F][None, :, :]).max(-1).min(-1)
        assert np.array_equal(np.sort(nonD[dist <= hh]), Z)


def _coulomb(ijk, S):
    return sum(1.0 / math.dist(ijk[a], ijk[b]) for a, b in itertools.combinations(S, 2))


@pytest.mark.parametrize("shape", [(9, 8), (8, 8), (8, 7)])
def test_rectangle_placement_is_global_minimum(shape):
    """On cfg1's rectangular interface shapes the R10 placement equals the
    brute-force global minimum of the Coulomb energy over all C(|F|,4) subsets
    (unique minimum = the 4 corners)."""
    a, b = shape
    jj, ii = np.meshgrid(np.arange(b), np.arange(a), indexing="ij")
    ijk = np.stack([ii.ravel(), jj.ravel(), np.zeros(a * b, int)], 1)
    F = np.arange(a * b)
    X = mortar.place_mortars(F, ijk, 4)
    P = ijk.astype(float)
    D = np.sqrt(((P[:, None] - P[None]) ** 2).sum(-1))
    np.fill_diagonal(D, np.inf)
    inv = 1.0 / D
    # vectorised brute force over all 4-subsets
    idx = np.array(list(itertools.combinations(range(a * b), 4)))
    E = np.zeros(len(idx))
    for x, y in itertools.combinations(range(4), 2):
        E += inv[idx[:, x], idx[:, y]]
    m = E.min()
    winners = idx[E <= m * (1 + 1e-12)]
    corners = sorted([0, a - 1, a * (b - 1), a * b - 1])
    assert len(winners) == 1 and sorted(winners[0]) == corners
    assert sorted(X) == corners


def test_gaussian_two_node_closed_form():
    # own-node weight with two mortars = 1/(1+e^{-1/4})
    # (tests/golden/gauss_two_node.json)
    g = _golden("gauss_two_node.json")
    ijk = np.array(g["mortars_ijk"] + [g["probe_ijk"]])
    W = mortar.gaussian_weights(np.array([0, 1, 2]), ijk, [0, 1], g["beta"])
    assert abs(W[0, 0] - 1.0 / (1.0 + math.exp(-0.25))) <= 1e-15
    assert abs(W[0, 0] - g["w_own"]) <= 1e-15


def test_mortar_partition_of_unity_and_nu1(porous20):
    p, s, h = porous20
    for F, W in zip(h.dec.interfaces, h.mor.weights):
        assert np.abs(W.sum(1) - 1.0).max() <= 1e-15 * 4
        assert np.all(W > 0)
    d = h.dec
    m1 = mortar.Mortars(d, s.mesh.node_ijk, 1, 4.0)
    for W in m1.weights:
        assert np.all(W == 1.0)           # PLMM reduction, bitwise


def test_full_cap_places_every_node(cfg1):
    _, s, h = cfg1
    F = h.dec.interfaces[0]
    assert mortar.place_mortars(F, s.mesh.node_ijk, 10 ** 6) == list(map(int, F))


# ---- Algebraic mortars (eq:algebra via the Remark P:356; reading R25) -----
def _alg_case(h, s, ci, n):
    F = h.dec.interfaces[ci]
    X = mortar.place_mortars(F, s.mesh.node_ijk, n)
    M = mortar.algebraic_block(F, s.A, X)
    dofs = (3 * np.asarray(F)[:, None] + np.arange(3)[None, :]).ravel()
    Acc = s.A[dofs][:, dofs].toarray()
    pos = {int(y): f for f, y in enumerate(F)}
    con = np.array([3 * pos[int(x)] + g for x in X for g in range(3)])
    free = np.setdiff1d(np.arange(dofs.size), con)
    return F, X, M, Acc, con, free


@pytest.mark.parametrize("ci", [0, 3, 7])
def test_algebraic_mortars_constraints_and_harmonicity(porous20, ci):
    """Each column meets its 0/1 mortar constraints exactly and is A^{c}_{c}-
    harmonic on the free interface DOFs (the Remark's local problem)."""
    p, s, h = porous20
    F, X, M, Acc, con, free = _alg_case(h, s, ci, 4)
    assert np.array_equal(M[con], np.eye(len(con)))
    res = Acc[free] @ M
    assert np.abs(res).max() <= 1e-12 * np.abs(Acc).max() * max(1.0, np.abs(M).max())


def test_algebraic_mortars_minimise_interface_energy(porous20):
    """The constrained solve is the minimiser of x^T A^{c}_{c} x under the
    0/1 constraints: any admissible perturbation raises the energy."""
    p, s, h = porous20
    F, X, M, Acc, con, free = _alg_case(h, s, 1, 4)
    rng = np.random.default_rng(3)
    for q in range(M.shape[1]):
        e0 = M[:, q] @ Acc @ M[:, q]
        for _ in range(5):
            d = np.zeros(M.shape[0])
            d[free] = 1e-3 * rng.standard_normal(free.size)
            x = M[:, q] + d
            assert x @ Acc @ x > e0


def test_algebraic_full_cap_is_identity(cfg1):
    """nu = |F| (every interface node a mortar): no free DOFs, M = I."""
    _, s, h = cfg1
    F = h.dec.interfaces[2]
    X = mortar.place_mortars(F, s.mesh.node_ijk, 10 ** 6)
    M = mortar.algebraic_block(F, s.A, X)
    assert np.array_equal(M, np.eye(3 * F.size))


def test_algebraic_hplmm_projection_and_gmres():
    """With Algebraic mortars the two-level operator keeps the M_G projection
    identity M_G^-1 A^ P^ z = P^ z, and GMRES converges (cube8)."""
    import scipy.sparse as sp
    from oracle import gmres, hplmm
    from workloads import make_problem
    p = make_problem("cube8", mortar="algebraic")
    s, h = hplmm.setup(p)
    h.set_rhs(s.b)
    P = sp.hstack([h.PB, h.P_C()]).tocsc()
    z = np.random.default_rng(5).standard_normal(P.shape[1])
    Pz = P @ z
    assert np.linalg.norm(h.apply_MG(s.A @ Pz) - Pz) <= 1e-10 * np.linalg.norm(Pz)
    x, it, hist, rr, conv = gmres.gmres(s.A, s.b, h.apply_M, tol=1e-8)
    assert conv and it < 60


# ---- mortar placement sweeps (eq:node_init + the sweep of P:142; R10) -----
def _pot_np(P, y, others):
    """sum over the other mortar nodes of 1/||y - x|| (numpy, any order)."""
    d = np.sqrt(((P[others] - P[y]) ** 2).sum(-1))
    return float(np.sum(1.0 / d))


def _fixpoint_violations(F, ijk, X):
    """Nodes i of placement X for which some unchosen y in F lowers the
    potential of the other mortar nodes by more than the R10 tie band."""
    P = ijk.astype(np.float64)
    bad = []
    for i in range(len(X)):
        others = np.array([x for t, x in enumerate(X) if t != i])
        cur = _pot_np(P, X[i], others)
        cand = np.array([y for y in F if y not in set(others.tolist())])
        d = np.sqrt(((P[cand][:, None, :] - P[others][None, :, :]) ** 2).sum(-1))
        best = (1.0 / d).sum(1).min()
        if best < cur * (1.0 - 2e-12):
            bad.append(i)
    return bad


@functools.lru_cache(maxsize=None)
def _decomp(name):
    from oracle import fem
    from workloads import make_problem
    p = make_problem(name)
    s = fem.build_system(p)
    return s, decomp.Decomposition(s, p.contact_h)


@pytest.mark.parametrize("name", ["porous20", "cfg2"])
def test_placement_n2_is_farthest_pair(name):
    """n = 2: the sweep cannot improve on the farthest pair (R10 (ii)), so the
    result is the brute-force farthest pair by integer d^2, lowest ids."""
    s, d = _decomp(name)
    ijk = s.mesh.node_ijk
    for F in d.interfaces:
        if F.size <= 2:
            continue
        P = ijk[F].astype(np.int64)
        D2 = ((P[:, None, :] - P[None, :, :]) ** 2).sum(-1)
        m = D2.max()
        a, b = np.argwhere(np.triu(D2 == m, 1))[0]     # row-major: lowest (a, b)
        assert mortar.place_mortars(F, ijk, 2) == [int(F[a]), int(F[b])]


@pytest.mark.parametrize("name", ["porous20", "cfg2"])
@pytest.mark.parametrize("n", [3, 4, 8])
def test_placement_is_sweep_fixpoint(name, n):
    """the sweeps stop when no mortar node moves -- i.e. the returned
    placement is a fixpoint: no single-node move to an unchosen interface node
    lowers that node's potential sum_{j != i} 1/||y - x_j|| (brute force, numpy,
    independent summation).  The greedy start alone is NOT a fixpoint on a
    number of these interfaces (checked below), so dropping the sweeps fails."""
    s, d = _decomp(name)
    ijk = s.mesh.node_ijk
    moved = 0
    for F in d.interfaces:
        if F.size <= n:
            continue
        X = mortar.place_mortars(F, ijk, n)
        assert len(set(X)) == n and set(X) <= set(map(int, F))
        assert _fixpoint_violations(list(map(int, F)), ijk, X) == []
        X0 = mortar.place_mortars(F, ijk, n, max_sweeps=0)
        moved += X0 != X
    assert moved > 0
