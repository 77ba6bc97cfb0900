"""Mortar nodes and Gaussian mortar functions (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §3.3 "Mortar nodes and mortar functions":
  * placement: first two = farthest pair of F^{c_j}; then
    x_{m_{i+1}} = argmin_{y in F} sum_{j<=i} 1/||y - x_{m_j}||   (eq:node_init,
    P:137-141); then sweeps that move each node to the argmin of the potential
    of all OTHER nodes until nothing changes;
  * Gaussian mortars eta_{m_i gamma}^{(d)} = delta_{d gamma} alpha_i/sum_j alpha_j,
    alpha_i(x) = exp(-||x-x_{m_i}||^2 / (beta min_j ||x_{m_i}-x_{m_j}||^2))
    (eq:gauss), beta = 4.
  * Algebraic mortars (eq:algebra) built as in the Remark:
    column (m_i, gamma) of the interface block M^{c} solves the interface
    matrix A^{c}_{c} = A^[F_c, F_c] with Dirichlet constraints on the mortar
    nodes -- 1 for component gamma of m_i, 0 for every other mortar-node
    component -- i.e. x_free = -(A~)^-1 e_1 expanded with the 0/1 values
    (reading R25: A^{c}_{c} is the principal interface block of A^; all 3
    components of every mortar node are constrained; global x/y/z frame).
Every interface is stored as a dense block M^{c} of 3|F_c| x 3 nu_c: row 3f + d
(f-th node of F_c, component d), column 3i + gamma (mortar i, component
gamma).  Gaussian blocks are component-diagonal: M[3f+d, 3i+g] = W[f,i] d_{dg}.
Readings: R9 (nu_c = min(n, |F_c|)), R10 (deterministic placement: integer d^2,
IEEE 1/sqrt, sequential sums in chosen order, lowest id on ties, ascending
sweep order, move only on a > 1e-12 relative improvement, <= 20 sweeps; nu=|F|
=> all nodes ascending; nu=1 => node nearest the centroid), R11 (min over
j != i; nu=1 => w == 1).
"""
from __future__ import annotations

import math

import numpy as np


def _d2(a, b) -> int:
    return int((a[0] - b[0]) ** 2 + (a[1] - b[1]) ** 2 + (a[2] - b[2]) ** 2)


def _potential(y, X, skip=-1) -> float:
    """sum_j 1/||y - x_j|| over X in order (j != skip), sequential fp64 sum."""
    s = 0.0
    for j, x in enumerate(X):
        if j == skip:
            continue
        s += 1.0 / math.sqrt(float(_d2(y, x)))
    return s


def place_mortars(F: np.ndarray, ijk: np.ndarray, n: int, max_sweeps: int = 20):
    """Mortar node ids (a list in placement order) on interface node set F
    (ascending node ids) with lattice coords ijk[F]."""
    F = [int(p) for p in F]
    P = {p: tuple(int(v) for v in ijk[p]) for p in F}
    nu = min(n, len(F))
    if nu == len(F):
        return list(F)
    if nu == 1:
        m = len(F)
        S = [sum(P[p][a] for p in F) for a in range(3)]
        best, bd = None, None
        for p in F:                          # integer |F|^2 * d^2 to centroid
            d = sum((m * P[p][a] - S[a]) ** 2 for a in range(3))
            if bd is None or d < bd:
                best, bd = p, d
        return [best]
    # farthest pair, lowest (id_a, id_b) lexicographic
    best, bd = None, -1
    for ia, a in enumerate(F):
        for b in F[ia + 1:]:
            d = _d2(P[a], P[b])
            if d > bd:
                best, bd = (a, b), d
    X = [best[0], best[1]]
    # greedy Coulomb argmin (eq:node_init)
    while len(X) < nu:
        chosen = set(X)
        xs = [P[x] for x in X]
        arg, val = None, None
        for y in F:
            if y in chosen:
                continue
            v = _potential(P[y], xs)
            if val is None or v < val:
                arg, val = y, v
        X.append(arg)
    # sweeps in ascending mortar index (R10)
    for _ in range(max_sweeps):
        moved = False
        for i in range(nu):
            others = set(X[:i] + X[i + 1:])
            xs = [P[x] for x in X]
            cur = _potential(P[X[i]], xs, skip=i)
            arg, val = None, None
            for y in F:
                if y in others:
                    continue
                v = _potential(P[y], xs, skip=i)
                if val is None or v < val:
                    arg, val = y, v
            if val < cur * (1.0 - 1e-12):
                X[i] = arg
                moved = True
        if not moved:
            break
    return X


def gaussian_weights(F: np.ndarray, ijk: np.ndarray, mortars, beta: float) -> np.ndarray:
    """W[y, i] = eta_{m_i}(y) for y in F (eq:gauss with R11).  Evaluated with a
    max-exponent shift (identical in exact arithmetic)."""
    F = np.asarray(F)
    nu = len(mortars)
    if nu == 1:
        return np.ones((F.size, 1))
    xm = ijk[np.asarray(mortars)].astype(np.int64)
    dmin2 = np.empty(nu)
    for i in range(nu):
        dmin2[i] = min(_d2(xm[i], xm[j]) for j in range(nu) if j != i)
    y = ijk[F].astype(np.int64)
    d2 = ((y[:, None, :] - xm[None, :, :]) ** 2).sum(-1).astype(np.float64)
    e = -d2 / (beta * dmin2[None, :])
    alpha = np.exp(e - e.max(axis=1, keepdims=True))
    return alpha / alpha.sum(axis=1, keepdims=True)


def gaussian_block(W: np.ndarray) -> np.ndarray:
    """3|F| x 3nu block of component-diagonal Gaussian mortars."""
    nf, nu = W.shape
    M = np.zeros((3 * nf, 3 * nu))
    for g in range(3):
        M[g::3, g::3] = W
    return M


def algebraic_block(F: np.ndarray, A, mortars) -> np.ndarray:
    """Algebraic mortars by the Remark, steps (1)-(4) as written:
    (1) drop the rows of the 0/1-constrained DOFs (all components of the
    mortar nodes) from A^{c}_{c}; (2) take the column of the 1-constraint;
    (3) drop the constrained columns -> A~; (4) x = -(A~)^-1 e_1, expanded by
    the 0/1 values.  A: the (Dirichlet-constrained) fine matrix A^ (sparse)."""
    F = np.asarray(F)
    dofs = (3 * F[:, None] + np.arange(3)[None, :]).ravel()
    Acc = A[dofs][:, dofs].toarray()
    pos = {int(y): f for f, y in enumerate(F)}
    con = np.array([3 * pos[int(x)] + g for x in mortars for g in range(3)], dtype=np.int64)
    free = np.setdiff1d(np.arange(dofs.size), con)
    nu = len(mortars)
    M = np.zeros((dofs.size, 3 * nu))
    for q in range(3 * nu):              # q = 3 i + gamma, i.e. con[q]
        M[con[q], q] = 1.0
        if free.size:
            e1 = Acc[np.ix_(free, [con[q]])][:, 0]
            At = Acc[np.ix_(free, free)]
            M[free, q] = -np.linalg.solve(At, e1)
    return M


# ----------------------------------------------------------------------------
# Algebraic mortars on the interface surface (reading R29, mortar = "surface")
# ----------------------------------------------------------------------------
# eq:algebra is the (D-1)-dimensional elasticity problem on the
# interface Gamma^{c} with tangential derivatives only, zero stress on the
# interface boundary and 0/1 constraints at the mortar nodes.  Discretised on
# the voxel faces shared by a solid voxel of each grain of the interface's pair
# (all four face nodes in F_c): Q1 on the unit square, 2x2 Gauss, all three
# displacement components; strain = sym(grad_t eta) with the tangential
# gradient only:  e_aa = d_a u_a, e_bb = d_b u_b, g_ab = d_b u_a + d_a u_b,
# g_an = d_a u_n, g_bn = d_b u_n  (a, b in-plane axes, n the face normal);
# isotropic lambda, mu from the mean E of the two voxels and the uniform nu.
# A translation-free tie TIE * mu_bar * sum (eta_p - eta_q)^2 over the node
# pairs of F_c coupled in A^ (the R7 interface graph, connected) attaches
# nodes that lie on no shared face; mu_bar = mean E over solid voxels / (2(1+nu)).
SURFACE_TIE = 0.1


def surface_face_matrix(E: float, nu: float) -> np.ndarray:
    """12 x 12 stiffness of one interface face, local components (a, b, n) per
    node, nodes in corner order (0,0), (1,0), (0,1), (1,1) of (a, b)."""
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    D = np.diag([lam + 2 * mu, lam + 2 * mu, mu, mu, mu])
    D[0, 1] = D[1, 0] = lam
    g = 0.5 / math.sqrt(3.0)
    K = np.zeros((12, 12))
    corners = [(0, 0), (1, 0), (0, 1), (1, 1)]
    for s_ in (0.5 - g, 0.5 + g):
        for t_ in (0.5 - g, 0.5 + g):
            B = np.zeros((5, 12))
            for k, (da, db) in enumerate(corners):
                fa = s_ if da else 1.0 - s_
                fb = t_ if db else 1.0 - t_
                dNa = (1.0 if da else -1.0) * fb      # d/ds
                dNb = fa * (1.0 if db else -1.0)      # d/dt
                B[0, 3 * k + 0] = dNa
                B[1, 3 * k + 1] = dNb
                B[2, 3 * k + 0] = dNb
                B[2, 3 * k + 1] = dNa
                B[3, 3 * k + 2] = dNa
                B[4, 3 * k + 2] = dNb
            K += 0.25 * B.T @ D @ B
    return K


def surface_faces(prob, lat_id, pair, pos):
    """Faces of interface (pair, node positions pos) as (local node indices,
    components (a, b, n), E of the face)."""
    solid = np.asarray(prob.solid) > 0
    grain = np.asarray(prob.grain)
    comp_of_axis = (2, 1, 0)          # array axes (z, y, x) -> component index
    g1, g2 = pair
    out = []
    for ax in range(3):
        o0, o1 = [a for a in range(3) if a != ax]
        sl1 = [slice(None)] * 3
        sl2 = [slice(None)] * 3
        sl1[ax] = slice(0, -1)
        sl2[ax] = slice(1, None)
        both = solid[tuple(sl1)] & solid[tuple(sl2)]
        ga, gb = grain[tuple(sl1)], grain[tuple(sl2)]
        hit = both & (((ga == g1) & (gb == g2)) | ((ga == g2) & (gb == g1)))
        for v in np.argwhere(hit):
            v = tuple(int(t) for t in v)
            w = list(v)
            w[ax] += 1
            base = list(w)
            nodes = []
            for da, db in ((0, 0), (1, 0), (0, 1), (1, 1)):
                c = list(base)
                c[o0] += da
                c[o1] += db
                nodes.append(int(lat_id[c[0], c[1], c[2]]))
            if not all(q in pos for q in nodes):
                continue
            E = 0.5 * (float(prob.E[v]) + float(prob.E[tuple(w)]))
            out.append(([pos[q] for q in nodes],
                        (comp_of_axis[o0], comp_of_axis[o1], comp_of_axis[ax]), E))
    return out


def surface_block(F, faces, ties, nu, mu_bar, mortars) -> np.ndarray:
    """3|F| x 3nu block: the constrained solves of the Remark on the
    surface operator K (faces + tie) instead of A^{c}_{c} (reading R29)."""
    F = np.asarray(F)
    pos = {int(y): f for f, y in enumerate(F)}
    n3 = 3 * F.size
    K = np.zeros((n3, n3))
    for nodes, (ca, cb, cn), E in faces:
        Kf = surface_face_matrix(E, nu)
        idx = np.array([3 * nodes[k] + c for k in range(4) for c in (ca, cb, cn)])
        K[np.ix_(idx, idx)] += Kf
    tau = SURFACE_TIE * mu_bar
    for f, q in ties:                      # each unordered pair once
        for c in range(3):
            K[3 * f + c, 3 * f + c] += tau
            K[3 * q + c, 3 * q + c] += tau
            K[3 * f + c, 3 * q + c] -= tau
            K[3 * q + c, 3 * f + c] -= tau
    con = np.array([3 * pos[int(x)] + g for x in mortars for g in range(3)], dtype=np.int64)
    free = np.setdiff1d(np.arange(n3), con)
    M = np.zeros((n3, con.size))
    for q in range(con.size):
        M[con[q], q] = 1.0
        if free.size:
            M[free, q] = -np.linalg.solve(K[np.ix_(free, free)], K[np.ix_(free, [con[q]])][:, 0])
    return M


class Mortars:
    """Mortar nodes + mortar blocks for every interface; coarse column ordering
    R13: interface id -> mortar index (placement order) -> gamma in {x,y,z}.
    kind: "gaussian" (eq:gauss, the paper's choice for its results) or
    "algebraic" (eq:algebra via the Remark; needs A)."""

    def __init__(self, decomp, node_ijk, n_mortar: int, beta: float, kind: str = "gaussian",
                 A=None, system=None):
        self.kind = kind
        if kind == "surface":
            prob = system.mesh.prob
            solid = np.asarray(prob.solid) > 0
            mu_bar = float(np.asarray(prob.E)[solid].mean()) / (2.0 * (1.0 + prob.nu))
            rp, ci = system.row_ptr, system.col_idx
        self.nodes = []
        self.weights = []       # Gaussian W[f, i] (kind == "gaussian")
        self.blocks = []        # 3|F| x 3nu per interface (both kinds)
        self.offset = [0]
        for F in decomp.interfaces:
            X = place_mortars(F, node_ijk, n_mortar)
            self.nodes.append(X)
            if kind == "gaussian":
                W = gaussian_weights(F, node_ijk, X, beta)
                self.weights.append(W)
                self.blocks.append(gaussian_block(W))
            elif kind == "algebraic":
                self.blocks.append(algebraic_block(F, A, X))
            elif kind == "surface":
                ci_ = len(self.nodes) - 1
                pos = {int(y): f for f, y in enumerate(F)}
                faces = surface_faces(prob, system.mesh.lat_id, tuple(decomp.iface_pair[ci_]), pos)
                ties = [(pos[int(y)], pos[int(q)]) for y in F for q in ci[rp[y]:rp[y + 1]]
                        if int(q) in pos and int(q) > int(y)]
                self.blocks.append(surface_block(F, faces, ties, prob.nu, mu_bar, X))
            else:
                raise ValueError(kind)
            self.offset.append(self.offset[-1] + len(X))
        self.offset = np.array(self.offset, dtype=np.int64)
        self.n_mortar_nodes = int(self.offset[-1])
        self.n_mortar_dofs = 3 * self.n_mortar_nodes
