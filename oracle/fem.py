"""Q1 hexahedral FEM for linear elasticity on a voxel grid (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §2: eq:Linear-elastic, eq:BC, eq:stiff_iso
(P:69-71), "Galerkin FEM over a Cartesian fine grid ... bilinear/trilinear"
 -> eq:ls_all  A^ x^ = b^.
Readings: R2 (2x2x2 Gauss, unit voxel, lambda/mu from per-voxel E and uniform
nu), R3 (node-major DOFs 3*node+c, nodes in ascending lattice key
i+(nx+1)(j+(ny+1)k), col ascending), R4 (Dirichlet nodes kept as identity 3x3
rows, couplings removed, RHS lifted).
"""
from __future__ import annotations

import itertools
import math

import numpy as np
import scipy.sparse as sp


# --------------------------------------------------------------------------
# element matrix  (eq:stiff_iso P:69-71; R2)
# --------------------------------------------------------------------------
def lame(E: float, nu: float) -> tuple[float, float]:
    """Lame parameters from (E, nu)."""
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    return lam, mu


def elasticity_D(E: float, nu: float) -> np.ndarray:
    """6x6 isotropic stiffness C_ijkl = lam d_ij d_kl + mu(d_ik d_jl + d_il d_jk)
    in Voigt form, strain order [exx, eyy, ezz, gyz, gxz, gxy] (engineering
    shear strains)."""
    lam, mu = lame(E, nu)
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[0, 0] = D[1, 1] = D[2, 2] = lam + 2.0 * mu
    D[3, 3] = D[4, 4] = D[5, 5] = mu
    return D


def _corner(a: int) -> tuple[int, int, int]:
    """Local hex node a = dx + 2dy + 4dz (R2/R3)."""
    return a & 1, (a >> 1) & 1, (a >> 2) & 1


def shape_grad(xi: np.ndarray) -> np.ndarray:
    """Gradients (8 x 3) of the trilinear shape functions
    N_a = prod_d (corner_d ? xi_d : 1-xi_d) on the unit cube."""
    G = np.zeros((8, 3))
    for a in range(8):
        c = _corner(a)
        f = [xi[d] if c[d] else 1.0 - xi[d] for d in range(3)]
        df = [1.0 if c[d] else -1.0 for d in range(3)]
        G[a, 0] = df[0] * f[1] * f[2]
        G[a, 1] = f[0] * df[1] * f[2]
        G[a, 2] = f[0] * f[1] * df[2]
    return G


def strain_B(xi: np.ndarray) -> np.ndarray:
    """6 x 24 strain-displacement matrix, DOF 3a+c."""
    G = shape_grad(xi)
    B = np.zeros((6, 24))
    for a in range(8):
        gx, gy, gz = G[a]
        B[0, 3 * a + 0] = gx
        B[1, 3 * a + 1] = gy
        B[2, 3 * a + 2] = gz
        B[3, 3 * a + 1] = gz; B[3, 3 * a + 2] = gy   # gyz
        B[4, 3 * a + 0] = gz; B[4, 3 * a + 2] = gx   # gxz
        B[5, 3 * a + 0] = gy; B[5, 3 * a + 1] = gx   # gxy
    return B


def element_K0(nu: float, order: int = 2) -> np.ndarray:
    """K0 = int_[0,1]^3 B^T D(E=1,nu) B dV by order^3 Gauss-Legendre (R2:
    order 2, points 0.5 +- 0.5/sqrt(3), weights 1/8)."""
    pts, wts = np.polynomial.legendre.leggauss(order)
    pts = 0.5 + 0.5 * pts
    wts = 0.5 * wts
    D = elasticity_D(1.0, nu)
    K = np.zeros((24, 24))
    for (i, wi), (j, wj), (k, wk) in itertools.product(
            zip(range(order), wts), zip(range(order), wts), zip(range(order), wts)):
        B = strain_B(np.array([pts[i], pts[j], pts[k]]))
        K += (wi * wj * wk) * (B.T @ D @ B)
    return K


# --------------------------------------------------------------------------
# mesh (O1; R3)
# --------------------------------------------------------------------------
class Mesh:
    """Solid nodes = lattice points touching >= 1 solid voxel; node id = rank
    of the lattice key i + (nx+1)(j + (ny+1)k) (R3)."""

    def __init__(self, prob):
        self.prob = prob
        nx, ny, nz = prob.nx, prob.ny, prob.nz
        self.lat_shape = (nz + 1, ny + 1, nx + 1)
        solid = prob.solid > 0
        sn = np.zeros(self.lat_shape, dtype=bool)
        for dz, dy, dx in itertools.product((0, 1), repeat=3):
            sn[dz:dz + nz, dy:dy + ny, dx:dx + nx] |= solid
        self.node_key = np.flatnonzero(sn.ravel()).astype(np.int64)
        self.n_nodes = self.node_key.size
        lat_id = -np.ones(sn.size, dtype=np.int64)
        lat_id[self.node_key] = np.arange(self.n_nodes)
        self.lat_id = lat_id.reshape(self.lat_shape)
        k, rem = np.divmod(self.node_key, (nx + 1) * (ny + 1))
        j, i = np.divmod(rem, nx + 1)
        self.node_ijk = np.stack([i, j, k], axis=1).astype(np.int64)
        # solid voxels and their 8 node ids (local node a = dx+2dy+4dz)
        vk, vj, vi = np.nonzero(solid)
        self.vox = np.stack([vi, vj, vk], axis=1)
        self.vox_nodes = np.stack(
            [self.lat_id[vk + _corner(a)[2], vj + _corner(a)[1], vi + _corner(a)[0]]
             for a in range(8)], axis=1)
        self.vox_E = prob.E[vk, vj, vi].astype(np.float64)
        self.vox_grain = prob.grain[vk, vj, vi].astype(np.int64)
        # Dirichlet flags / data per node
        flat = lambda a: a.reshape(-1, *a.shape[3:])[self.node_key]
        self.dirichlet = flat(prob.node_dirichlet).astype(bool)
        self.u_D = flat(prob.node_u).astype(np.float64)
        self.f = flat(prob.node_f).astype(np.float64)

    @property
    def n_dof(self) -> int:
        return 3 * self.n_nodes


# --------------------------------------------------------------------------
# assembly (O3; eq:ls_all; R3, R4)
# --------------------------------------------------------------------------
def _bsr(row_ptr, col, val, n):
    return sp.bsr_matrix((val, col, row_ptr), shape=(3 * n, 3 * n))


def assemble_full(mesh: Mesh):
    """Unconstrained A_full = sum_e E_e K0 scattered in node-major 3x3 blocks.

    Pattern: block (p,q) exists iff p and q share a solid voxel.  Values are
    accumulated in ascending local-pair order (a, b)."""
    K0 = element_K0(mesh.prob.nu)
    n = mesh.n_nodes
    vn = mesh.vox_nodes
    keys = np.unique(np.concatenate(
        [vn[:, a] * n + vn[:, b] for a in range(8) for b in range(8)]))
    rows = keys // n
    cols = keys % n
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    val = np.zeros((keys.size, 3, 3))
    for a in range(8):
        for b in range(8):
            pos = np.searchsorted(keys, vn[:, a] * n + vn[:, b])
            val[pos] += mesh.vox_E[:, None, None] * K0[3 * a:3 * a + 3, 3 * b:3 * b + 3]
    return row_ptr, cols.astype(np.int64), val


class System:
    """A^ (BSR, Dirichlet-constrained) and b^ of eq:ls_all."""

    def __init__(self, mesh: Mesh):
        self.mesh = mesh
        n = mesh.n_nodes
        rp, ci, va = assemble_full(mesh)
        self.full = _bsr(rp, ci, va, n)            # unconstrained (pins only)
        D = mesh.dirichlet
        # RHS lift: b_free = f_free - A_fD u_D ;  b_D = u_D     (R4)
        uD = np.where(D[:, None], mesh.u_D, 0.0).ravel()
        b = mesh.f.ravel() - self.full @ uD
        b = b.reshape(n, 3)
        b[D] = mesh.u_D[D]
        self.b = b.ravel().copy()
        # structural removal of Dirichlet couplings; identity diagonal block
        rows = np.repeat(np.arange(n), np.diff(rp))
        keep = (~D[rows] & ~D[ci]) | (D[rows] & (rows == ci))
        va = va.copy()
        va[D[rows] & (rows == ci)] = np.eye(3)
        rows, ci, va = rows[keep], ci[keep], va[keep]
        row_ptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(row_ptr, rows + 1, 1)
        self.row_ptr = np.cumsum(row_ptr)
        self.col_idx = ci
        self.val = va
        self.A = _bsr(self.row_ptr, self.col_idx, self.val, n).tocsr()

    @property
    def n_dof(self):
        return self.mesh.n_dof

    @property
    def nnzb(self):
        return int(self.col_idx.size)


def assemble_rows(mesh: Mesh, nodes):
    """Block rows of the constrained A^ and entries of b^ for selected nodes,
    one node at a time straight from the element sum (eq:stiff_iso; R3, R4):
    row p = sum over the solid voxels v touching p (p = local node a of v) of
    E_v K0[a, b] scattered to the node of local index b; Dirichlet columns
    dropped (their u_D moved to the right-hand side); a Dirichlet row is the
    identity with b_p = u_D(p).  A second route to the same rows as System
    (for sampled checks where the full assembly is too large).

    Returns [(cols ascending int64, blocks (len, 3, 3), b_p (3,))]."""
    K0 = element_K0(mesh.prob.nu)
    prob = mesh.prob
    out = []
    for p in np.asarray(nodes, dtype=np.int64):
        if mesh.dirichlet[p]:
            out.append((np.array([p]), np.eye(3)[None], mesh.u_D[p].copy()))
            continue
        i, j, k = (int(t) for t in mesh.node_ijk[p])
        acc = {}
        for a in range(8):
            dx, dy, dz = _corner(a)
            vi, vj, vk = i - dx, j - dy, k - dz
            if not (0 <= vi < prob.nx and 0 <= vj < prob.ny and 0 <= vk < prob.nz):
                continue
            if not prob.solid[vk, vj, vi]:
                continue
            E = float(prob.E[vk, vj, vi])
            for b in range(8):
                cx, cy, cz = _corner(b)
                q = int(mesh.lat_id[vk + cz, vj + cy, vi + cx])
                blk = E * K0[3 * a:3 * a + 3, 3 * b:3 * b + 3]
                acc[q] = acc[q] + blk if q in acc else blk.copy()
        bp = mesh.f[p].copy()
        cols = []
        for q in sorted(acc):
            if mesh.dirichlet[q]:
                bp -= acc[q] @ mesh.u_D[q]
            else:
                cols.append(q)
        out.append((np.array(cols, dtype=np.int64), np.array([acc[q] for q in cols]), bp))
    return out


def build_system(prob) -> System:
    return System(Mesh(prob))


def rigid_body_modes(node_ijk: np.ndarray) -> np.ndarray:
    """Six rigid-body modes (3 translations, 3 infinitesimal rotations) as
    columns (n_dof x 6)."""
    x = node_ijk.astype(np.float64)
    n = x.shape[0]
    R = np.zeros((n, 3, 6))
    for c in range(3):
        R[:, c, c] = 1.0
    # rotations about x, y, z: u = w x r
    R[:, 1, 3] = -x[:, 2]; R[:, 2, 3] = x[:, 1]
    R[:, 0, 4] = x[:, 2];  R[:, 2, 4] = -x[:, 0]
    R[:, 0, 5] = -x[:, 1]; R[:, 1, 5] = x[:, 0]
    return R.reshape(3 * n, 6)
