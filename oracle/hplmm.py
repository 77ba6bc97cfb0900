"""The hPLMM two-level preconditioner (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §4 "Multiscale preconditioner":
  eq:multi_precond   M^-1 = M_G^-1 + M_L^-1 (I - A^ M_G^-1)       [O16]
  eq:local_smoother  M_L = n_st stages of a base smoother M_l:
                                 M_CG (default, n_st = 1 => M_L = M_CG, R20)
                                 or ILU(0) (oracle/ilu.py, R26-R28)
  eq:mg_struct / eq:WQP  M_G^-1 = P^ (R^ A^ P^)^-1 R^, R^ = P^T,
                                 P^ = W Q P                                  [O13]
  eq:reduced_defs    Q = diag(I, Q^o), Q^o from mortar blocks M^{m_i}
                                 (horizontal concatenation per interface, R12)
  eq:all_prolong     P = [B C; I O],
                                 c^{g_i} = (A^{g_i}_{g_i})^-1 b^{g_i}           (eq:col_cg)
                                 p_k^{g_i} = -(A^{g_i}_{g_i})^-1 Abar^{g_i}_{m_j} R^{m_j}_m e_k
                                                                          (eq:col_pk)
  eq:local_smoother_CG M_CG^-1 = M_zeta^-1 + M_g^-1 (I - A^ M_zeta^-1)
  eq:Mg_Mz           additive Schwarz  sum_i E_i (R_i A^ E_i)^-1 R_i

W is absorbed: every vector stays in the original (node-major) DOF order, so
P^ column k = q_k + sum_g E_g p_k^g with q_k = Q^o e_k on interface DOFs.
Readings: R13 (coarse order), R14 (option B: a shape vector is built in EVERY
grain structurally coupled to the mortar's interface), R15 (correction columns
only for grains with b[I_g] != 0), R16 (A^o = blockdiag(S, D_c) with
S = P_B^T A^ P_B symmetrised from its lower triangle, D_c[g] = b_g . c_g),
R17 (dense Cholesky of S), R18 (M_g on grain-interior DOFs I_g), R19 (plain
additive overlap sum, ascending interface id), R21 (M_G first; M_zeta first),
R30 (update_matrix: M_G reused across a perturbed A^, local solves refreshed).
"""
from __future__ import annotations

import time

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from .decomp import CLASS_G, Decomposition, node_dofs
from .fem import System, build_system
from .ilu import ILU0, block_pattern_csr, local_smoother
from .mortar import Mortars


class _Local:
    """Exact local solve with (R_s A^ E_s)^-1 by a sparse LU factorisation
    (the paper's precomputed LU)."""

    def __init__(self, A, dofs):
        self.dofs = dofs
        self.n = dofs.size
        self.lu = splu(A[dofs][:, dofs].tocsc()) if self.n else None

    def solve(self, r):
        if self.n == 0:
            return np.zeros_like(r)
        return self.lu.solve(r)


class HPLMM:
    def __init__(self, system: System, n_mortar: int = 4, beta: float = 4.0,
                 contact_h: int = 1, mortar: str = "gaussian", smoother: str = "cg",
                 n_st: int = 1):
        if smoother not in ("cg", "ilu0") or n_st < 1:
            raise ValueError("smoother must be 'cg' or 'ilu0' and n_st >= 1")
        self.smoother, self.n_st = smoother, int(n_st)
        self._params = dict(n_mortar=n_mortar, beta=beta, contact_h=contact_h, mortar=mortar,
                            smoother=smoother, n_st=n_st)
        self.sys = system
        self.timings = {}      # wall seconds of the setup phases (bench's cpu baseline)
        t0 = time.perf_counter()
        A = system.A
        self.A = A
        n_dof = system.n_dof
        mesh = system.mesh
        self.dec = Decomposition(system, contact_h)
        self.mor = Mortars(self.dec, mesh.node_ijk, n_mortar, beta, kind=mortar, A=A,
                           system=system)
        dec, mor = self.dec, self.mor
        Nm = mor.n_mortar_dofs
        self.Nm = Nm

        # Q^o (eq:reduced_defs, R12/R13): column 3*(off_c + i) + gamma,
        # rows 3*F[f] + d, values M^{c}[3f + d, 3i + gamma]
        r, c, v = [], [], []
        for ci, F in enumerate(dec.interfaces):
            M = mor.blocks[ci]
            rows = (3 * np.asarray(F)[:, None] + np.arange(3)[None, :]).ravel()
            for q in range(M.shape[1]):
                nz = M[:, q] != 0.0
                r.append(rows[nz])
                c.append(np.full(int(nz.sum()), 3 * mor.offset[ci] + q))
                v.append(M[nz, q])
        self.Qo = sp.csc_matrix((np.concatenate(v), (np.concatenate(r), np.concatenate(c))),
                                shape=(n_dof, Nm)) if r else sp.csc_matrix((n_dof, Nm))

        t1 = time.perf_counter()
        # grain-interior DOF sets and their factors (eq:permute_blk_2, R18)
        self.grain_dofs = [node_dofs(nodes) for nodes in dec.grain_nodes]
        self.grain_solve = [_Local(A, d) for d in self.grain_dofs]
        # contact grids (eq:Mg_Mz, R8/R19)
        self.contact_dofs = [node_dofs(nodes) for nodes in dec.contact_nodes]
        self.contact_solve = [_Local(A, d) for d in self.contact_dofs]
        # ILU(0) base smoother (R26): scalar pattern = all 9 entries of
        # every stored block, natural DOF order
        self.ilu = (ILU0(block_pattern_csr(system.row_ptr, system.col_idx, system.val,
                                           mesh.n_nodes))
                    if smoother == "ilu0" else None)
        t2 = time.perf_counter()

        # cols_g (R14 option B, structural): every mortar column of an interface
        # that has a node coupled (a block of A^) to a class-G node of grain g.
        rp, ci_ = system.row_ptr, system.col_idx
        self.grain_cols = []
        for g, nodes in enumerate(dec.grain_nodes):
            ifs = set()
            for p in nodes:
                if dec.node_class[p] != CLASS_G:
                    continue
                for q in ci_[rp[p]:rp[p + 1]]:
                    if dec.node_iface[q] >= 0:
                        ifs.add(int(dec.node_iface[q]))
            cols = [np.arange(3 * mor.offset[c], 3 * mor.offset[c + 1]) for c in sorted(ifs)]
            self.grain_cols.append(np.concatenate(cols).astype(np.int64) if cols
                                   else np.zeros(0, np.int64))

        # shape vectors (eq:col_pk): B_g = -A_g^-1 (A^[I_g,:] Q^o[:, cols_g])
        self.B = []
        rows, cols, vals = [], [], []
        for g in range(dec.n_grains):
            dg, cg = self.grain_dofs[g], self.grain_cols[g]
            if dg.size == 0 or cg.size == 0:
                self.B.append(np.zeros((dg.size, cg.size)))
                continue
            Rg = (A[dg] @ self.Qo[:, cg]).toarray()
            Bg = -self.grain_solve[g].solve(Rg)
            self.B.append(Bg)
            rows.append(np.repeat(dg.astype(np.int32), cg.size))     # int32: cfg3 has
            cols.append(np.tile(cg.astype(np.int32), dg.size))       # 0.25 G entries
            vals.append(Bg.ravel())
        if rows:
            rows, cols, vals = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
            PB = sp.csc_matrix((vals, (rows, cols)), shape=(n_dof, Nm))
            del rows, cols, vals
        else:
            PB = sp.csc_matrix((n_dof, Nm))
        self.PB = (self.Qo + PB).tocsc()
        del PB
        self.PBT = self.PB.T          # CSR view of the same arrays

        # coarse mortar block S = P_B^T A^ P_B (eq:mg_struct, R16), formed a
        # block of columns of P_B at a time (the sparse intermediate A^ P_B of
        # the whole P_B is ~10 GB at cfg3), symmetrised from its lower
        # triangle; dense Cholesky (R17)
        S = np.zeros((Nm, Nm))
        for j0 in range(0, Nm, 2048):
            J = slice(j0, min(Nm, j0 + 2048))
            S[:, J] = (self.PBT @ (A @ self.PB[:, J])).toarray()
        # S = tril(S) + tril(S, -1)^T, block by block in place: S[I, J] = S[J, I]^T, I < J
        for i0 in range(0, Nm, 2048):
            I = slice(i0, min(Nm, i0 + 2048))
            for j0 in range(i0, Nm, 2048):
                J = slice(j0, min(Nm, j0 + 2048))
                if j0 == i0:
                    blk = S[I, J]
                    S[I, J] = np.tril(blk) + np.tril(blk, -1).T
                else:
                    S[I, J] = S[J, I].T
        self.S = S
        self.S_chol = sla.cho_factor(self.S, lower=True) if Nm else None
        self.corr = []          # set by set_rhs
        t3 = time.perf_counter()
        # T_ML-like: local (grain + contact-grid) factorisations; T_MG-like:
        # decomposition, mortars, Q^o, shape vectors, S and its factor
        self.timings = {"T_ML": t2 - t1, "T_MG": (t1 - t0) + (t3 - t2)}

    # ------------------------------------------------------------------
    def update_matrix(self, system: System):
        """Reuse of M_G for a perturbed A^ (reading R30): the
        linear system becomes `system` (same mesh, pattern and decomposition;
        new values, e.g. locally degraded moduli), M_G keeps the P^_B and S
        built from the ORIGINAL matrix, and everything local follows the new
        one: the residual operator A^, the exact grain / contact-grid solves
        of M_g and M_zeta (eq:Mg_Mz) and, through set_rhs, the correction
        columns c^g = (A_g)^-1 b^g (eq:col_cg).  GMRES on the new system with
        this preconditioner still converges to the new solution; only the
        iteration count feels the stale coarse space."""
        if self.smoother != "cg":
            raise ValueError("update_matrix: contact-grain smoother only")
        if system.n_dof != self.sys.n_dof or not np.array_equal(system.col_idx, self.sys.col_idx):
            raise ValueError("update_matrix: the block pattern must not change")
        self.sys = system
        self.A = system.A
        self.grain_solve = [_Local(self.A, d) for d in self.grain_dofs]
        self.contact_solve = [_Local(self.A, d) for d in self.contact_dofs]
        self.corr = []

    def refresh_coarse(self):
        """"Otherwise, M_G must be updated periodically": M_G rebuilt
        for the CURRENT system -- by definition the setup of eq:mg_struct /
        eq:col_pk on that system (same geometry, decomposition and mortar
        nodes: they do not depend on the matrix values)."""
        self.__init__(self.sys, **self._params)

    def set_rhs(self, b: np.ndarray):
        """Correction vectors c^g = A_g^-1 b^g (eq:col_cg) for grains with
        b[I_g] != 0 (R15); D_c[g] = b^g . c^g (R16)."""
        self.corr = []
        for g in range(self.dec.n_grains):
            dg = self.grain_dofs[g]
            bg = b[dg]
            if dg.size == 0 or not np.any(bg != 0.0):
                continue
            cg = self.grain_solve[g].solve(bg)
            self.corr.append((g, cg, float(bg @ cg)))

    @property
    def n_coarse(self):
        return self.Nm + len(self.corr)

    def P_C(self) -> sp.csc_matrix:
        n = self.sys.n_dof
        if not self.corr:
            return sp.csc_matrix((n, 0))
        r = np.concatenate([self.grain_dofs[g] for g, _, _ in self.corr])
        c = np.concatenate([np.full(self.grain_dofs[g].size, j)
                            for j, (g, _, _) in enumerate(self.corr)])
        v = np.concatenate([cg for _, cg, _ in self.corr])
        return sp.csc_matrix((v, (r, c)), shape=(n, len(self.corr)))

    def coarse_matrix_literal(self) -> np.ndarray:
        """A^o = R^ A^ P^ with P^ = [P_B, P_C], dense (eq:mg_struct, pins only)."""
        P = sp.hstack([self.PB, self.P_C()]).tocsc()
        return (P.T @ (self.A @ P)).toarray()

    # ------------------------------------------------------------------
    def restrict(self, r):
        """r_c = P^T r: mortar part P_B^T r, correction part c_g^T r[I_g]."""
        rm = self.PBT @ r
        rc = np.array([cg @ r[self.grain_dofs[g]] for g, cg, _ in self.corr])
        return rm, rc

    def apply_MG(self, r):
        """M_G^-1 r = P^ (A^o)^-1 P^T r (eq:mg_struct) with A^o = blockdiag(S, D_c)."""
        rm, rc = self.restrict(r)
        ym = sla.cho_solve(self.S_chol, rm) if self.Nm else rm
        x = self.PB @ ym
        for j, (g, cg, Dc) in enumerate(self.corr):
            x[self.grain_dofs[g]] += cg * (rc[j] / Dc)
        return x

    def apply_Mzeta(self, r):
        """M_zeta^-1 r = sum_c E_c (A^[zeta_c, zeta_c])^-1 r[zeta_c] (eq:Mg_Mz)."""
        z = np.zeros_like(r)
        for d, s in zip(self.contact_dofs, self.contact_solve):
            if d.size:
                z[d] += s.solve(r[d])
        return z

    def apply_Mg(self, r):
        """M_g^-1 r = sum_g E_g (A_g)^-1 r[I_g] (eq:Mg_Mz, R18)."""
        z = np.zeros_like(r)
        for d, s in zip(self.grain_dofs, self.grain_solve):
            if d.size:
                z[d] += s.solve(r[d])
        return z

    def apply_MCG(self, r):
        """M_CG^-1 r = z1 + M_g^-1 (r - A^ z1), z1 = M_zeta^-1 r (eq:local_smoother_CG)."""
        z1 = self.apply_Mzeta(r)
        return z1 + self.apply_Mg(r - self.A @ z1)

    def apply_Ml(self, r):
        """The base smoother M_l^-1 r: M_CG (eq:local_smoother_CG) or ILU(0) (R27)."""
        return self.apply_MCG(r) if self.smoother == "cg" else self.ilu.solve(r)

    def apply_ML(self, r):
        """M_L^-1 r with n_st stages of M_l (eq:local_smoother, R28)."""
        return local_smoother(self.A, self.apply_Ml, r, self.n_st)

    def apply_M(self, r):
        """M^-1 r = y + M_L^-1 (r - A^ y), y = M_G^-1 r (eq:multi_precond)."""
        y = self.apply_MG(r)
        return y + self.apply_ML(r - self.A @ y)


def setup(prob, **kw) -> tuple[System, HPLMM]:
    s = build_system(prob)
    h = HPLMM(s, n_mortar=kw.get("n_mortar", prob.n_mortar), beta=kw.get("beta", prob.beta),
              contact_h=kw.get("contact_h", prob.contact_h),
              mortar=kw.get("mortar", getattr(prob, "mortar", "gaussian")),
              smoother=kw.get("smoother", "cg"), n_st=kw.get("n_st", 1))
    return s, h
