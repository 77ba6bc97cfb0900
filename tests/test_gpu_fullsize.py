"""GPU parity at BASELINE.json's full sizes, in the launch configuration
bench.py times (default options: supernodal local factors, TMA SpMV).

cfg2 (configs[1], 265k DOF): the oracle runs in full (setup ~1 min), so every
operator and the GMRES solve are compared element by element, as for the
small cases in test_gpu_parity.py.

cfg3 (configs[2], 2.16M DOF, the bench workload): the oracle assembles A^
(~35 s) and decomposes the mesh; compared are the full SpMV, grain-smoother
solves on sampled grains against SuperLU on the oracle's A^[I_g, I_g], the
identity M_g^-1 A^ z = z for z supported on grain interiors (eq:Mg_Mz with
disjoint grains, R18), and the final solve through its true residual computed
with the oracle's A^.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


EPS = np.finfo(np.float64).eps / 2


@pytest.fixture(scope="module")
def cfg2():
    import __graft_entry__
    __graft_entry__.build()
    from oracle import hplmm
    from paper_2509_19777_b200 import Solver
    from workloads import make_problem
    p = make_problem("cfg2")
    s, h = hplmm.setup(p)
    sv = Solver(p).assemble(0).setup()
    ev = np.linalg.eigvalsh(h.S)
    floor = 10.0 * (ev[-1] / ev[0]) * EPS
    return p, s, h, sv, floor


@pytest.mark.parametrize("op", ["SPMV", "MZETA", "MGRAIN", "MCG", "MG", "MINV"])
def test_cfg2_operators(cfg2, op):
    p, s, h, sv, floor = cfg2
    sv.set_rhs(dev(s.b))
    h.set_rhs(s.b)
    v = np.random.default_rng(12345).standard_normal(s.n_dof)
    ref = {"SPMV": lambda u: s.A @ u, "MZETA": h.apply_Mzeta, "MGRAIN": h.apply_Mg,
           "MCG": h.apply_MCG, "MG": h.apply_MG, "MINV": h.apply_M}[op](v)
    out = sv.apply(op, dev(v)).cpu().numpy()
    tol = 1e-12 if op in ("SPMV", "MZETA", "MGRAIN", "MCG") else max(1e-12, floor)
    assert rel(out, ref) <= tol, (rel(out, ref), tol)


def test_cfg2_solve(cfg2):
    from oracle import gmres
    p, s, h, sv, floor = cfg2
    h.set_rhs(s.b)
    xo, ito, histo, rro, convo = gmres.gmres(s.A, s.b, h.apply_M, tol=p.tol)
    x, rep, hist = sv.solve(dev(s.b), tol=p.tol)
    x = x.cpu().numpy()
    assert rep["converged"] == 1 and convo
    assert abs(rep["iterations"] - ito) <= 1, (rep["iterations"], ito)
    assert rel(x, xo) <= 1e-8
    assert np.linalg.norm(s.b - s.A @ x) / np.linalg.norm(s.b) < p.tol


@pytest.fixture(scope="module")
def cfg3():
    import __graft_entry__
    __graft_entry__.build()
    from oracle import decomp, fem
    from paper_2509_19777_b200 import Solver
    from workloads import make_problem
    p = make_problem("cfg3")
    s = fem.build_system(p)
    d = decomp.Decomposition(s, p.contact_h)
    sv = Solver(p).assemble(0).setup()
    return p, s, d, sv


def test_cfg3_spmv(cfg3):
    p, s, d, sv = cfg3
    v = np.random.default_rng(12345).standard_normal(s.n_dof)
    assert rel(sv.apply("SPMV", dev(v)).cpu().numpy(), s.A @ v) <= 1e-12
    # the solve's element-by-element operator vs the stored blocks and the
    # oracle's A^, row by row (summation order only)
    scale = abs(s.A) @ np.abs(v)
    ye = sv.apply("SPMV", dev(v)).cpu().numpy()
    assert sv.report()["fine_operator"] == 0
    assert np.all(np.abs(ye - sv.apply("SPMV_BSR", dev(v)).cpu().numpy()) <= 1e-13 * scale)
    assert np.all(np.abs(ye - s.A @ v) <= 1e-13 * scale)
    b = sv.export("RHS")
    assert np.abs(b - s.b).max() <= 1e-13 * np.abs(s.b).max()


def test_cfg3_grain_smoother_sampled(cfg3):
    """M_g^-1 v restricted to I_g equals A^[I_g,I_g]^-1 v[I_g] (grains are
    disjoint, eq:Mg_Mz / R18): sampled grains against SuperLU."""
    import scipy.sparse.linalg as spla
    from oracle.decomp import node_dofs
    p, s, d, sv = cfg3
    A = s.A.tocsr()
    v = np.random.default_rng(12345).standard_normal(s.n_dof)
    out = sv.apply("MGRAIN", dev(v)).cpu().numpy()
    grains = [g for g in range(len(d.grain_nodes)) if d.grain_nodes[g].size]
    for g in [grains[i] for i in np.linspace(0, len(grains) - 1, 6).astype(int)]:
        dofs = node_dofs(d.grain_nodes[g])
        Ag = A[dofs][:, dofs].tocsc()
        lu = spla.splu(Ag)
        ref = lu.solve(v[dofs])
        # two backward-stable solves differ by ~kappa_1(A_g) u (lognormal E, sigma = 1)
        inv = spla.LinearOperator(Ag.shape, matvec=lu.solve, rmatvec=lambda y: lu.solve(y, trans="T"))
        kappa = spla.norm(Ag, 1) * spla.onenormest(inv)
        tol = max(1e-12, 10 * kappa * EPS)
        assert rel(out[dofs], ref) <= tol, (g, rel(out[dofs], ref), tol)


def test_cfg3_contact_smoother_full(cfg3):
    """M_zeta^-1 v in full at cfg3 -- the contact batch, the largest launch of
    the bench step, in its bench launch shape (8 warps x 2 CTAs per SM): all
    contact grids solved by SuperLU on the oracle's A^[zeta_c, zeta_c] and
    summed in ascending interface order (eq:Mg_Mz, R8, R19)."""
    import scipy.sparse.linalg as spla
    from oracle.decomp import node_dofs
    p, s, d, sv = cfg3
    assert sv.report()["sn_shape_contact"] == 8
    A = s.A.tocsr()
    v = np.random.default_rng(12345).standard_normal(s.n_dof)
    ref = np.zeros(s.n_dof)
    for nodes in d.contact_nodes:
        if nodes.size:
            dofs = node_dofs(nodes)
            ref[dofs] += spla.splu(A[dofs][:, dofs].tocsc()).solve(v[dofs])
    out = sv.apply("MZETA", dev(v)).cpu().numpy()
    assert rel(out, ref) <= 1e-12, rel(out, ref)


def test_cfg3_grain_identity(cfg3):
    """M_g^-1 A^ z = z for z supported on the grain interiors (all grains)."""
    from oracle.decomp import node_dofs
    p, s, d, sv = cfg3
    z = np.zeros(s.n_dof)
    rng = np.random.default_rng(5)
    for nodes in d.grain_nodes:
        if nodes.size:
            dofs = node_dofs(nodes)
            z[dofs] = rng.standard_normal(dofs.size)
    Az = s.A @ z
    out = sv.apply("MGRAIN", dev(Az)).cpu().numpy()
    assert rel(out, z) <= 1e-9, rel(out, z)


def test_cfg3_solve(cfg3):
    p, s, d, sv = cfg3
    x, rep, hist = sv.solve(dev(s.b), tol=p.tol)
    x = x.cpu().numpy()
    assert rep["converged"] == 1
    assert np.linalg.norm(s.b - s.A @ x) / np.linalg.norm(s.b) < p.tol


# ---- ILU(0) base smoother, n_st = 6 at full size ---------------------
def _ilu_full_checks(p, s, sv, rows_sample=None):
    from tests.test_gpu_ilu import block_factors
    L, U = block_factors(sv, s)
    A = s.A.tocsr()
    # ILU(0) defining equations (L U)_ij = a_ij on the stored pattern, on all or
    # sampled block rows
    rp, ci = s.row_ptr, s.col_idx
    nodes = np.arange(rp.size - 1) if rows_sample is None else rows_sample
    dofs = (3 * nodes[:, None] + np.arange(3)).ravel()
    LUr = (L[dofs] @ U).tocsr()
    Ar = A[dofs]
    cols = [(3 * ci[rp[q]:rp[q + 1]][:, None] + np.arange(3)).ravel() for q in nodes]
    rr = np.concatenate([np.full(c.size, 3 * i + a) for i, c in enumerate(cols) for a in range(3)])
    cc = np.concatenate([c for c in cols for a in range(3)])
    d = np.asarray(LUr[rr, cc]).ravel() - np.asarray(Ar[rr, cc]).ravel()
    assert np.abs(d).max() <= 1e-12 * np.abs(s.val).max()
    # the apply is U^-1 L^-1 on the whole vector: L (U z) = v
    v = np.random.default_rng(12345).standard_normal(s.n_dof)
    z = sv.apply("MILU", dev(v)).cpu().numpy()
    assert rel(L @ (U @ z), v) <= 1e-12
    x, rep, _ = sv.solve(dev(s.b), tol=p.tol)
    x = x.cpu().numpy()
    assert rep["converged"] == 1
    assert np.linalg.norm(s.b - s.A @ x) / np.linalg.norm(s.b) < p.tol
    return rep


def test_cfg2_ilu(cfg2):
    from paper_2509_19777_b200 import Solver
    p, s, h, _, _ = cfg2
    sv = Solver(p, smoother="ilu0", n_st=6).assemble(0).setup()
    _ilu_full_checks(p, s, sv)


def test_cfg3_ilu(cfg3):
    from paper_2509_19777_b200 import Solver
    p, s, d, _ = cfg3
    sv = Solver(p, smoother="ilu0", n_st=6).assemble(0).setup()
    sample = np.random.default_rng(9).choice(s.row_ptr.size - 1, 4000, replace=False)
    _ilu_full_checks(p, s, sv, np.sort(sample))

