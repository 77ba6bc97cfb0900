"""GPU parity of the subtree-parallel supernodal solves (hplmm_options.sn_split).

A batch with too few subdomains shares its largest ones between teams of up to
2^L CTAs: the top L levels of each nested-dissection tree are cut, the members
sweep their subtrees and exchange the separators' x rows.  The operator is the
same A_s^-1 (eq:Mg_Mz); only the order in which the subtrees' updates of a
separator are added differs, so every apply is held to the same 1e-12 against
the oracle as the one-CTA-per-subdomain path, for every cut depth and both
launch shapes, and the solve to iterations +-1 / x <= 1e-8.
"""
import numpy as np
import pytest

from tests.conftest import oracle_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = ["cube8", "cfg1", "porous20"]
_solvers = {}


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def split_case(name, split, shape=0):
    if (name, split, shape) not in _solvers:
        import __graft_entry__
        __graft_entry__.build()
        from paper_2509_19777_b200 import Solver
        p, s, h = oracle_case(name)
        sv = Solver(p, sn_split=split, sn_shape=shape).assemble(0).setup()
        _solvers[(name, split, shape)] = (p, s, h, sv)
    return _solvers[(name, split, shape)]


@pytest.mark.parametrize("case", CASES)
def test_split_off_has_no_teams(case):
    p, s, h, sv = split_case(case, -1)
    r = sv.report()
    assert r["sn_teams_grain"] == 0 and r["sn_teams_contact"] == 0 and r["sn_team_max"] == 1, r


@pytest.mark.parametrize("shape", [16, 8])
@pytest.mark.parametrize("split", [1, 2, 3])
@pytest.mark.parametrize("case", CASES)
def test_split_local_solves_match_oracle(case, split, shape):
    """M_zeta, M_g and M_CG with the largest subdomains cut `split` levels deep
    (sn_split > 0 forces the cuts; these cases have far fewer subdomains than
    CTAs, so every subdomain whose tree has a separator is shared)."""
    p, s, h, sv = split_case(case, split, shape)
    r = sv.report()
    assert r["sn_teams_grain"] > 0, r
    assert case == "cube8" or r["sn_teams_contact"] > 0, r
    assert 2 <= r["sn_team_max"] <= 2 ** split, r
    v = np.random.default_rng(12345).standard_normal(s.n_dof)
    for op, ref in (("MZETA", h.apply_Mzeta), ("MGRAIN", h.apply_Mg), ("MCG", h.apply_MCG)):
        out = sv.apply(op, dev(v)).cpu().numpy()
        assert rel(out, ref(v)) <= 1e-12, (op, rel(out, ref(v)))
    # repeated launches reuse the one-shot exchange flags
    a = sv.apply("MGRAIN", dev(v)).cpu().numpy()
    b = sv.apply("MGRAIN", dev(v)).cpu().numpy()
    assert np.array_equal(a, b)


@pytest.mark.parametrize("split", [2, 3])
@pytest.mark.parametrize("case", CASES)
def test_split_matches_unsplit(case, split):
    """Team solves against the one-CTA-per-subdomain solves of the same
    factors: the two differ only in where a separator's updates are summed."""
    p, s, h, sv = split_case(case, split)
    _, _, _, s0 = split_case(case, -1)
    v = np.random.default_rng(7).standard_normal(s.n_dof)
    for op in ("MZETA", "MGRAIN"):
        a = sv.apply(op, dev(v)).cpu().numpy()
        b = s0.apply(op, dev(v)).cpu().numpy()
        assert rel(a, b) <= 1e-13, (op, rel(a, b))


@pytest.mark.parametrize("split", [0, 3])
@pytest.mark.parametrize("case", CASES)
def test_split_solve_matches_oracle(case, split):
    """GMRES through the device-resident graph with team solves inside it
    (cooperative launches captured in the WHILE bodies)."""
    from oracle import gmres
    p, s, h, sv = split_case(case, split)
    h.set_rhs(s.b)
    xo, ito, histo, rro, convo = gmres.gmres(s.A, s.b, h.apply_M, tol=1e-8)
    x, rep, hist = sv.solve(dev(s.b), tol=1e-8)
    x = x.cpu().numpy()
    assert rep["converged"] == 1 and convo
    assert abs(rep["iterations"] - ito) <= 1, (rep["iterations"], ito)
    assert rel(x, xo) <= 1e-8
    k = min(len(hist), len(histo)) - 2
    assert np.allclose(hist[:k], histo[:k], rtol=1e-6, atol=1e-14)
    # the solve ran as one graph launch (no silent fall-back to the host loop)
    assert rep["kernel_launches"] > 0


def test_split_cfg2_golden():
    """cfg2 (64 grains, 203 contact grids on 148 SMs: teams form by default)
    against the oracle's stored full-size run (tests/golden/cfg2_oracle.*)."""
    import json
    import os
    from paper_2509_19777_b200 import Solver
    from workloads import make_problem
    gold = os.path.join(os.path.dirname(__file__), "golden")
    meta = json.load(open(os.path.join(gold, "cfg2_oracle.json")))
    p = make_problem("cfg2")
    sv = Solver(p).assemble(0).setup()
    r = sv.report()
    assert r["sn_teams_grain"] > 0 and r["sn_teams_contact"] > 0, r
    b = torch.from_numpy(sv.export("RHS")).cuda()
    x, rep, hist = sv.solve(b, tol=p.tol)
    assert rep["converged"] == 1
    assert abs(rep["iterations"] - meta["iterations"]) <= 1, (rep["iterations"], meta["iterations"])
