"""The C ABI used from plain C (tests/c/setup_bsr_solve.c, compiled here with
the system C compiler against include/hplmm.h -- no ctypes), fed with the
ORACLE's BSR matrix: the north star's hplmm_setup(A in 3x3-block CSR,
subdomain partition, material and BC data) = hplmm_setup_bsr, then
hplmm_solve(b, tol) -> x, iterations, history (eq:ls_all P:75-77, GMRES P:482).

CPU (no GPU): the program compiles and links, and fails loudly with
HPLMM_ERR_CUDA (no CPU fallback); a caller pattern / numbering that is not the
geometry's (R3/R4) is rejected with HPLMM_ERR_ARG before any device work.
GPU: the C program's x and iteration count match the oracle's GMRES.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

from tests.conftest import oracle_case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2509_19777_b200")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    import __graft_entry__
    __graft_entry__.build()
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    out = str(tmp_path_factory.mktemp("cbin") / "setup_bsr_solve")
    subprocess.run([cc, "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "setup_bsr_solve.c"), "-L", PKG, "-lhplmm",
                    "-Wl,-rpath," + PKG, "-o", out], check=True)
    return out


def _write_case(d, name):
    """Raw arrays of the problem and of the ORACLE's A^, b^ (oracle/fem.py)."""
    p, s, h = oracle_case(name)
    os.makedirs(d, exist_ok=True)
    w = lambda f, a, t: np.ascontiguousarray(a, dtype=t).tofile(os.path.join(d, f))
    w("solid.u8", p.solid, np.uint8)
    w("E.f64", p.E, np.float64)
    w("grain.i32", p.grain, np.int32)
    w("dir.u8", p.node_dirichlet, np.uint8)
    w("node_u.f64", p.node_u, np.float64)
    w("node_f.f64", p.node_f, np.float64)
    w("row_ptr.i32", s.row_ptr, np.int32)
    w("col_idx.i32", s.col_idx, np.int32)
    w("val.f64", s.val, np.float64)
    w("node_ijk.i32", s.mesh.node_ijk, np.int32)
    w("b.f64", s.b, np.float64)
    with open(os.path.join(d, "dims.txt"), "w") as f:
        f.write(f"{p.nx} {p.ny} {p.nz} {p.n_grains} {s.mesh.n_nodes} {s.nnzb} {p.nu!r}\n")
    return p, s, h


def _run(exe, d, tol=1e-8):
    r = subprocess.run([exe, d, repr(tol)], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout.strip(), r.stderr


def test_c_client_builds_and_fails_loudly_without_gpu(exe, tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    d = str(tmp_path / "cube8")
    _write_case(d, "cube8")
    code, out, err = _run(exe, d)
    assert code == 3 and out.startswith("status -2"), (code, out, err)   # HPLMM_ERR_CUDA


def _bsr(s):
    return dict(row_ptr=s.row_ptr, col_idx=s.col_idx, val=s.val, node_ijk=s.mesh.node_ijk)


@pytest.mark.parametrize("mutation", ["col", "rowptr", "ijk", "nrows", "dirichlet_coupling"])
def test_setup_bsr_rejects_foreign_pattern(mutation):
    """ERR_ARG (status -1) for a BSR whose numbering or pattern is not the
    one the geometry defines (R3, R4); checked before any GPU work."""
    import __graft_entry__
    __graft_entry__.build()
    from paper_2509_19777_b200 import HPLMMError, Solver
    p, s, h = oracle_case("porous20")
    A = {k: np.array(v, copy=True) for k, v in _bsr(s).items()}
    r = 40
    lo, hi = int(A["row_ptr"][r]), int(A["row_ptr"][r + 1])
    if mutation == "col":
        A["col_idx"][hi - 1] += 1 if A["col_idx"][hi - 1] + 1 < s.mesh.n_nodes else -1
    elif mutation == "rowptr":
        A["row_ptr"][r + 1] -= 1
    elif mutation == "ijk":
        A["node_ijk"][r, 0] += 1
    elif mutation == "nrows":
        n = s.mesh.n_nodes - 1
        A = dict(row_ptr=A["row_ptr"][:n + 1], col_idx=A["col_idx"][:A["row_ptr"][n]],
                 val=A["val"][:A["row_ptr"][n]], node_ijk=A["node_ijk"][:n])
    else:   # keep a Dirichlet coupling the R4 pattern removes: one extra block
        d = int(np.flatnonzero(s.mesh.dirichlet)[0])
        q = next(int(c) for c in s.full.indices[s.full.indptr[3 * d]:s.full.indptr[3 * d + 1]] // 3
                 if c // 3 != d)
        rows = [list(A["col_idx"][A["row_ptr"][i]:A["row_ptr"][i + 1]]) for i in range(s.mesh.n_nodes)]
        rows[d] = sorted(rows[d] + [q])
        A["row_ptr"] = np.concatenate([[0], np.cumsum([len(x) for x in rows])])
        A["col_idx"] = np.concatenate(rows)
        A["val"] = np.zeros((A["col_idx"].size, 3, 3))
    with pytest.raises(HPLMMError) as ei:
        Solver(p, bsr=A)
    assert ei.value.status == -1, str(ei.value)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cube8", "porous20", "cfg1"])
def test_c_client_solves_oracle_matrix(exe, tmp_path, name):
    from oracle import gmres
    d = str(tmp_path / name)
    p, s, h = _write_case(d, name)
    code, out, err = _run(exe, d)
    assert code == 0, (out, err)
    f = out.split()
    rep = {f[i]: f[i + 1] for i in range(0, len(f) - 1, 2)}
    assert int(rep["status"]) == 0 and int(rep["converged"]) == 1
    assert int(rep["fine_operator"]) == 1          # the caller's stored blocks
    x = np.fromfile(os.path.join(d, "x.f64"))
    hist = np.fromfile(os.path.join(d, "hist.f64"))
    h.set_rhs(s.b)
    xo, it, ho, rr, conv = gmres.gmres(s.A, s.b, h.apply_M, tol=1e-8)
    assert abs(int(rep["iterations"]) - it) <= 1
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
    k = min(len(hist), len(ho))
    assert np.allclose(hist[:k], np.asarray(ho)[:k], rtol=1e-6, atol=0)
    assert np.linalg.norm(s.b - s.A @ x) < 1e-8 * np.linalg.norm(s.b)


@pytest.mark.gpu
def test_solver_from_bsr_matches_own_assembly():
    """The binding's Solver(bsr=...) on the oracle's matrix and the library's own
    assembly give the same operators (SPMV, M^-1) to 1e-12."""
    from paper_2509_19777_b200 import Solver
    from workloads import random_vector
    p, s, h = oracle_case("porous20")
    a = Solver(p, bsr=_bsr(s))
    b = Solver(p, operator="bsr").assemble(0).setup()
    v = random_vector(s.n_dof)
    for op in ("SPMV", "MZETA", "MGRAIN", "MCG"):
        ya, yb = a.apply(op, v), b.apply(op, v)
        assert np.linalg.norm(ya - yb) <= 1e-12 * np.linalg.norm(yb), op
    a.set_rhs(s.b)
    b.set_rhs(s.b)
    ya, yb = a.apply("MINV", v), b.apply("MINV", v)
    assert np.linalg.norm(ya - yb) <= 1e-10 * np.linalg.norm(yb)
