"""C-ABI library: loads, exports every declared symbol, and its HOST integer
setup (hplmm_create: no GPU work) is bit-exact with the oracle.

North_star parity contract: "bit-exact on all integer and indexing work (voxel
mesh, connectivity, partition, sparsity patterns)".  Mortar placement (R10) is
included: its IEEE-fixed potentials make it an integer decision.
"""
import ctypes
import os
import re

import numpy as np
import pytest

from tests.conftest import oracle_case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2509_19777_b200 import hplmm
    return hplmm.load()


def test_exports_every_header_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "hplmm.h")).read()
    names = set(re.findall(r"\b(hplmm_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 14
    for n in sorted(names):
        assert hasattr(lib, n), n
    from paper_2509_19777_b200 import hplmm
    assert names == set(hplmm.EXPORTED)


def test_gpu_entry_fails_loudly_without_device(lib):
    """No CPU fallback: on a box without a GPU hplmm_assemble must error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2509_19777_b200 import Solver, HPLMMError
    from workloads import make_problem
    s = Solver(make_problem("cube8"))
    with pytest.raises(HPLMMError):
        s.assemble()


def test_invalid_options_rejected(lib):
    from paper_2509_19777_b200 import Solver, HPLMMError
    from workloads import make_problem
    with pytest.raises(HPLMMError):
        Solver(make_problem("cube8"), restart=0)


def _csr(lists):
    ptr = np.zeros(len(lists) + 1, np.int64)
    ptr[1:] = np.cumsum([len(x) for x in lists])
    val = np.concatenate([np.asarray(x, np.int64) for x in lists]) if lists else np.zeros(0)
    return ptr, val


@pytest.mark.parametrize("case", ["cube8", "cfg1", "porous20"])
def test_integer_artifacts_bit_exact(lib, case):
    from paper_2509_19777_b200 import Solver
    p, s, h = oracle_case(case)
    sv = Solver(p)
    d = h.dec
    eq = lambda a, b: np.array_equal(np.asarray(a, np.int64), np.asarray(b, np.int64))
    assert eq(sv.export("NODE_KEY"), s.mesh.node_key)
    assert eq(sv.export("ROW_PTR"), s.row_ptr)
    assert eq(sv.export("COL_IDX"), s.col_idx)
    assert eq(sv.export("NODE_CLASS"), d.node_class)
    assert eq(sv.export("NODE_IFACE"), d.node_iface)
    assert eq(sv.export("NODE_OWNER"), d.owner)
    ptr, nodes = _csr(d.interfaces)
    assert eq(sv.export("IFACE_PTR"), ptr) and eq(sv.export("IFACE_NODES"), nodes)
    ptr, nodes = _csr(d.contact_nodes)
    assert eq(sv.export("CONTACT_PTR"), ptr) and eq(sv.export("CONTACT_NODES"), nodes)
    ptr, nodes = _csr(h.mor.nodes)
    assert eq(sv.export("MORTAR_PTR"), ptr) and eq(sv.export("MORTAR_NODES"), nodes)
    ptr, cols = _csr(h.grain_cols)
    assert eq(sv.export("GRAIN_COLS_PTR"), ptr) and eq(sv.export("GRAIN_COLS"), cols)
    r = sv.report()
    assert r["n_interfaces"] == d.n_interfaces and r["n_mortar_dofs"] == h.Nm


@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_mortar_placement_other_n_bit_exact(lib, n):
    from paper_2509_19777_b200 import Solver
    from oracle import mortar
    p, s, h = oracle_case("porous20")
    sv = Solver(p, n_mortar=n)
    m = mortar.Mortars(h.dec, s.mesh.node_ijk, n, 4.0)
    ptr, nodes = _csr(m.nodes)
    assert np.array_equal(sv.export("MORTAR_PTR"), ptr)
    assert np.array_equal(sv.export("MORTAR_NODES"), nodes)


def test_binding_struct_layout_matches_header(tmp_path):
    """The ctypes structs of the binding have the C layout of include/hplmm.h
    (size and every field offset, compiled with the system C compiler) and
    the enums' values agree."""
    import shutil
    import subprocess
    from paper_2509_19777_b200 import hplmm
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {"hplmm_problem": hplmm.Problem, "hplmm_options": hplmm.Options,
               "hplmm_report": hplmm.Report, "hplmm_bsr": hplmm.Bsr}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "hplmm.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    for op, v in hplmm.OP.items():
        lines.append(f'printf("op {op} %d\\n", (int)HPLMM_OP_{op});')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln:
            a, b, c = ln.split()
            got[(a, b)] = int(c)
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
    for op, v in hplmm.OP.items():
        assert got[("op", op)] == v, op
