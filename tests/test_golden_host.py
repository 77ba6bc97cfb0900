"""Full-size integer parity on the CPU: the library's host setup
(hplmm_create: mesh numbering R3, BSR pattern R4, node classes R6, interfaces
R7, contact grids R8, mortar placement eq:node_init/R10, shape-vector column
sets R14) against SHA-256 digests of the ORACLE's arrays at cfg2 and cfg3
(BASELINE.json configs[1], configs[2] -- the bench workload), written by
tests/golden/make_golden.py (calls only oracle/).  Bit-exact, as the north star
requires for all integer and indexing work.  No GPU work is involved.
"""
import hashlib
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def golden(name):
    path = os.path.join(HERE, "golden", f"{name}_oracle.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return json.load(open(path))


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_full_size_integer_artifacts_bit_exact(name):
    import __graft_entry__
    __graft_entry__.build()
    from paper_2509_19777_b200 import Solver
    from workloads import make_problem
    g = golden(name)
    sv = Solver(make_problem(name))
    r = sv.report()
    assert 3 * r["n_nodes"] == g["n_dof"] and r["nnzb"] == g["nnzb"]
    assert r["n_interfaces"] == g["n_interfaces"] and r["n_mortar_dofs"] == g["Nm"]
    for art, digest in g["int_sha256"].items():
        a = np.ascontiguousarray(np.asarray(sv.export(art), np.int64))
        assert hashlib.sha256(a.tobytes()).hexdigest() == digest, art


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_golden_self_consistent(name):
    """The stored oracle run is a converged GMRES(50) history (R22)."""
    g = golden(name)
    assert g["converged"] and len(g["hist"]) == g["iterations"]
    assert g["hist"][-1] < 1e-8 and g["final_true_relres"] < 1e-8
    assert all(b <= a * (1 + 1e-12) for a, b in zip(g["hist"], g["hist"][1:]))   # monotone
