"""GPU parity at the two largest BASELINE.json configs (cfg4 = configs[3],
5.6M DOF; cfg5 = configs[4], 13.2M DOF, ~150 GB of device memory at peak) --
in a module of their own so that the cfg2/cfg3 fixtures of
test_gpu_fullsize.py are released first.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


# ---- cfg4 (configs[3], 5.6M DOF) and cfg5 (configs[4], 13.2M DOF) -----------
# The full oracle assembly is too slow / large here, so the oracle supplies
# sampled rows (oracle.fem.assemble_rows, pinned against the full assembly in
# tests/test_oracle_fem.py): SpMV and b^ on the sampled rows, and the residual
# b^ - A^ x of the GPU solution on those rows (||r_S|| <= ||r|| < tol ||b||).
@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["cfg4", "cfg5"])
def test_large_config_sampled(cfg):
    import __graft_entry__
    __graft_entry__.build()
    from oracle.fem import Mesh, assemble_rows
    from paper_2509_19777_b200 import Solver
    from workloads import make_problem
    p = make_problem(cfg)
    mesh = Mesh(p)
    sv = Solver(p).assemble(0)
    assert sv.n_dof == mesh.n_dof
    nodes = np.sort(np.random.default_rng(11).choice(mesh.n_nodes, 3000, replace=False))
    rows = assemble_rows(mesh, nodes)
    rp, ci = sv.export("ROW_PTR"), sv.export("COL_IDX")
    for q, (cols, _, _) in zip(nodes, rows):
        assert np.array_equal(cols, ci[rp[q]:rp[q + 1]])   # pattern, bit-exact
    b = sv.export("RHS")
    bS = np.concatenate([bp for _, _, bp in rows])
    dofs = (3 * nodes[:, None] + np.arange(3)).ravel()
    assert np.abs(b[dofs] - bS).max() <= 1e-13 * np.abs(b).max()

    def rows_times(v):
        return np.concatenate([np.einsum("kij,kj->i", blk, v.reshape(-1, 3)[cols])
                               for cols, blk, _ in rows])
    v = np.random.default_rng(12345).standard_normal(sv.n_dof)
    y = sv.apply("SPMV", dev(v)).cpu().numpy()
    ref = rows_times(v)
    assert rel(y[dofs], ref) <= 1e-12
    sv.setup()
    x, rep, _ = sv.solve(dev(b), tol=p.tol)
    x = x.cpu().numpy()
    assert rep["converged"] == 1 and rep["final_true_relres"] < p.tol
    rS = bS - rows_times(x)
    assert np.linalg.norm(rS) < p.tol * np.linalg.norm(b)
