"""Thin ctypes binding of libhplmm (include/hplmm.h).

Argument marshalling only: every step of the hot path runs in the CUDA
library.  There is no CPU fallback -- if ``libhplmm.so`` is missing or no GPU
is usable, calls raise.  Vectors may be NumPy arrays (host) or torch CUDA
tensors (device, float64, contiguous); the library detects which.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HPLMM_LIB: an alternative in-tree build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("HPLMM_LIB") or os.path.join(_HERE, "libhplmm.so")

# status codes / ops / artifacts (mirror include/hplmm.h)
OK, NOT_CONVERGED = 0, 1
ERR_NAMES = {-1: "ERR_ARG", -2: "ERR_CUDA", -3: "ERR_OOM", -4: "ERR_SINGULAR_LOCAL",
             -5: "ERR_SINGULAR_COARSE", -6: "ERR_NONFINITE", -7: "ERR_STATE"}
OP = dict(SPMV=0, MG=1, MZETA=2, MGRAIN=3, MCG=4, MINV=5, RESTRICT=6, PROLONG=7, COARSE=8,
          MILU=9, ML=10, SPMV_BSR=11)
ART = dict(NODE_KEY=0, ROW_PTR=1, COL_IDX=2, NODE_CLASS=3, NODE_IFACE=4, NODE_OWNER=5,
           IFACE_PTR=6, IFACE_NODES=7, CONTACT_PTR=8, CONTACT_NODES=9, MORTAR_PTR=10,
           MORTAR_NODES=11, GRAIN_COLS_PTR=12, GRAIN_COLS=13, VAL=14, RHS=15, S=16,
           MORTAR_W=17, ILU=18)
_ART_DTYPE = {0: np.int64, 14: np.float64, 15: np.float64, 16: np.float64, 17: np.float64,
              18: np.float64}
SMOOTHER = dict(cg=0, ilu0=1)

EXPORTED = ["hplmm_default_options", "hplmm_create", "hplmm_assemble", "hplmm_set_matrix",
            "hplmm_setup", "hplmm_update_moduli", "hplmm_refresh_coarse", "hplmm_set_rhs", "hplmm_solve", "hplmm_solve_many", "hplmm_apply",
            "hplmm_apply_many",
            "hplmm_export", "hplmm_setup_bsr", "hplmm_assemble_bsr", "hplmm_free_bsr",
            "hplmm_get_report", "hplmm_profile", "hplmm_kernel_stats", "hplmm_destroy",
            "hplmm_last_error"]


class Problem(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("solid", C.c_void_p), ("E", C.c_void_p), ("nu", C.c_double),
                ("grain", C.c_void_p), ("n_grains", C.c_int32),
                ("node_dirichlet", C.c_void_p), ("node_u", C.c_void_p), ("node_f", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("n_mortar", C.c_int32), ("beta", C.c_double), ("contact_h", C.c_int32),
                ("restart", C.c_int32), ("max_iter", C.c_int32), ("n_st", C.c_int32),
                ("coarse_refine", C.c_int32), ("local_factor", C.c_int32),
                ("coarse_solver", C.c_int32), ("mortar_kind", C.c_int32),
                ("smoother", C.c_int32), ("operator_kind", C.c_int32),
                ("sn_shape", C.c_int32), ("sn_split", C.c_int32), ("host_loop", C.c_int32),
                ("rhs_block", C.c_int32)]


class Bsr(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("nnzb", C.c_int64), ("row_ptr", C.c_void_p),
                ("col_idx", C.c_void_p), ("val", C.c_void_p), ("node_ijk", C.c_void_p)]


class Report(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("nnzb", C.c_int64), ("n_grains", C.c_int32),
                ("n_interfaces", C.c_int32), ("n_mortar_dofs", C.c_int32),
                ("n_coarse", C.c_int32), ("local_bytes", C.c_int64),
                ("coarse_bytes", C.c_int64), ("prolong_nnz", C.c_int64),
                ("iterations", C.c_int32), ("converged", C.c_int32), ("hist_len", C.c_int32),
                ("err_index", C.c_int32), ("final_true_relres", C.c_double),
                ("t_host_setup_s", C.c_double), ("t_assemble_s", C.c_double),
                ("t_setup_local_s", C.c_double), ("t_setup_coarse_s", C.c_double),
                ("t_rhs_s", C.c_double), ("t_solve_s", C.c_double), ("t_update_s", C.c_double),
                ("kernel_launches", C.c_int64), ("fine_operator", C.c_int32),
                ("sn_shape_grain", C.c_int32), ("sn_shape_contact", C.c_int32),
                ("sn_teams_grain", C.c_int32), ("sn_teams_contact", C.c_int32),
                ("sn_team_max", C.c_int32), ("sn_xg_grain", C.c_int32),
                ("sn_xg_contact", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libhplmm.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not found: build it with "
                           "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    vp, i32, dbl = C.c_void_p, C.c_int32, C.c_double
    sig = {
        "hplmm_default_options": (None, [vp]),
        "hplmm_create": (C.c_int, [vp, vp, vp]),
        "hplmm_assemble": (C.c_int, [vp, i32, vp]),
        "hplmm_set_matrix": (C.c_int, [vp, vp, vp]),
        "hplmm_setup": (C.c_int, [vp, vp]),
        "hplmm_update_moduli": (C.c_int, [vp, vp, vp]),
        "hplmm_refresh_coarse": (C.c_int, [vp, vp]),
        "hplmm_set_rhs": (C.c_int, [vp, vp, vp]),
        "hplmm_solve": (C.c_int, [vp, vp, dbl, vp, vp, vp, i32, vp]),
        "hplmm_solve_many": (C.c_int, [vp, i32, vp, dbl, vp, vp, vp]),
        "hplmm_apply": (C.c_int, [vp, i32, vp, vp, vp]),
        "hplmm_apply_many": (C.c_int, [vp, i32, i32, vp, C.c_int64, vp, C.c_int64, vp]),
        "hplmm_export": (C.c_int, [vp, i32, vp, C.c_int64, vp]),
        "hplmm_setup_bsr": (C.c_int, [vp, vp, vp, i32, vp, vp]),
        "hplmm_assemble_bsr": (C.c_int, [vp, i32, vp, vp]),
        "hplmm_free_bsr": (None, [vp, vp]),
        "hplmm_get_report": (C.c_int, [vp, vp]),
        "hplmm_profile": (C.c_int, [vp, i32, i32]),
        "hplmm_kernel_stats": (C.c_int, [vp, i32, vp, vp, vp]),
        "hplmm_destroy": (None, [vp]),
        "hplmm_last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


class HPLMMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{ERR_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(st, allow=(OK,)):
    if st not in allow:
        raise HPLMMError(st, load().hplmm_last_error().decode())
    return st


def _ptr(a):
    """(pointer, keepalive) for a NumPy array or a torch tensor."""
    if a is None:
        return None, None
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a)
        return a.ctypes.data, a
    # torch tensor
    if not a.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return a.data_ptr(), a


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return 0
    return int(getattr(stream, "cuda_stream", stream))


def default_options(**kw) -> Options:
    o = Options()
    load().hplmm_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


OPERATOR = {"ebe": 0, "bsr": 1}   # hplmm_options.operator_kind


def _problem(prob):
    """(hplmm_problem, keepalive arrays) of a ``workloads.Problem``-like object."""
    arr = lambda a, dt: np.ascontiguousarray(a, dtype=dt)
    solid = arr(prob.solid, np.uint8)
    E = arr(prob.E, np.float64)
    grain = arr(prob.grain, np.int32)
    ndir = arr(prob.node_dirichlet, np.uint8)
    nu_ = arr(prob.node_u, np.float64)
    nf = arr(prob.node_f, np.float64)
    p = Problem(prob.nx, prob.ny, prob.nz, solid.ctypes.data, E.ctypes.data, float(prob.nu),
                grain.ctypes.data, int(prob.n_grains), ndir.ctypes.data, nu_.ctypes.data,
                nf.ctypes.data)
    return p, [solid, E, grain, ndir, nu_, nf]


def assemble_bsr(prob, device: int = 0):
    """hplmm_assemble_bsr: the library's A^ (row_ptr, col_idx, val (nnzb,3,3),
    node_ijk (n,3)) and b^ as host NumPy copies."""
    lib = load()
    p, keep = _problem(prob)
    A = C.POINTER(Bsr)()
    b = C.POINTER(C.c_double)()
    _check(lib.hplmm_assemble_bsr(C.byref(p), device, C.byref(A), C.byref(b)))
    try:
        a = A.contents
        n, nb = a.n_nodes, a.nnzb
        cp = lambda ptr, ct, cnt: np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), (cnt,)).copy()
        out = dict(row_ptr=cp(a.row_ptr, C.c_int32, n + 1), col_idx=cp(a.col_idx, C.c_int32, nb),
                   val=cp(a.val, C.c_double, 9 * nb).reshape(nb, 3, 3),
                   node_ijk=cp(a.node_ijk, C.c_int32, 3 * n).reshape(n, 3),
                   b=np.ctypeslib.as_array(b, (3 * n,)).copy())
    finally:
        lib.hplmm_free_bsr(A, b)
    return out


class Solver:
    """Handle over one voxel problem (a ``workloads.Problem``-like object)."""

    def __init__(self, prob, n_mortar=None, beta=None, contact_h=None, restart=None,
                 max_iter=None, coarse_refine=0, local_factor=None, coarse_solver=None,
                 mortar=None, smoother=None, n_st=None, operator=None, sn_shape=None,
                 sn_split=None, host_loop=None, rhs_block=None, bsr=None, device=0, stream=None):
        """bsr: optional dict(row_ptr, col_idx, val, node_ijk=None) -- the
        caller's matrix A^ (host NumPy or torch CUDA arrays): the handle is
        then built by hplmm_setup_bsr (create + pattern check + assemble +
        values + setup, on `device`) and is ready to solve."""
        lib = load()
        self._lib = lib
        p, self._keep = _problem(prob)
        o = default_options()
        for k, v in dict(n_mortar=n_mortar if n_mortar is not None else getattr(prob, "n_mortar", None),
                         beta=beta if beta is not None else getattr(prob, "beta", None),
                         contact_h=contact_h if contact_h is not None else getattr(prob, "contact_h", None),
                         restart=restart if restart is not None else getattr(prob, "restart", None),
                         max_iter=max_iter if max_iter is not None else getattr(prob, "maxit", None)).items():
            if v is not None:
                setattr(o, k, v)
        o.coarse_refine = int(coarse_refine)
        if local_factor is not None:
            o.local_factor = int(local_factor)
        if coarse_solver is not None:
            o.coarse_solver = int(coarse_solver)
        mk = mortar if mortar is not None else getattr(prob, "mortar", "gaussian")
        o.mortar_kind = {"gaussian": 0, "algebraic": 1, "surface": 2}[mk]
        if smoother is not None:
            o.smoother = SMOOTHER[smoother] if isinstance(smoother, str) else int(smoother)
        if n_st is not None:
            o.n_st = int(n_st)
        if operator is not None:
            o.operator_kind = OPERATOR[operator] if isinstance(operator, str) else int(operator)
        if sn_shape is not None:
            o.sn_shape = int(sn_shape)
        if sn_split is not None:
            o.sn_split = int(sn_split)
        if host_loop is not None:
            o.host_loop = int(host_loop)
        if rhs_block is not None:
            o.rhs_block = int(rhs_block)
        self.options = o
        h = C.c_void_p()
        if bsr is None:
            _check(lib.hplmm_create(C.byref(p), C.byref(o), C.byref(h)))
        else:
            dt = dict(row_ptr=np.int32, col_idx=np.int32, val=np.float64, node_ijk=np.int32)
            conv = {k: (np.ascontiguousarray(bsr[k], dtype=t)
                        if isinstance(bsr.get(k), np.ndarray) else bsr.get(k)) for k, t in dt.items()}
            ptrs = {k: _ptr(v) for k, v in conv.items()}
            n = int(conv["row_ptr"].shape[0]) - 1
            A = Bsr(n, int(conv["col_idx"].shape[0]), ptrs["row_ptr"][0], ptrs["col_idx"][0],
                    ptrs["val"][0], ptrs["node_ijk"][0])
            _check(lib.hplmm_setup_bsr(C.byref(A), C.byref(p), C.byref(o), int(device),
                                       _stream(stream), C.byref(h)))
        self._h = h
        self._keep = []
        r = self.report()
        self.n_nodes = r["n_nodes"]
        self.n_dof = 3 * self.n_nodes
        self.nnzb = r["nnzb"]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.hplmm_destroy(h)
            self._h = None

    # ---- lifecycle -----------------------------------------------------
    def assemble(self, device: int = 0, stream=None):
        _check(self._lib.hplmm_assemble(self._h, device, _stream(stream)))
        return self

    def set_matrix(self, val, stream=None):
        p, k = _ptr(val)
        _check(self._lib.hplmm_set_matrix(self._h, p, _stream(stream)))

    def setup(self, stream=None):
        _check(self._lib.hplmm_setup(self._h, _stream(stream)))
        return self

    def update_moduli(self, E, stream=None):
        """Reuse M_G for perturbed voxel moduli E (host array, [z][y][x])."""
        E = np.ascontiguousarray(E, dtype=np.float64)
        _check(self._lib.hplmm_update_moduli(self._h, E.ctypes.data_as(C.c_void_p), _stream(stream)))
        return self

    def refresh_coarse(self, stream=None):
        """Rebuild M_G (shape vectors, S, S^-1) for the current A^."""
        _check(self._lib.hplmm_refresh_coarse(self._h, _stream(stream)))
        return self

    def set_rhs(self, b, stream=None):
        p, k = _ptr(b)
        _check(self._lib.hplmm_set_rhs(self._h, p, _stream(stream)))

    def solve(self, b, tol=1e-8, x=None, hist_cap=1024, stream=None):
        """Returns (x, report dict, history ndarray).  b/x: NumPy (host) or
        torch CUDA tensors (device)."""
        if x is None:
            x = np.zeros(self.n_dof) if isinstance(b, np.ndarray) else b.new_zeros(self.n_dof)
        pb, kb = _ptr(b)
        px, kx = _ptr(x)
        hist = np.zeros(max(hist_cap, 1))
        rep = Report()
        st = self._lib.hplmm_solve(self._h, pb, float(tol), px, C.byref(rep), hist.ctypes.data,
                                   hist_cap, _stream(stream))
        _check(st, allow=(OK, NOT_CONVERGED))
        if isinstance(x, np.ndarray) and kx is not x:
            x[:] = kx
        return x, rep.as_dict(), hist[:rep.hist_len].copy()

    def solve_many(self, B, tol=1e-8, X=None, stream=None):
        """B: (nrhs, n_dof) NumPy or torch CUDA array; returns (X, [report dicts])."""
        nrhs = int(B.shape[0])
        if X is None:
            X = np.zeros_like(B) if isinstance(B, np.ndarray) else B.new_zeros(B.shape)
        pb, kb = _ptr(B)
        px, kx = _ptr(X)
        reps = (Report * max(nrhs, 1))()
        st = self._lib.hplmm_solve_many(self._h, nrhs, pb, float(tol), px, reps, _stream(stream))
        _check(st, allow=(OK, NOT_CONVERGED))
        if isinstance(X, np.ndarray) and kx is not X:
            X[:] = kx
        return X, [reps[i].as_dict() for i in range(nrhs)]

    def apply_many(self, op, V, out=None, stream=None):
        """V: (ncols <= 4, n_dof) NumPy or torch CUDA array, rows = vectors;
        out[c] = op applied to V[c] through one block application."""
        opi = OP[op] if isinstance(op, str) else int(op)
        if out is None:
            out = np.zeros_like(V) if isinstance(V, np.ndarray) else V.new_zeros(V.shape)
        pi, ki = _ptr(V)
        po, ko = _ptr(out)
        ld = int(V.shape[1])
        _check(self._lib.hplmm_apply_many(self._h, opi, int(V.shape[0]), pi, ld, po,
                                          int(out.shape[1]), _stream(stream)))
        if isinstance(out, np.ndarray) and ko is not out:
            out[:] = ko
        return out

    def apply(self, op, v, out=None, stream=None):
        opi = OP[op] if isinstance(op, str) else int(op)
        r = self.report()
        n_out = {OP["RESTRICT"]: r["n_coarse"], OP["COARSE"]: r["n_mortar_dofs"]}.get(opi, self.n_dof)
        if out is None:
            out = np.zeros(n_out) if isinstance(v, np.ndarray) else v.new_zeros(n_out)
        pi, ki = _ptr(v)
        po, ko = _ptr(out)
        _check(self._lib.hplmm_apply(self._h, opi, pi, po, _stream(stream)))
        return out

    def export(self, art):
        a = ART[art] if isinstance(art, str) else int(art)
        n = C.c_int64()
        _check(self._lib.hplmm_export(self._h, a, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=_ART_DTYPE.get(a, np.int32))
        _check(self._lib.hplmm_export(self._h, a, out.ctypes.data, out.nbytes, C.byref(n)))
        return out

    def report(self) -> dict:
        r = Report()
        _check(self._lib.hplmm_get_report(self._h, C.byref(r)))
        return r.as_dict()

    def profile(self, enable=True, reset=True):
        _check(self._lib.hplmm_profile(self._h, int(enable), int(reset)))

    def kernel_stats(self, kernel: int):
        ms = C.c_double()
        n = C.c_int64()
        by = C.c_int64()
        _check(self._lib.hplmm_kernel_stats(self._h, kernel, C.byref(ms), C.byref(n), C.byref(by)))
        return ms.value, n.value, by.value
