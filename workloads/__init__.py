"""Seeded synthetic voxel workloads (input generators only).

This module is shared by the oracle (``oracle/``), the tests and ``bench.py``.
It holds NONE of the method's arithmetic: it only draws voxel images, material
fields, grain labels and boundary data, i.e. the *problem statement* of
PAPER.md §2 (eq:Linear-elastic / eq:BC) on a Cartesian voxel grid
 with a Cartesian decomposition (§3.1).

The recipes are the readings of BASELINE.json ``configs`` written down in
SURVEY.md §8(d) (also restated in DESIGN.md "Input recipe"):

* cfg1  solid 16^3, E=1, nu=0.3, bottom clamped, unit downward traction on top,
        2x2x2 blocks.
* cfg2  porous 48^3 (Gaussian random field, sigma=3, porosity 0.35), top
        u=(0,0,-0.48), 4x4x4 blocks.
* cfg3  porous 96^3 (porosity 0.30), lognormal E (sigma=4 field), nu=0.25, top
        shear u=(0.96,0,0), 8x8x8 blocks.
* cfg4  porous 128^3 (porosity 0.20) + 6 planar fractures E=1e-6, x faces
        compressed, 8x8x8 blocks.
* cfg5  porous 192^3 (porosity 0.50), two-phase E in {1,100}, torsion, 12^3 blocks.
* cube8 solid 8^3, 2x2x2 blocks (the tiny case used by the dense brute-force pins).

Array conventions: voxel arrays are indexed ``[z][y][x]`` (x fastest, z
vertical, bottom at z=0); node arrays live on the ``(nz+1, ny+1, nx+1)``
lattice. A Dirichlet node prescribes all 3 displacement components.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = ["Problem", "make_problem", "CONFIGS", "random_vector", "load_cases", "perturbed_moduli"]


@dataclass
class Problem:
    name: str
    nx: int
    ny: int
    nz: int
    solid: np.ndarray          # uint8 [nz,ny,nx]
    E: np.ndarray              # float64 [nz,ny,nx] (read where solid)
    nu: float
    grain: np.ndarray          # int32 [nz,ny,nx], -1 where void
    n_grains: int
    node_dirichlet: np.ndarray  # uint8 [nz+1,ny+1,nx+1]
    node_u: np.ndarray         # float64 [nz+1,ny+1,nx+1,3]
    node_f: np.ndarray         # float64 [nz+1,ny+1,nx+1,3]
    block: int                 # Cartesian block edge s (voxels)
    # method parameters (BASELINE configs)
    n_mortar: int = 4
    beta: float = 4.0
    mortar: str = "gaussian"     # or "algebraic" (eq:algebra via the Remark)
    contact_h: int = 1
    restart: int = 50
    tol: float = 1e-8
    maxit: int = 300
    meta: dict = field(default_factory=dict)


# ----------------------------------------------------------------------------
# field generators
# ----------------------------------------------------------------------------
def _smooth_field(seed: int, L: int, sigma: float) -> np.ndarray:
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(seed)
    return gaussian_filter(rng.standard_normal((L, L, L)), sigma=sigma, mode="wrap")


def _porous_mask(seed: int, L: int, sigma: float, porosity: float) -> np.ndarray:
    """Solid mask: threshold a smoothed Gaussian field at the porosity quantile,
    keep the largest 6-connected solid component touching z=0 (6-connectivity:
    edge/corner-only contacts would be zero-energy hinges)."""
    from scipy.ndimage import label
    g = _smooth_field(seed, L, sigma)
    void = g < np.quantile(g, porosity)
    solid = ~void
    lab, nlab = label(solid)  # default structure = 6-connectivity in 3-D
    bottom = np.unique(lab[0][lab[0] > 0])
    if bottom.size == 0:
        raise RuntimeError("no solid component touches z=0")
    sizes = np.bincount(lab.ravel())
    keep = bottom[np.argmax(sizes[bottom])]
    return (lab == keep).astype(np.uint8)


def _cartesian_grains(solid: np.ndarray, s: int) -> tuple[np.ndarray, int]:
    """Grain of a solid voxel = its Cartesian block id bx + a(by + a*bz), then
    compacted to 0..n-1 in ascending block id (empty blocks dropped, R5)."""
    nz, ny, nx = solid.shape
    ax, ay = -(-nx // s), -(-ny // s)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    bid = (i // s) + ax * ((j // s) + ay * (k // s))
    bid = np.where(solid > 0, bid, -1)
    used = np.unique(bid[bid >= 0])
    remap = -np.ones(int(bid.max()) + 2, dtype=np.int64)
    remap[used] = np.arange(used.size)
    grain = np.where(bid >= 0, remap[np.maximum(bid, 0)], -1).astype(np.int32)
    return grain, int(used.size)


def _solid_nodes(solid: np.ndarray) -> np.ndarray:
    nz, ny, nx = solid.shape
    sn = np.zeros((nz + 1, ny + 1, nx + 1), dtype=bool)
    s = solid > 0
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                sn[dz:dz + nz, dy:dy + ny, dx:dx + nx] |= s
    return sn


def _fractures(L: int, seed: int, nfrac: int = 6) -> np.ndarray:
    """Voxel-centre c is in disc fracture (n, p, R) if |n.(c-p)| <= ||n||_inf/2
    and the in-plane distance <= R."""
    rng = np.random.default_rng(seed)
    k, j, i = np.meshgrid(np.arange(L), np.arange(L), np.arange(L), indexing="ij")
    c = np.stack([i + 0.5, j + 0.5, k + 0.5], axis=-1)
    frac = np.zeros((L, L, L), dtype=bool)
    for _ in range(nfrac):
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        p = rng.uniform(0, L, 3)
        R = rng.uniform(16, 40)
        d = c - p
        dn = d @ n
        inplane = np.linalg.norm(d - dn[..., None] * n, axis=-1)
        frac |= (np.abs(dn) <= 0.5 * np.abs(n).max()) & (inplane <= R)
    return frac


# ----------------------------------------------------------------------------
# configurations
# ----------------------------------------------------------------------------
def _base(name, solid, E, nu, s, h, **kw) -> Problem:
    nz, ny, nx = solid.shape
    grain, ng = _cartesian_grains(solid, s)
    return Problem(name=name, nx=nx, ny=ny, nz=nz, solid=solid.astype(np.uint8),
                   E=np.where(solid > 0, E, 0.0).astype(np.float64), nu=float(nu),
                   grain=grain, n_grains=ng,
                   node_dirichlet=np.zeros((nz + 1, ny + 1, nx + 1), np.uint8),
                   node_u=np.zeros((nz + 1, ny + 1, nx + 1, 3)),
                   node_f=np.zeros((nz + 1, ny + 1, nx + 1, 3)),
                   block=s, contact_h=h, **kw)


def _clamp_bottom(p: Problem, sn: np.ndarray):
    p.node_dirichlet[0][sn[0]] = 1
    p.node_u[0][sn[0]] = 0.0


def _prescribe(p: Problem, sl, sn, u):
    """Dirichlet u on lattice slice ``sl`` where a solid node exists; a node
    already clamped at the bottom keeps u=0 (bottom wins, R4)."""
    m = sn[sl] & (p.node_dirichlet[sl] == 0)
    p.node_dirichlet[sl][m] = 1
    p.node_u[sl][m] = np.asarray(u, dtype=np.float64)


def _solid_cube(name: str, L: int, s: int, h: int) -> Problem:
    solid = np.ones((L, L, L), np.uint8)
    p = _base(name, solid, np.ones((L, L, L)), 0.3, s, h)
    sn = _solid_nodes(solid)
    _clamp_bottom(p, sn)
    # unit downward traction t=(0,0,-1) on the top face as consistent nodal
    # loads: each exposed top voxel face gives -1/4 to each of its 4 corners.
    top = solid[L - 1] > 0
    f = p.node_f[L]
    for dy in (0, 1):
        for dx in (0, 1):
            f[dy:dy + L, dx:dx + L, 2] += np.where(top, -0.25, 0.0)
    return p


def _cfg2() -> Problem:
    L = 48
    solid = _porous_mask(2, L, 3.0, 0.35)
    p = _base("cfg2", solid, np.ones((L, L, L)), 0.3, 12, 2)
    sn = _solid_nodes(solid)
    _clamp_bottom(p, sn)
    _prescribe(p, np.s_[L], sn, (0.0, 0.0, -0.01 * L))
    return p


def _cfg3() -> Problem:
    L = 96
    solid = _porous_mask(3, L, 3.0, 0.30)
    z = _smooth_field(1003, L, 4.0)
    z = (z - z.mean()) / z.std()
    p = _base("cfg3", solid, np.exp(z), 0.25, 12, 2)
    sn = _solid_nodes(solid)
    _clamp_bottom(p, sn)
    _prescribe(p, np.s_[L], sn, (0.01 * L, 0.0, 0.0))
    return p


def _cfg4() -> Problem:
    L = 128
    solid = _porous_mask(4, L, 3.0, 0.20)
    E = np.where(_fractures(L, 1004), 1e-6, 1.0)
    p = _base("cfg4", solid, E, 0.3, 16, 2)
    sn = _solid_nodes(solid)
    _clamp_bottom(p, sn)
    _prescribe(p, np.s_[:, :, 0], sn, (0.005 * L, 0.0, 0.0))
    _prescribe(p, np.s_[:, :, L], sn, (-0.005 * L, 0.0, 0.0))
    return p


def _cfg5() -> Problem:
    L = 192
    solid = _porous_mask(5, L, 3.0, 0.50)
    g2 = _smooth_field(1005, L, 3.0)
    med = np.median(g2[solid > 0])
    p = _base("cfg5", solid, np.where(g2 > med, 100.0, 1.0), 0.3, 16, 2)
    sn = _solid_nodes(solid)
    _clamp_bottom(p, sn)
    theta = 0.01
    j, i = np.meshgrid(np.arange(L + 1), np.arange(L + 1), indexing="ij")
    m = sn[L] & (p.node_dirichlet[L] == 0)
    p.node_dirichlet[L][m] = 1
    u = np.stack([-theta * (j - L / 2), theta * (i - L / 2), np.zeros_like(i, dtype=float)], -1)
    p.node_u[L][m] = u[m]
    return p


def _porous_small(name: str, L: int, s: int, h: int, seed: int, porosity: float) -> Problem:
    """Small porous cases for parity tests (same generator as cfg2)."""
    solid = _porous_mask(seed, L, 2.0, porosity)
    z = _smooth_field(seed + 1000, L, 2.0)
    z = (z - z.mean()) / z.std()
    p = _base(name, solid, np.exp(0.5 * z), 0.3, s, h)
    sn = _solid_nodes(solid)
    _clamp_bottom(p, sn)
    _prescribe(p, np.s_[L], sn, (0.01 * L, 0.0, -0.01 * L))
    return p


CONFIGS = {
    "cube8": lambda: _solid_cube("cube8", 8, 4, 1),
    "cfg1": lambda: _solid_cube("cfg1", 16, 8, 1),
    "cfg2": _cfg2,
    "cfg3": _cfg3,
    "cfg4": _cfg4,
    "cfg5": _cfg5,
    # small ragged porous case: 20^3 with 8-voxel blocks -> 3x3x3 blocks, the
    # last one ragged (4 voxels); used for parity over several tiles + tails.
    "porous20": lambda: _porous_small("porous20", 20, 8, 1, 7, 0.3),
}


def make_problem(name: str, **overrides) -> Problem:
    p = CONFIGS[name]()
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def load_cases(p: Problem, k: int) -> list:
    """k load cases on one problem (the paper's multi-RHS reuse):
    same geometry, material, decomposition and Dirichlet node set, different
    loads.  Case 0 is ``p`` itself; case c >= 1 cyclically shifts the
    components of the prescribed displacement on every Dirichlet node that is
    not clamped at the bottom (shear x -> y -> z ...) and adds seeded nodal
    forces 1e-3 N(0,1) (seed 2000 + c) on every lattice node.  Only the
    right-hand side b^ changes from case to case (eq:ls_all)."""
    import copy
    out = [p]
    for c in range(1, k):
        q = copy.deepcopy(p)
        q.name = f"{p.name}_load{c}"
        u = np.asarray(p.node_u)
        q.node_u = np.roll(u, c, axis=-1).copy()
        q.node_u[0] = u[0]                       # the bottom clamp keeps u = 0
        rng = np.random.default_rng(2000 + c)
        q.node_f = np.asarray(p.node_f) + 1e-3 * rng.standard_normal(np.shape(p.node_f))
        out.append(q)
    return out


def random_vector(n: int, seed: int = 12345) -> np.ndarray:
    """N(0,1) parity input (default_rng(12345))."""
    return np.random.default_rng(seed).standard_normal(n)


def perturbed_moduli(prob: "Problem", kind: str = "crack", seed: int = 11) -> np.ndarray:
    """New per-voxel Young's moduli for the reuse of M_G across a perturbed A^
    (P:743): same geometry, grains and boundary data.

    * ``crack``: a localised degradation -- the solid voxels of a thin slanted
      band through the middle of the sample lose 3 decades of stiffness (the
      "local cracks" of P:743);
    * ``global``: E scaled voxel by voxel by a seeded, spatially uncorrelated
      factor in [0.8, 1.25] -- global AND rough (the case where, per P:819,
      "M_G must be updated");
    * ``smooth``: E scaled by a smooth field in [0.8, 1.25] (one period of a
      sine product across the sample: "global but not too severe").
    """
    E = np.array(prob.E, dtype=np.float64, copy=True)
    nz, ny, nx = E.shape
    if kind == "crack":
        z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        band = np.abs((z - nz // 2) + (x - nx // 2) // 3) <= 0
        band &= (y >= ny // 4) & (y < ny - ny // 4)
        E[band] *= 1e-3
    elif kind == "global":
        rng = np.random.default_rng(seed)
        E *= np.exp(rng.uniform(np.log(0.8), np.log(1.25), E.shape))
    elif kind == "smooth":
        z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        f = np.sin(2 * np.pi * x / nx) * np.cos(2 * np.pi * y / ny) * np.sin(2 * np.pi * (z + 0.25 * nz) / nz)
        E *= np.exp(np.log(1.25) * f)
    else:
        raise ValueError(kind)
    return E
