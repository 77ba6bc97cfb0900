"""Domain decomposition: node classes, contact interfaces, contact grids (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §3.1 "Domain decomposition": grain grids Omega^{g_i}
(Cartesian decomposition), contact interfaces Gamma^{c_j} shared by
grain grids, contact grids Omega^{zeta_k} by morphological dilation of each
interface, never merged.  §3.2 notation: C^{g_i}, G^{c_j}.
eq:permute_blk_2: grain blocks A^{g_i}_{g_i}.

Readings: R5 (grain = block id), R6 (a node shared by >= 2
grains is an interface node of the pair of its two smallest grain ids;
Dirichlet nodes are never interface nodes and are owned by their lowest grain),
R7 (interface = connected component of one pair's interface nodes under the
A^ node-coupling graph; ids ordered by (g1, g2, smallest node id)), R8
(contact grid = non-Dirichlet nodes within Chebyshev node distance h of the
interface), R18 (M_g subdomain = grain-interior DOFs I_g incl. owned Dirichlet
nodes).
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

CLASS_G, CLASS_I, CLASS_D = 0, 1, 2


class Decomposition:
    def __init__(self, system, contact_h: int):
        mesh = system.mesh
        prob = mesh.prob
        n = mesh.n_nodes
        self.n_grains = int(prob.n_grains)
        # G(p): sorted grain ids of the solid voxels around node p (O4)
        nx, ny, nz = prob.nx, prob.ny, prob.nz
        gpad = -np.ones((nz + 2, ny + 2, nx + 2), dtype=np.int64)
        gpad[1:-1, 1:-1, 1:-1] = prob.grain
        i, j, k = mesh.node_ijk.T
        around = np.stack([gpad[k + dz, j + dy, i + dx]
                           for dz, dy, dx in itertools.product((0, 1), repeat=3)], 1)
        around = np.sort(around, axis=1)
        self.node_grains = []
        first = np.full(n, -1, np.int64)
        second = np.full(n, -1, np.int64)
        count = np.zeros(n, np.int64)
        for p in range(n):
            g = np.unique(around[p][around[p] >= 0])
            count[p] = g.size
            first[p] = g[0]
            if g.size >= 2:
                second[p] = g[1]
        D = mesh.dirichlet
        cls = np.where(D, CLASS_D, np.where(count >= 2, CLASS_I, CLASS_G))
        self.node_class = cls.astype(np.int64)
        self.owner = np.where(cls == CLASS_I, -1, first)        # G and D nodes
        self.pair = np.where((cls == CLASS_I)[:, None], np.stack([first, second], 1), -1)

        # interfaces: connected components per grain pair (R7)
        rp, ci = system.row_ptr, system.col_idx
        rows = np.repeat(np.arange(n), np.diff(rp))
        isI = cls == CLASS_I
        same = isI[rows] & isI[ci] & (self.pair[rows, 0] == self.pair[ci, 0]) & \
            (self.pair[rows, 1] == self.pair[ci, 1])
        G = sp.coo_matrix((np.ones(same.sum()), (rows[same], ci[same])), shape=(n, n))
        ncomp, lab = connected_components(G, directed=False)
        inodes = np.flatnonzero(isI)
        comps = {}
        for p in inodes:                       # ascending node id
            comps.setdefault(lab[p], []).append(p)
        keyed = sorted(comps.values(),
                       key=lambda F: (self.pair[F[0], 0], self.pair[F[0], 1], F[0]))
        self.interfaces = [np.array(F, dtype=np.int64) for F in keyed]
        self.iface_pair = np.array([self.pair[F[0]] for F in self.interfaces],
                                   dtype=np.int64).reshape(-1, 2)
        self.node_iface = -np.ones(n, np.int64)
        for c, F in enumerate(self.interfaces):
            self.node_iface[F] = c

        # grain-interior node sets I_g (class G or D, owner g), ascending (R18)
        self.grain_nodes = [np.flatnonzero((self.owner == g) & (cls != CLASS_I))
                            for g in range(self.n_grains)]

        # contact grids (R8): Chebyshev dilation by h of each interface
        lat = mesh.lat_id
        self.contact_h = int(contact_h)
        h = self.contact_h
        self.contact_nodes = []
        for F in self.interfaces:
            ijk = mesh.node_ijk[F]
            lo = np.maximum(ijk.min(0) - h, 0)
            hi = np.minimum(ijk.max(0) + h, np.array(lat.shape[::-1]) - 1)
            sub = lat[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
            cand = sub[sub >= 0]
            cand = cand[~D[cand]]
            cijk = mesh.node_ijk[cand]
            dist = np.abs(cijk[:, None, :] - ijk[None, :, :]).max(axis=2).min(axis=1)
            self.contact_nodes.append(np.sort(cand[dist <= h]))

    @property
    def n_interfaces(self):
        return len(self.interfaces)


def node_dofs(nodes: np.ndarray) -> np.ndarray:
    """DOFs 3*node + c of a node list (node-major, R3)."""
    nodes = np.asarray(nodes, dtype=np.int64)
    return (3 * nodes[:, None] + np.arange(3)[None, :]).ravel()
