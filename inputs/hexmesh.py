"""Doubly periodic planar regular-hexagon Voronoi mesh -- INPUT GENERATION ONLY.

Stand-in for the paper's MPAS meshes (Table 1), as BASELINE.json
configs 1, 2 and 5 prescribe ("Doubly periodic planar regular-hexagon Voronoi
mesh"); the SPEC's ``build_periodic_hex_mesh`` is the interface.
Pointy-top cells in odd-r offset rows: cell (i, j) -> c = j*nx + i, centre
x = (i + (j mod 2)/2) dc, y = j dc sqrt(3)/2; L_x = nx dc, L_y = ny dc sqrt(3)/2
(ny must be even for periodicity).  Edge slots CCW: E, NE, NW, W, SW, SE.
"""
from __future__ import annotations

import numpy as np

from .trisk_mesh import Mesh, PlanarTorus, build_trisk_mesh

SQ3 = np.sqrt(3.0)


def hex_adjacency(nx: int, ny: int):
    """Return (cell_nbrs, cell_verts) for the odd-r periodic hex grid."""
    if nx < 4 or ny < 4 or ny % 2:
        raise ValueError("periodic hex mesh needs nx >= 4, ny >= 4 and ny even")
    jj, ii = np.divmod(np.arange(nx * ny, dtype=np.int64), nx)
    odd = (jj & 1).astype(np.int64)

    def cid(i, j):
        return (j % ny) * nx + (i % nx)

    E = cid(ii + 1, jj)
    NE = cid(ii + odd, jj + 1)
    NW = cid(ii - 1 + odd, jj + 1)
    W = cid(ii - 1, jj)
    SW = cid(ii - 1 + odd, jj - 1)
    SE = cid(ii + odd, jj - 1)
    nbrs = np.stack([E, NE, NW, W, SW, SE], axis=1)
    c = np.arange(nx * ny, dtype=np.int64)
    verts = np.stack([2 * c, 2 * c + 1, 2 * W, 2 * SW + 1, 2 * SW, 2 * SE + 1], axis=1)
    return nbrs, verts


def build_periodic_hex_mesh(nx: int, ny: int, dc: float) -> Mesh:
    """Periodic regular hex mesh with nx*ny cells, 3nx*ny edges, 2nx*ny vertices."""
    nbrs, verts = hex_adjacency(nx, ny)
    nC = nx * ny
    Lx, Ly = nx * dc, ny * dc * SQ3 / 2.0
    jj, ii = np.divmod(np.arange(nC, dtype=np.int64), nx)
    xc = (ii + 0.5 * (jj & 1)) * dc
    yc = jj * (dc * SQ3 / 2.0)
    cell_pos = np.stack([xc, yc, np.zeros(nC)], axis=1)
    R = dc / SQ3
    vpos = np.empty((2 * nC, 3))
    vpos[0::2, 0] = np.mod(xc + 0.5 * dc, Lx)
    vpos[0::2, 1] = np.mod(yc + 0.5 * R, Ly)
    vpos[1::2, 0] = xc
    vpos[1::2, 1] = np.mod(yc + R, Ly)
    vpos[:, 2] = 0.0
    n_on = np.full(nC, 6, dtype=np.int32)
    return build_trisk_mesh(nbrs, verts, n_on, cell_pos, vpos, PlanarTorus(Lx, Ly))
