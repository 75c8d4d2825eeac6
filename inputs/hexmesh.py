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


def build_periodic_hex_mesh_fast(nx: int, ny: int, dc: float) -> Mesh:
    """Same periodic hex mesh, assembled directly from the lattice (fast at 16.8 M cells).

    Numbering: edge 3c+k joins c to its E (k=0), NE (k=1), NW (k=2) neighbour with c = c0, so n_e
    points at 0, 60, 120 degrees; vertex 2c is the 30-degree corner of c, 2c+1 the 90-degree one.
    Geometry uses the closed forms of the regular hexagon (A_i = sqrt3/2 dc^2, l_e = dc/sqrt3,
    d_e = dc, kite = A_v/3 = sqrt3/12 dc^2) and weightsOnEdge the same kite-fraction
    construction as trisk_mesh.build_trisk_mesh.  Pinned by the same tests (P7, P19).
    """
    nbrs, verts = hex_adjacency(nx, ny)
    nC = nx * ny
    nE, nV = 3 * nC, 2 * nC
    c = np.arange(nC, dtype=np.int64)
    E, NE, NW, W, SW, SE = (nbrs[:, k] for k in range(6))
    eoc = np.stack([3 * c, 3 * c + 1, 3 * c + 2, 3 * W, 3 * SW + 1, 3 * SE + 2], axis=1)
    coe = np.empty((nE, 2), dtype=np.int64)
    coe[:, 0] = np.repeat(c, 3)
    coe[0::3, 1] = E
    coe[1::3, 1] = NE
    coe[2::3, 1] = NW
    voe = np.empty((nE, 2), dtype=np.int64)
    voe[0::3] = np.stack([2 * SE + 1, 2 * c], axis=1)         # (v0, v1): v1 on the +t_e side
    voe[1::3] = np.stack([2 * c, 2 * c + 1], axis=1)
    voe[2::3] = np.stack([2 * c + 1, 2 * W], axis=1)
    cov = np.empty((nV, 3), dtype=np.int64)
    cov[0::2] = np.stack([c, E, NE], axis=1)                  # CCW around the 30-degree corner
    cov[1::2] = np.stack([c, NE, NW], axis=1)                 # CCW around the 90-degree corner
    eov = np.empty((nV, 3), dtype=np.int64)
    eov[0::2] = np.stack([3 * c, 3 * E + 2, 3 * c + 1], axis=1)
    eov[1::2] = np.stack([3 * c + 1, 3 * NW, 3 * c + 2], axis=1)
    A = SQ3 / 2.0 * dc * dc
    Av = SQ3 / 4.0 * dc * dc
    kite = Av / 3.0
    lv = dc / SQ3
    # weightsOnEdge: walk c0 from the edge's slot k and c1 from slot k+3 (all cells identical)
    maxE2 = 10
    eoeT = np.empty((maxE2, nE), dtype=np.int32)
    Wt = np.empty((nE, maxE2), dtype=np.float64)
    eocT = [np.ascontiguousarray(eoc[:, s]) for s in range(6)]
    for k in range(3):
        col = 0
        for cells, js, n_e in ((None, k, 1.0), (nbrs[:, k], k + 3, -1.0)):
            sumR = 0.0
            for m in range(1, 6):
                sumR = sumR + kite / A
                s = (js + m) % 6
                n_ep = 1.0 if s < 3 else -1.0
                eoeT[col, k::3] = eocT[s] if cells is None else eocT[s][cells]
                Wt[k::3, col] = n_e * n_ep * (0.5 - sumR) * lv / dc
                col += 1
    eoe = eoeT.T
    Lx, Ly = nx * dc, ny * dc * SQ3 / 2.0
    jj, ii = np.divmod(c, nx)
    xc = (ii + 0.5 * (jj & 1)) * dc
    yc = jj * (dc * SQ3 / 2.0)
    R = dc / SQ3
    xv = np.empty(nV)
    yv = np.empty(nV)
    xv[0::2] = np.mod(xc + 0.5 * dc, Lx)
    yv[0::2] = np.mod(yc + 0.5 * R, Ly)
    xv[1::2] = xc
    yv[1::2] = np.mod(yc + R, Ly)
    ang = np.deg2rad([0.0, 60.0, 120.0])
    nrm = np.zeros((nE, 3))
    nrm[:, 0] = np.tile(np.cos(ang), nC)
    nrm[:, 1] = np.tile(np.sin(ang), nC)
    ept = np.zeros((nE, 3))
    ept[:, 0] = np.mod(np.repeat(xc, 3) + 0.5 * dc * nrm[:, 0], Lx)
    ept[:, 1] = np.mod(np.repeat(yc, 3) + 0.5 * dc * nrm[:, 1], Ly)
    i32 = np.int32
    return Mesh(
        nCells=nC, nEdges=nE, nVertices=nV, maxEdges=6, maxEdges2=maxE2,
        nEdgesOnCell=np.full(nC, 6, dtype=i32), edgesOnCell=eoc.astype(i32), cellsOnCell=nbrs.astype(i32),
        verticesOnCell=verts.astype(i32), cellsOnEdge=coe.astype(i32), verticesOnEdge=voe.astype(i32),
        nEdgesOnEdge=np.full(nE, maxE2, dtype=i32), edgesOnEdge=eoe.astype(i32), weightsOnEdge=Wt,
        edgesOnVertex=eov.astype(i32), cellsOnVertex=cov.astype(i32),
        kiteAreasOnVertex=np.full((nV, 3), kite), areaCell=np.full(nC, A), areaTriangle=np.full(nV, Av),
        dvEdge=np.full(nE, lv), dcEdge=np.full(nE, float(dc)),
        xCell=xc, yCell=yc, zCell=np.zeros(nC), xVertex=xv, yVertex=yv, zVertex=np.zeros(nV),
        edgeNormal=nrm, edgePoint=ept, fVertex=np.zeros(nV), bottomDepth=np.ones(nC),
        kind="planar", Lx=Lx, Ly=Ly, radius=0.0,
    )
