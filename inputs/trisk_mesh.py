"""Generic TRiSK (Voronoi C-grid) mesh builder -- INPUT GENERATION ONLY.

This module builds the static mesh arrays that both the oracle (``oracle/``) and
the CUDA library (``paper_2405_10505_b200``) consume.  It holds none of the
method's arithmetic (no tendencies, no time stepping, no LTS logic): it only
turns a cell adjacency + geometry into the MPAS-style connectivity, lengths,
areas, kite areas and ``weightsOnEdge`` that a TRiSK mesh file carries.

Conventions (Fig. ``fig:trisk``):
  * ``cellsOnEdge[e] = (c0, c1)``; the fixed normal n_e points from c0 to c1, so
    n_{e,c0} = +1, n_{e,c1} = -1 (P:L961 defines n_{e,i} as the outward sign).
  * t_e = k x n_e; ``verticesOnEdge[e] = (v0, v1)`` with v1 on the +t_e
    side.
  * ``edgesOnCell``/``verticesOnCell``/``cellsOnCell`` are counter-clockwise;
    vertex slot j lies between edge slots j and j+1.
  * ``cellsOnVertex`` is counter-clockwise around the vertex, and
    ``edgesOnVertex[v][k]`` is the edge between ``cellsOnVertex[v][k]`` and
    ``cellsOnVertex[v][k+1]``; ``kiteAreasOnVertex`` is aligned with
    ``cellsOnVertex``.
  * ``areaCell`` = sum of the cell's kites, ``areaTriangle`` = sum of the
    vertex's kites, so the three domain sums agree to rounding.
  * ``weightsOnEdge`` (the flux-mapping operator M_e of P:L1057-1059, "defined
    in Ringler 2010"): MPAS normalisation F_perp_e = sum_j W_{e,j} F_{eoe_j},
    built by the kite-fraction construction
        W_{e,e'} = n_{e,i} n_{e',i} (1/2 - sum_v R_{i,v}) l_{e'} / d_e,
    R_{i,v} = kite_{v,i}/A_i, summing over the vertices of cell i passed when
    walking counter-clockwise from e to e' (the vertex right after e counted).
    ``edgesOnEdge`` lists c0's edges (CCW, starting after e) then c1's.  The
    oracle pins these weights (uniform-flow reconstruction, antisymmetry of
    l_e d_e W, PV consistency) rather than trusting this code.
"""
from __future__ import annotations

import dataclasses
import numpy as np

I32 = np.int32
F64 = np.float64


@dataclasses.dataclass
class Mesh:
    nCells: int
    nEdges: int
    nVertices: int
    maxEdges: int
    maxEdges2: int
    nEdgesOnCell: np.ndarray      # [nCells] int32
    edgesOnCell: np.ndarray       # [nCells, maxEdges] int32 (-1 padded)
    cellsOnCell: np.ndarray       # [nCells, maxEdges] int32 (-1 padded)
    verticesOnCell: np.ndarray    # [nCells, maxEdges] int32 (-1 padded)
    cellsOnEdge: np.ndarray       # [nEdges, 2] int32
    verticesOnEdge: np.ndarray    # [nEdges, 2] int32
    nEdgesOnEdge: np.ndarray      # [nEdges] int32
    edgesOnEdge: np.ndarray       # [nEdges, maxEdges2] int32 (-1 padded)
    weightsOnEdge: np.ndarray     # [nEdges, maxEdges2] f64 (0 padded)
    edgesOnVertex: np.ndarray     # [nVertices, 3] int32
    cellsOnVertex: np.ndarray     # [nVertices, 3] int32
    kiteAreasOnVertex: np.ndarray  # [nVertices, 3] f64
    areaCell: np.ndarray          # [nCells] f64
    areaTriangle: np.ndarray      # [nVertices] f64
    dvEdge: np.ndarray            # [nEdges] f64  (l_e, primal edge length)
    dcEdge: np.ndarray            # [nEdges] f64  (d_e, cell-centre distance)
    xCell: np.ndarray
    yCell: np.ndarray
    zCell: np.ndarray
    xVertex: np.ndarray
    yVertex: np.ndarray
    zVertex: np.ndarray
    edgeNormal: np.ndarray        # [nEdges, 3] f64, unit n_e (tangent plane)
    edgePoint: np.ndarray         # [nEdges, 3] f64
    fVertex: np.ndarray           # [nVertices] f64 (set by the config)
    bottomDepth: np.ndarray       # [nCells] f64 H > 0, z_b = -H (set by the config)
    kind: str = "planar"          # "planar" | "sphere"
    Lx: float = 0.0
    Ly: float = 0.0
    radius: float = 0.0

    def arrays(self) -> dict:
        return {f.name: getattr(self, f.name) for f in dataclasses.fields(self)}


class PlanarTorus:
    """Doubly periodic plane [0,Lx) x [0,Ly); displacements by minimum image."""

    kind = "planar"

    def __init__(self, Lx: float, Ly: float):
        self.Lx, self.Ly = float(Lx), float(Ly)

    def disp(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        """Vector from a to b (shape [...,3]) under the minimum-image rule."""
        d = b - a
        d[..., 0] -= self.Lx * np.round(d[..., 0] / self.Lx)
        d[..., 1] -= self.Ly * np.round(d[..., 1] / self.Ly)
        return d

    def dist(self, a, b):
        d = self.disp(a, b)
        return np.sqrt(d[..., 0] ** 2 + d[..., 1] ** 2)

    def midpoint(self, a, b):
        return a + 0.5 * self.disp(a, b)

    def tri_area(self, a, b, c):
        """Unsigned area of the planar triangle (a,b,c), via displacements from a."""
        u = self.disp(a, b)
        v = self.disp(a, c)
        return 0.5 * np.abs(u[..., 0] * v[..., 1] - u[..., 1] * v[..., 0])

    def signed_tri_area(self, a, b, c):
        """Signed area, positive for counter-clockwise (a,b,c); equals tri_area for CCW triangles."""
        u = self.disp(a, b)
        v = self.disp(a, c)
        cr = u[..., 0] * v[..., 1] - u[..., 1] * v[..., 0]
        return np.where(cr >= 0, 0.5 * np.abs(cr), -(0.5 * np.abs(cr)))

    def tangent_dir(self, p, a, b):
        d = self.disp(a, b)
        return d / np.linalg.norm(d, axis=-1, keepdims=True)


class Sphere:
    """Sphere of radius R; points stored as 3-vectors of norm R."""

    kind = "sphere"

    def __init__(self, R: float):
        self.R = float(R)

    def _unit(self, a):
        return a / np.linalg.norm(a, axis=-1, keepdims=True)

    def dist(self, a, b):
        ua, ub = self._unit(a), self._unit(b)
        cr = np.linalg.norm(np.cross(ua, ub), axis=-1)
        dt = np.sum(ua * ub, axis=-1)
        return self.R * np.arctan2(cr, dt)

    def midpoint(self, a, b):
        return self.R * self._unit(self._unit(a) + self._unit(b))

    def tri_area(self, a, b, c):
        """Spherical triangle area (Eriksson 1990 / van Oosterom-Strackee)."""
        ua, ub, uc = self._unit(a), self._unit(b), self._unit(c)
        num = np.abs(np.sum(ua * np.cross(ub, uc), axis=-1))
        den = 1.0 + np.sum(ua * ub, axis=-1) + np.sum(ub * uc, axis=-1) + np.sum(uc * ua, axis=-1)
        return 2.0 * np.arctan2(num, den) * self.R ** 2

    def signed_tri_area(self, a, b, c):
        """Signed spherical area, positive for (a,b,c) counter-clockwise seen from outside; equals
        tri_area for such triangles."""
        ua, ub, uc = self._unit(a), self._unit(b), self._unit(c)
        trip = np.sum(ua * np.cross(ub, uc), axis=-1)
        area = self.tri_area(a, b, c)
        return np.where(trip >= 0, area, -area)

    def tangent_dir(self, p, a, b):
        """Unit tangent at point p pointing along the great circle from a to b."""
        up = self._unit(p)
        d = self._unit(b) - self._unit(a)
        d = d - np.sum(d * up, axis=-1, keepdims=True) * up
        return d / np.linalg.norm(d, axis=-1, keepdims=True)


def build_trisk_mesh(cell_nbrs: np.ndarray, cell_verts: np.ndarray, n_on_cell: np.ndarray,
                     cell_pos: np.ndarray, vert_pos: np.ndarray, geom) -> Mesh:
    """Assemble a TRiSK mesh from a CCW cell adjacency.

    cell_nbrs[c, j]  : neighbour across edge slot j (CCW), -1 padded
    cell_verts[c, j] : vertex between edge slots j and j+1, -1 padded
    n_on_cell[c]     : number of edges of cell c
    cell_pos, vert_pos : [n,3] coordinates (planar z = 0)
    """
    nC, maxE = cell_nbrs.shape
    n_on_cell = n_on_cell.astype(I32)
    nV = vert_pos.shape[0]
    slot = np.arange(maxE)[None, :]
    valid = slot < n_on_cell[:, None]

    # ---- edges: one per unordered neighbour pair, c0 = smaller index ----
    cc = np.repeat(np.arange(nC, dtype=np.int64)[:, None], maxE, axis=1)
    nb = cell_nbrs.astype(np.int64)
    own = valid & (cc < nb)
    c0 = cc[own]
    c1 = nb[own]
    nE = c0.size
    key_e = c0 * nC + c1                      # sorted already (row-major scan, c0 ascending, slot order)
    order = np.argsort(key_e, kind="stable")
    key_sorted = key_e[order]
    edge_ids = np.empty(nE, dtype=np.int64)
    edge_ids[order] = np.arange(nE)
    # map every (c, j) to its edge id
    lo = np.minimum(cc, nb)
    hi = np.maximum(cc, nb)
    key_all = np.where(valid, lo * nC + hi, -1)
    pos = np.searchsorted(key_sorted, key_all[valid])
    if not np.all(key_sorted[pos] == key_all[valid]):
        raise ValueError("neighbour relation is not symmetric")
    eoc = np.full((nC, maxE), -1, dtype=np.int64)
    eoc[valid] = order[pos]
    # edge numbering: follow the owner scan order (c0 ascending, then slot)
    # order[pos] gives the index in the 'own' scan -> that IS the edge id.
    edgesOnCell = eoc.astype(I32)
    cellsOnEdge = np.stack([c0, c1], axis=1).astype(I32)

    # slot of each edge inside c0 and c1
    e_slot = np.full((nE, 2), -1, dtype=np.int64)
    ci, sj = np.nonzero(valid)
    ev = eoc[ci, sj]
    is0 = cellsOnEdge[ev, 0] == ci
    e_slot[ev[is0], 0] = sj[is0]
    e_slot[ev[~is0], 1] = sj[~is0]
    assert np.all(e_slot >= 0)

    # ---- verticesOnEdge: walk CCW around c0: edge slot j goes from vertex j-1 to vertex j ----
    j0 = e_slot[:, 0]
    n0 = n_on_cell[c0]
    v_after = cell_verts[c0, j0]
    v_before = cell_verts[c0, (j0 - 1) % n0]
    verticesOnEdge = np.stack([v_before, v_after], axis=1).astype(I32)   # v1 on +t_e side

    # ---- geometry per edge ----
    pc0 = cell_pos[c0]
    pc1 = cell_pos[c1]
    dcEdge = geom.dist(pc0, pc1)
    dvEdge = geom.dist(vert_pos[verticesOnEdge[:, 0]], vert_pos[verticesOnEdge[:, 1]])
    edgePoint = geom.midpoint(pc0, pc1)
    edgeNormal = geom.tangent_dir(edgePoint, pc0, pc1)

    # ---- kites per (cell, vertex slot): quad (x_i, x_e(j), x_v(j), x_e(j+1)) ----
    kiteOnCell = np.zeros((nC, maxE), dtype=F64)
    for j in range(maxE):
        m = j < n_on_cell
        cidx = np.nonzero(m)[0]
        nj = n_on_cell[cidx]
        ea = eoc[cidx, j]
        eb = eoc[cidx, (j + 1) % nj]
        vv = cell_verts[cidx, j]
        xi = cell_pos[cidx]
        xa = edgePoint[ea]
        xb = edgePoint[eb]
        xv = vert_pos[vv]
        # signed (counter-clockwise positive) sub-triangles: where an obtuse Delaunay triangle puts
        # the vertex beyond the edge, one part is negative and the kites still tile the domain
        kiteOnCell[cidx, j] = geom.signed_tri_area(xi, xa, xv) + geom.signed_tri_area(xi, xv, xb)
    areaCell = np.zeros(nC, dtype=F64)
    for j in range(maxE):
        areaCell = areaCell + np.where(valid[:, j], kiteOnCell[:, j], 0.0)

    # ---- vertex records: each (c, j) contributes (v, c, nbr_j, nbr_{j+1}) ----
    rec_c = ci
    rec_j = sj
    rec_v = cell_verts[rec_c, rec_j].astype(np.int64)
    rec_n = n_on_cell[rec_c]
    rec_nb = cell_nbrs[rec_c, rec_j]                  # across edge j (toward v)
    rec_e = eoc[rec_c, rec_j]
    rec_k = kiteOnCell[rec_c, rec_j]
    # cellsOnVertex CCW: [c, nbr_j, nbr_{j+1}]; take the record with the smallest c as owner
    o = np.lexsort((rec_c, rec_v))
    rv = rec_v[o]
    first = np.ones(o.size, dtype=bool)
    first[1:] = rv[1:] != rv[:-1]
    counts = np.diff(np.append(np.nonzero(first)[0], o.size))
    if not np.all(counts == 3) or np.count_nonzero(first) != nV:
        raise ValueError("every vertex must be shared by exactly 3 cells")
    owner = o[first]                                  # record index per vertex (v ascending)
    cv0 = rec_c[owner]
    cv1 = rec_nb[owner]
    cv2 = cell_nbrs[cv0, (rec_j[owner] + 1) % rec_n[owner]]
    cellsOnVertex = np.stack([cv0, cv1, cv2], axis=1).astype(I32)
    # kites aligned with cellsOnVertex: lookup record (v, c)
    key_rec = rec_v * nC + rec_c
    ordk = np.argsort(key_rec)
    ks = key_rec[ordk]
    kiteAreasOnVertex = np.zeros((nV, 3), dtype=F64)
    vidx = np.arange(nV, dtype=np.int64)
    for k in range(3):
        kk = vidx * nC + cellsOnVertex[:, k]
        p = np.searchsorted(ks, kk)
        assert np.all(ks[p] == kk)
        kiteAreasOnVertex[:, k] = rec_k[ordk[p]]
    areaTriangle = (kiteAreasOnVertex[:, 0] + kiteAreasOnVertex[:, 1]) + kiteAreasOnVertex[:, 2]
    # edgesOnVertex[k] between cellsOnVertex[k] and cellsOnVertex[k+1]
    def edge_between(a, b):
        lo_, hi_ = np.minimum(a, b).astype(np.int64), np.maximum(a, b).astype(np.int64)
        kk = lo_ * nC + hi_
        p = np.searchsorted(key_sorted, kk)
        assert np.all(key_sorted[p] == kk)
        return order[p]
    edgesOnVertex = np.stack([edge_between(cellsOnVertex[:, 0], cellsOnVertex[:, 1]),
                              edge_between(cellsOnVertex[:, 1], cellsOnVertex[:, 2]),
                              edge_between(cellsOnVertex[:, 2], cellsOnVertex[:, 0])], axis=1).astype(I32)

    # ---- edgesOnEdge / weightsOnEdge (kite-fraction construction, MPAS normalisation) ----
    maxE2 = 2 * (maxE - 1)
    nEoE = (n_on_cell[c0] - 1) + (n_on_cell[c1] - 1)
    eoe = np.full((nE, maxE2), -1, dtype=np.int64)
    W = np.zeros((nE, maxE2), dtype=F64)
    eidx = np.arange(nE)
    base = np.zeros(nE, dtype=np.int64)
    for side in range(2):
        ci_ = cellsOnEdge[:, side].astype(np.int64)
        n_i = n_on_cell[ci_]
        je = e_slot[:, side]
        n_e_i = 1.0 if side == 0 else -1.0
        A_i = areaCell[ci_]
        sumR = np.zeros(nE, dtype=F64)
        for m in range(1, maxE):
            act = m < n_i
            if not np.any(act):
                break
            a = eidx[act]
            vslot = (je[a] + m - 1) % n_i[a]
            sumR[a] = sumR[a] + kiteOnCell[ci_[a], vslot] / A_i[a]
            s = (je[a] + m) % n_i[a]
            ep = eoc[ci_[a], s]
            n_ep_i = np.where(cellsOnEdge[ep, 0] == ci_[a], 1.0, -1.0)
            col = base[a] + (m - 1)
            eoe[a, col] = ep
            W[a, col] = n_e_i * n_ep_i * (0.5 - sumR[a]) * dvEdge[ep] / dcEdge[a]
        base = base + (n_i - 1)

    if geom.kind == "planar":
        Lx, Ly, R = geom.Lx, geom.Ly, 0.0
    else:
        Lx, Ly, R = 0.0, 0.0, geom.R
    return Mesh(
        nCells=nC, nEdges=nE, nVertices=nV, maxEdges=maxE, maxEdges2=maxE2,
        nEdgesOnCell=n_on_cell.astype(I32), edgesOnCell=edgesOnCell,
        cellsOnCell=np.where(valid, cell_nbrs, -1).astype(I32),
        verticesOnCell=np.where(valid, cell_verts, -1).astype(I32),
        cellsOnEdge=cellsOnEdge, verticesOnEdge=verticesOnEdge,
        nEdgesOnEdge=nEoE.astype(I32), edgesOnEdge=eoe.astype(I32), weightsOnEdge=W,
        edgesOnVertex=edgesOnVertex, cellsOnVertex=cellsOnVertex,
        kiteAreasOnVertex=kiteAreasOnVertex, areaCell=areaCell, areaTriangle=areaTriangle,
        dvEdge=dvEdge, dcEdge=dcEdge,
        xCell=cell_pos[:, 0].copy(), yCell=cell_pos[:, 1].copy(), zCell=cell_pos[:, 2].copy(),
        xVertex=vert_pos[:, 0].copy(), yVertex=vert_pos[:, 1].copy(), zVertex=vert_pos[:, 2].copy(),
        edgeNormal=edgeNormal, edgePoint=edgePoint,
        fVertex=np.zeros(nV, dtype=F64), bottomDepth=np.ones(nC, dtype=F64),
        kind=geom.kind, Lx=Lx, Ly=Ly, radius=R,
    )
