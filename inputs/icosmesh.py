"""Quasi-uniform spherical Voronoi mesh: the dual of the icosahedral geodesic grid -- INPUT ONLY.

BASELINE config 3 ("dual of the icosahedral geodesic grid at subdivision level 8 (655,362 cells,
1,966,080 edges)").  Level-L subdivision of the icosahedron gives 10*4^L + 2 generators (cell
centres, 12 of them pentagons), 20*4^L triangles whose circumcentres are the Voronoi vertices,
and 30*4^L edges.  Geometry (great-circle lengths, spherical polygon and kite areas, tangent
normals, weightsOnEdge) comes from the generic TRiSK builder with the Sphere geometry.
"""
from __future__ import annotations

import numpy as np

from .trisk_mesh import Mesh, Sphere, build_trisk_mesh

EARTH_R = 6371.0e3


def icosahedron():
    p = (1.0 + np.sqrt(5.0)) / 2.0
    v = np.array([[-1, p, 0], [1, p, 0], [-1, -p, 0], [1, -p, 0], [0, -1, p], [0, 1, p], [0, -1, -p], [0, 1, -p],
                  [p, 0, -1], [p, 0, 1], [-p, 0, -1], [-p, 0, 1]], dtype=np.float64)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4], [11, 10, 2],
                  [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9], [4, 9, 5],
                  [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v, f


def subdivide(v, f, levels):
    """Split every triangle into 4 (edge midpoints pushed to the unit sphere), `levels` times."""
    for _ in range(levels):
        nv = v.shape[0]
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        e.sort(axis=1)
        key = e[:, 0] * nv + e[:, 1]
        uk, inv = np.unique(key, return_inverse=True)
        a, b = uk // nv, uk % nv
        mid = v[a] + v[b]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        nf = f.shape[0]
        m01 = nv + inv[:nf]
        m12 = nv + inv[nf:2 * nf]
        m20 = nv + inv[2 * nf:]
        f = np.concatenate([np.stack([f[:, 0], m01, m20], 1), np.stack([f[:, 1], m12, m01], 1),
                            np.stack([f[:, 2], m20, m12], 1), np.stack([m01, m12, m20], 1)])
        v = np.concatenate([v, mid])
    return v, f


def mesh_from_sphere_triangulation(v, f, radius: float = EARTH_R) -> Mesh:
    """TRiSK mesh of the Voronoi dual of a Delaunay triangulation of the unit sphere: generators
    v [n,3] (unit vectors), triangles f [m,3]; Voronoi vertices at the triangle circumcentres."""
    f = np.array(f, dtype=np.int64, copy=True)
    # orient every triangle counter-clockwise seen from outside
    nrm = np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]])
    flip = np.sum(nrm * v[f[:, 0]], axis=1) < 0
    f[flip] = f[flip][:, [0, 2, 1]]
    nC, nT = v.shape[0], f.shape[0]
    # circumcentres (Voronoi vertices) on the sphere
    cc = np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]])
    cc /= np.linalg.norm(cc, axis=1, keepdims=True)
    # records (cell c, next CCW neighbour a, following neighbour b, triangle t)
    rc = np.concatenate([f[:, 0], f[:, 1], f[:, 2]])
    ra = np.concatenate([f[:, 1], f[:, 2], f[:, 0]])
    rb = np.concatenate([f[:, 2], f[:, 0], f[:, 1]])
    rt = np.concatenate([np.arange(nT)] * 3)
    key = rc * nC + ra
    order = np.argsort(key)
    ks = key[order]
    deg = np.bincount(rc, minlength=nC)
    maxE = int(deg.max())
    nbrs = np.full((nC, maxE), -1, dtype=np.int64)
    verts = np.full((nC, maxE), -1, dtype=np.int64)
    # start each cell's walk at the neighbour of its first record; step to the next CCW neighbour
    first = np.full(nC, -1, dtype=np.int64)
    first[rc[::-1]] = ra[::-1]
    cur = first
    cells = np.arange(nC)
    for j in range(maxE):
        act = j < deg
        p = np.searchsorted(ks, cells[act] * nC + cur[act])
        rec = order[p]
        nbrs[act, j] = cur[act]
        verts[act, j] = rt[rec]                  # triangle (c, nbr_j, nbr_{j+1}): vertex between edges j, j+1
        nxt = cur.copy()
        nxt[act] = rb[rec]
        cur = nxt
    return build_trisk_mesh(nbrs, verts, deg.astype(np.int32), v * radius, cc * radius, Sphere(radius))


def build_icosahedral_mesh(level: int, radius: float = EARTH_R) -> Mesh:
    v, f = subdivide(*icosahedron(), level)
    return mesh_from_sphere_triangulation(v, f, radius)
