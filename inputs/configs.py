"""Seeded synthetic workloads (BASELINE.json configs) -- INPUT GENERATION ONLY.

The paper measures on DelBay2km / DelBay125m with hurricane-Sandy forcing
(Table 1); those meshes and data are not available, so these
seeded synthetic inputs stand in for them.  Every recipe
follows SURVEY.md 8(d) and the readings Q19-Q28; nothing here computes any
part of the FB-LTS method (no tendencies, no labels, no stepping).  The random
numbers are drawn with ``numpy.random.default_rng(seed)``.
"""
from __future__ import annotations

import dataclasses
import json
import os
import types

import numpy as np

from .hexmesh import build_periodic_hex_mesh, build_periodic_hex_mesh_fast
from .icosmesh import EARTH_R, build_icosahedral_mesh
from .trisk_mesh import Mesh

G = 9.81              # reading Q28
F_PLANE = 1.0e-4      # f-plane configs 1, 2, 5
RHO0 = 1000.0         # reading Q19
TAU_X = 0.1           # N m^-2, reading Q19
OMEGA = 7.292115e-5   # s^-1, reading Q28 (f = 2 Omega sin(latitude) on the sphere)
BETA = (0.531, 0.531, 0.313)

_HERE = os.path.dirname(os.path.abspath(__file__))
DT_TABLE = os.path.join(os.path.dirname(_HERE), "configs", "dt.json")


def periodic_step(x, L, W, n_images=2):
    """Smooth periodic plateau: ~1 on [L/2, L), ~0 on [0, L/2) (reading Q20)."""
    s = np.zeros_like(x)
    for m in range(-n_images, n_images + 1):
        s += 0.5 * (np.tanh((x - L / 2 + m * L) / W) - np.tanh((x - L + m * L) / W))
    return s


def grf_periodic(nx, ny, dx, dy, corr_len, rng):
    """Zero-mean, unit-variance periodic Gaussian random field with Gaussian covariance.

    Spectral synthesis on the (row, column) lattice of the mesh (reading Q22).
    """
    kx = 2 * np.pi * np.fft.fftfreq(nx, d=dx)
    ky = 2 * np.pi * np.fft.fftfreq(ny, d=dy)
    k2 = ky[:, None] ** 2 + kx[None, :] ** 2
    amp = np.exp(-k2 * corr_len ** 2 / 8.0)          # sqrt of a Gaussian spectrum
    noise = rng.standard_normal((ny, nx))
    f = np.fft.ifft2(np.fft.fft2(noise) * amp).real
    f -= f.mean()
    f /= f.std()
    return f.reshape(-1)


def periodic_gaussians(mesh: Mesh, centres, amps, sigma, cutoff=10.0):
    """Sum of Gaussian bumps with 3x3 periodic images (reading Q23); terms beyond cutoff*sigma
    (< 2e-22 relative) are skipped by windowing the rows when cells are stored row by row."""
    eta = np.zeros(mesh.nCells)
    rows_sorted = bool(np.all(np.diff(mesh.yCell) >= 0))
    for (cx, cy), a in zip(centres, amps):
        for my in (-1, 0, 1):
            yc = cy + my * mesh.Ly
            if rows_sorted:
                lo = np.searchsorted(mesh.yCell, yc - cutoff * sigma, side="left")
                hi = np.searchsorted(mesh.yCell, yc + cutoff * sigma, side="right")
            else:
                lo, hi = 0, mesh.nCells
            if hi <= lo:
                continue
            x = mesh.xCell[lo:hi]
            dy = mesh.yCell[lo:hi] - yc
            for mx in (-1, 0, 1):
                dx = x - (cx + mx * mesh.Lx)
                eta[lo:hi] += a * np.exp(-(dx * dx + dy * dy) / (2.0 * sigma * sigma))
    return eta


@dataclasses.dataclass
class Case:
    name: str
    mesh: Mesh
    h0: np.ndarray
    u0: np.ndarray
    fine_mask: np.ndarray
    tau_n: np.ndarray
    M: int
    dt: float
    n_steps: int
    g: float = G
    rho0: float = RHO0
    beta: tuple = BETA
    slow: bool = True
    seed: int = 0
    r: int = 2


def load_dt(name, default):
    try:
        with open(DT_TABLE) as f:
            return float(json.load(f)[name]["dt"])
    except (OSError, KeyError, ValueError):
        return default


def lattice_positions(nx, ny, dc):
    """Cell centres of the odd-r periodic hex lattice, the formula of hexmesh.build_periodic_hex_mesh(_fast):
    (x, y) = ((i + (j mod 2)/2) dc, j dc sqrt(3)/2) for cell c = j nx + i."""
    c = np.arange(nx * ny, dtype=np.int64)
    jj, ii = np.divmod(c, nx)
    xc = (ii + 0.5 * (jj & 1)) * dc
    yc = jj * (dc * np.sqrt(3.0) / 2.0)
    return xc, yc, nx * dc, ny * dc * np.sqrt(3.0) / 2.0


def shelf_fields(xc, yc, Lx, Ly, nx, ny, dc, rng, *, n_tiles=1, H_lo=10.0, H_hi=4000.0, W=20e3, rough=0.05,
                 corr=20e3, fine_H=250.0, bumps_per_tile=8, sigma=40e3, amp=(0.5, 2.0)):
    """Bathymetry H, initial surface eta and the fine mask of the shelf recipe on the lattice cells
    (readings Q20-Q23); draws from rng in a fixed order (GRF, then the bumps)."""
    Lt = Lx / n_tiles
    S = periodic_step(np.mod(xc, Lt), Lt, W)
    H = H_lo + (H_hi - H_lo) * S
    if rough:
        xi = grf_periodic(nx, ny, dc, dc * np.sqrt(3) / 2, corr, rng)
        H = H * (1.0 + rough * xi)
    centres, amps = [], []
    for t in range(n_tiles):
        cx = rng.uniform(t * Lt, (t + 1) * Lt, bumps_per_tile)
        cy = rng.uniform(0, Ly, bumps_per_tile)
        centres += list(zip(cx, cy))
        amps += list(rng.uniform(amp[0], amp[1], bumps_per_tile))
    grid = types.SimpleNamespace(nCells=xc.size, xCell=xc, yCell=yc, Lx=Lx, Ly=Ly)
    eta = periodic_gaussians(grid, centres, amps, sigma)
    return H, eta, H > fine_H


def shelf_case(name, nx, ny, dc, seed, *, n_tiles=1, H_lo=10.0, H_hi=4000.0, W=20e3,
               rough=0.05, corr=20e3, fine_H=250.0, bumps_per_tile=8, sigma=40e3,
               amp=(0.5, 2.0), forcing=True, M=4, n_steps=200, dt=None, slow=True,
               builder="generic") -> Case:
    """Continental-shelf case (configs 2 and 5; reduced sizes for parity tests).

    H(x) = [H_lo + (H_hi - H_lo) S(x mod L_tile; W)] (1 + rough xi), xi a GRF
    (readings Q20-Q22); fine = H > fine_H (Q21); Gaussian bumps (Q23);
    tau = (0.1, 0) N m^-2 projected on n_e (Q19).
    """
    rng = np.random.default_rng(seed)
    mesh = (build_periodic_hex_mesh_fast if builder == "lattice" else build_periodic_hex_mesh)(nx, ny, dc)
    H, eta, fine = shelf_fields(mesh.xCell, mesh.yCell, mesh.Lx, mesh.Ly, nx, ny, dc, rng, n_tiles=n_tiles,
                                H_lo=H_lo, H_hi=H_hi, W=W, rough=rough, corr=corr, fine_H=fine_H,
                                bumps_per_tile=bumps_per_tile, sigma=sigma, amp=amp)
    mesh.bottomDepth = H
    mesh.fVertex = np.full(mesh.nVertices, F_PLANE)
    h0 = H + eta
    u0 = np.zeros(mesh.nEdges)
    tau_n = TAU_X * mesh.edgeNormal[:, 0] if forcing else np.zeros(mesh.nEdges)
    if dt is None:
        dt = load_dt(name, 0.5 * dc / np.sqrt(G * H_hi * 1.1))
    return Case(name=name, mesh=mesh, h0=h0, u0=u0, fine_mask=fine, tau_n=tau_n, M=M,
                dt=dt, n_steps=n_steps, seed=seed, slow=slow)


def config1(seed=1, dt=None, nx=32, ny=32) -> Case:
    """BASELINE config 1: 32x32 periodic hex, dc = 10 km, 100 m / 4000 m halves joined by a
    tanh ramp (reading Q20: W = 25 km), fine = H > 2000 m, M = 4, 1 m bump (sigma 40 km)."""
    rng = np.random.default_rng(seed)
    dc = 10e3
    mesh = build_periodic_hex_mesh(nx, ny, dc)
    H = 100.0 + 3900.0 * periodic_step(mesh.xCell, mesh.Lx, 25e3)
    mesh.bottomDepth = H
    mesh.fVertex = np.full(mesh.nVertices, F_PLANE)
    c = (rng.uniform(0, mesh.Lx), rng.uniform(0, mesh.Ly))
    h0 = H + periodic_gaussians(mesh, [c], [1.0], 40e3)
    if dt is None:
        dt = load_dt("config1", 80.0)
    return Case(name="config1", mesh=mesh, h0=h0, u0=np.zeros(mesh.nEdges), fine_mask=H > 2000.0,
                tau_n=np.zeros(mesh.nEdges), M=4, dt=dt, n_steps=100, seed=seed)


def config2(seed=2, dt=None) -> Case:
    """BASELINE config 2: 512x512, dc = 2 km, shelf + 5 % roughness, 8 bumps, forcing, 200 steps."""
    return shelf_case("config2", 512, 512, 2e3, seed, n_steps=200, dt=dt)


def config5(seed=5, dt=None, nx=4096, ny=4096) -> Case:
    """BASELINE config 5: 4096x4096, dc = 500 m, config 2's profile per 256-km x-tile (8 tiles)."""
    n_tiles = max(1, int(round(nx * 500.0 / 256e3)))
    return shelf_case("config5", nx, ny, 500.0, seed, n_tiles=n_tiles, n_steps=50, dt=dt, builder="lattice")


WEAK_MARGIN = 16     # rows of neighbouring blocks in a weak piece: >= 2 halo rings + 5r label rings + 4


@dataclasses.dataclass
class Piece:
    """Rank `rank`'s piece of the weak-scaled config 5 (reading Q25): the N x 1 stack in y of the
    config-5 block, 4096 x 4096N cells; the piece holds rows [r 4096 - m, (r+1) 4096 + m) of it as a
    closed y-periodic strip (the wrap joins the two far margin rows only).  owner / gid per piece cell
    (fblts_set_partition); block_cell maps a piece cell to its config-5 block cell, own its owned cells."""
    case: Case
    owner: np.ndarray
    gid: np.ndarray
    block_cell: np.ndarray
    own: np.ndarray


def config5_weak_piece(rank, nranks, seed=5, nx=4096, ny=4096, margin=WEAK_MARGIN, dt=None) -> Piece:
    """Weak scaling of config 5 (BASELINE "Weak/strong scaling at 1/2/4/8"; reading Q25: a 4096 x 4096
    block per GPU, composition preserved): the whole mesh is the config-5 block repeated nranks times in
    y -- every field periodic with the block, so each block evolves exactly as config 5 does on its own
    and rank r's owned rows must reproduce the one-GPU config-5 state bit for bit.  Each rank builds only
    its piece: the block's fields (the config-5 recipe and seed, drawn on the block's lattice) indexed by
    row, on a (ny + 2 margin)-row lattice mesh.  INPUT GENERATION ONLY."""
    if margin % 2 or margin < 14:
        raise ValueError("margin must be even (row parity) and >= 14")
    n_tiles = max(1, int(round(nx * 500.0 / 256e3)))
    xc, yc, Lx, Ly = lattice_positions(nx, ny, 500.0)
    H_b, eta_b, fine_b = shelf_fields(xc, yc, Lx, Ly, nx, ny, 500.0, np.random.default_rng(seed), n_tiles=n_tiles)
    nyp = ny + 2 * margin if nranks > 1 else ny
    mesh = build_periodic_hex_mesh_fast(nx, nyp, 500.0)
    j, i = np.divmod(np.arange(nx * nyp, dtype=np.int64), nx)
    grow = (rank * ny - (margin if nranks > 1 else 0) + j) % (ny * nranks)     # row in the whole mesh
    bcell = (grow % ny) * nx + i
    mesh.bottomDepth = H_b[bcell]
    mesh.fVertex = np.full(mesh.nVertices, F_PLANE)
    owner = (grow // ny).astype(np.int32)
    gid = grow * nx + i
    if dt is None:
        dt = load_dt("config5", 0.5 * 500.0 / np.sqrt(G * 4000.0 * 1.1))
    case = Case(name="config5_weak", mesh=mesh, h0=H_b[bcell] + eta_b[bcell], u0=np.zeros(mesh.nEdges),
                fine_mask=fine_b[bcell], tau_n=TAU_X * mesh.edgeNormal[:, 0], M=4, dt=dt, n_steps=50, seed=seed)
    return Piece(case=case, owner=owner, gid=gid, block_cell=bcell, own=np.nonzero(owner == rank)[0])


def small_shelf(seed=7, nx=48, ny=40, dc=2e3, **kw) -> Case:
    """Reduced shelf case for parity tests: config 2's recipe with every length scale (ramp width,
    roughness correlation length, bump width) shrunk by L_x / 1024 km so the regions keep their shape."""
    s = nx * dc / 1024e3
    kw.setdefault("n_steps", 100)
    kw.setdefault("W", 20e3 * s)
    kw.setdefault("corr", 20e3 * s)
    kw.setdefault("sigma", 40e3 * s)
    return shelf_case("small_shelf", nx, ny, dc, seed, **kw)


def config3(seed=3, dt=None, level=8, n_steps=500) -> Case:
    """BASELINE config 3: icosahedral level-8 dual on R = 6371 km, H = 4000 m, f = 2 Omega sin(phi),
    global FB-RK(3,2) (no fine cells), u = 0, 16 Gaussian bumps U[10, 100] m with a 300-km
    great-circle sigma (reading Q23), 500 steps.  dt: 0.9 x the oracle-bisected Courant limit
    nu_loc (configs/dt.json "config3", measured on a lower level of the same recipe) applied to
    this mesh's max sqrt(g H)/d_e."""
    rng = np.random.default_rng(seed)
    mesh = build_icosahedral_mesh(level)
    H = np.full(mesh.nCells, 4000.0)
    mesh.bottomDepth = H
    lat_v = np.arcsin(np.clip(mesh.zVertex / mesh.radius, -1.0, 1.0))
    mesh.fVertex = 2.0 * OMEGA * np.sin(lat_v)
    c = rng.standard_normal((16, 3))
    c /= np.linalg.norm(c, axis=1, keepdims=True)
    amps = rng.uniform(10.0, 100.0, 16)
    x = np.stack([mesh.xCell, mesh.yCell, mesh.zCell], axis=1) / mesh.radius
    eta = np.zeros(mesh.nCells)
    sigma = 300e3
    for k in range(16):
        d = mesh.radius * np.arccos(np.clip(x @ c[k], -1.0, 1.0))
        eta += amps[k] * np.exp(-(d * d) / (2.0 * sigma * sigma))
    if dt is None:
        try:
            with open(DT_TABLE) as f:
                nu = float(json.load(f)["config3"]["nu_loc_limit"])
        except (OSError, KeyError, ValueError):
            nu = 1.5767175 * 0.8
        cmax = np.max(np.sqrt(G * np.maximum(H[mesh.cellsOnEdge[:, 0]], H[mesh.cellsOnEdge[:, 1]])) / mesh.dcEdge)
        dt = 0.9 * nu / cmax
    return Case(name="config3", mesh=mesh, h0=H + eta, u0=np.zeros(mesh.nEdges),
                fine_mask=np.zeros(mesh.nCells, dtype=bool), tau_n=np.zeros(mesh.nEdges), M=1, dt=dt,
                n_steps=n_steps, seed=seed)


def config4(seed=4, dt=None, dx_scale=1.0, n_lloyd=50, M=8, n_steps=100, verbose=False) -> Case:
    """BASELINE config 4: variable-resolution spherical centroidal Voronoi mesh (inputs/scvt.py):
    seeded points, a fixed 50 Lloyd iterations under rho ~ dx^-4, dx = 30 km globally refined to
    2 km in a seeded disk of 500 km diameter (tanh transition, 150 km); N from the resolution spec
    (reading Q24, ~0.8 M cells).  Shelf bathymetry across the disk (Q24): along a seeded direction
    s through the disk centre H_shelf = 5 + 3995 (1 + tanh(s / 50 km)) / 2, blended to 4000 m
    outside the disk by w = (1 - tanh((d - 250 km) / 50 km)) / 2.  f = 2 Omega sin(phi) (Q28).  Fine
    region = cells whose target dx < 15 km (Q24), M = 8, r = 2.  u = 0, a 1 m Gaussian surge
    (sigma 50 km, great-circle) at a seeded point of the disk.  dt: 0.9 x the oracle-bisected
    Courant limit nu_loc (configs/dt.json "config4", measured on the dx_scale = 8 reduction of the
    same recipe) applied to this mesh's max_e sqrt(g max H) dt_e / d_e, with dt_e = dt / M on the
    edges touching a fine cell (the F_E rule, reading Q7).

    dx_scale multiplies the two resolutions (and the fine threshold) only: the disk, the
    transition and the shelf keep their size, so a reduced case has the same geometry with
    dx_scale^2 fewer background cells (dx_scale = 8: ~10 k cells, for the parity tests)."""
    from .scvt import Refinement, build_scvt
    rng = np.random.default_rng(seed)
    centre = rng.standard_normal(3)
    centre /= np.linalg.norm(centre)
    ref = Refinement(centre, dx_coarse=30e3 * dx_scale, dx_fine=2e3 * dx_scale, beta=250e3, alpha=150e3)
    mesh, _ = build_scvt(ref, rng, n_lloyd=n_lloyd, verbose=verbose)
    R = mesh.radius
    x = np.stack([mesh.xCell, mesh.yCell, mesh.zCell], axis=1) / R
    # shelf across the disk along a seeded tangent direction t at the centre
    t = np.cross(centre, rng.standard_normal(3))
    t /= np.linalg.norm(t)
    s = R * np.arcsin(np.clip(x @ t, -1.0, 1.0))
    H_shelf = 5.0 + 3995.0 * 0.5 * (1.0 + np.tanh(s / 50e3))
    d = ref.dist(x)
    w = 0.5 * (1.0 - np.tanh((d - ref.beta) / 50e3))      # 1 inside the disk, 0 outside (shelf scale)
    H = 4000.0 + (H_shelf - 4000.0) * w
    mesh.bottomDepth = H
    lat_v = np.arcsin(np.clip(mesh.zVertex / R, -1.0, 1.0))
    mesh.fVertex = 2.0 * OMEGA * np.sin(lat_v)
    fine = ref.dx(x) < 15e3 * dx_scale
    # surge centre: uniform in the disk (radius beta) around the disk centre
    a = rng.uniform(0.0, 2.0 * np.pi)
    rr = ref.beta * np.sqrt(rng.uniform(0.0, 1.0))
    e1 = np.cross(centre, t)
    pc = np.cos(rr / R) * centre + np.sin(rr / R) * (np.cos(a) * t + np.sin(a) * e1)
    ds = R * np.arccos(np.clip(x @ pc, -1.0, 1.0))
    eta = 1.0 * np.exp(-(ds * ds) / (2.0 * 50e3 * 50e3))
    if dt is None:
        try:
            with open(DT_TABLE) as f:
                nu = float(json.load(f)["config4"]["nu_loc_limit"])
        except (OSError, KeyError, ValueError):
            nu = 1.0
        c0, c1 = mesh.cellsOnEdge[:, 0], mesh.cellsOnEdge[:, 1]
        ce = np.sqrt(G * np.maximum(H[c0], H[c1])) / mesh.dcEdge
        ce = np.where(fine[c0] | fine[c1], ce / M, ce)
        dt = 0.9 * nu / np.max(ce)
    return Case(name="config4", mesh=mesh, h0=H + eta, u0=np.zeros(mesh.nEdges), fine_mask=fine,
                tau_n=np.zeros(mesh.nEdges), M=M, dt=dt, n_steps=n_steps, seed=seed)


CD_BOTTOM = 2.5e-3            # bottom-drag coefficient C_D (synthetic hurricane runs, N4)
CW_WIND = 1.225 / 1000.0 * 1.5e-3   # C_W = (rho_air / rho_0) C_d10 (constant-drag reading, N4)


def hurricane_wind(mesh, centre, vmax=40.0, rmax=40e3, alpha=0.5, inflow_deg=20.0):
    """Synthetic stationary hurricane wind u_W (no Sandy data): a Rankine-type
    vortex, azimuthal speed V(r) = vmax r / rmax inside rmax and vmax (rmax / r)^alpha outside,
    counter-clockwise (northern hemisphere), turned inward by inflow_deg.  Returns the per-edge
    normal and tangential components (u_W . n_e, u_W . t_e) at the edge points; planar periodic
    meshes use the minimum-image displacement from the centre.  INPUT GENERATION ONLY."""
    p = mesh.edgePoint[:, :2]
    d = p - np.asarray(centre)[None, :2]
    if mesh.kind == "planar":
        d[:, 0] -= mesh.Lx * np.round(d[:, 0] / mesh.Lx)
        d[:, 1] -= mesh.Ly * np.round(d[:, 1] / mesh.Ly)
    r = np.hypot(d[:, 0], d[:, 1])
    V = np.where(r < rmax, vmax * r / rmax, vmax * (rmax / np.maximum(r, 1e-9)) ** alpha)
    er = d / np.maximum(r, 1e-9)[:, None]
    eth = np.stack([-er[:, 1], er[:, 0]], axis=1)
    a = np.deg2rad(inflow_deg)
    w = V[:, None] * (np.cos(a) * eth - np.sin(a) * er)
    n = mesh.edgeNormal[:, :2]
    t = np.stack([-n[:, 1], n[:, 0]], axis=1)          # t_e = k x n_e
    return np.sum(w * n, axis=1), np.sum(w * t, axis=1)


def hurricane_case(seed=8, nx=64, ny=48, dt=25.0, sal=0.1, **kw) -> Case:
    """The reduced shelf case driven by a synthetic stationary hurricane over the shelf break:
    bottom drag C_D, wind C_W |u_W - u| (u_W - u) / h, SAL coefficient sal in the fast term
    (eq. hurricane_model / hurricane_fast_terms).  Case.hurricane holds the terms."""
    c = small_shelf(seed=seed, nx=nx, ny=ny, dt=dt, **kw)
    rng = np.random.default_rng(seed + 100)
    centre = (0.5 * c.mesh.Lx + rng.uniform(-0.1, 0.1) * c.mesh.Lx, rng.uniform(0.3, 0.7) * c.mesh.Ly)
    rmax = 0.06 * c.mesh.Lx
    uw_n, uw_t = hurricane_wind(c.mesh, centre, rmax=rmax)
    c.tau_n = np.zeros(c.mesh.nEdges)
    c.hurricane = {"sal": sal, "cd": CD_BOTTOM, "cw": CW_WIND, "uw_n": uw_n, "uw_t": uw_t}
    return c
