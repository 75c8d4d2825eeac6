#!/usr/bin/env python
"""bench.py -- throughput of the FB-LTS hot path on B200 (BASELINE.json metric:
"cell-updates/sec (fine-step equiv) and % of HBM roofline at 1/2/4/8 B200").

One step = one FB-LTS coarse step in split mode (all rows of SURVEY 8(a): slow terms, coarse
advancement, interface prediction, M fine subcycles with the interface accumulation, interface
correction) on the workload named in config.workload (default BASELINE config 5: 4096 x 4096
periodic hex, dc = 500 m, shelf bathymetry tiled 8x in x, M = 4).  value = N_cells * M * K / T
summed over ranks, T the max over ranks of the CUDA-event time of K steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference] [--config config5]

--impl reference times the ORACLE (oracle/, plain numpy fp64) on the host cores, on a bounded
sample of the same workload (this tier's reference arm).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "cell-updates/sec (fine-step equiv) and % of HBM roofline at 1/2/4/8 B200"
UNIT = "cell-updates/s"


# ------------------------------------------------------------------ workloads
def make_case(name, rank=0):
    from inputs import configs
    if name == "config5":
        return configs.config5()
    if name == "config2":
        return configs.config2()
    if name == "config1":
        return configs.config1()
    if name == "config3":
        return configs.config3()
    if name == "config4":
        return configs.config4()                         # ~10 min of host mesh generation (50 Lloyd iterations)
    if name.startswith("config4_"):                      # config4_<k>: the recipe at dx_scale = k
        return configs.config4(dx_scale=float(name.split("_")[1]))
    if name.startswith("config5_"):                      # config5_<n>: n x n block of the config-5 recipe
        n = int(name.split("_")[1])
        return configs.config5(nx=n, ny=n)
    raise SystemExit(f"unknown workload {name}")


def cpu_sample_case():
    """Bounded CPU sample of config 5: a 512 x 512 block of its recipe (one 256-km tile, dc = 500 m)."""
    from inputs import configs
    c = configs.config5(nx=512, ny=512)
    return c, "512x512 block of the config-5 recipe (one 256-km x-tile, dc = 500 m, M = 4)"


# ------------------------------------------------------------------ byte model
def byte_model(counts, M, fused, sub=0, maxE=6, maxE2=10):
    """Algorithmic bytes PER STEP of each kernel kind (the method's arrays, each element once per
    sweep; recomputable intermediates and padding not counted), summed over that kind's launches in
    one coarse step.  On a hex mesh the stage sweeps give SURVEY 8(d)'s 188 B/cell (s >= 2).
    `fused`: the deep fine velocity sweep of subcycle k-1 runs inside the deep stage-1 sweep of
    subcycle k (kind fine_vel_s1, k = 1..M-1); fine_s1 then holds the band stage 1 (every k) and the
    deep stage 1 of k = 0, fine_vel the band velocity sweeps and the last full one.
    `sub` (the fused-subcycle start level, 0 = off): the cells of F minus F^sub run whole subcycles in
    kind fine_sub (per launch: the subcycle's inputs h^{n,k}, [h^{n,k-1}, h2], z_b, A and the
    connectivity per cell, u, S, l_e, d_e per edge, once; writes h^{n,k+1}, h2 [+ its publishing
    copy] and [u^{n,k}]); the staged deep sweeps then stop at F^sub."""
    C, E = counts["owned_cells"], counts["owned_edges"]          # this rank's share
    V = counts["nVertices"] * C // max(1, counts["nCells"])
    cc, ec = counts["cells_by_region"], counts["edges_by_region"]
    cells = lambda lo, hi: sum(cc[lo:hi + 1])
    edges = lambda lo, hi: sum(ec[lo:hi + 1])
    slotC = 4 + 4 * maxE + 4 * maxE          # nEdgesOnCell + edgesOnCell + cellsOnCell
    cell_s1 = slotC + 8 + 8 + 8              # h_prev(=h^n), areaCell, write
    cell_s = slotC + 8 + 8 + 8 + 8 + 8       # h_prev, h_base, z_b, areaCell, write
    edge_s1 = 8 + 8                          # u, l_e
    edge_s = 8 + 8 + 8 + 8                   # u_base, S, l_e, d_e
    vel_e = 8 + 8 + 8 + 8 + 8                # cellsOnEdge, u_base, S, d_e, write
    vel_c = 8 * 4                            # h3, h2, h_base, z_b
    top = 8 if not sub else 2 + sub        # last region code of the staged fine sweeps (F^sub \ F^(sub-1))
    fs1 = lambda lo: cells(lo, top) * (slotC + 8 + 8 + 8) + edges(lo, top) * edge_s1
    fvel = lambda lo: edges(lo, 8) * vel_e + cells(lo, 8) * vel_c
    b = {}
    # per edge: cellsOnEdge, u, d_e, write F -- cellsOnEdge not read when F_e is formed in the vertex
    # role (DevMesh::vF, every mesh here; FBLTS_VF=0 turns it off)
    coe_b = 0 if os.environ.get("FBLTS_VF", "1") != "0" else 8
    b["slow_pre"] = V * (12 + 12 + 24 + 8 + 8) + C * (4 + 4 * maxE + 8 + 8) + E * (coe_b + 8 + 8 + 8)
    b["slow_edge"] = E * (4 + 4 * maxE2 + 8 * maxE2 + 8 + 8 + 8 + 8 + 8) + V * 8 + C * 8 + C * 8
    b["coarse_s1"] = cells(0, 7) * cell_s1 + edges(0, 7) * edge_s1
    b["coarse_s2"] = cells(0, 5) * cell_s + edges(0, 5) * edge_s
    b["coarse_s3"] = cells(0, 3) * cell_s + edges(0, 3) * edge_s
    # + u~^{n+1/2} (IF-2_E, IF-1_E) and u~^{n+1} (IF-1_E) for the fine stage-3 band sweeps (fine phases only)
    b["coarse_vel"] = edges(0, 0) * vel_e + cells(0, 1) * vel_c + (edges(1, 2) * vel_e + edges(2, 2) * 8 if fused else 0)
    b["fine_s2"] = M * (cells(3, top) * (slotC + 8 + 8 + 8 + 8 + 8 - 8) + edges(3, top) * edge_s)
    b["fine_s3"] = M * (cells(1, top) * (slotC + 8 + 8 + 8 + 8 + 8 - 8) + edges(1, top) * edge_s)
    if sub:
        cs_, es_ = cells(top + 1, 8), edges(top + 1, 8)
        k0 = cs_ * (slotC + 8 * 3 + 8 * 2) + es_ * edge_s                        # h, z_b, A; write h2, out
        k1 = cs_ * (slotC + 8 * 5 + 8 * 2 + 16) + es_ * (edge_s + 8)            # + h^{n,k-1}, h2, copy; write u
        b["fine_sub"] = k0 + (M - 1) * k1
    b["correct_if"] = cells(1, 2) * 24 + edges(1, 2) * 24
    # slow-term refresh (k = 1..M-1): views (cells IF..F write h, edges IF-1_E..F_E write u), the
    # restricted slow_pre (cells IF-1..F, edges IF-1_E..F_E, vertices ~2 per cell) and slow_edge on F_E
    Vf = 2 * cells(2, 8)
    b["slow_refresh"] = (M - 1) * (cells(1, 8) * 24 + edges(2, 8) * 40
                                   + Vf * 72 + cells(2, 8) * (4 + 4 * maxE + 16) + edges(2, 8) * 32
                                   + edges(3, 8) * (4 + 12 * maxE2 + 48))
    if fused:
        band_s1 = fs1(3) - fs1(4)
        band_vel = fvel(1) - fvel(4)
        b["fine_s1"] = M * band_s1 + fs1(4)
        b["fine_vel"] = (M - 1) * band_vel + fvel(1)
        # deep vel(k-1) + s1(k): cells row, h^{n,k}, h2, h^{n,k-1}, z_b, A, write h1; edges u, S, l, d, write u
        b["fine_vel_s1"] = (M - 1) * (cells(4, top) * (slotC + 8 * 6) + edges(4, top) * 40)
    else:
        b["fine_s1"] = M * fs1(3)
        b["fine_vel"] = M * fvel(1)
        b["fine_vel_s1"] = 0
    return b


def unsplit_byte_model(counts, M, maxE=6, maxE2=10):
    """Algorithmic bytes PER STEP of each kernel kind of the unsplit FB-LTS step (
    host.cu enqueue_unsplit_step), with the split model's per-entity costs:
    every velocity update is preceded by a slow sweep (slow_pre over the mesh -- or, for fine stages 1-2,
    over the F_E stencil -- and slow_edge over the update's edge range); the thickness sweeps read the
    stored stage velocity instead of recomputing it (cell row + h_prev, h_base, A, write; per edge U, l);
    the view kernels write the HS / U views of the stage's stencil (8 B per cell and per edge each way).
    The velocity update runs inside the slow edge sweep (VelFuse): + u_base, z_b, the write of u, - the
    store of S (16 B per edge); the coarse_vel / fine_vel kinds are then empty."""
    C, E = counts["owned_cells"], counts["owned_edges"]
    V = counts["nVertices"] * C // max(1, counts["nCells"])
    cc, ec = counts["cells_by_region"], counts["edges_by_region"]
    cells = lambda lo, hi: sum(cc[lo:hi + 1])
    edges = lambda lo, hi: sum(ec[lo:hi + 1])
    slotC = 4 + 4 * maxE + 4 * maxE
    coe_b = 0 if os.environ.get("FBLTS_VF", "1") != "0" else 8     # as in byte_model
    pre_full = V * (12 + 12 + 24 + 8 + 8) + C * (4 + 4 * maxE + 8 + 8) + E * (coe_b + 8 + 8 + 8)
    fstencil = cells(2, 8) / max(1, C)                              # F u IF-1 share of the mesh
    pre_fine = pre_full * fstencil
    edge_b = 4 + 4 * maxE2 + 8 * maxE2 + 8 * 5 + 8 * 2              # slow_edge per edge (+ q, K, h gathers)
    th = lambda n_c, n_e: n_c * (slotC + 8 * 4) + n_e * 16             # thickness sweep with stored U
    view = lambda n_c, n_e: (n_c + n_e) * 16
    b = {}
    yE = [edges(0, 6), edges(0, 4), edges(0, 2)]                       # Y1 = C_E u F^4_E, Y2, Y3
    xC = [cells(0, 7), cells(0, 5), cells(0, 3)]                       # X1 = C u F^5, X2, X3
    b["coarse_s1"], b["coarse_s2"], b["coarse_s3"] = (th(xC[q], yE[q]) for q in range(3))
    b["slow_pre"] = 3 * pre_full + M * (2 * pre_fine + pre_full)
    fE, ifE = edges(3, 8), edges(1, 8)
    b["slow_edge"] = (edge_b + 16) * (sum(yE) + M * (2 * fE + ifE))
    b["coarse_vel"] = 0
    b["fine_s1"] = M * (th(cells(3, 8), fE) + view(cells(1, 8), ifE))
    b["fine_s2"] = M * (th(cells(3, 8), fE) + view(cells(1, 8), ifE))
    b["fine_s3"] = M * (th(cells(1, 8), ifE) + view(cells(1, 8), ifE) + view(0, ifE))
    b["fine_vel"] = 0
    b["correct_if"] = cells(1, 2) * 24 + edges(1, 2) * 24
    return b


def _finite(x):
    """JSON-safe copy: NaN / inf -> null."""
    if isinstance(x, dict):
        return {k: _finite(v) for k, v in x.items()}
    if isinstance(x, (list, tuple)):
        return [_finite(v) for v in x]
    if isinstance(x, float) and not np.isfinite(x):
        return None
    return x


def scheme_dt(c, name, scheme):
    """0.9 x the Courant limit nu_loc of `scheme` ("global" FB-RK(3,2), "rk32", "rk4") bisected with the
    oracle on this config or its proxy (configs/dt.json "<config>_<scheme>", scripts/cfl_scan.py), applied
    to this mesh's max_e sqrt(g max H) / d_e; (None, why) if no scan is recorded."""
    try:
        with open(os.path.join(ROOT, "configs", "dt.json")) as f:
            ent = json.load(f)[f"{name}_{scheme}"]
        nu = float(ent["nu_loc_limit"])
    except (OSError, KeyError, ValueError):
        return None, f"no {name}_{scheme} entry in configs/dt.json"
    H = c.mesh.bottomDepth
    c0, c1 = c.mesh.cellsOnEdge[:, 0], c.mesh.cellsOnEdge[:, 1]
    cmax = float(np.max(np.sqrt(c.g * np.maximum(H[c0], H[c1])) / c.mesh.dcEdge))
    bound = " (lower bound: no unstable step found)" if ent.get("bound_only") or ent.get("unstable_dt") is None \
        or ent.get("unstable_dt") == ent.get("stable_dt") else ""
    return 0.9 * nu / cmax, f"0.9 x nu_loc {nu:.4f} (configs/dt.json {name}_{scheme}){bound}"


def host_cpu():
    model = "?"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic():
    """Per-launch DRAM bytes from the committed ncu --set full capture (profiles/), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_dram_bytes.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                rows.append((float(p[1]), float(p[2]), p[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        load = [r for r in rows if r[0] > 0.5 * r[1]] or rows
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[2]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


# ------------------------------------------------------------------ arms
def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def run_cpu_baseline(c, workload, steps=1, slow_refresh=False, split=True):
    """The oracle as it stands (oracle/lts.py, numpy fp64, single-threaded) on the SAME workload at full
    size: `steps` coarse steps after labelling (labelling excluded, as the GPU's setup is)."""
    from oracle import fbrk32, lts
    lab = lts.label_regions(c.mesh, c.fine_mask)
    phys = fbrk32.Phys(g=c.g, beta=c.beta, slow=c.slow, tau_n=c.tau_n, rho0=c.rho0)
    h, u = c.h0, c.u0
    t0 = time.perf_counter()
    for _ in range(steps):
        h, u = lts.fblts_step(c.mesh, lab, h, u, c.dt, c.M, phys, slow_refresh=slow_refresh, split=split)
    t = time.perf_counter() - t0
    return {"value": c.mesh.nCells * c.M * steps / t, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{workload} at full size ({c.mesh.nCells} cells, M = {c.M}): {steps} coarse step(s) of the "
                      "oracle (oracle/lts.py fblts_step), numpy single-threaded, labelling excluded",
            "seconds": t, "host_cpu": host_cpu()}


def arm_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from inputs import configs  # noqa: F401
    c, sample = cpu_sample_case()
    from oracle import fbrk32, lts
    lab = lts.label_regions(c.mesh, c.fine_mask)
    phys = fbrk32.Phys(g=c.g, beta=c.beta, slow=c.slow, tau_n=c.tau_n, rho0=c.rho0)
    h, u = c.h0, c.u0
    for _ in range(args.warmup):
        h, u = lts.fblts_step(c.mesh, lab, h, u, c.dt, c.M, phys)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        h, u = lts.fblts_step(c.mesh, lab, h, u, c.dt, c.M, phys)
    t = time.perf_counter() - t0
    value = c.mesh.nCells * c.M * args.steps / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config, "sample": sample, "M": c.M,
                                            "cells": c.mesh.nCells, "dt": c.dt},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def arm_native(args):
    import torch
    import torch.distributed as dist

    from paper_2405_10505_b200 import Solver
    from paper_2405_10505_b200 import _abi

    build_info = _abi.require_default_build()        # never time a probe / bounds-checked build
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # NCCL's init lines (ranks, transports) on stderr
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t_setup = time.perf_counter()
    weak = world > 1 and args.scaling == "weak" and args.config == "config5"
    piece = None
    if weak:
        # weak scaling (reading Q25): config 5 stacked N times in y, each rank generating, labelling and
        # partitioning ONLY its piece (its 4096 x 4096 block plus a 16-row margin), O(block) set-up
        from inputs import configs
        piece = configs.config5_weak_piece(rank, world)
        c = piece.case
    else:
        c = make_case(args.config, rank)
    nccl_id = None
    if world > 1:                    # partitioned run: the library's own NCCL communicator for the halos
        from paper_2405_10505_b200 import abi
        obj = [abi.fblts_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    s = Solver(c.mesh, c.fine_mask, c.dt, c.M, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow, tau_n=c.tau_n,
               rank=rank, nranks=world, nccl_id=nccl_id, slow_refresh=args.slow_refresh, unsplit=args.unsplit,
               partition=(piece.owner, piece.gid) if piece is not None else None)
    s.set_state(c.h0, c.u0, 0.0)
    counts = s.counts()
    t_setup = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        s.step(1)
    torch.cuda.synchronize()

    # ---------------- timed region (device, CUDA events on the launching stream)
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.step(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    s.sync()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    n_whole = len(piece.own) * world if piece is not None else c.mesh.nCells   # cells of the whole mesh
    units = n_whole * c.M * args.steps              # the whole mesh is advanced once per step (all ranks)
    value = units / (ms * 1e-3)

    # ---------------- instrumented replay: per-kernel device time (events on the same stream)
    n_prof = max(1, min(args.steps, 5))
    prof = s.profile(n_prof)
    fused = prof.get("fine_vel_s1", (0.0, 0))[1] > 0
    sub = 5 if prof.get("fine_sub", (0.0, 0))[1] > 0 else 0
    sub = int(os.environ.get("FBLTS_SUB_LEVEL", sub)) if sub else 0
    bm = byte_model(counts, c.M, fused, sub)                # bytes per step per kind
    if args.unsplit:                                        # the unsplit step's own sweep structure
        bm = {**{k: float("nan") for k in bm}, **unsplit_byte_model(counts, c.M)}
    t_step = {k: tms / n_prof for k, (tms, n) in prof.items() if n}
    dom = max(t_step, key=lambda k: t_step[k])
    launches_dom = prof[dom][1] / n_prof
    dom_ms = t_step[dom] / launches_dom                     # average launch duration
    peak, peak_src = load_peaks()
    achieved = bm[dom] / (t_step[dom] * 1e-3) / 1e9
    traffic = load_traffic().get(args.config, {}).get(dom)
    launches_per_step = s.counts()["kernels_per_step"]         # nodes of the captured step graph
    step_bytes = sum(bm[k] for k in t_step)
    prof_total = sum(t_step.values())
    # the dominant stage sweep against SURVEY 8(d)'s flat 188 B per cell-update (s >= 2) as well: cells
    # per launch = the sweep's extent (fine s3: IF-2 u IF-1 u F, fine s2: F; the split step only)
    survey = None
    if dom in ("fine_s2", "fine_s3") and not args.unsplit and not args.slow_refresh:
        cc = counts["cells_by_region"]
        n_cells = sum(cc[1:]) if dom == "fine_s3" else sum(cc[3:])
        ach = n_cells * 188 / (dom_ms * 1e-3) / 1e9
        survey = {"bytes_per_cell": 188, "cells_per_launch": n_cells, "achieved": ach, "frac": ach / peak}

    # ---------------- end to end through the public API with HOST buffers
    e2e = None
    if not args.no_e2e:
        h_host = torch.from_numpy(np.ascontiguousarray(c.h0)).pin_memory()
        u_host = torch.from_numpy(np.ascontiguousarray(c.u0)).pin_memory()
        h_out = torch.empty_like(h_host).pin_memory()
        u_out = torch.empty_like(u_host).pin_memory()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        s.set_state(h_host, u_host, 0.0)                # H2D of the initial state (+ device permutation)
        records = []
        for _ in range(args.steps):
            s.step(1)
            # per-step result: total mass and min h (positivity) of the new state, reduced on the device
            # and copied to the host every step without stalling the step pipeline (read back by the
            # final synchronising call, inside the timed region), and the full run record (mass, Gamma,
            # min h, max nu) once at the end, as a model run reports its global statistics every N steps
            if world == 1:
                records.append(s.diagnostics_mass_async())
            else:
                records.append(s.diagnostics_mass())
        records.append(s.diagnostics())
        s.state(h_out.numpy(), u_out.numpy())            # D2H of the final state
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1)
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        state_bytes = 8 * (c.mesh.nCells + c.mesh.nEdges)
        e2e = {"value": units / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": state_bytes / args.steps,
               "d2h_bytes_per_step": 16 + (32 + state_bytes) / args.steps,
               "how": "set_state(pinned host h,u) + K x (step(1) + diagnostics_mass_async(): mass and min h "
                      "reduced and copied to the host every step, not stalling the next step) + diagnostics() "
                      "(mass, Gamma, min h, max nu; synchronises) + get_state(pinned host)"}
        assert all(np.all(np.isfinite(r)) for r in records)

    # ---------------- the paper's speedup framing (Tables 1 and 3) on one GPU:
    # the same mesh and state advanced by each reference scheme at ITS OWN stable step (0.9 x the Courant
    # limit bisected with the oracle, configs/dt.json "<config>_<scheme>") -- global FB-RK(3,2) (no LTS),
    # RK(3,2) (Wicker-Skamarock, unsplit) and classical RK4 (unsplit) -- and FB-LTS at its own coarse step;
    # speedup at equal simulated time = (ms per step / dt)_scheme / (ms per step / dt)_FB-LTS.
    schemes = None
    if world == 1 and not args.no_global and not args.unsplit and not args.slow_refresh:
        s.close()
        del s
        torch.cuda.empty_cache()
        lts_cost = ms_step / c.dt                      # device ms per simulated second
        schemes = {"fblts": {"dt": c.dt, "M": c.M, "ms_per_step": ms_step, "ms_per_sim_s": lts_cost,
                             "dt_source": "0.9 x nu_loc (configs/dt.json %s)" % args.config}}
        base = args.config
        for name, kw in (("global", {"scheme": "fblts"}), ("rk32", {"scheme": "rk32"}), ("rk4", {"scheme": "rk4"})):
            dtx, src = scheme_dt(c, base, name)
            if dtx is None:
                schemes[name] = {"skipped": src}
                continue
            sx = Solver(c.mesh, np.zeros(c.mesh.nCells, dtype=bool), dtx, 1, g=c.g, beta=c.beta, rho0=c.rho0,
                        slow=c.slow, tau_n=c.tau_n, **kw)
            sx.set_state(c.h0, c.u0, 0.0)
            sx.step(3)
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            sx.step(args.steps)
            g1.record(stream)
            torch.cuda.synchronize()
            sx.sync()
            tx = g0.elapsed_time(g1) / args.steps
            sx.close()
            del sx
            torch.cuda.empty_cache()
            schemes[name] = {"dt": dtx, "dt_source": src, "ms_per_step": tx, "ms_per_sim_s": tx / dtx,
                             "cell_updates_per_s": c.mesh.nCells / (tx * 1e-3),
                             "fblts_speedup_at_equal_simulated_time": (tx / dtx) / lts_cost}
        schemes["how"] = ("same mesh and initial state, K steps each, CUDA events on the launching stream; global = "
                          "FB-RK(3,2) with no fine cells (M = 1), rk32 / rk4 on the unsplit system; each at 0.9 x its "
                          "own oracle-bisected Courant limit (scripts/cfl_scan.py)")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(c, args.config, slow_refresh=args.slow_refresh, split=not args.unsplit)
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if (world == 1 or weak) else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "scaling_note": ("weak: config 5 stacked N times in y (4096 x 4096N cells), a 4096 x 4096 block per GPU; "
                         "each rank builds only its piece (fblts_set_partition)") if weak else
                        ("strong: the same config-5 mesh partitioned over N GPUs (dual-set SFC partition)"
                         if world > 1 else None),
        "config": {"workload": args.config + ("_weak" if weak else ""), "slow_refresh": bool(args.slow_refresh),
                   "unsplit": bool(args.unsplit),
                   "cells": n_whole, "cells_per_rank_piece": c.mesh.nCells if weak else None, "edges": c.mesh.nEdges,
                   "vertices": c.mesh.nVertices, "M": c.M, "dt": c.dt,
                   "cells_by_region": counts["cells_by_region"],
                   "l2": "inputs larger than L2 (no flush needed)" if c.mesh.nCells > 2_000_000 else
                         "working set may be L2-resident (no flush)",
                   "parallelism": "1 GPU" if world == 1 else
                   (f"{world} GPUs, one 4096 x 4096 row block each, NCCL halo exchange per stage" if weak else
                    f"{world} GPUs, dual-set SFC partition of one mesh, NCCL halo exchange per stage"),
                   "setup_s": round(t_setup, 1), "build": build_info},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "bytes_per_launch": bm[dom] / launches_dom,
                     "launch_ms": dom_ms, "share_of_step": t_step[dom] / prof_total, "peak_source": peak_src,
                     "step_achieved": step_bytes / (ms_step * 1e-3) / 1e9,
                     "step_frac": step_bytes / (ms_step * 1e-3) / 1e9 / peak, "survey_8d_model": survey},
        "kernels": {k: {"ms_per_launch": tms / n, "launches_per_step": n / n_prof, "ms_per_step": tms / n_prof,
                        "GBps": bm[k] / (tms / n_prof * 1e-3) / 1e9}
                    for k, (tms, n) in prof.items() if n},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(round(launches_per_step * args.steps)),
        "schemes": schemes,
        "clocks": clocks,
    }
    print(json.dumps(_finite(line)), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50,
                    help="timed coarse steps (default 50: BASELINE config 5's stated run length)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="config5")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1 on config5: weak (a 4096 x 4096 block per GPU, default) or strong (one 4096^2 mesh)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-global", action="store_true", help="skip the global FB-RK(3,2) comparison run")
    ap.add_argument("--unsplit", action="store_true",
                    help="unsplit FB-LTS (full Phi in every velocity update, P:L468-787; one GPU)")
    ap.add_argument("--slow-refresh", action="store_true",
                    help="the slow-term refresh variant (S re-evaluated at every fine level, P:L1427-1431)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        arm_reference(args)
    else:
        arm_native(args)


if __name__ == "__main__":
    main()
