"""Solver: a thin object wrapper over the C ABI (marshalling + torch-owned device memory).

    s = Solver(mesh, fine_mask, dt=..., M=4)       # upload, label, reorder, bind workspace
    s.set_state(h0, u0)                            # host arrays, original order
    s.step(100)                                    # enqueued on torch's current stream
    h, u, t = s.state()                            # host arrays, original order
    mass, gamma, hmin, numax = s.diagnostics()

PyTorch supplies only the device workspace (one uint8 tensor), the stream and,
for several ranks, the process group; every step of the method runs in
libfblts.so's CUDA kernels.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _abi as abi


class Solver:
    def __init__(self, mesh, fine_mask, dt, M, *, g=9.81, beta=(0.531, 0.531, 0.313), rho0=1000.0, r=2,
                 slow=True, tau_n=None, device=None, stream=None, rank=0, nranks=1, nccl_id=None, scheme="fblts",
                 slow_refresh=False, hurricane=None, unsplit=False, pv="centered", vorticity=False,
                 partition=None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2405_10505_b200.Solver needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.nCells, self.nEdges, self.nVertices = int(mesh.nCells), int(mesh.nEdges), int(mesh.nVertices)
        self.ctx = abi.fblts_create(dt, M, g=g, beta=beta, rho0=rho0, r=r, slow=slow, device=self.device.index,
                                    stream=self.stream.cuda_stream, rank=rank, nranks=nranks, nccl_id=nccl_id,
                                    scheme=scheme, slow_refresh=slow_refresh,
                                    sal=(hurricane or {}).get("sal", 0.0), unsplit=unsplit, pv=pv,
                                    vorticity=vorticity)
        self.rank, self.nranks = rank, nranks
        try:
            abi.fblts_upload_mesh(self.ctx, mesh)
            if partition is not None:          # (owner, gid): `mesh` is this rank's piece (fblts_set_partition)
                abi.fblts_set_partition(self.ctx, partition[0], partition[1])
            abi.fblts_set_regions(self.ctx, fine_mask)
            nbytes = abi.fblts_workspace_size(self.ctx)
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            abi.fblts_bind_workspace(self.ctx, self.workspace.data_ptr(), nbytes)
            abi.fblts_set_forcing(self.ctx, tau_n)
            if hurricane is not None:       # dict(sal, cd, cw, uw_n, uw_t), inputs.configs.hurricane_case
                abi.fblts_set_hurricane(self.ctx, hurricane["uw_n"], hurricane["uw_t"], hurricane["cd"],
                                        hurricane["cw"])
        except Exception:
            abi.fblts_destroy(self.ctx)
            self.ctx = None
            raise
        self.dt, self.M = dt, M
        self._pending = []              # arrays filled by outstanding diagnostics_async calls

    # --- setup queries
    def labels(self):
        return abi.fblts_get_labels(self.ctx, self.nCells, self.nEdges)

    def counts(self):
        c = abi.fblts_get_counts(self.ctx)
        return {"nCells": int(c[0]), "nEdges": int(c[1]), "nVertices": int(c[2]),
                "cells_by_region": c[3:12].tolist(), "edges_by_region": c[12:21].tolist(),
                "owned_cells": int(c[21]), "owned_edges": int(c[22]), "kernels_per_step": int(c[23]),
                "tiles": int(c[24]), "tile_halo_cells": int(c[25]), "tile_edges": int(c[26]),
                "tile_smem_bytes": int(c[27]), "sub_tiles": int(c[28]), "sub_halo_cells": int(c[29]),
                "sub_foreign_edges": int(c[30]), "sub_smem_bytes": int(c[31])}

    # --- state and stepping
    def set_state(self, h, u, t=0.0):
        abi.fblts_set_state(self.ctx, h, u, t)

    def set_vorticity(self, eta):
        """Prognostic absolute vorticity per vertex (vorticity=True contexts; Theorem 2 companion)."""
        abi.fblts_set_vorticity(self.ctx, eta, self.nVertices)

    def vorticity(self):
        return abi.fblts_get_vorticity(self.ctx, self.nVertices)

    def set_forcing(self, tau_n):
        abi.fblts_set_forcing(self.ctx, tau_n)

    def step(self, n_coarse=1):
        abi.fblts_step(self.ctx, n_coarse)

    def sync(self):
        abi.fblts_sync(self.ctx)
        self._pending.clear()

    def state(self, h_out=None, u_out=None):
        h = np.empty(self.nCells) if h_out is None else h_out
        u = np.empty(self.nEdges) if u_out is None else u_out
        t = abi.fblts_get_state(self.ctx, h, u)
        self._pending.clear()
        return h, u, t

    def diagnostics(self):
        d = abi.fblts_diagnostics(self.ctx)
        self._pending.clear()
        return d

    def pv_volume(self):
        """sum_v A_v h_v q_v, the volume integral of PV (Remark rmk:volume_conservation_pv)."""
        return abi.fblts_diagnostics_pv(self.ctx)

    def diagnostics_mass(self):
        """(total mass, min h) of the current state: the cell part of diagnostics(), same bits."""
        return abi.fblts_diagnostics_mass(self.ctx)

    def diagnostics_mass_async(self):
        """(mass, min h) of the current state without synchronising: valid after the next sync() / state()."""
        out = np.full(2, np.nan)
        self._pending.append(out)
        abi.fblts_diagnostics_mass_async(self.ctx, out)
        return out

    def diagnostics_async(self):
        """(mass, Gamma, min h, max nu) of the current state, filled in without synchronising: the
        returned array holds the values after the next sync() / state() / diagnostics()."""
        out = np.full(4, np.nan)
        self._pending.append(out)
        abi.fblts_diagnostics_async(self.ctx, out)
        return out

    def profile(self, n_coarse):
        ms, cnt = abi.fblts_profile(self.ctx, n_coarse)
        return {abi.fblts_kernel_name(k): (float(ms[k]), int(cnt[k])) for k in range(abi.NUM_KERNELS)}

    def close(self):
        if self.ctx is not None:
            abi.fblts_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SolverGroup:
    """n partitions of one mesh driven together on ONE device (loopback halo exchange through
    device copies, fblts_step_group).  Exercises the partitioned multi-rank path -- dual-set
    partition, local numbering, halo lists, pack/unpack, per-rank diagnostics -- without NCCL."""

    def __init__(self, mesh, fine_mask, dt, M, nranks, **kw):
        self.solvers = [Solver(mesh, fine_mask, dt, M, rank=r, nranks=nranks, **kw) for r in range(nranks)]
        self.nCells, self.nEdges = int(mesh.nCells), int(mesh.nEdges)

    @classmethod
    def from_pieces(cls, pieces, dt, M, **kw):
        """Rank r's context from its own piece (inputs.configs.Piece: mesh, fine mask, owner, gid) --
        the distributed set-up of fblts_set_partition, exercised in one process.  State I/O per rank."""
        g = cls.__new__(cls)
        n = len(pieces)
        g.solvers = [Solver(p.case.mesh, p.case.fine_mask, dt, M, rank=r, nranks=n, partition=(p.owner, p.gid), **kw)
                     for r, p in enumerate(pieces)]
        g.nCells = g.nEdges = None
        return g

    def set_state(self, h, u, t=0.0):
        for s in self.solvers:
            s.set_state(h, u, t)

    def step(self, n_coarse=1):
        abi.fblts_step_group([s.ctx for s in self.solvers], n_coarse)

    def state(self):
        h, u = np.full(self.nCells, np.nan), np.full(self.nEdges, np.nan)
        t = None
        for s in self.solvers:
            t = abi.fblts_get_state(s.ctx, h, u)      # each rank fills its owned entries
        return h, u, t

    def diagnostics(self):
        return abi.fblts_diagnostics_group([s.ctx for s in self.solvers])

    def counts(self):
        return [s.counts() for s in self.solvers]

    def close(self):
        for s in self.solvers:
            s.close()
