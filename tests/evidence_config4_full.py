"""BASELINE config 4 at full size on one GPU: build the variable-resolution SCVT (N from the
resolution spec, ~0.8 M cells, 50 Lloyd iterations -- about ten minutes of host time), compare one
FB-LTS coarse step (M = 8) with the oracle element by element, check conservation over the
config's 100 coarse steps on the GPU, and time the step.  Writes a JSON summary (argument 1,
default gpurun_out/config4_full.json).  Development/evidence script: calls inputs/, oracle/ and
the library through its Python binding.

usage: python tests/evidence_config4_full.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from inputs import configs                     # noqa: E402
from oracle import diagnostics as dg           # noqa: E402
from oracle import fbrk32, lts                 # noqa: E402


def main(out):
    import torch
    from paper_2405_10505_b200 import Solver
    t0 = time.time()
    c = configs.config4(verbose=True)
    m = c.mesh
    res = {"config": "config4", "cells": m.nCells, "edges": m.nEdges, "vertices": m.nVertices,
           "maxEdges": m.maxEdges, "fine_cells": int(np.count_nonzero(c.fine_mask)), "M": c.M, "dt": c.dt,
           "build_s": round(time.time() - t0, 1)}
    print(res, flush=True)
    lab = lts.label_regions(m, c.fine_mask)
    phys = fbrk32.Phys(g=c.g, beta=c.beta, slow=c.slow, tau_n=c.tau_n, rho0=c.rho0)
    t1 = time.time()
    ho, uo = lts.run(m, lab, c.h0, c.u0, c.dt, c.M, phys, 1)
    res["oracle_step_s"] = round(time.time() - t1, 1)
    s = Solver(m, c.fine_mask, c.dt, c.M, g=c.g, beta=c.beta, rho0=c.rho0, slow=c.slow, tau_n=c.tau_n)
    s.set_state(c.h0, c.u0)
    s.step(1)
    hg, ug, _ = s.state()
    res["eps_h"] = float(np.max(np.abs(hg - ho)) / np.max(np.abs(ho)))
    res["eps_u"] = float(np.max(np.abs(ug - uo)) / np.max(np.abs(uo)))
    res["bitwise"] = bool(np.array_equal(hg, ho) and np.array_equal(ug, uo))
    res["counts"] = s.counts()
    # conservation over the config's 100 coarse steps (from the initial state)
    s.set_state(c.h0, c.u0)
    d0 = s.diagnostics()
    s.step(c.n_steps)
    d1 = s.diagnostics()
    fscale = float(np.sum(m.areaTriangle * np.abs(m.fVertex)))
    res["mass_drift"] = abs(d1[0] - d0[0]) / d0[0]
    res["circulation_drift"] = abs(d1[1] - d0[1]) / fscale
    res["min_h"], res["max_nu"] = d1[2], d1[3]
    # timing (CUDA events on the launching stream)
    st = torch.cuda.current_stream()
    s.step(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.step(20)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res["ms_per_coarse_step"] = ms
    res["cell_updates_per_s"] = m.nCells * c.M / (ms * 1e-3)
    prof = s.profile(3)
    res["kernels_ms_per_step"] = {k: v[0] / 3 for k, v in prof.items() if v[1]}
    s.close()
    print(json.dumps(res, indent=1), flush=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    assert res["eps_h"] <= 1e-11 and res["eps_u"] <= 1e-11
    assert res["mass_drift"] <= 1e-13 and res["circulation_drift"] <= 1e-13


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/config4_full.json")
