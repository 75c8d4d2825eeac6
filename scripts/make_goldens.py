"""Full-size, full-length oracle goldens for the GPU parity gate (north_star: "GPU FB-LTS
bit-faithful to the oracle within the stated tolerance on all five configs", SURVEY 8(c)
"after each config's stated step count").

Calls only ``inputs/`` (seeded case generation, no method arithmetic) and ``oracle/`` (the
literal numpy transcription of P:L302-787).  Nothing here touches the CUDA path.  For each
BASELINE config it runs the oracle for the config's stated number of coarse steps and writes
``tests/golden/full_<config>.json`` with

* an input fingerprint (sha256 of h0, u0, the fine mask and the mesh arrays the step reads, and
  dt): the GPU test regenerates the case on the GPU box and first checks that its inputs are the
  same bytes, so an input-generation difference can never pass for a parity failure;
* the sha256 of the final h and u (fp64, little endian, original mesh order): the GPU test
  asserts bit-for-bit equality (canonical arithmetic);
* strided samples of h and u (float.hex, exact) and the oracle's norms max|h|, max|h - H|,
  max|u|: the GPU test asserts the contract tolerance (1e-11, reading Q26) sample-wise on
  h, on eta = h - H and on u, independently of the hash;
* mass and absolute vorticity at t0 and at the end (oracle/diagnostics.py).

Usage: python scripts/make_goldens.py config2 [config3 config4 config5 ...]
Run times on one core (numpy): config1 ~10 s, config2 ~7 min, config3 ~10 min, config4 ~20 min
(incl. ~5 min of SCVT generation), config5 ~2 h and ~30 GB.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from inputs import configs                     # noqa: E402
from oracle import diagnostics as dg           # noqa: E402
from oracle import fbrk32, lts                 # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
N_SAMPLES = 2000                               # per field; stride = the next odd number >= n / N_SAMPLES

MESH_FIELDS = ("nEdgesOnCell", "edgesOnCell", "cellsOnCell", "cellsOnEdge", "verticesOnEdge",
               "nEdgesOnEdge", "edgesOnEdge", "weightsOnEdge", "edgesOnVertex", "cellsOnVertex",
               "kiteAreasOnVertex", "areaCell", "areaTriangle", "dvEdge", "dcEdge", "fVertex",
               "bottomDepth")


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind == "f":
        a = a.astype("<f8", copy=False)
    elif a.dtype.kind in "iu":
        a = a.astype("<i8", copy=False)
    elif a.dtype.kind == "b":
        a = a.astype("u1", copy=False)
    return hashlib.sha256(a.tobytes()).hexdigest()


def input_fingerprint(c) -> dict:
    """sha256 per input array (shared test helper semantics; documented in tests/test_gpu_full.py)."""
    fp = {"h0": sha(c.h0), "u0": sha(c.u0), "fine_mask": sha(c.fine_mask), "tau_n": sha(c.tau_n)}
    for f in MESH_FIELDS:
        fp["mesh." + f] = sha(getattr(c.mesh, f))
    fp["dt"] = float(c.dt).hex()
    fp["M"] = int(c.M)
    return fp


def stride_of(n: int) -> int:
    s = max(1, -(-n // N_SAMPLES))
    return s if s % 2 else s + 1


def make_case(name: str):
    return {"config1": configs.config1, "config2": configs.config2, "config3": configs.config3,
            "config4": configs.config4, "config5": configs.config5}[name]()


def run_oracle(c, verbose=True):
    phys = fbrk32.Phys(g=c.g, beta=c.beta, slow=c.slow, tau_n=c.tau_n, rho0=c.rho0)
    h, u = c.h0.copy(), c.u0.copy()
    t0 = time.time()
    if not np.any(c.fine_mask):
        # no fine cells: global FB-RK(3,2) (the oracle's LTS reduces to it bitwise, pin P2)
        for n in range(c.n_steps):
            h, u = fbrk32.fbrk32_step(c.mesh, h, u, c.dt, phys)
            if verbose and (n + 1) % 10 == 0:
                print(f"  {c.name}: step {n + 1}/{c.n_steps}  {time.time() - t0:.0f} s", flush=True)
        return h, u, None
    lab = lts.label_regions(c.mesh, c.fine_mask)
    for n in range(c.n_steps):
        h, u = lts.fblts_step(c.mesh, lab, h, u, c.dt, c.M, phys)
        if verbose and ((n + 1) % 10 == 0 or c.mesh.nCells > 4_000_000):
            print(f"  {c.name}: step {n + 1}/{c.n_steps}  {time.time() - t0:.0f} s", flush=True)
    return h, u, lab


def main(names):
    os.makedirs(GOLDEN, exist_ok=True)
    for name in names:
        t0 = time.time()
        c = make_case(name)
        t_gen = time.time() - t0
        print(f"{name}: {c.mesh.nCells} cells, {c.mesh.nEdges} edges, M = {c.M}, {c.n_steps} steps, "
              f"dt = {c.dt!r}; generated in {t_gen:.0f} s", flush=True)
        fp = input_fingerprint(c)
        m0 = dg.total_mass(c.mesh, c.h0)
        g0 = dg.total_abs_vorticity(c.mesh, c.u0)
        t1 = time.time()
        h, u, lab = run_oracle(c)
        t_run = time.time() - t1
        assert np.all(np.isfinite(h)) and np.all(np.isfinite(u)), name
        sc, se = stride_of(c.mesh.nCells), stride_of(c.mesh.nEdges)
        ic, ie = np.arange(0, c.mesh.nCells, sc), np.arange(0, c.mesh.nEdges, se)
        out = {
            "what": "oracle final state after the config's stated coarse steps (scripts/make_goldens.py; "
                    "oracle/lts.py fblts_step P:L551-787, or oracle/fbrk32.py fbrk32_step P:L302-326 when "
                    "there are no fine cells)",
            "config": name, "seed": int(c.seed), "nCells": int(c.mesh.nCells), "nEdges": int(c.mesh.nEdges),
            "M": int(c.M), "n_steps": int(c.n_steps), "dt": float(c.dt).hex(),
            "n_fine": int(np.count_nonzero(c.fine_mask)),
            "inputs": fp,
            "h_sha256": sha(h), "u_sha256": sha(u),
            "max_abs_h": float(np.max(np.abs(h))).hex(),
            "max_abs_eta": float(np.max(np.abs(h - c.mesh.bottomDepth))).hex(),
            "max_abs_u": float(np.max(np.abs(u))).hex(),
            "cell_stride": int(sc), "edge_stride": int(se),
            "h_samples": [float(x).hex() for x in h[ic]],
            "u_samples": [float(x).hex() for x in u[ie]],
            "mass0": float(m0).hex(), "mass": float(dg.total_mass(c.mesh, h)).hex(),
            "gamma0": float(g0).hex(), "gamma": float(dg.total_abs_vorticity(c.mesh, u)).hex(),
            "oracle_seconds": round(t_run, 1),
        }
        if lab is not None:
            out["labels_sha256"] = {"cell": sha(lab.cell), "edge": sha(lab.edge)}
        path = os.path.join(GOLDEN, f"full_{name}.json")
        with open(path, "w") as f:
            json.dump(out, f, indent=0)
        print(f"{name}: wrote {path} (oracle {t_run:.0f} s, mass drift "
              f"{abs(dg.total_mass(c.mesh, h) - m0) / m0:.2e})", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["config1", "config2", "config3"])
