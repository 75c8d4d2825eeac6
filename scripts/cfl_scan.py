"""Delta-t selection by bisection on the ORACLE (SURVEY 8(c) reading Q12; the paper's own procedure
"running the model at increasing time-steps until it becomes unstable").

Calls only inputs/ and oracle/; writes configs/dt.json.  Predicate: 300 coarse steps, unstable if
any value is non-finite or max|u| > 5 m/s.  Bracket [0.5, 1.0] x the step at which
nu_loc = nu_max of the scheme (FB-RK(3,2): 3.8621532/sqrt(6); RK(3,2): sqrt(3)/sqrt(6); RK4:
2 sqrt(2)/sqrt(6)); when the top of the bracket is still stable the bracket is widened (x 1.25, up to
8 times) until a step is unstable, then bisected; if no unstable step is ever found the entry records
unstable_dt = null and the scheme's dt is a lower bound.  The run uses dt = 0.9 x the largest stable
step found.

Schemes (suffix of the entry name): none = FB-LTS (frozen slow terms, the paper's split mode);
_refresh = FB-LTS with the slow-term refresh at every fine level; _global = global
FB-RK(3,2) (split, no fine cells, M = 1); _rk32 = global RK(3,2) (Wicker-Skamarock, unsplit,
P:L283-285); _rk4 = global classical RK4 (unsplit).

usage: python scripts/cfl_scan.py config1 [config2 config5 config5_rk4 ...]
"""
import fcntl
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from inputs import configs                      # noqa: E402
from oracle import diagnostics as dg            # noqa: E402
from oracle import fbrk32, lts                  # noqa: E402

NU_MAX_FBRK = 3.8621532 / np.sqrt(6.0)
NU_MAX_RK4 = 2.0 * np.sqrt(2.0) / np.sqrt(6.0)
NU_MAX_RK32 = np.sqrt(3.0) / np.sqrt(6.0)
SCHEMES = ("refresh", "global", "rk32", "rk4")
OUT = configs.DT_TABLE


def stable(case, lab, dt, steps=300, scheme="fblts"):
    phys = fbrk32.Phys(g=case.g, beta=case.beta, slow=case.slow, tau_n=case.tau_n, rho0=case.rho0)
    h, u = case.h0.copy(), case.u0.copy()
    with np.errstate(all="ignore"):
        for _ in range(steps):
            if scheme == "rk4":
                h, u = fbrk32.rk4_step(case.mesh, h, u, dt, phys)
            elif scheme == "rk32":
                h, u = fbrk32.rk32_step(case.mesh, h, u, dt, phys)
            elif scheme == "global":
                h, u = fbrk32.fbrk32_step(case.mesh, h, u, dt, phys)
            else:
                h, u = lts.fblts_step(case.mesh, lab, h, u, dt, case.M, phys, slow_refresh=scheme == "refresh")
            if not (np.all(np.isfinite(u)) and np.all(np.isfinite(h))) or np.max(np.abs(u)) > 5.0:
                return False
    return True


def scan(name, case, iters=6, scheme="fblts", widen=8):
    """scheme rk4 / rk32 / global: a global reference scheme (no fine cells, M = 1), bracket top at
    its own imaginary-axis limit in units of the hex gravity-wave Courant number."""
    if scheme in ("rk4", "rk32", "global"):
        case.fine_mask = np.zeros(case.mesh.nCells, dtype=bool)
        case.M = 1
    lab = lts.label_regions(case.mesh, case.fine_mask)
    nu1 = dg.rest_courant(case.mesh, lab, 1.0, case.M, case.g)
    nu_top = {"rk4": NU_MAX_RK4, "rk32": NU_MAX_RK32}.get(scheme, NU_MAX_FBRK)
    top = nu_top / nu1
    lo, hi = 0.5 * top, 1.0 * top
    t0 = time.time()
    if not stable(case, lab, lo, scheme=scheme):
        raise RuntimeError(f"{name}: unstable at the bracket bottom {lo:.3f} s")
    n_widen = 0
    while stable(case, lab, hi, scheme=scheme):        # widen until the top is unstable
        lo = hi
        if n_widen == widen:
            hi = None
            break
        hi *= 1.25
        n_widen += 1
        print(f"  {name}: stable at {lo:.3f} s, widening to {hi:.3f} s  ({time.time() - t0:.0f} s)", flush=True)
    if hi is not None:
        for _ in range(iters):
            mid = 0.5 * (lo + hi)
            if stable(case, lab, mid, scheme=scheme):
                lo = mid
            else:
                hi = mid
            print(f"  {name}: [{lo:.3f}, {hi:.3f}] s  ({time.time() - t0:.0f} s)", flush=True)
    dt = 0.9 * lo
    return {"dt": dt, "stable_dt": lo, "unstable_dt": hi, "nu_loc_limit": lo * nu1,
            "nu_loc_run": dt * nu1, "bracket_top_dt": top, "widened": n_widen,
            "bound_only": hi is None, "predicate": "300 steps, finite, max|u| <= 5",
            "M": case.M, "nCells": case.mesh.nCells, "scan_seconds": round(time.time() - t0)}


def main(names):
    for name in names:
        scheme, base = "fblts", name
        for sch in SCHEMES:
            if name.endswith("_" + sch):
                scheme, base = sch, name[:-len(sch) - 1]
        if base == "config1":
            case = configs.config1(dt=1.0)
        elif base == "config2":
            case = configs.config2(dt=1.0)
        elif base == "config3":
            # the level-5 dual (10,242 cells) of the config-3 recipe; the Courant limit nu_loc
            # is applied to the level-8 mesh by inputs.configs.config3
            case = configs.config3(level=5, dt=1.0)
        elif base == "config4_full":
            # the full config-4 mesh (N = 796,141): ~30 min of oracle time per 300-step trial
            case = configs.config4(dt=1.0)
        elif base == "config3_full":
            case = configs.config3(dt=1.0)
        elif base == "config4":
            # the dx_scale = 8 reduction of the config-4 recipe (~12 k cells, same disk, shelf and
            # M = 8); the Courant limit nu_loc is applied to the full mesh by inputs.configs.config4
            case = configs.config4(dx_scale=8, dt=1.0)
        elif base == "config5":
            # proxy: one 256-km tile of config 5 (same dc, profile, roughness recipe, M) in x,
            # 128 km in y; the full 4096^2 mesh is too large for 300 oracle steps per trial.
            # bump density kept: 8 bumps per 256 x 1773 km tile -> 1 bump on the 256 x 128 km proxy
            case = configs.shelf_case("config5_proxy", 512, 296, 500.0, 5, n_tiles=1, n_steps=50, dt=1.0,
                                      bumps_per_tile=1)
        else:
            raise SystemExit(f"unknown config {name}")
        res = scan(name, case, scheme=scheme)
        res["scheme"] = scheme
        if base == "config5":
            res["proxy"] = "512x296 cells (one 256-km x-tile, 128 km in y, dc = 500 m, 1 bump, seed 5)"
        print(name, res, flush=True)
        with open(OUT + ".lock", "w") as lk:            # several scans may run side by side
            fcntl.flock(lk, fcntl.LOCK_EX)
            table = json.load(open(OUT)) if os.path.exists(OUT) else {}
            table[name] = res
            with open(OUT, "w") as f:
                json.dump(table, f, indent=2, sort_keys=True)
                f.write("\n")


if __name__ == "__main__":
    main(sys.argv[1:] or ["config1"])
