"""Check the chosen coarse step on the FULL mesh of a config whose Courant limit was bisected on a
reduced proxy (reading Q12; configs 3 and 4): the oracle runs the scan's stability predicate (300
coarse steps, finite, max|u| <= 5 m/s) at the run's dt.  Calls only inputs/ and oracle/; records the
outcome in configs/dt.json under "<config>_full_check".

usage: python scripts/cfl_verify.py config3 | config4
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
from oracle import lts                          # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from cfl_scan import OUT, stable                # noqa: E402


def main(name):
    c = {"config3": configs.config3, "config4": configs.config4}[name]()
    lab = lts.label_regions(c.mesh, c.fine_mask)
    t0 = time.time()
    ok = stable(c, lab, c.dt, steps=300)
    res = {"dt": c.dt, "nCells": c.mesh.nCells, "M": c.M, "stable_300_steps": bool(ok),
           "nu_loc_run": dg.rest_courant(c.mesh, lab, c.dt, c.M, c.g), "seconds": round(time.time() - t0),
           "predicate": "300 steps, finite, max|u| <= 5 (oracle, full mesh)"}
    print(name, res, flush=True)
    with open(OUT + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        table = json.load(open(OUT))
        table[f"{name}_full_check"] = res
        with open(OUT, "w") as f:
            json.dump(table, f, indent=2, sort_keys=True)
            f.write("\n")


if __name__ == "__main__":
    main(sys.argv[1])
