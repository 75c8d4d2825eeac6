"""Quick device timing of the FB-LTS step on a config (development aid, not the bench)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import configs  # noqa: E402
from paper_2405_10505_b200 import Solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
t0 = time.time()
if name == "config2":
    c = configs.config2()
elif name == "config1":
    c = configs.config1()
elif name.startswith("hex"):
    n = int(name[3:])
    c = configs.shelf_case("config5", n, n, 500.0, 5, n_tiles=max(1, int(round(n * 500 / 256e3))), n_steps=50)
t1 = time.time()
s = Solver(c.mesh, c.fine_mask, c.dt, c.M, tau_n=c.tau_n)
t2 = time.time()
print(f"{name}: cells={c.mesh.nCells} gen={t1-t0:.1f}s setup={t2-t1:.1f}s dt={c.dt:.3f} counts={s.counts()}", flush=True)
s.set_state(c.h0, c.u0)
st = torch.cuda.current_stream()
s.step(3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
s.step(steps)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"{name}: {ms:.3f} ms/coarse step, {c.mesh.nCells * c.M / (ms * 1e-3):.3e} cell-updates/s (fine-step equiv)")
prof = s.profile(5)
tot = sum(v[0] for v in prof.values())
for k, (t, n) in prof.items():
    if n:
        print(f"  {k:12s} {t / 5:9.3f} ms/step  {n // 5:3d} launches/step  {100 * t / tot:5.1f}%")
print("diag", s.diagnostics())
