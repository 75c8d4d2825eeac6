"""Development aid: time the public-API calls that make up bench.py's e2e number (set_state from
pinned host buffers, step, diagnostics, get_state) on a hex mesh of the config-5 recipe."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import configs  # noqa: E402
from paper_2405_10505_b200 import Solver  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
c = configs.shelf_case("config5", n, n, 500.0, 5, n_tiles=max(1, int(round(n * 500 / 256e3))), n_steps=50)
s = Solver(c.mesh, c.fine_mask, c.dt, c.M, tau_n=c.tau_n)
h = torch.from_numpy(np.ascontiguousarray(c.h0)).pin_memory()
u = torch.from_numpy(np.ascontiguousarray(c.u0)).pin_memory()
ho, uo = torch.empty_like(h).pin_memory(), torch.empty_like(u).pin_memory()
s.set_state(h, u)
s.step(3)
torch.cuda.synchronize()


def t(f, k=5):
    best = 1e9
    for _ in range(k):
        torch.cuda.synchronize()
        a = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - a)
    return best * 1e3


print(f"cells {c.mesh.nCells}: set_state {t(lambda: s.set_state(h, u)):.2f} ms, step {t(lambda: s.step(1)):.2f} ms, "
      f"diagnostics {t(lambda: s.diagnostics()):.3f} ms, get_state {t(lambda: s.state(ho.numpy(), uo.numpy())):.2f} ms, "
      f"state bytes {8 * (c.mesh.nCells + c.mesh.nEdges) / 1e6:.0f} MB")
