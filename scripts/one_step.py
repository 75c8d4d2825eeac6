"""Development aid for ncu captures: build a config (default config5), set the state and run a few
coarse steps through the public API (no timing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs import configs  # noqa: E402
from paper_2405_10505_b200 import Solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if name.startswith("config5_"):                     # config5_<n>: n x n block of the config-5 recipe
    c = configs.config5(nx=int(name.split("_")[1]), ny=int(name.split("_")[1]))
else:
    c = getattr(configs, name)()
s = Solver(c.mesh, c.fine_mask, c.dt, c.M, g=c.g, beta=c.beta, rho0=c.rho0, tau_n=c.tau_n)
s.set_state(c.h0, c.u0)
s.step(n)
torch.cuda.synchronize()
print("diag", s.diagnostics())
