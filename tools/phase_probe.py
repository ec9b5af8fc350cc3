"""Per-phase timing probe: python tools/phase_probe.py CONFIG [key=value ...]
keys: passes, newton, steps, warm.  Prints ms per phase per stage."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2007_00094_b200 import Solver  # noqa: E402
from paper_2007_00094_b200 import problems as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
kw = dict(a.split("=") for a in sys.argv[2:])
passes = int(kw.get("passes", 2))
newton = int(kw.get("newton", 2))
steps = int(kw.get("steps", 20))
warm = int(kw.get("warm", 20))
ps = P.make_config(cfg)
st = torch.cuda.Stream()
s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary, limiter_passes=passes, newton_steps=newton,
           stream=st.cuda_stream)
s.set_state(ps.U0)
for _ in range(warm):
    s.ssp_rk3_step_async()
s.sync()
s.enable_timers(True)
t0 = s.timers
for _ in range(steps):
    s.ssp_rk3_step_async()
s.sync()
t1 = s.timers
per = {k: (t1[k] - t0[k]) / (3 * steps) * 1e3 for k in t0}
tot = sum(per.values())
print(cfg, f"passes={passes} newton={newton}", " ".join(f"{k}={v:.3f}" for k, v in per.items()),
      f"total={tot:.3f} ms/stage -> {ps.matrices.n / (tot * 1e-3):.3e} node-upd/s")
