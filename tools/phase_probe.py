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
uni = int(kw.get("uni", -1))  # 0: identical-state shortcuts forced off (bench.py's general path)
st = torch.cuda.Stream()
if cfg.startswith("c5w"):  # bench.py's default path: per-rank setup in lexicographic order, one rank (c5w160 = 160^3)
    from paper_2007_00094_b200.distributed import ShardedSolver

    lp = P.periodic_fourier_box_local(int(cfg[3:] or 320), 0, 1)
    s = ShardedSolver([lp.local], limiter_passes=passes, newton_steps=newton, stream=st.cuda_stream)
    s.set_state(lp.U0)
    n_nodes = s.n
else:
    ps = P.make_config(cfg)
    s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary, limiter_passes=passes, newton_steps=newton,
               stream=st.cuda_stream)
    s.set_state(ps.U0)
    n_nodes = ps.matrices.n
if uni >= 0:
    s.set_uniform_shortcuts(uni)
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
print(cfg, f"passes={passes} newton={newton} uni={uni}", " ".join(f"{k}={v:.3f}" for k, v in per.items()),
      f"total={tot:.3f} ms/stage -> {n_nodes / (tot * 1e-3):.3e} node-upd/s")
