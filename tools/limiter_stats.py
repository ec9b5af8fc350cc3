"""How often the limiter passes are trivial: fraction of real off-diagonal
slots with min(l) == 1 after pass 0 and after the last pass, over a run.
python tools/limiter_stats.py CONFIG STEPS [EVERY]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2007_00094_b200 import Solver  # noqa: E402
from paper_2007_00094_b200 import problems as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
every = int(sys.argv[3]) if len(sys.argv) > 3 else 50
ps = P.make_config(cfg)
s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
s.set_state(ps.U0)
for k in range(steps + 1):
    if k % every == 0:
        l0 = s.fetch("l_prev")
        l1 = s.fetch("l")
        d = s.fetch("d")
        real = (d > 0)  # off-diagonal real slots (d_ij > 0 unless both states coincide)
        print(f"step {k}: slots {real.sum()}, pass0 ml==1: {np.mean(l0[real] == 1.0):.4f}, "
              f"last ml==1: {np.mean(l1[real] == 1.0):.4f}, ml==0: {np.mean(l0[real] == 0.0):.4f}", flush=True)
    if k < steps:
        s.ssp_rk3_step()
