"""Run a few RK steps of a config for ncu capture: python tools/ncu_stage.py CONFIG STEPS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_00094_b200 import Solver  # noqa: E402
from paper_2007_00094_b200 import problems as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5m"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if cfg == "c5w":  # bench.py's default path: per-rank setup, one rank
    from paper_2007_00094_b200.distributed import ShardedSolver

    lp = P.periodic_fourier_box_local(320, 0, 1)
    s = ShardedSolver([lp.local])
    s.set_state(lp.U0)
else:
    ps = P.make_config(cfg)
    s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    s.set_state(ps.U0)
for _ in range(steps):
    s.ssp_rk3_step()
print("ok", cfg, steps, s.tau_last)
