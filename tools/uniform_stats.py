"""Fraction of stencil edges whose two states are bitwise equal (U_i == U_j),
and of rows whose whole stencil is uniform, over a run:
python tools/uniform_stats.py CONFIG STEPS EVERY"""
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
M = ps.matrices
rows = np.repeat(np.arange(M.n), np.diff(M.indptr))
up = M.indices > rows
ri, rj = rows[up], M.indices[up]
s = Solver(M, c_cfl=ps.c_cfl, boundary=ps.boundary)
s.set_state(ps.U0)
for k in range(steps + 1):
    if k % every == 0:
        U = s.get_state()
        eq = np.all(U[ri] == U[rj], axis=1)
        bad = np.zeros(M.n, dtype=bool)
        np.logical_or.at(bad, ri, ~eq)
        np.logical_or.at(bad, rj, ~eq)
        print(f"{cfg} step {k}: edges U_i==U_j {eq.mean():.4f}, uniform stencils {1 - bad.mean():.4f}", flush=True)
    if k < steps:
        s.ssp_rk3_step()
