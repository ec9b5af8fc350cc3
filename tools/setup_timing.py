"""Setup-time breakdown of a config: python tools/setup_timing.py CONFIG"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_00094_b200 import Solver  # noqa: E402
from paper_2007_00094_b200 import problems as P  # noqa: E402
from paper_2007_00094_b200.stepper import cm_permutation  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5m"
t0 = time.time()
ps = P.make_config(cfg)
t1 = time.time()
perm, _ = cm_permutation(ps.matrices)
t2 = time.time()
s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary, cm_perm=perm)
t3 = time.time()
s.set_state(ps.U0)
t4 = time.time()
s.ssp_rk3_step()
t5 = time.time()
print(f"{cfg}: n={ps.matrices.n} nnz={ps.matrices.nnz} problem={t1 - t0:.1f}s rcm={t2 - t1:.1f}s "
      f"create={t3 - t2:.1f}s set_state={t4 - t3:.1f}s first_step={t5 - t4:.2f}s")
