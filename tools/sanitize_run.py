"""One small run per config for compute-sanitizer: python tools/sanitize_run.py CONFIG
(c1: the smoke case; c2s / c5s: small C2 / C5; group: 3 same-device ranks with overlap)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_00094_b200 import Solver  # noqa: E402
from paper_2007_00094_b200 import problems as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
ranks = 1
if cfg == "c1":
    ps = P.isentropic_vortex(32)
elif cfg == "c2s":
    ps = P.mach3_disc(20, seed=3)
elif cfg == "c5s":
    ps = P.periodic_fourier_box(12)
elif cfg == "group":
    ps = P.mach3_disc(20, seed=3)
    ranks = 3
else:
    raise SystemExit(f"unknown config {cfg}")
for uni in (0, 1):  # the general path and the identical-state shortcut variants
    s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary, ranks=ranks)
    s.set_uniform_shortcuts(uni)
    s.enable_graphs(False)  # every kernel launched directly (the sanitizer sees each one)
    s.set_state(ps.U0)
    for _ in range(2):
        s.ssp_rk3_step()
    s.euler_step()
    s.get_state()
    s.close()
print("ok", cfg)
