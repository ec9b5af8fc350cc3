"""One-rank NCCL check (the pool has one GPU): python -m torch.distributed.run --nnodes=1
--nproc-per-node 1 --master-addr 127.0.0.1 --master-port P tools/nccl1_check.py

Runs the NCCL transport of the library with a communicator of one rank -- unique id,
ncclCommInitRank, the tau allreduce(min) on every stage, CUDA-graph capture of steps that
contain NCCL calls, the collective set_state verdict and get_state's all_gather -- and
compares the result bit for bit with the single-process solver.  Peer send/recv needs a
second GPU and is covered only by the same-device group tests."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2007_00094_b200 import Solver  # noqa: E402
from paper_2007_00094_b200 import problems as P  # noqa: E402
from paper_2007_00094_b200.distributed import DistributedSolver, ShardedSolver  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
assert dist.get_world_size() == 1
steps = 4

# per-rank setup (bench.py's c5w path)
lp = P.periodic_fourier_box_local(24, 0, 1)
a = ShardedSolver(lp.local, c_cfl=lp.c_cfl, boundary=lp.boundary, nccl=True)
b = ShardedSolver([lp.local], c_cfl=lp.c_cfl, boundary=lp.boundary)
a.set_state(lp.U0)
b.set_state(lp.U0)
for _ in range(steps):
    a.ssp_rk3_step_async()
    b.ssp_rk3_step_async()
ta, tb = a.sync(), b.sync()
Ua, Ub = a.get_state(), b.get_state()
assert ta == tb and np.array_equal(Ua.view(np.int64), Ub.view(np.int64)), "ShardedSolver(nccl) != group"
ta, tb = a.ssp_rk3_step(), b.ssp_rk3_step()  # synchronous entry point
assert ta == tb and np.array_equal(a.get_state(), b.get_state())
a.close()
b.close()

# global setup (DistributedSolver: CM ranges, all_gather get_state)
ps = P.isentropic_vortex(32)
d = DistributedSolver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
d.set_state(ps.U0)
s.set_state(ps.U0)
for _ in range(steps):
    td, ts = d.ssp_rk3_step(), s.ssp_rk3_step()
    assert td == ts
assert np.array_equal(d.get_state().view(np.int64), s.get_state().view(np.int64)), "DistributedSolver != Solver"
bad = ps.U0.copy()
bad[5, 0] = -1.0
try:
    d.set_state(bad)
    raise SystemExit("inadmissible set_state accepted")
except Exception as exc:  # AdmissibilityError on every rank
    assert "admissib" in str(exc).lower() or "density" in str(exc).lower() or "state" in str(exc).lower(), exc
d.close()
s.close()
dist.destroy_process_group()
print("nccl1 ok")
