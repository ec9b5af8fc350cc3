"""The NCCL transport with a one-rank communicator (tools/nccl1_check.py), launched as
bench.py's multi-GPU arm is launched: torch.distributed.run, one process per GPU."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_nccl_transport_one_rank():
    env = dict(os.environ)
    env.pop("EF_B200_LIB", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "tools", "nccl1_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0 and "nccl1 ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
