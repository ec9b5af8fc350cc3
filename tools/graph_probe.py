"""A/B of CUDA-graph step replay: node-updates/s/stage with graphs on and off,
for the async chain (device-resident) and the synchronous API (one tau
readback per step).  python tools/graph_probe.py [config ...]"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2007_00094_b200 import Solver  # noqa: E402
from paper_2007_00094_b200 import problems as P  # noqa: E402


def rate(s, n, steps, sync_api):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        if sync_api:
            s.ssp_rk3_step()
        else:
            s.ssp_rk3_step_async()
    s.sync()
    dt = time.perf_counter() - t0
    return n * 3 * steps / dt


def main():
    configs = sys.argv[1:] or ["c1", "c2"]
    out = {}
    for name in configs:
        ps = P.make_config(name)
        steps = 400 if name == "c1" else 100
        res = {}
        for graphs in (False, True):
            s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
            s.enable_graphs(graphs)
            s.set_state(ps.U0)
            for _ in range(5):
                s.ssp_rk3_step()
            for sync_api in (False, True):
                key = ("graphs" if graphs else "direct") + ("_sync" if sync_api else "_async")
                res[key] = max(rate(s, ps.matrices.n, steps, sync_api) for _ in range(3))
            s.close()
        out[name] = res
        print(json.dumps({name: res}), flush=True)


if __name__ == "__main__":
    main()
