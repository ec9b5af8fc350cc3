"""Benchmark: fp64 Q1 node-updates per second per SSP-RK3 stage (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5w|c5|c1|c2|c3|c3m|c4|c4m|c5m] [--impl ours|reference]

Workload (config.workload): BASELINE.json configs[4], the largest
single-GPU configuration, as its weak-scaling series `c5w`: the 3D periodic Q1
hex box n^3 with n = round(320 N^(1/3)) (320^3 = 32.8M nodes and 885M stencil
entries at N = 1; 403^3 / 508^3 / 640^3 at N = 2 / 4 / 8), seeded smooth
random state from 8 Fourier modes, synthetic (generated mesh; no dataset
exists).  Every N runs the same code path: per-rank setup (each rank builds
its x-slab of the box in the box's lexicographic node order, ShardedSolver).
`--config c5` runs the same 320^3 problem through the global-setup Solver in
the reference's Cuthill-McKee order (bit-identical to the reference's own
output at 64^3 x 50 steps, tests/test_gpu_stated.py).
A step is one SSP-RK3 step (3 forward-Euler stages) over the whole mesh.

value     device-resident throughput: N_nodes * 3 * K / (CUDA-event time of K
          RK steps on the launching stream), max over ranks; the library's
          default path (exact identical-state fast paths chosen per step; on
          C5 no state is ever bitwise identical to a neighbour's, so this is
          the general path).
general_path  the same metric over K/2 steps with those fast paths forced off.
e2e       the same metric through the public API with host buffers: every step
          set_state(pinned host U) -> ssp_rk3_step() -> get_state(pinned host U).
roofline  dominant kernel (per-phase CUDA-event timing pass on the general
          path): algorithmic bytes from the reference's traffic model
          (perf.py:47-89) / kernel time, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the CPU oracle (C restatement of the reference stage, all host
          threads) on a bounded sample of the same workload.
--impl reference  times that CPU port alone (the reference itself is pure
          Python and does not exist on the GPU box).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

METRIC = "fp64 Q1 node-updates/sec per SSP-RK3 stage"
UNIT = "node-updates/s"
CONFIG_NAMES = {
    "c5w": "C5 3D periodic Fourier box, weak scaling: round(320 N^(1/3))^3 nodes (~32.8M per GPU)",
    "c1": "C1 2D isentropic vortex 129x129, CFL 0.5",
    "c2": "C2 2D Mach-3 flow past a disc, ~1.24M Q1 nodes, shuffled ids + RCM",
    "c3": "C3 3D Sod box 512x128x128 (jittered)",
    "c4": "C4 3D Mach-3 flow past a cylinder, extruded O-grid 255x255 layers, 67M nodes (per-rank z-slabs; 8 GPUs)",
    "c4m": "C4-shaped 3D Mach-3 cylinder, extruded O-grid 100x50 (~2.1M nodes)",
    "c5": "C5 3D periodic Fourier box 320^3 (32.8M nodes)",
    "c3m": "C3-shaped 3D Sod box 256x64x64 (jittered, 1.05M nodes)",
    "c5m": "C5-shaped 3D periodic Fourier box 160^3 (4.1M nodes)",
}


def l2_note(ws_mb: float) -> str:
    if ws_mb > 126.0:
        return "no flush: per-step working set (~%.0f MB) > 126 MB L2" % ws_mb
    # only the small C1 case: its stages read what the previous stage wrote, so
    # an L2 flush between steps would not model the solver; reported as such
    return "no flush: per-step working set (~%.0f MB) fits in the 126 MB L2 (L2-resident)" % ws_mb


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th is not None:
            self.th.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


# above this size the CPU oracle (and the reference arm) time the same generator's
# mid-size instance: the port's per-rank arrays need ~3 KB/node of host memory
CPU_MAX_NODES = 5_000_000
# configs whose ranks are built from their own rows (no rank holds the global matrix)
PER_RANK = ("c5w", "c4")
FORCE_NCCL = os.environ.get("EF_BENCH_NCCL") == "1"
CPU_SAMPLE_OF = {"c3": "c3m", "c4": "c4m", "c5": "c5m"}


def weak_side(world: int) -> int:
    """C5 weak scaling (BASELINE configs[4]): 320^3 nodes per GPU."""
    return int(round(320 * world ** (1.0 / 3.0)))


def build_problem(name: str, world: int = 1):
    from paper_2007_00094_b200 import problems as P

    if name == "c5w":
        return P.periodic_fourier_box(weak_side(world))
    return P.make_config(name)


def cpu_info() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_rate(ps, budget_s: float, threads: int, max_steps: int = 1000):
    """Oracle (C port of the reference stage) throughput on a bounded sample."""
    import oracle as O

    o = O.OracleSolver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary, threads=threads)
    o.set_state(ps.U0)
    o.ssp_rk3_step()  # warm-up
    steps = 0
    t0 = time.perf_counter()
    while steps < max_steps:
        o.ssp_rk3_step()
        steps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return ps.matrices.n * 3 * steps / dt, steps, dt


def cpu_sample_problem(config: str):
    """The bounded CPU sample of a config: the same generator at a size the
    C port's host arrays (~3 KB/node) and a few minutes of CPU time allow."""
    from paper_2007_00094_b200 import problems as P

    if config in ("c5", "c5w", "c5m"):
        return "the c5 generator at 128^3 (periodic Fourier box)", P.periodic_fourier_box(128)
    name = CPU_SAMPLE_OF.get(config, config)
    return f"the {name} mesh", build_problem(name)


def run_reference(args, rank, world):
    """--impl reference: the CPU port of the reference stage (oracle/idp_oracle.c;
    the reference itself is pure Python and cannot travel to the GPU box) on all
    host threads, W warm-up + K timed SSP-RK3 steps of the bounded sample, each
    leg capped at ~2 minutes of wall time."""
    if rank != 0:
        return
    import oracle as O

    label, ps = cpu_sample_problem(args.config)
    threads = os.cpu_count() or 1
    o = O.OracleSolver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary, threads=threads)
    o.set_state(ps.U0)
    warm = 0
    t0 = time.perf_counter()
    while warm < args.warmup and time.perf_counter() - t0 < 60.0:
        o.ssp_rk3_step()
        warm += 1
    steps = 0
    t0 = time.perf_counter()
    while steps < max(1, args.steps):
        o.ssp_rk3_step()
        steps += 1
        if time.perf_counter() - t0 >= 120.0:
            break
    dt = time.perf_counter() - t0
    rate = ps.matrices.n * 3 * steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True,
        "scaling": "weak" if args.config == "c5w" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": CONFIG_NAMES[args.config], "nodes": int(ps.matrices.n),
                   "nnz": int(ps.matrices.nnz), "sample": label},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "cpu": cpu_info(),
                         "sample": f"{steps} SSP-RK3 steps of {label} ({ps.matrices.n} nodes) after {warm} "
                                   f"warm-up steps, oracle/idp_oracle.c, {threads} threads"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def kernel_launches() -> int:
    from paper_2007_00094_b200 import _lib

    return int(_lib.load().ef_kernel_launches())


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2007_00094_b200 import Solver
    from paper_2007_00094_b200.perf import KERNEL_OF_PHASE, PHASES, predict_traffic, stage_doubles_per_nnz

    dist = world > 1 or FORCE_NCCL  # (EF_BENCH_NCCL=1: the N > 1 code path with a one-rank communicator)
    torch.cuda.set_device(local_rank)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    if args.config in PER_RANK:
        # per-rank setup: each rank generates only its rows (an x-slab of the box in
        # its lexicographic order / a z-slab of the extruded O-grid) and its ghost
        # layer; NCCL halos for N > 1
        from paper_2007_00094_b200 import problems as P
        from paper_2007_00094_b200.distributed import ShardedSolver

        if args.config == "c5w":
            ps = P.periodic_fourier_box_local(weak_side(world), rank, world)
        else:
            ps = P.mach3_cylinder_local(255, 255, rank, world)
        solver = ShardedSolver(ps.local, c_cfl=ps.c_cfl, boundary=ps.boundary, device=local_rank,
                               stream=stream.cuda_stream, nccl=dist)
        n_nodes, dim = ps.local.n_global, ps.local.dim
        mat = None
    else:
        ps = build_problem(args.config, world)
        mat = ps.matrices
        if dist:  # one rank per GPU: contiguous CM ranges, NCCL halo exchange + tau allreduce
            from paper_2007_00094_b200.distributed import DistributedSolver

            solver = DistributedSolver(mat, c_cfl=ps.c_cfl, boundary=ps.boundary, device=local_rank,
                                       stream=stream.cuda_stream)
        else:
            solver = Solver(mat, c_cfl=ps.c_cfl, boundary=ps.boundary, device=local_rank,
                            stream=stream.cuda_stream)
        n_nodes = mat.n
        dim = mat.dim
    card = solver.standard_card
    nnz = solver.nnz_owned
    solver.set_state(ps.U0)
    for _ in range(args.warmup):
        solver.ssp_rk3_step_async()
    solver.sync()
    # the sync above re-decides the identical-state shortcut mode from the warm-up steps'
    # sample; two more untimed steps capture that mode's CUDA graph outside the timed region
    # (a capture costs ~10 ms: nothing on C5, half of C1's 100 timed steps)
    for _ in range(2):
        solver.ssp_rk3_step_async()
    solver.sync()
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = kernel_launches()
    vol0 = solver.comm.sync_volume
    e0.record(stream)
    for _ in range(args.steps):
        solver.ssp_rk3_step_async()
    e1.record(stream)
    launches = kernel_launches() - launches0
    halo_bytes = 8.0 * (solver.comm.sync_volume - vol0) / (3 * args.steps)  # received per stage, this rank
    torch.cuda.synchronize()
    if dist:
        torch.distributed.barrier()
    clocks = sampler.stop()
    solver.sync()  # raises on any latched error of the timed steps
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    node_updates = n_nodes * 3 * args.steps  # the whole mesh, split over the ranks
    value = node_updates / (ms * 1e-3)
    ms_per_step = ms / args.steps

    # the same metric with the identical-state shortcuts forced off:
    # how much of `value` comes from bitwise-uniform regions of the flow
    gsteps = max(1, args.steps // 2)
    solver.set_uniform_shortcuts(0)
    for _ in range(2):
        solver.ssp_rk3_step_async()
    solver.sync()
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(gsteps):
        solver.ssp_rk3_step_async()
    e1.record(stream)
    torch.cuda.synchronize()
    solver.sync()
    gms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([gms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        gms = float(t.item())
    general = {"value": n_nodes * 3 * gsteps / (gms * 1e-3), "steps": gsteps,
               "note": "identical-state shortcuts off (exact either way); P=0 limiter skips stay on"}

    # per-phase kernel times: events between the kernels of every stage, no host
    # syncs inside the pass (the library folds them in when the timers are read).
    # Timed on the general path (identical-state shortcuts off): the roofline
    # measures the kernels on the reference's full work -- with the shortcuts
    # on, the model's bytes are not all moved and its "achieved" GB/s would
    # overstate the memory system (C2 exceeds 100%)
    solver.set_uniform_shortcuts(0)
    solver.enable_timers(True)
    base = solver.timers
    tsteps = 5
    for _ in range(tsteps):
        solver.ssp_rk3_step_async()
    solver.sync()
    after = solver.timers
    solver.enable_timers(False)
    solver.set_uniform_shortcuts(-1)
    stages = 3 * tsteps
    per_launch = {k: (after[k] - base[k]) / stages for k in PHASES}
    passes = solver.limiter_passes
    if passes > 1:
        per_launch["step5"] /= (passes - 1)
    model = predict_traffic(dim, card)
    phase_bytes = {k: 8.0 * model[k] * nnz for k in PHASES}
    # dominant single kernel (step0 is fused into k_final; step5 is two kernels)
    dom = max((k for k in PHASES if k not in ("step0", "step5")), key=lambda k: per_launch[k])
    peak, peak_kind = peaks()
    achieved = phase_bytes[dom] / per_launch[dom] / 1e9
    stage_bytes = 8.0 * stage_doubles_per_nnz(dim, card, passes) * nnz
    stage_s = (ms * 1e-3) / (3 * args.steps)
    gstage_s = 1.0 / (general["value"] / n_nodes)  # seconds per stage
    traffic = None  # dram read + write bytes per launch from the committed ncu --set full capture
    prof = {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            allprof = json.load(fh)
            prof = (allprof.get(args.config) or allprof.get("c5" if args.config == "c5w" else args.config, {})
                    ).get(KERNEL_OF_PHASE[dom], {})
        traffic = prof.get("traffic_bytes")
    except Exception:
        traffic = None
    # Composite roof of the stage: per kernel the larger of its fp64-pipe busy time and its
    # DRAM bytes / peak, both from the committed ncu capture of this config, over the ncu
    # durations of the same capture (B200 issues 64 fp64 FMA per SM and clock, so the
    # arithmetic-heavy kernels of an exactly rounded fp64 scheme sit on that pipe, not on HBM)
    composite = None
    try:
        kp = allprof.get(args.config) or allprof.get("c5" if args.config == "c5w" else args.config, {})
        ks = {k: v for k, v in kp.items() if "#" not in k and v.get("duration_ns")}
        if ks:
            t_meas = sum(v["duration_ns"] * 1e-9 for v in ks.values())
            t_roof = sum(max(v["duration_ns"] * 1e-9 * v["fp64_pipe_active"], v["traffic_bytes"] / (peak * 1e9))
                         for v in ks.values())
            composite = {"frac": t_roof / t_meas, "roof_ms": t_roof * 1e3, "ncu_ms": t_meas * 1e3,
                         "dram_bytes": sum(v["traffic_bytes"] for v in ks.values()),
                         "source": "profiles/ncu_traffic.json (ncu --set full, one stage; not a live timing)"}
    except Exception:
        composite = None
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "kernel": KERNEL_OF_PHASE[dom], "phase": dom,
        "kernel_ms": per_launch[dom] * 1e3, "algorithmic_bytes_per_launch": phase_bytes[dom],
        "peak_kind": peak_kind,
        # co-limiter from the same ncu capture: the edge kernels are fp64-issue bound
        "fp64_pipe_active": prof.get("fp64_pipe_active"), "warps_active": prof.get("warps_active"),
        "phase_ms": {k: round(v * 1e3, 4) for k, v in per_launch.items()},
        "path": "general (identical-state shortcuts off; zero-P limiter skips and the 3D fast accept stay on)",
        "stage": {"algorithmic_bytes": stage_bytes, "achieved": stage_bytes / gstage_s / 1e9,
                  "frac": stage_bytes / gstage_s / 1e9 / peak, "timing": "general_path steps",
                  "doubles_per_nnz": stage_doubles_per_nnz(dim, card, passes),
                  # the same model bytes over the headline `value`'s own stage time
                  "frac_of_value": stage_bytes / stage_s / 1e9 / peak,
                  "composite_fp64_hbm": composite},
    }

    # e2e through the public API with pinned host buffers
    nv = dim + 2
    io_rows = ps.local.n_owned if args.config in PER_RANK else n_nodes  # a rank's state I/O
    host = torch.empty((io_rows, nv), dtype=torch.float64).pin_memory()
    Uh = host.numpy()
    solver.set_state(ps.U0)
    solver.get_state(out=Uh)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(e2e_steps):
        solver.set_state(Uh)
        solver.ssp_rk3_step()
        solver.get_state(out=Uh)
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    e2e_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": n_nodes * 3 * e2e_steps / (e2e_ms * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": int(io_rows * nv * 8), "d2h_bytes_per_step": int(io_rows * nv * 8),
           "steps": e2e_steps, "wall_s": wall}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if args.config == "c5w" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": CONFIG_NAMES[args.config], "nodes": int(n_nodes), "nnz_rank0": int(nnz),
                   "dim": dim, "pad_width": solver.pad_width, "standard_card": card,
                   "c_cfl": ps.c_cfl, "limiter_passes": passes, "newton_steps": solver.newton_steps,
                   "parallelism": (f"{'slab (per-rank setup)' if args.config in PER_RANK else 'cm-range'} "
                                   f"partition x{world}, NCCL halo" if world > 1 else "single"),
                   "ghost_fraction_rank0": (solver.n_local - solver.n_owned) / max(solver.n_owned, 1),
                   "halo_bytes_per_stage_rank0": halo_bytes,
                   "l2": l2_note(nnz * (4 + 1 + 8 * (2 * dim + 1 + 1 + passes)) / 1e6)},
        "roofline": roofline,
        "general_path": general,
        "e2e": e2e,
        "clocks": clocks,
        "gpu_launches": int(launches),
    }
    solver.close()
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        if n_nodes > CPU_MAX_NODES:  # the oracle's host memory: the same generator at a bounded size
            del ps, mat
            label, ps = cpu_sample_problem(args.config)
        else:
            label = f"the {args.config} mesh"
        rate, steps, dt = cpu_oracle_rate(ps, args.cpu_seconds, threads, max_steps=args.steps)
        # one host thread on a small instance of the same generator (the reference's
        # default Solver(workers=1), stepper.py:96)
        from paper_2007_00094_b200 import problems as P
        small = P.periodic_fourier_box(48) if args.config.startswith("c5") else build_problem(
            args.config if args.config == "c1" else "c1")
        rate1, steps1, _ = cpu_oracle_rate(small, 0.5 * args.cpu_seconds, 1, max_steps=args.steps)
        line["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": threads, "kind": "port", "cpu": cpu_info(),
            "sample": f"{steps} SSP-RK3 steps of {label} ({ps.matrices.n} nodes) after 1 warm-up step, "
                      f"oracle/idp_oracle.c (C restatement of the reference stage), {threads} threads",
            "workers_1": {"value": rate1, "cores": 1,
                          "sample": f"{steps1} SSP-RK3 steps, {small.matrices.n} nodes, 1 thread"}}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None, choices=sorted(CONFIG_NAMES),
                    help="default: c5w (C5 weak scaling, 320^3 per GPU)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config is None:
        args.config = "c5w"
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1 or FORCE_NCCL:
        import torch

        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1 or FORCE_NCCL:
            import torch

            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
