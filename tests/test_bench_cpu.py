"""bench.py's host-side pieces (no GPU): the weak-scaling sizes, the bounded
CPU samples, and the reference arm's JSON line (the CPU port of the stage)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_weak_scaling_sizes():
    # BASELINE.json configs[4]: 320^3 at 1 GPU up to 640^3 at 8 GPUs (~32.8M nodes per GPU)
    assert [bench.weak_side(n) for n in (1, 2, 4, 8)] == [320, 403, 508, 640]
    for n in (1, 2, 4, 8):
        assert abs(bench.weak_side(n) ** 3 / n / 320 ** 3 - 1.0) < 0.01


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "node-updates/s"
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["steps"] == 2 and line["warmup"] == 1
    assert line["metric"] == bench.METRIC and line["higher_is_better"] is True
