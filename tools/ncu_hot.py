"""Hottest SASS lines (stall samples) of one kernel with their neighbours:
python tools/ncu_hot.py REP KERNEL_REGEX [N] [CONTEXT]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 12
ctx = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
S = hdr.index("Warp Stall Sampling (All Samples)")


def f(x):
    try:
        return float(x)
    except Exception:
        return None


data, seen = [], set()
for r in rows[2:]:
    if len(r) > S and f(r[S]) is not None and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
tot = sum(f(r[S]) for r in data)
print(f"{len(data)} SASS lines, {tot:.0f} samples")
for v, k in sorted(((f(r[S]), k) for k, r in enumerate(data)), reverse=True)[:n]:
    for q in range(max(0, k - ctx), min(len(data), k + 1)):
        mark = ">" if q == k else " "
        print(f"{mark}{f(data[q][S]) / tot * 100:5.1f}% [{q:5d}] {data[q][1].strip()[:84]}")
    if ctx:
        print("-")
