"""Executed CALL sites (slow paths) and total instructions of a kernel in an ncu report:
python tools/ncu_calls.py REPORT KERNEL_REGEX"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
src = hdr.index("Source")


def num(x):
    try:
        return float(x)
    except Exception:
        return 0.0


data = [r for r in rows[2:] if len(r) > ie]
tot = sum(num(r[ie]) for r in data)
print(f"warp instructions executed: {tot:.4g} over {len(data)} SASS lines")
calls = [(num(r[ie]), k, r[src].strip()) for k, r in enumerate(data) if "CALL" in r[src]]
for v, k, s in sorted(calls, reverse=True)[:15]:
    print(f"{v:12.0f}  [{k:5d}] {s[:60]}")
ops = {}
for r in data:
    op = r[src].strip().split()[0] if r[src].strip() else ""
    if op.startswith("@"):
        op = r[src].strip().split()[1]
    op = op.split(".")[0]
    ops[op] = ops.get(op, 0) + num(r[ie])
print("top opcodes:", ", ".join(f"{k}={v / tot * 100:.1f}%" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:14]))
