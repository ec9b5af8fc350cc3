"""Hot path of one kernel from an ncu --import-source report: the SASS instructions that hold
at least THR of the kernel's stall samples, plus (optional 4th argument) every load / store on
the hot path, in program order: python tools/ncu_hot_lines.py REP KERNEL_REGEX [THR] [mem]"""
import csv
import re
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
seen, data = set(), []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] in seen:
        continue
    seen.add(r[0])
    try:
        data.append((r[col["Source"]].strip(), float(r[col["Instructions Executed"]]),
                     float(r[col["Warp Stall Sampling (All Samples)"]])))
    except ValueError:
        pass
entry = max(d[1] for d in data)
ts = sum(d[2] for d in data)
print(f"# {kern}: {len(data)} SASS instructions, {sum(d[1] for d in data):.4g} executed, {entry:.4g} warps")
print("# index  share of stall samples  executed / warps  instruction")
for idx, (s, n, st) in enumerate(data):
    op = re.sub(r"^@!?U?P\d+\s+", "", s).split()[0].split(".")[0]
    mem = len(sys.argv) > 4 and op in ("LDG", "STG", "LDGSTS", "LDS", "STL", "LDL") and n / entry > 0.5
    if st / ts >= thr or mem:
        print(f"{idx:5d}  {st / ts:6.3f}  {n / entry:5.2f}  {s[:96]}")
