"""Executed warp instructions of one kernel per source line: joins the SASS rows of an
ncu --import-source report with the line table of the same kernel in the library
(nvdisasm -g): python tools/ncu_lines.py REP KERNEL_REGEX MANGLED_PREFIX [LIB] [N]"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, kern, mangled = sys.argv[1], sys.argv[2], sys.argv[3]
lib = sys.argv[4] if len(sys.argv) > 4 else "paper_2007_00094_b200/libef_b200.so"
n = int(sys.argv[5]) if len(sys.argv) > 5 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
seen, dyn = set(), []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] in seen:
        continue
    seen.add(r[0])
    try:
        dyn.append((r[col["Source"]].strip(), float(r[col["Instructions Executed"]])))
    except ValueError:
        pass
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.startswith("ef_kernels.") and f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.split("\n")
start = end = None
for i, l in enumerate(sass):
    if l.startswith(".text." + mangled):
        start = i
    elif start is not None and l.startswith("\t.section"):
        end = i
        break
cur, stat = None, []
for l in sass[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", l)
    if m:
        stat.append((cur, m.group(1).strip()))
print(f"dynamic rows {len(dyn)}, static instructions {len(stat)}")
assert len(dyn) == len(stat), "kernel mismatch"
tot = sum(v for _, v in dyn)
per = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for (src, v), (ln, ins) in zip(dyn, stat):
    per[ln] += v
    t = ins.split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[ln][op] += v
byfile = collections.Counter()
for k, v in per.items():
    byfile[k[0]] += v
print("total warp instructions", f"{tot:.4g}", {k: f"{v / tot * 100:.1f}%" for k, v in byfile.most_common(6)})
for k, v in per.most_common(n):
    print(f"{k[0]}:{k[1]:<5d} {v / tot * 100:5.2f}%  " + " ".join(f"{o}={x / tot * 100:.2f}" for o, x in ops[k].most_common(6)))
