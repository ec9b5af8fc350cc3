"""Executed-instruction and stall mix by opcode class of one kernel from an
ncu --import-source report: python tools/ncu_opmix.py REP KERNEL_REGEX"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(r, h):
    try:
        return float(r[col[h]])
    except Exception:
        return 0.0


seen = set()
ex = defaultdict(float)
st = defaultdict(lambda: defaultdict(float))
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] in seen:
        continue
    seen.add(r[0])
    op = r[col["Source"]].strip().split()[0] if r[col["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[col["Source"]].strip().split()[1]
    cls = op.split(".")[0]
    ex[cls] += num(r, "Instructions Executed")
    for h in stalls:
        st[cls][h] += num(r, h)
tot = sum(ex.values())
tots = sum(sum(v.values()) for v in st.values())
print(f"warp instructions executed {tot:.4g}; stall samples {tots:.4g}")
for cls, v in sorted(ex.items(), key=lambda kv: -kv[1])[:28]:
    s = st[cls]
    top = sorted(s.items(), key=lambda kv: -kv[1])[:3]
    print(f"{cls:10} {v / tot * 100:5.1f}% inst  {sum(s.values()) / tots * 100:5.1f}% samples  " +
          " ".join(f"{k[6:]}={x / tots * 100:.1f}" for k, x in top))
