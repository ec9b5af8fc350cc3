import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
def num(x):
    try:
        return float(x)
    except Exception:
        return None
data = [r for r in rows[2:] if len(r) > si and num(r[si]) is not None]
tot = sum(num(r[si]) for r in data if len(r) > si)
top = sorted(((num(r[si]), i, r[1]) for i, r in enumerate(data) if len(r) > si), reverse=True)[:n]
print(f"total samples {tot:.0f} over {len(data)} SASS lines")
for v, i, src in top:
    print(f"{v/tot*100:5.1f}%  [{i:5d}] {src.strip()[:90]}")
