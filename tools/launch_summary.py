"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(list)
for d in data:
    if d["Metric Name"] == "gpu__time_duration.sum":
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name].append(float(d["Metric Value"].replace(",", "")) * (1e-3 if d["Metric Unit"] == "ns" else 1.0))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':36s} {'launches':>8s} {'mean us':>10s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:36s} {len(v):8d} {sum(v)/len(v):10.1f} {sum(v)/tot*100:6.1f}%")
