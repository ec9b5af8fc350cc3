"""Per-kernel DRAM bytes per launch from an `ncu --set full` report -> profiles/ncu_traffic.json.

python tools/ncu_traffic.py REPORT.ncu-rep CONFIG
Keys are the short kernel names (`k_edge_lim` = the first limiter pass, which
forms P; `k_edge_lim#2` = a later pass; repeated launches get `#2`, `#3`...)."""
import csv
import json
import os
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(r, name):
    i = hdr.index(name)
    return float(r[i].replace(",", "")) * scale.get(units[i], 1.0)


res = {}
for r in rows[2:]:
    full = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
    name = full.split("<")[0]
    targs = [a.strip() for a in full.split("<", 1)[1].rstrip(">").split(",")] if "<" in full else []
    if name == "k_edge_lim" and len(targs) > 1 and targs[1] == "0":
        name = "k_edge_lim#2"  # a later pass; the first pass (P) is `k_edge_lim`
    key, k = name, 2
    while key in res:
        key = f"{name}#{k}"
        k += 1
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    pct = lambda name: float(r[hdr.index(name)].replace(",", "")) / 100.0  # noqa: E731
    res[key] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
                "fp64_pipe_active": pct("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "warps_active": pct("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "duration_ns": float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
                * {"us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(units[hdr.index("gpu__time_duration.sum")], 1.0)}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
allres = json.load(open(path)) if os.path.exists(path) else {}
allres[cfg] = res
json.dump(allres, open(path, "w"), indent=1)
print(json.dumps(res, indent=1))
