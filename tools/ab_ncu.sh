#!/bin/bash
# A/B of one kernel at locked base clocks (free of the power-cap noise of in-situ timing; for
# comparisons only, never a bench value): KERNEL=regex CFG=c5m tools/ab_ncu.sh TAG...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in "$@"; do
  EF_B200_LIB=$PWD/build/lib_$v.so timeout 600 ncu --clock-control base --metrics gpu__time_duration.sum,smsp__inst_executed.sum \
    -k regex:${KERNEL:-k_edge_visc} --launch-skip ${SKIP:-4} --launch-count ${COUNT:-4} --csv --log-file gpurun_out/ab_$v.csv \
    python tools/ncu_stage.py ${CFG:-c5m} 2 > gpurun_out/ab_$v.log 2>&1
  python - "$v" <<'PY'
import csv, sys
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/ab_{v}.csv")) if len(r) > 10 and r[0].isdigit()]
out = {}
for r in rows:
    out.setdefault((r[4][:40], r[-3]), []).append(float(r[-1].replace(",", "")))
print(v, {k: [round(x, 1) for x in vals] for k, vals in out.items()})
PY
done
