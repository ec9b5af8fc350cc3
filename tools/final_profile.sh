#!/bin/bash
# End-of-round measurement campaign: bench lines, reference arm, launch list and
# one ncu --set full stage capture of the headline config.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
run() { local tag=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/fin_$tag.json 2> gpurun_out/fin_$tag.err; echo "$tag rc=$?"; }
run c5w
run c5 --config c5 --no-cpu
run ref --impl reference
run c2 --config c2 --no-cpu --steps 200
run c3 --config c3 --no-cpu --steps 20
run c4m --config c4m --no-cpu --steps 50
run c1 --config c1 --no-cpu --steps 100
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_c5_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/fin_ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --launch-skip 23 --launch-count 8 \
  -o gpurun_out/fin_c5w_stage -f python tools/ncu_stage.py c5w 2 > gpurun_out/fin_ncu_full.log 2>&1; echo "ncu full rc=$?"
