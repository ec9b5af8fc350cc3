#!/bin/bash
# one ncu --set full capture (with source) of the kernels of one stage: tools/ncu_stage_src.sh CONFIG TAG [SKIP]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
cfg=${1:-c5m}; tag=${2:-stage}; skip=${3:-23}
timeout 1500 ncu --set full --clock-control none --import-source on --launch-skip $skip --launch-count 8 \
  -o gpurun_out/stage_$tag -f python tools/ncu_stage.py $cfg 2 > gpurun_out/ncu_stage_$tag.log 2>&1; echo "ncu rc=$?"
