#!/bin/bash
# ncu --set full (source) of k_edge_visc for each build/lib_<v>.so
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in ${VARIANTS}; do
  EF_B200_LIB=$PWD/build/lib_$v.so timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:${KERNEL:-k_edge_visc} --launch-skip ${SKIP:-4} --launch-count 1 -o gpurun_out/${KERNEL:-k_edge_visc}_$v -f \
    python tools/ncu_stage.py ${CFG:-c5m} 2 > gpurun_out/ncu_$v.log 2>&1; echo "ncu $v rc=$?"
done
