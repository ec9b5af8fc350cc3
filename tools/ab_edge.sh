#!/bin/bash
# A/B of the 3D edge kernel variants: phase probe + one ncu --set full capture of k_edge_visc each
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out build
for v in ${VARIANTS}; do
  echo "== $v"; EF_B200_LIB=$PWD/build/lib_$v.so timeout 600 python tools/phase_probe.py ${CFG:-c5m} 2>&1 | tail -1
done
if [ "${NCU:-1}" = 1 ]; then
for v in ${VARIANTS}; do
  EF_B200_LIB=$PWD/build/lib_$v.so timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:k_edge_visc --launch-skip 4 --launch-count 1 -o gpurun_out/edge_$v -f \
    python tools/ncu_stage.py ${CFG:-c5m} 2 > gpurun_out/ncu_edge_$v.log 2>&1; echo "ncu $v rc=$?"
done
fi
