#!/bin/bash
# phase probe of every build/lib_*.so on CFG (default c5m), twice each (interleaved)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for rep in 1 2; do
  for f in build/lib_*.so; do
    v=$(basename $f .so); v=${v#lib_}
    echo -n "$rep $v: "; EF_B200_LIB=$PWD/$f timeout 300 python tools/phase_probe.py ${CFG:-c5m} steps=10 warm=5 2>&1 | tail -1
  done
done
