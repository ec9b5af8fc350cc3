#!/bin/bash
# function-level + parity tests, then the phase probe of the working build and of build/lib_*.so variants
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_functions.py tests/test_gpu_parity.py -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_fn.log 2>&1; echo "pytest rc=$?"
tail -12 gpurun_out/pytest_fn.log
for c in ${PROBES:-c5m}; do
  echo -n "probe $c: "; timeout 600 python tools/phase_probe.py $c 2>&1 | tail -1
  for v in ${VARIANTS}; do
    echo -n "  $v: "; EF_B200_LIB=$PWD/build/lib_$v.so timeout 600 python tools/phase_probe.py $c 2>&1 | tail -1
  done
done
