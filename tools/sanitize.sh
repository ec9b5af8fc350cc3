#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck on small runs of every kernel
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in c1 c2s c5s group; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_run.py $cfg > gpurun_out/san_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_${cfg}.log | tail -1)"
  done
done
