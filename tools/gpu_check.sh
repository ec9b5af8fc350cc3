#!/bin/bash
# tests + the default bench line (+ optional phase probe): GPU session helper
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-chk}
if [ "${TESTS:-1}" = 1 ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
  tail -15 gpurun_out/pytest_$TAG.log
fi
if [ "${BENCH:-1}" = 1 ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1]); print('%.4g'%d['value'], '%.2f'%d['ms_per_step'], d['roofline']['phase_ms'], d['roofline']['stage']['frac'], d['clocks'])" 2>&1 | tail -2
fi
for c in ${PROBES}; do
  echo -n "probe $c: "; timeout 600 python tools/phase_probe.py $c 2>&1 | tail -1
done
