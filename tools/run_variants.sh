#!/bin/bash
# run bench for each build/lib_<tag>.so given as args; print value + phase ms
for v in "$@"; do
  EF_B200_LIB=$PWD/build/lib_$v.so python bench.py --steps ${STEPS:-100} --no-cpu --e2e-steps 5 ${BENCH_ARGS} > gpurun_out/var_$v.log 2>&1
  echo "== $v rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/var_$v.log').read().strip().splitlines()[-1]); print('%.4g'%d['value'], '%.3f'%d['ms_per_step'], d['roofline']['phase_ms'])" 2>&1 | tail -2
done
