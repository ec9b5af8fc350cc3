#!/bin/bash
# default bench line (no CPU leg) of build/lib_TAG.so variants: tools/bench_variants.sh TAG...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in "$@"; do
  EF_B200_LIB=$PWD/build/lib_$v.so timeout 900 python bench.py --no-cpu ${BENCH_ARGS} > gpurun_out/benchv_$v.json 2> gpurun_out/benchv_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/benchv_$v.json').read().strip().splitlines()[-1]); print('$v', '%.4g'%d['value'], '%.4g'%d['general_path']['value'], d['roofline']['phase_ms'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
