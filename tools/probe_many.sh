#!/bin/bash
# phase probes of build/lib_TAG.so variants: CFGS="c5m c2" tools/probe_many.sh TAG...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for c in ${CFGS:-c5m}; do
  for v in "$@"; do
    echo -n "$c $v: "; EF_B200_LIB=$PWD/build/lib_$v.so timeout 600 python tools/phase_probe.py $c ${PROBE_ARGS} 2>&1 | tail -1
  done
done
