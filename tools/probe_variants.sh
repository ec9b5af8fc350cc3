#!/bin/bash
# tools/probe_variants.sh CONFIG TAG... : phase probe for each build/lib_TAG.so
cfg=$1; shift
for v in "$@"; do
  echo -n "$v: "; EF_B200_LIB=$PWD/build/lib_$v.so python tools/phase_probe.py $cfg ${PROBE_ARGS} 2>&1 | tail -1
done
