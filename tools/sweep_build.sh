#!/bin/bash
# build register-cap variants for tools/probe_variants.sh: TAG=FLAGS pairs
cd "$(dirname "$0")/.."
build() { bash tools/variants.sh "$1" "$2" && echo "built $1"; }
export -f build
printf '%s\n' "$@" | xargs -P 4 -I{} bash -c 'v="{}"; build "${v%%=*}" "${v#*=}"'
