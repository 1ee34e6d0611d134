#!/bin/bash
# interleaved A/B of an environment switch: bash tools/gpu/env_ab.sh VAR=value [configs...]
kv=$1; shift
for rep in 1 2 3; do
  echo -n "base "; python tools/perf_probe.py "$@"
  echo -n "$kv "; env $kv python tools/perf_probe.py "$@"
done
