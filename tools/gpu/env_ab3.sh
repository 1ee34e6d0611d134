#!/bin/bash
# interleaved A/B/C of environment settings: bash tools/gpu/env_ab3.sh "VAR=a" "VAR=b" -- configs...
vals=(); while [ "$1" != "--" ]; do vals+=("$1"); shift; done; shift
for rep in 1 2 3; do
  echo -n "base "; python tools/perf_probe.py "$@"
  for kv in "${vals[@]}"; do echo -n "$kv "; env $kv python tools/perf_probe.py "$@"; done
done
