#!/bin/bash
# repeat the C++ drop-in test: failures per mode
for mode in default no_single; do
  f=0
  for i in $(seq 1 ${REPS:-25}); do
    if [ $mode = no_single ]; then out=$(RGG_NO_SINGLE=1 ./oracle/_ref/test_gpu_engine tests/golden/scenarios 2>&1); else out=$(./oracle/_ref/test_gpu_engine tests/golden/scenarios 2>&1); fi
    if echo "$out" | grep -q "FAIL"; then f=$((f+1)); echo "$out" | grep FAIL | head -3; fi
  done
  echo "$mode: $f failures of ${REPS:-25}"
done
