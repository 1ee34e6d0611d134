#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "single or replay or eager or resolve or handoffs or degenerate or obstacles" > gpurun_out/single_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/single_tests.log
for r in 1 2; do
  echo "default: $(timeout 300 python tools/gpu/single_probe.py 2>&1 | tail -1)" >> gpurun_out/single_ab3.log
  echo "no_single: $(RGG_NO_SINGLE=1 timeout 300 python tools/gpu/single_probe.py 2>&1 | tail -1)" >> gpurun_out/single_ab3.log
done
bash tools/gpu/single_ncu.sh
