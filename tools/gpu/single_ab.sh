#!/bin/bash
# A/B of the single-move kernel against the batched pipeline for n == 1 (RGG_NO_SINGLE)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "single or replay or eager or resolve or handoffs" > gpurun_out/single_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/single_tests.log
for r in 1 2; do
  echo "default: $(timeout 300 python tools/gpu/e2e_small.py 2>&1 | tail -1)" >> gpurun_out/single_ab.log
  echo "no_single: $(RGG_NO_SINGLE=1 timeout 300 python tools/gpu/e2e_small.py 2>&1 | tail -1)" >> gpurun_out/single_ab.log
done
