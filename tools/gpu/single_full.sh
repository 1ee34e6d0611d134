#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/full_tests.log
for r in 1 2; do
  echo "default: $(timeout 300 python tools/gpu/single_probe.py 2>&1 | tail -1)" >> gpurun_out/single_ab4.log
  echo "no_single: $(RGG_NO_SINGLE=1 timeout 300 python tools/gpu/single_probe.py 2>&1 | tail -1)" >> gpurun_out/single_ab4.log
done
