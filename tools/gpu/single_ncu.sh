#!/bin/bash
mkdir -p gpurun_out
for m in default no_single; do
  if [ $m = no_single ]; then export RGG_NO_SINGLE=1; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sn_$m.csv \
     python tools/gpu/single_steps.py c2 > /dev/null 2>&1
done
