python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c5 c3; do RGG_DEBUG_TIMELINE=1 python tools/timeline.py $c 2> gpurun_out/tl_$c.txt; echo $c; python tools/timeline.py --parse gpurun_out/tl_$c.txt; done
python tools/perf_probe.py c5 c2 c3 c4
RGG_EARLY_TOUCH_MIN=256 python tools/perf_probe.py c5 c3
