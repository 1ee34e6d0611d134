set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
RGG_DEBUG_TIMELINE=1 python tools/timeline.py c5 2> gpurun_out/tl_c5_bin.txt; python tools/timeline.py --parse gpurun_out/tl_c5_bin.txt
RGG_DEBUG_TIMELINE=1 python tools/timeline.py c3 2> gpurun_out/tl_c3_bin.txt; python tools/timeline.py --parse gpurun_out/tl_c3_bin.txt
python tools/perf_probe.py c5 c2 c3 c4
RGG_NO_SMALL_BIN=1 python tools/perf_probe.py c2 c4
