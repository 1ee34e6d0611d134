for rep in 1 2; do for cs in 128 64 32; do echo -n "cell $cs "; RGG_CELL_SIZE=$cs python tools/perf_probe.py c5 c3 c2 c4; done; done
