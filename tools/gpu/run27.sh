bash tools/gpu/ktimes.sh var6 nar5 nar6
bash tools/gpu/ab.sh var6 nar5 nar6
for rep in 1; do for cs in 64 32; do echo -n "cell $cs "; RGG_CELL_SIZE=$cs RGG_GPU_LIB=tools/gpu/var6/librgg_gpu.so python tools/perf_probe.py c5 c3 c2 c4; done; done
