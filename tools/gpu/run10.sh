bash tools/gpu/ab.sh var2 var3
for cs in 64 32; do echo "cell $cs"; RGG_CELL_SIZE=$cs RGG_GPU_LIB=tools/gpu/var3/librgg_gpu.so python tools/perf_probe.py c5 c3 c2 c4; done
