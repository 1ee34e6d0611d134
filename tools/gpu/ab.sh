# interleaved A/B of prebuilt engine libraries: bash tools/gpu/ab.sh var1 var2 ...
for rep in 1 2 3; do
  for v in "$@"; do
    echo -n "$v "; RGG_GPU_LIB=tools/gpu/$v/librgg_gpu.so python tools/perf_probe.py c5 c3 c2 c4
  done
done
