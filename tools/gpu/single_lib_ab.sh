# interleaved single-move latency A/B of prebuilt libraries: bash tools/gpu/single_lib_ab.sh varA varB
for rep in 1 2 3; do
  for v in "$@"; do echo -n "$v "; RGG_GPU_LIB=tools/gpu/$v/librgg_gpu.so python tools/gpu/single_probe.py; done
done
