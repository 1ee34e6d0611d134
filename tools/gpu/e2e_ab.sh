# interleaved e2e A/B of prebuilt libraries: bash tools/gpu/e2e_ab.sh varA varB
for rep in 1 2 3; do
  for v in "$@"; do echo -n "$v "; RGG_GPU_LIB=tools/gpu/$v/librgg_gpu.so python tools/gpu/e2e_c5c.py; done
done
