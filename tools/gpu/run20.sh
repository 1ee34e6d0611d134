for env in "" "RGG_L2_PREFETCH=1" "RGG_L2_PREFETCH=1 RGG_NARROW_REV=1" "RGG_NARROW_REV=1"; do
  for rep in 1 2; do echo -n "[$env] "; env $env RGG_GPU_LIB=tools/gpu/var7/librgg_gpu.so python tools/perf_probe.py c5 c3 c2 c4; done
done
