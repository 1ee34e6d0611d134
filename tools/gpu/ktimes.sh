# per-kernel ncu durations of c5 updates for each prebuilt variant: bash tools/gpu/ktimes.sh var2 var4
for v in "$@"; do
  RGG_GPU_LIB=tools/gpu/$v/librgg_gpu.so ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     -k 'regex:pose_kernel|bin_|touch|narrow_|apply_warp|gray_' --log-file gpurun_out/kt_$v.csv \
     python tools/step_once.py 4 ${CFG:-c5} > /dev/null 2>&1
  echo -n "$v: "; python tools/gpu/ktimes.py gpurun_out/kt_$v.csv 1
done
