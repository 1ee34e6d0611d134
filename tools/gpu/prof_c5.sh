# ncu --set full of the 3rd c5 update's kernels, then launch list of a short bench
set -x
ncu --set full --clock-control none --import-source on -k 'regex:pose_kernel|bin_|touch|narrow_kernel|apply_warp|gray_' \
    --launch-skip 16 --launch-count 8 -f -o gpurun_out/c5_prof python tools/step_once.py 4 c5 > gpurun_out/ncu_c5.log 2>&1
tail -3 gpurun_out/ncu_c5.log
ncu -i gpurun_out/c5_prof.ncu-rep --page raw --csv > gpurun_out/c5_raw.csv 2>/dev/null
ncu -i gpurun_out/c5_prof.ncu-rep --page source --csv --print-source cuda,sass -k regex:narrow > gpurun_out/c5_src_narrow.csv 2>/dev/null
ncu -i gpurun_out/c5_prof.ncu-rep --page source --csv --print-source cuda,sass -k regex:apply > gpurun_out/c5_src_apply.csv 2>/dev/null
ncu -i gpurun_out/c5_prof.ncu-rep --page source --csv --print-source cuda,sass -k regex:cells_touch > gpurun_out/c5_src_touch.csv 2>/dev/null
ls -la gpurun_out/
