ncu --set full --clock-control none --import-source on -k 'regex:pose_kernel|bin_|touch|narrow_kernel|apply_warp|gray_' \
    --launch-skip 25 --launch-count 6 -f -o gpurun_out/c2_prof python tools/step_once.py 6 c2 > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc $?"
ncu -i gpurun_out/c2_prof.ncu-rep --page raw --csv > gpurun_out/c2_raw.csv 2>/dev/null
