# ncu --set full of the 3rd c5 update's kernels (gray list in the update), the source pages
# of the classify kernels, then the launch list of a short bench: bash tools/gpu/prof_c5.sh
set -x
ncu --set full --clock-control none --import-source on -k 'regex:pose_kernel|bin_|touch|narrow_|apply_warp|gray_' \
    --launch-skip 18 --launch-count 9 -f -o gpurun_out/c5_prof python tools/step_once.py 4 c5 gray > gpurun_out/ncu_c5.log 2>&1
tail -3 gpurun_out/ncu_c5.log
ncu -i gpurun_out/c5_prof.ncu-rep --page raw --csv > gpurun_out/c5_raw.csv 2>/dev/null
for k in narrow_over narrow_under apply touch; do
  ncu -i gpurun_out/c5_prof.ncu-rep --page source --csv --print-source cuda,sass -k regex:$k > gpurun_out/c5_src_$k.csv 2>/dev/null
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c5_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench.log 2>&1
ls -la gpurun_out/ | head -30
