# one bench line + reference arm + ncu launch list + ncu --set full of a c5 and a c2 update
# (gray list in the update), with the classify kernels' source pages (profiles/r2*)
start=$(date +%s)
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $? in $(( $(date +%s) - start )) s"
tail -3 gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench.log 2>&1; echo "launch list rc $?"
K='regex:pose_kernel|bin_|touch|narrow_|apply_warp|gray_'
ncu --set full --clock-control none --import-source on -k "$K" \
    --launch-skip 18 --launch-count 9 -f -o gpurun_out/c5_prof python tools/step_once.py 4 c5 gray > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc $?"
for k in narrow_over narrow_under apply touch pose; do
  ncu -i gpurun_out/c5_prof.ncu-rep --page source --csv --print-source cuda,sass -k regex:$k > gpurun_out/c5_src_$k.csv 2>/dev/null
done
ncu --set full --clock-control none --import-source on -k "$K" \
    --launch-skip 16 --launch-count 8 -f -o gpurun_out/c2_prof python tools/step_once.py 4 c2 gray > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc $?"
