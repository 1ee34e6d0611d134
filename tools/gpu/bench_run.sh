start=$(date +%s)
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $? in $(( $(date +%s) - start )) s"
tail -3 gpurun_out/bench.err
start=$(date +%s)
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $? in $(( $(date +%s) - start )) s"
tail -3 gpurun_out/bench_ref.err
