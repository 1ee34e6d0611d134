start=$(date +%s)
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $? in $(( $(date +%s) - start )) s"
tail -5 gpurun_out/bench.err
