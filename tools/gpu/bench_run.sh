python -m pytest tests -m gpu -x -q 2>&1 | tail -2
/usr/bin/time -v python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -5 gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
tail -3 gpurun_out/bench_ref.err
