# repeat the bench under faulthandler to catch an intermittent native crash
for i in 1 2 3 4; do
  python -X faulthandler bench.py --steps 5 --warmup 3 --cpu-sample-s 2 > gpurun_out/br_$i.json 2> gpurun_out/br_$i.err
  echo "run $i rc=$?"
done
