python -X faulthandler bench.py --no-cpu-baseline --no-extras --steps 3 --warmup 3 2>&1 | tail -3 | cut -c1-1500
