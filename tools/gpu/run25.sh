python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/gpu/ktimes.sh var6 var9 var10
bash tools/gpu/ab.sh var6 var9 var10
