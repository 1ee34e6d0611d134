python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/gpu/ktimes.sh var6 var8a var8b
bash tools/gpu/ab.sh var6 var8a var8b
