python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/gpu/ktimes.sh var2 var3 var4
bash tools/gpu/ab.sh var2 var4
