python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/gpu/ktimes.sh var5b var6
bash tools/gpu/ab.sh var5b var6
