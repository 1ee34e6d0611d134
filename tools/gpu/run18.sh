bash tools/gpu/ktimes.sh var5b var6
bash tools/gpu/ab.sh var5b var6
