#!/bin/bash
# Rebuild the in-tree native libraries; non-zero exit on any failure.
set -e
cd "$(dirname "$0")"
python -m paper_2603_28674_b200.build --force
python - <<'PY'
import ctypes, os
for f in ["paper_2603_28674_b200/lib/librgg_gpu.so", "paper_2603_28674_b200/lib/librgg_build.so"]:
    ctypes.CDLL(os.path.abspath(f))
print("build ok")
PY
