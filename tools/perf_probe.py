"""Per-update latency of several configs (diagnostic; device-resident moves, L2 flushed):
python tools/perf_probe.py c2 c5 c3"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

out = {}
for cfg in sys.argv[1:] or ["c2", "c5"]:
    r = bench.measure_extra(cfg, 12345, 0, steps=20, warmup=5)
    out[cfg] = round(r["per_update_ms"], 4)
print(json.dumps(out))
