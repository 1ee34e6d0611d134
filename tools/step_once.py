"""Replay a few updates of a config through the engine (profiling driver: launch lists / ncu):
python tools/step_once.py STEPS CONFIG [gray]."""
import sys
sys.path.insert(0, '.')
from paper_2603_28674_b200 import engine as E, producer
import bench
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cfg = sys.argv[2] if len(sys.argv) > 2 else 'c2'
rm, obs, _ = bench.tile_workload(cfg, 0, 12345, steps)
lv = producer.layout_for(rm, obs)
ids, rts = bench.world_moves(cfg, 1, 12345, steps)
eng = E.GpuEngine(lv)
for it in range(steps):
    eng.batch_update((ids[it], rts[it]), per_move=True, gray_list=len(sys.argv) > 3 and sys.argv[3] == "gray")
print("done", eng.last_stats())
