import sys, numpy as np
sys.path.insert(0, '.')
from paper_2603_28674_b200 import engine as E, producer
import bench
rm, obs, _ = bench.tile_workload('c2', 0, 12345, 30)
lv = producer.layout_for(rm, obs)
ids, rts = bench.world_moves('c2', 1, 12345, 30)
eng = E.GpuEngine(lv)
for it in range(6): eng.batch_update((ids[it], rts[it]), per_move=True)
