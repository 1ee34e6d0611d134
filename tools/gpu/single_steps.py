"""One c2 batch, then 10 single update_obstacle calls (for an ncu launch list)."""
import sys
sys.path.insert(0, '.')
import bench
from paper_2603_28674_b200 import engine as E, producer
cfg = sys.argv[1] if len(sys.argv) > 1 else 'c2'
rm, obs, _ = bench.tile_workload(cfg, 0, 12345, 30)
lv = producer.layout_for(rm, obs)
ids, rts = bench.world_moves(cfg, 1, 12345, 30)
eng = E.GpuEngine(lv, allow_wide=True)
eng.batch_update((ids[0], rts[0]), per_move=True)
for j in range(10):
    eng.update_obstacle(int(ids[1][j]), rts[1][j])
