"""Single-move latency: host wall time of update_obstacle and the device time of its
graph (last_stats total_ms, events bracketing the update), warm L2 and flushed."""
import statistics, sys, time
sys.path.insert(0, '.')
import torch
import bench
from paper_2603_28674_b200 import engine as E, producer
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
out = {}
for cfg in ('c2', 'c5'):
    rm, obs, _ = bench.tile_workload(cfg, 0, 12345, 30)
    lv = producer.layout_for(rm, obs)
    ids, rts = bench.world_moves(cfg, 1, 12345, 30)
    eng = E.GpuEngine(lv, allow_wide=True)
    eng.batch_update((ids[0], rts[0]), per_move=True)
    for fl in (False, True):
        wall, dev = [], []
        for it in range(200):
            j = it % len(ids[1])
            if fl:
                flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng.update_obstacle(int(ids[1][j]), rts[1][j])
            wall.append(time.perf_counter() - t0)
            dev.append(eng.last_stats()['total_ms'])
        out[(cfg, 'flush' if fl else 'warm')] = (round(1e3 * statistics.median(wall[20:]), 4),
                                                 round(1e3 * statistics.median(dev[20:]), 4))
print(out)
