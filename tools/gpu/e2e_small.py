"""Host-API latency of small batches (c2 64 moves, c4 16 moves, c1-like single moves), L2 flushed."""
import statistics, sys, time
sys.path.insert(0, '.')
import torch
import bench
from paper_2603_28674_b200 import engine as E, producer
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
out = {}
for cfg in ('c2', 'c4'):
    rm, obs, _ = bench.tile_workload(cfg, 0, 12345, 30)
    lv = producer.layout_for(rm, obs)
    ids, rts = bench.world_moves(cfg, 1, 12345, 30)
    eng = E.GpuEngine(lv)
    ts, t1 = [], []
    for it in range(30):
        flush.zero_(); torch.cuda.synchronize()
        t0 = time.perf_counter(); eng.batch_update((ids[it], rts[it]), per_move=True); ts.append(time.perf_counter() - t0)
        flush.zero_(); torch.cuda.synchronize()
        t0 = time.perf_counter(); eng.update_obstacle(int(ids[it][0]), rts[it][0]); t1.append(time.perf_counter() - t0)
    out[cfg] = (round(1e3 * statistics.median(ts[5:]), 4), round(1e3 * statistics.median(t1[5:]), 4))
print(out)
