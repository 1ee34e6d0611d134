"""Small-batch latency: host wall time of batch_update and its device time (last_stats
total_ms), L2 flushed, for c2 (64 moves), c4 (7 moves) and c4 with 16 / 32 moves."""
import statistics, sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
from paper_2603_28674_b200 import engine as E, producer
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
out = {}
for cfg, take in (('c2', 64), ('c4', 7), ('c5', 16), ('c5', 32), ('c5', 64)):
    rm, obs, _ = bench.tile_workload(cfg, 0, 12345, 30)
    lv = producer.layout_for(rm, obs)
    ids, rts = bench.world_moves(cfg, 1, 12345, 30)
    eng = E.GpuEngine(lv, allow_wide=True)
    wall, dev = [], []
    for it in range(30):
        i0 = (it * take) % ids.shape[1]
        mi, mr = np.ascontiguousarray(ids[it][i0:i0 + take]), np.ascontiguousarray(rts[it][i0:i0 + take])
        flush.zero_(); torch.cuda.synchronize()
        t0 = time.perf_counter(); eng.batch_update((mi, mr), per_move=True, gray_list=True); wall.append(time.perf_counter() - t0)
        dev.append(eng.last_stats()['total_ms'])
    out[f"{cfg}x{take}"] = (round(1e3 * statistics.median(wall[5:]), 2), round(1e3 * statistics.median(dev[5:]), 2))
print(out)
