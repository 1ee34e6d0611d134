"""c5 e2e split: batch_update (host moves in, reports out) and gray_ids_view (pinned DMA),
against the device time of the same update (last_stats total_ms)."""
import sys, time, statistics
sys.path.insert(0, '.')
import torch
import bench
from paper_2603_28674_b200 import engine as E, producer
rm, obs, _ = bench.tile_workload('c5', 0, 12345, 14)
lv = producer.layout_for(rm, obs)
ids, rts = bench.world_moves('c5', 1, 12345, 14)
eng = E.GpuEngine(lv)
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
T = {"update": [], "gray_view": [], "device": [], "total": []}
for it in range(14):
    flush.zero_(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = eng.batch_update((ids[it], rts[it]), per_move=True, gray_list=True)
    t1 = time.perf_counter()
    g = eng.gray_ids_view()
    t2 = time.perf_counter()
    if it >= 4:
        T["update"].append(t1 - t0); T["gray_view"].append(t2 - t1); T["total"].append(t2 - t0)
        T["device"].append(eng.last_stats()["total_ms"] * 1e-3)
print({k: round(1e3 * statistics.median(v), 4) for k, v in T.items()}, len(g))
