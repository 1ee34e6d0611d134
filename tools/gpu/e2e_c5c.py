"""c5 e2e: batch_update then gray_ids_view, each timed; the view timed twice (the second
call shows the call overhead alone)."""
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
T = {"update": [], "view1": [], "view2": [], "device": []}
for it in range(14):
    flush.zero_(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = eng.batch_update((ids[it], rts[it]), per_move=True, gray_list=True)
    t1 = time.perf_counter()
    g = eng.gray_ids_view()
    t2 = time.perf_counter()
    g2 = eng.gray_ids_view()
    t3 = time.perf_counter()
    if it >= 4:
        T["update"].append(t1 - t0); T["view1"].append(t2 - t1); T["view2"].append(t3 - t2)
        T["device"].append(eng.last_stats()["total_ms"] * 1e-3)
print({k: round(1e3 * statistics.median(v), 4) for k, v in T.items()}, len(g), int(g[-1]))
