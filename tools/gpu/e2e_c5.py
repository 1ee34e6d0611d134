"""Where the c5 host-API (e2e) time goes: batch_update alone, gray_ids into pageable and pinned memory."""
import sys, time, statistics
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2603_28674_b200 import engine as E, producer
rm, obs, _ = bench.tile_workload('c5', 0, 12345, 12)
lv = producer.layout_for(rm, obs)
ids, rts = bench.world_moves('c5', 1, 12345, 12)
eng = E.GpuEngine(lv)
pin = torch.empty(lv.N, dtype=torch.int32, pin_memory=True).numpy()
t_up, t_gp, t_gpin, t_dev = [], [], [], []
for it in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = eng.batch_update((ids[it], rts[it]), per_move=True, gray_list=True)
    t1 = time.perf_counter()
    g = eng.gray_ids()
    t2 = time.perf_counter()
    n = eng.unknown_count()
    t3 = time.perf_counter()
    E.library().rgg_gpu_gray_ids(eng.handle, pin.ctypes.data, n, (E.C.c_int32 * 1)())
    t4 = time.perf_counter()
    if it >= 2:
        t_up.append(t1 - t0); t_gp.append(t2 - t1); t_gpin.append(t4 - t3)
print(f"batch_update {1e3*statistics.median(t_up):.3f} ms | gray_ids pageable {1e3*statistics.median(t_gp):.3f} ms "
      f"| gray_ids pinned {1e3*statistics.median(t_gpin):.3f} ms | n_gray {n}")
