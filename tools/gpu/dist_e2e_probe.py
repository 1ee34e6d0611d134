"""Where the N>1 e2e step's host time goes (world-1 NCCL group, c5): per-call wall times."""
import os, sys, time, statistics
sys.path.insert(0, '.')
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch, torch.distributed as dist
import bench
from paper_2603_28674_b200 import engine as E, producer
from paper_2603_28674_b200.dist import DistributedUpdater
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=dev)
rm, obs, _ = bench.tile_workload("c5", 0, 12345, 12)
lv = producer.layout_for(rm, obs)
ids_h, rts_h = bench.world_moves("c5", 1, 12345, 12)
eng = E.GpuEngine(lv, device=0)
up = DistributedUpdater(eng, dev, gray_cap=eng.n_owned)
m = ids_h.shape[1]
pin_ids = torch.empty((m,), dtype=torch.int32, pin_memory=True)
pin_rts = torch.empty((m, 12), dtype=torch.float64, pin_memory=True)
T = {k: [] for k in ("h2d", "update", "reports", "gray", "total")}
for it in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pin_ids.numpy()[:] = ids_h[it]; pin_rts.numpy()[:] = rts_h[it]
    ids_t = pin_ids.to(dev, non_blocking=True); rts_t = pin_rts.to(dev, non_blocking=True)
    t1 = time.perf_counter()
    c = up.update(ids_t, rts_t, per_move=True, gather_gray=True)
    t2 = time.perf_counter()
    r = c.cpu()
    t3 = time.perf_counter()
    g = up.gathered_gray()
    t4 = time.perf_counter()
    if it >= 2:
        for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
            T[k].append(1e3 * v)
print({k: round(statistics.median(v), 3) for k, v in T.items()}, len(g))
dist.destroy_process_group()
