"""A/B the classify stage: per-move counters on/off, under tests on/off (c2)."""
import os, sys, statistics, numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_28674_b200 import engine as E, producer
import bench
rm, obs, _ = bench.tile_workload('c2', 0, 12345, 30)
lv = producer.layout_for(rm, obs)
ids, rts = bench.world_moves('c2', 1, 12345, 30)
flush = torch.empty(512 * 1024 * 1024 // 4, device='cuda')
for use_under in (True, False):
    for per_move in (True, False):
        eng = E.GpuEngine(lv, use_under=use_under)
        for it in range(3):
            eng.batch_update((ids[it], rts[it]), per_move=per_move)
        cls = []
        for it in range(3, 15):
            flush.zero_(); torch.cuda.synchronize()
            eng.batch_update((ids[it], rts[it]), per_move=per_move)
            cls.append(eng.last_stats()['classify_ms'] * 1e3)
        print(os.environ.get('RGG_PIPELINE', '4'), 'under', use_under, 'per_move', per_move,
              'classify us %.1f' % statistics.median(cls), flush=True)
