import sys, time, json, statistics, numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_28674_b200 import engine as E, producer
import bench
rm, obs, _ = bench.tile_workload('c2', 0, 12345, 30)
lv = producer.layout_for(rm, obs)
ids, rts = bench.world_moves('c2', 1, 12345, 30)
flush = torch.empty(512*1024*1024//4, device='cuda')
for cell in (128, 64, 32):
    eng = E.GpuEngine(lv, cell_size=cell)
    for it in range(3): eng.batch_update((ids[it], rts[it]), per_move=True)
    res = {}
    for fl in (True, False):
        cls, tot = [], []
        for it in range(3, 23):
            if fl: flush.zero_(); torch.cuda.synchronize()
            eng.batch_update((ids[it], rts[it]), per_move=True)
            st = eng.last_stats(); cls.append(st['classify_ms']); tot.append(st['total_ms'])
        res['flush' if fl else 'warm'] = (round(statistics.median(cls)*1e3,1), round(statistics.median(tot)*1e3,1))
    print('cell', cell, 'classify/total us', res, 'dirty', st['dirty_cells'], flush=True)
