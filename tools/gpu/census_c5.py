"""The engine's census of one c5 update: pairs, hits, tests (rgg_gpu_census)."""
import sys
sys.path.insert(0, '.')
import torch
import bench
from paper_2603_28674_b200 import engine as E, producer
cfg = sys.argv[1] if len(sys.argv) > 1 else 'c5'
rm, obs, _ = bench.tile_workload(cfg, 0, 12345, 3)
lv = producer.layout_for(rm, obs)
ids, rts = bench.world_moves(cfg, 1, 12345, 3)
eng = E.GpuEngine(lv, allow_wide=True)
d_ids, d_rts = torch.from_numpy(ids).cuda(), torch.from_numpy(rts).cuda()
torch.cuda.synchronize()
for it in range(3):
    eng.update_device(d_ids[it].data_ptr(), d_rts[it].data_ptr(), ids.shape[1], per_move=True, census=(it == 2))
eng.sync()
print(cfg, eng.census())
