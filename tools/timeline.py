"""Per-kernel timeline of flushed-L2 updates (diagnostic).  Run with
RGG_DEBUG_TIMELINE=1; the engine prints one '[tl]' line per update on stderr,
tools/timeline.py --parse FILE averages them."""
import sys

import numpy as np

if len(sys.argv) > 2 and sys.argv[1] == '--parse':
    rows = {}
    arr = []
    for line in open(sys.argv[2]):
        if not line.startswith('[tl]'):
            continue
        head, arrive = line[4:].split('arrive')
        parts = [p.split() for p in head.split('|') if p.strip()]
        for p in parts:
            rows.setdefault(p[0], []).append([float(x) for x in p[1:]])
        arr.append([float(x) for x in arrive.split()])
    print(f'{len(arr)} updates (us from first pose warp): first start / last start / first end / last end / mean warp')
    for k, v in rows.items():
        m = np.median(np.array(v[2:]), 0)
        print(f'  {k:7s} ' + ' '.join(f'{x:7.1f}' for x in m))
    print('  arrive (before PDL wait) bin/touch/narrow/apply:', ' '.join(f'{x:6.1f}' for x in np.median(np.array(arr[2:]), 0)))
    sys.exit(0)

import torch

sys.path.insert(0, '.')
import bench
from paper_2603_28674_b200 import engine as E, producer

cfg = sys.argv[1] if len(sys.argv) > 1 else 'c2'
do_flush = 'noflush' not in sys.argv
steps = 12
rm, obs, _ = bench.tile_workload(cfg, 0, 12345, steps)
lv = producer.layout_for(rm, obs)
ids, rts = bench.world_moves(cfg, 1, 12345, steps)
eng = E.GpuEngine(lv)
d_ids = torch.from_numpy(np.ascontiguousarray(ids)).cuda()
d_rts = torch.from_numpy(np.ascontiguousarray(rts)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
for it in range(steps):
    if do_flush:
        flush.zero_()
    torch.cuda.synchronize()
    eng.update_device(d_ids[it].data_ptr(), d_rts[it].data_ptr(), ids.shape[1], per_move=True)
    eng.sync()
