"""Where does the host-API (e2e) time of a c2 update go?  Wall-clock probes of
the pieces of GpuEngine.batch_update (diagnostic only; bench.py is the number)."""
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import bench
from paper_2603_28674_b200 import engine as E, producer

cfg = sys.argv[1] if len(sys.argv) > 1 else 'c2'
steps = 40
rm, obs, _ = bench.tile_workload(cfg, 0, 12345, steps)
lv = producer.layout_for(rm, obs)
ids, rts = bench.world_moves(cfg, 1, 12345, steps)
eng = E.GpuEngine(lv)
lib = E.library()
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')


def wall(fn, reps=3, do_flush=False):
    out = []
    for r in range(reps):
        for it in range(steps):
            if do_flush:
                flush.zero_()
                torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(it)
            out.append(time.perf_counter() - t0)
    return 1e6 * statistics.median(out), 1e6 * statistics.mean(out)


d_ids = torch.from_numpy(np.ascontiguousarray(ids)).cuda()
d_rts = torch.from_numpy(np.ascontiguousarray(rts)).cuda()
res = {}
for fl in (False, True):
    tag = 'flush' if fl else 'warm'
    res[f'batch_update_{tag}'] = wall(lambda it: eng.batch_update((ids[it], rts[it]), per_move=True), do_flush=fl)
    res[f'batch_update_noreports_{tag}'] = wall(lambda it: eng.batch_update((ids[it], rts[it]), per_move=False), do_flush=fl)

    def dev(it):
        eng.update_device(d_ids[it].data_ptr(), d_rts[it].data_ptr(), ids.shape[1], per_move=True)
        eng.sync()
    res[f'update_device+sync_{tag}'] = wall(dev, do_flush=fl)
res['ctypes_trivial'] = wall(lambda it: eng.unknown_count())
reps = (E._Report * 64)()
h = eng._h
a_ids = [np.ascontiguousarray(ids[i]) for i in range(steps)]
a_rts = [np.ascontiguousarray(rts[i]) for i in range(steps)]
res['raw_ctypes_update'] = wall(lambda it: lib.rgg_gpu_update(h, a_ids[it].ctypes.data, a_rts[it].ctypes.data, 64, 3, reps))
res['raw_ctypes_update_flush'] = wall(lambda it: lib.rgg_gpu_update(h, a_ids[it].ctypes.data, a_rts[it].ctypes.data, 64, 3, reps), do_flush=True)

st = torch.cuda.ExternalStream(eng.stream())
if st is not None:
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(3):
        for it in range(steps):
            ev0.record(st)
            eng.update_device(d_ids[it].data_ptr(), d_rts[it].data_ptr(), ids.shape[1], per_move=True)
            ev1.record(st)
            ev1.synchronize()
            ts.append(ev0.elapsed_time(ev1) * 1e3)
    res['device_events_warm'] = (statistics.median(ts), statistics.mean(ts))
for k, v in res.items():
    print(f'{k:32s} median {v[0]:8.1f} us  mean {v[1]:8.1f} us')
