"""Eager-update probe: host-API wall time of a first (graph capture) and later eager
batches on c2, for the launch list under ncu (`--metrics gpu__time_duration.sum`)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_28674_b200 import engine as E  # noqa: E402
from paper_2603_28674_b200 import producer  # noqa: E402

rounds = 4
rm, obs, _ = bench.tile_workload("c2", 0, 1234, rounds + 1)
lv = producer.layout_for(rm, obs, with_poses=True)
ids, rts = bench.world_moves("c2", 1, 1234, rounds + 1)
eng = E.GpuEngine(lv, device=0)
eng.set_resolver(*lv.resolver)
for r in range(rounds + 1):
    t0 = time.perf_counter()
    reps = eng.batch_update((ids[r], rts[r]), lazy=False)
    ms = 1e3 * (time.perf_counter() - t0)
    print(f"eager batch {r}: {len(ids[r])} moves, {sum(x.resolve_checks for x in reps)} checks, {ms:.2f} ms", flush=True)
