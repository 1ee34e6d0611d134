"""Engine construction cost (rgg_gpu_create: Morton sort, SoA upload) at c2/c5 (diagnostic)."""
import sys
import time

sys.path.insert(0, '.')
import bench
from paper_2603_28674_b200 import engine as E, producer

for cfg in sys.argv[1:] or ['c2', 'c5']:
    t0 = time.perf_counter()
    rm, obs, _ = bench.tile_workload(cfg, 0, 12345, 2)
    t1 = time.perf_counter()
    lv = producer.layout_for(rm, obs)
    t2 = time.perf_counter()
    E.library()
    for rep in range(3):
        t3 = time.perf_counter()
        eng = E.GpuEngine(lv)
        t4 = time.perf_counter()
        del eng
    print(f"{cfg}: roadmap {t1 - t0:.2f} s, producer {t2 - t1:.2f} s, rgg_gpu_create {1e3 * (t4 - t3):.1f} ms "
          f"(N={lv.N})")
