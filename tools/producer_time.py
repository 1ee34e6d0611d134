"""Producer wall time, host box fit vs GPU box fit (diagnostic)."""
import sys
import time

sys.path.insert(0, '.')
import bench
from paper_2603_28674_b200 import producer

for cfg in sys.argv[1:] or ['c2', 'c5']:
    rm, obs, _ = bench.tile_workload(cfg, 0, 12345, 2)
    for gpu in (False, True, True):
        t = time.perf_counter()
        producer.build_layout(rm.robot_he, rm.nodes, rm.edges, rm.eps, rm.max_segments, gpu_fit=gpu)
        print(f"{cfg}: gpu_fit={gpu} {time.perf_counter() - t:.3f} s")
