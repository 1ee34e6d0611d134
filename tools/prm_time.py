"""GPU kNN of build_prm (csrc/rgg_prm.cu) at table3's 10,000 nodes and at the 1M-edge
configs' 87,000 nodes (diagnostic)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2603_28674_b200 import prm  # noqa: E402

for n, k, half in ((10000, 8, 10.0), (87000, 20, 71.0)):
    lo, hi = prm.dof_bounds_free_flying([-half, -half, -half, half, half, half])
    nodes = prm.sample_nodes(106, n, lo, hi)
    for rep in range(3):
        t0 = time.perf_counter()
        edges, ms = prm.knn_edges(nodes, k, return_ms=True)
        t1 = time.perf_counter()
        print(f"n={n} k={k}: {len(edges)} edges, device {ms:.2f} ms, call {1e3 * (t1 - t0):.2f} ms")
