"""Cost of the reference's CPU engines at c5 on the GPU box's host (diagnostic):
world build, grouped SequentialEngine / BatchEngine construction and a sample of
moves.  python tools/ref_c5_probe.py [c5] [moves]"""
import os
import resource
import subprocess
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from oracle import ref  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
nmv = int(sys.argv[2]) if len(sys.argv) > 2 else 64
print(subprocess.run("lscpu | grep -E 'Model name|^CPU\\(s\\)|Thread|Socket'; free -g", shell=True,
                     capture_output=True, text=True).stdout, flush=True)
rss = lambda: resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
t = time.time()
rm, obs, _ = bench.tile_workload(cfg, 0, 12345, 3)
print(f"roadmap {len(rm.nodes)} nodes {len(rm.edges)} edges: {time.time() - t:.1f} s", flush=True)
t = time.time()
w = ref.World.from_roadmap(rm.robot_he, rm.env, rm.nodes, rm.edges, rm.eps, rm.max_segments)
for he, ns in zip(obs.he, obs.spheres):
    w.add_obstacle(he, int(ns))
print(f"world {w.counts()}: {time.time() - t:.1f} s, maxrss {rss():.1f} GB", flush=True)
ids, rts = bench.world_moves(cfg, 1, 12345, 3)
for kind, threads in ((1, 1), (0, os.cpu_count()), (0, 1)):
    t = time.time()
    e = ref.Engine(w, kind=kind, threads=threads, group_size=64)
    print(f"engine kind {kind} threads {threads}: {e.groups} groups built in {time.time() - t:.1f} s, "
          f"maxrss {rss():.1f} GB", flush=True)
    us = e.run(ids[0][:nmv], rts[0][:nmv])
    print(f"  first {nmv} moves: {us * 1e-3:.1f} ms ({us / nmv * 1e-3:.2f} ms/move)", flush=True)
    if kind == 1:
        us = e.run(ids[0][nmv:], rts[0][nmv:])
        print(f"  remaining {len(ids[0]) - nmv} moves: {us * 1e-3:.1f} ms", flush=True)
        us = e.run(ids[1], rts[1])
        print(f"  full update 2: {us * 1e-3:.1f} ms", flush=True)
    del e
