#!/usr/bin/env python
"""bench.py — SerRGG edge classification on B200: edges classified/s and per-update latency.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Workload (BASELINE.json configs[1], "c2"): SE(2) warehouse roadmap, 10k nodes /
114k edges (N = 124,080 components incl. nodes), 64 moving yaw-rotated box
obstacles, a move script of W + K iterations.  One STEP = one update of the
obstacle set = one iteration of the script: all 64 obstacles re-posed through
``batch_update`` with per-move UpdateReports (the reference's 64 calls to
BatchEngine::update_obstacle, proj/src/engine_batch.cpp:145-215).  After each
step every one of the N labels is the reference's, so

    value = N_components x steps / device time          ("edges/s")
    per-update latency = ms_per_step

* ``value``: moves already resident in HBM, timed with CUDA events on the
  engine's stream, L2 flushed (512 MB write) between steps.
* ``e2e``: the same steps through the public API with HOST buffers
  (GpuEngine.batch_update -> rgg_gpu_update: H2D of the moves, D2H of the
  per-move reports), wall clock around the call.
* ``--impl reference``: the reference's own CPU SerRGG path (BatchEngine, AVX2
  backend, all host threads) from oracle/_ref on the same roadmap and moves.

N > 1 (torchrun, one rank per GPU, NCCL): weak scaling.  Rank r owns tile r of
an N-tile world (a c2 roadmap + 64 obstacles per tile, tiles side by side);
obstacle moves are broadcast from rank 0 every step (ncclBroadcast) and the
per-move report counters are summed onto every rank (ncclAllReduce).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASE_METRIC = "edges classified/sec and per-update latency (ms) at 1/2/4/8 B200 vs CPU ref"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="c2")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--seed", type=int, default=12345)
    p.add_argument("--cpu-sample-s", type=float, default=15.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--json-out", default="")
    p.add_argument("--clock-window-s", type=float, default=1.0)
    p.add_argument("--no-resolve", action="store_true", help="skip the exact-resolve measurement")
    p.add_argument("--extra-configs", default="c5,c4,c3",
                   help="comma list of configs also measured on rank 0 (N=1) and reported under 'extra'")
    return p.parse_args()


def tile_workload(config, rank, seed, iterations):
    """Rank r's tile: the config's roadmap shifted by r tiles in x, obstacles r*M..r*M+M-1."""
    from paper_2603_28674_b200 import producer, synth

    kind, nodes, k, half, m, ohalf = synth.CONFIGS[config]
    rm = synth.make_roadmap(kind, nodes, k, half, seed + 1000 * rank)
    obs = synth.make_obstacles(kind, m, seed + 1)
    shift = 2.0 * (ohalf + 5.0) * rank
    rm.nodes[:, 0] += shift
    rm.env[[0, 3]] += shift
    return rm, obs, shift


def world_moves(config, world, seed, iterations):
    """Moves of every tile, interleaved per iteration: [iteration][tile][obstacle]."""
    from paper_2603_28674_b200 import synth

    kind, nodes, k, half, m, ohalf = synth.CONFIGS[config]
    ids_all, rts_all = [], []
    for r in range(world):
        ids, rts = synth.make_moves(kind, m, iterations, ohalf, seed + 2 + 7919 * r)
        rts[:, 9] += 2.0 * (ohalf + 5.0) * r
        ids_all.append(ids.reshape(iterations, m) + r * m)
        rts_all.append(rts.reshape(iterations, m, 12))
    ids = np.stack(ids_all, 1).reshape(iterations, world * m).astype(np.int32)
    rts = np.stack(rts_all, 1).reshape(iterations, world * m, 12)
    k = synth.MOVES_PER_STEP.get(config)
    if k:  # iteration it moves obstacles [k*it, k*it + k) mod m of every tile
        sel = np.array([[r * m + (k * it + j) % m for r in range(world) for j in range(k)] for it in range(iterations)])
        ids = np.take_along_axis(ids, sel, 1).astype(np.int32)
        rts = np.take_along_axis(rts, sel[:, :, None], 1)
    return ids, rts


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_run(config, seed, iterations, sample_s, threads, engine_kind=0):
    """The reference's CPU SerRGG path on tile 0's roadmap + moves (oracle/_ref)."""
    from oracle import ref
    from paper_2603_28674_b200 import producer, synth

    rm, obs, _ = tile_workload(config, 0, seed, iterations)
    w = ref.World.from_roadmap(rm.robot_he, rm.env, rm.nodes, rm.edges, rm.eps, rm.max_segments)
    for he, ns in zip(obs.he, obs.spheres):
        w.add_obstacle(he, int(ns))
    ids, rts = world_moves(config, 1, seed, iterations)
    eng = ref.Engine(w, kind=engine_kind, threads=threads, group_size=64)
    n = w.counts()["N"]
    done, spent = 0, 0.0
    per_step = []
    for it in range(iterations):
        us = eng.run(ids[it], rts[it], lazy=True)
        per_step.append(us)
        spent += us * 1e-6
        done += 1
        if spent >= sample_s:
            break
    return n, done, spent, per_step, eng


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    iterations = args.warmup + args.steps
    n, done, spent, per_step, _ = cpu_reference_run(args.config, args.seed, iterations, 1e18, threads)
    timed = per_step[args.warmup:] or per_step
    t = sum(timed) * 1e-6
    value = n * len(timed) / t
    line = {
        "impl": "reference", "metric": BASE_METRIC, "value": value, "unit": "edges/s", "n_gpus": args.gpus,
        "steps": len(timed), "warmup": min(args.warmup, done), "ms_per_step": 1e3 * t / len(timed),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, n),
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": threads, "kind": "reference",
                         "sample": f"rgg::BatchEngine (AVX2, {threads} threads) on tile 0: {len(timed)} updates x "
                                   f"64 moves, oracle/_ref/librgg_ref.so"},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, n_components, world=1):
    from paper_2603_28674_b200 import synth

    kind, nodes, k, half, m, ohalf = synth.CONFIGS[args.config]
    mv = synth.MOVES_PER_STEP.get(args.config)
    step = (f"1 step = 1 update = {mv} of the {m} obstacles re-posed (rotating subset, ~5 % of cells dirty)"
            if mv else f"1 step = 1 update = all {m} obstacles re-posed")
    return {"workload": f"{args.config}: {'SE(2)' if kind == 'se2' else '3D'} roadmap {nodes} nodes k={k} "
                        f"({n_components} components incl. nodes) x {m} moving OBB obstacles per GPU tile; "
                        f"{step} (per-move reports)",
            "components_per_gpu": n_components, "obstacles_per_gpu": m, "moves_per_step": m * world,
            "l2": "flushed (512 MB write) between timed steps", "parallelism": f"tiles x{world} (weak)",
            "precision": "fp64-exact (reference op order, no FMA)"}


def measure_extra(config, seed, device, steps=10, warmup=3):
    """A further BASELINE config on one GPU (device-resident moves, L2 flushed between
    updates): per-update latency and edges/s, the flop/byte census of one update."""
    import torch

    from paper_2603_28674_b200 import engine as E
    from paper_2603_28674_b200 import producer, synth

    t0 = time.time()
    rm, obs, _ = tile_workload(config, 0, seed, warmup + steps)
    lv = producer.layout_for(rm, obs)
    build_s = time.time() - t0
    eng = E.GpuEngine(lv, device=device)
    ids_h, rts_h = world_moves(config, 1, seed, warmup + steps)
    dev = torch.device("cuda", device)
    ids_d = torch.from_numpy(ids_h).to(dev)
    rts_d = torch.from_numpy(rts_h).to(dev)
    m = ids_h.shape[1]
    stream = torch.cuda.ExternalStream(eng.stream(), device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    eng.set_phase_timing(False)
    for it in range(warmup):
        eng.update_device(ids_d[it].data_ptr(), rts_d[it].data_ptr(), m, per_move=True)
    torch.cuda.synchronize()
    ms = []
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.update_device(ids_d[warmup + k].data_ptr(), rts_d[warmup + k].data_ptr(), m, per_move=True)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    eng.set_phase_timing(True)
    eng.update_device(ids_d[warmup + steps - 1].data_ptr(), rts_d[warmup + steps - 1].data_ptr(), m, per_move=True)
    eng.sync()
    dirty = eng.last_stats()["dirty_cells"]
    eng.set_phase_timing(False)
    eng.update_device(ids_d[warmup + steps - 1].data_ptr(), rts_d[warmup + steps - 1].data_ptr(), m,
                      per_move=True, census=True)
    cen = eng.census()
    per = statistics.mean(ms)
    ncells = (lv.N + 127) // 128
    byts = cen["bytes_components"] + m * 768
    return {"workload": config_dict(argparse.Namespace(config=config), lv.N)["workload"],
            "components": lv.N, "moves_per_update": m, "per_update_ms": per,
            # incremental configs: the components of the dirty cells are the ones relabelled
            "value": (min(lv.N, dirty * 128) if synth.MOVES_PER_STEP.get(config) else lv.N) / (per * 1e-3),
            "value_all_components": lv.N / (per * 1e-3),
            "unit": "edges/s", "steps": steps, "build_s": round(build_s, 1),
            "dirty_cells": dirty, "dirty_fraction": dirty / max(1, ncells),
            "hbm_frac_of_update": byts / (per * 1e-3) / 1e9 / 6553.3,
            "census": {k: cen[k] for k in ("over_pairs", "sat_flops", "under_pairs", "seg_sphere_tests",
                                           "bytes_components")}}


def measure_resolve(config, seed, device, rounds=4, cpu=True):
    """The exact resolve on the GPU: resolve_all_unknown after
    each lazy update, and one eager update, through the host API; the reference's
    own resolve_all_unknown / eager update_obstacle on the same roadmap and moves."""
    import numpy as np

    from paper_2603_28674_b200 import engine as E
    from paper_2603_28674_b200 import producer

    rm, obs, _ = tile_workload(config, 0, seed, rounds + 1)
    lv = producer.layout_for(rm, obs, with_poses=True)
    ids, rts = world_moves(config, 1, seed, rounds + 1)
    eng = E.GpuEngine(lv, device=device)
    t0 = time.perf_counter()
    eng.set_resolver(*lv.resolver)
    upload_s = time.perf_counter() - t0
    gpu_ms, grays = [], []
    for r in range(rounds):
        eng.batch_update((ids[r], rts[r]))
        grays.append(eng.unknown_count())
        t0 = time.perf_counter()
        n = eng.resolve_all_unknown()
        gpu_ms.append(1e3 * (time.perf_counter() - t0))
        assert n == grays[-1]
    t0 = time.perf_counter()
    reps = eng.batch_update((ids[rounds], rts[rounds]), lazy=False)
    eager_ms = 1e3 * (time.perf_counter() - t0)
    checks = int(sum(r.resolve_checks for r in reps))
    out = {"what": "resolve_all_unknown after each lazy update (64 moves), then one eager update (64 moves, each "
                   "move's gray over-hits resolved before the next); host API wall time incl. gray compaction",
           "configs": int(lv.resolver[0][-1]), "pose_upload_s": round(upload_s, 3),
           "resolve_all": {"gray_per_call": grays, "gpu_ms": gpu_ms,
                           "gpu_components_per_s": sum(grays) / (1e-3 * sum(gpu_ms))},
           "eager_update": {"moves": int(len(ids[rounds])), "resolve_checks": checks, "gpu_ms": eager_ms}}
    if cpu:
        from oracle import ref

        w = ref.World.from_roadmap(rm.robot_he, rm.env, rm.nodes, rm.edges, rm.eps, rm.max_segments)
        for he, ns in zip(obs.he, obs.spheres):
            w.add_obstacle(he, int(ns))
        re = ref.Engine(w, kind=0, threads=os.cpu_count() or 1)
        cpu_ms = []
        for r in range(min(rounds, 2)):  # bounded sample
            re.run(ids[r], rts[r], lazy=True)
            t0 = time.perf_counter()
            re.resolve_all_unknown()
            cpu_ms.append(1e3 * (time.perf_counter() - t0))
        out["resolve_all"]["cpu_ref_ms"] = cpu_ms
        out["resolve_all"]["speedup"] = statistics.mean(cpu_ms) / statistics.mean(gpu_ms[: len(cpu_ms)])
        # lock-step check: same labels after the same lazy updates + resolves
        for r in range(min(rounds, 2), rounds):
            re.run(ids[r], rts[r], lazy=True)
            re.resolve_all_unknown()
        t0 = time.perf_counter()
        re.run(ids[rounds], rts[rounds], lazy=False)
        out["eager_update"]["cpu_ref_ms"] = 1e3 * (time.perf_counter() - t0)
        out["labels_equal_reference"] = bool(np.array_equal(eng.states(), re.states()))
    return out


def measure_prm(cpu=True, reps=3):
    """PRM construction: build_prm's kNN on the GPU (csrc/rgg_prm.cu)
    through the host API (nodes H2D, edges D2H inside the wall time), at table3's 10,000
    nodes (the reference's largest shipped roadmap, timed beside it) and at the 1M-edge
    configs' 87,000 nodes (k=20; the reference would take minutes, so not run)."""

    from paper_2603_28674_b200 import prm

    out = {"what": "rgg_prm_knn_edges: k nearest nodes under dof_distance2, (min, max) pairs sorted + unique; "
                   "host API wall time (H2D nodes, D2H edges) and device time"}
    scn = os.path.join(ROOT, "tests", "golden", "scenarios", "table3_roadmap_10000.scn")
    for name, n, k, half, seed in (("table3_roadmap_10000", 10000, 8, 10.0, 105),
                                   ("n87000_k20", 87000, 20, 71.0, 12345)):
        lo, hi = prm.dof_bounds_free_flying([-half] * 3 + [half] * 3)
        nodes = prm.sample_nodes(seed, n, lo, hi)
        prm.knn_edges(nodes, k)  # warm (allocations, module load)
        wall, dev = [], []
        for _ in range(reps):
            t0 = time.perf_counter()
            edges, ms = prm.knn_edges(nodes, k, return_ms=True)
            wall.append(1e3 * (time.perf_counter() - t0))
            dev.append(ms)
        r = {"nodes": n, "k": k, "dof": 6, "edges": int(len(edges)), "gpu_wall_ms": statistics.median(wall),
             "gpu_device_ms": statistics.median(dev),
             "pairs_per_s_device": n * (n - 1) / (1e-3 * statistics.median(dev))}
        if cpu and name.startswith("table3") and os.path.exists(scn):
            from oracle import ref

            rn, re_, _, _, sec = ref.build_prm(open(scn).read())
            r["cpu_ref_ms"] = 1e3 * sec
            r["cpu_ref_note"] = "rgg::build_prm (oracle/_ref), one thread as the reference runs it, kNN + sort"
            r["speedup_wall"] = 1e3 * sec / r["gpu_wall_ms"]
            r["edges_equal_reference"] = bool(np.array_equal(rn.view(np.uint64), nodes.view(np.uint64)) and
                                              np.array_equal(re_, edges))
        out[name] = r
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2603_28674_b200 import engine as E
    from paper_2603_28674_b200 import producer

    iterations = args.warmup + args.steps
    rm, obs, _ = tile_workload(args.config, rank, args.seed, iterations)
    obs_all = obs
    if world > 1:
        from paper_2603_28674_b200 import synth

        obs_all = synth.Obstacles(he=np.tile(obs.he, (world, 1)), spheres=np.tile(obs.spheres, world))
    lv = producer.layout_for(rm, obs_all)
    eng = E.GpuEngine(lv, device=local)
    N = lv.N
    m_step = len(obs.he) * world
    if rank == 0:
        ids_h, rts_h = world_moves(args.config, world, args.seed, iterations)
    else:
        ids_h = np.zeros((iterations, m_step), np.int32)
        rts_h = np.zeros((iterations, m_step, 12))
    dev = torch.device("cuda", local)
    stream = torch.cuda.ExternalStream(eng.stream(), device=dev)
    ids_d = torch.from_numpy(ids_h).to(dev)
    rts_d = torch.from_numpy(rts_h).to(dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    up = None
    if dist is not None:
        from paper_2603_28674_b200.dist import DistributedUpdater

        up = DistributedUpdater(eng, dev)

    def step_device(it):
        if up is None:
            eng.update_device(ids_d[it].data_ptr(), rts_d[it].data_ptr(), m_step, per_move=True)
        else:  # broadcast of the moves from rank 0, shard update, all-reduce of the report counters
            up.update(ids_d[it], rts_d[it], per_move=True, check=False)

    # N = 1: the engine's own stream carries everything; N > 1: the collectives run on
    # torch's current stream and DistributedUpdater orders the engine stream against it
    tstream = stream if dist is None else torch.cuda.current_stream(dev)

    # ---- warm-up (device path), then K timed steps with L2 flushed in between; the
    # per-kernel phase split is sampled afterwards (its events would serialise the
    # pipeline's programmatic launches inside the timed steps)
    eng.set_phase_timing(False)
    for it in range(args.warmup):
        step_device(it)
    torch.cuda.synchronize()
    eng.filter_stats(reset=True)
    if dist is not None:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    classify_ms, stats = [], []
    with ClockSampler(local) as clk:
        t_clock0 = time.perf_counter()
        for k in range(args.steps):
            with torch.cuda.stream(tstream):
                flush.zero_()
            ev[k][0].record(tstream)
            step_device(args.warmup + k)
            ev[k][1].record(tstream)
        torch.cuda.synchronize()
        # keep the same load under the sampler for >= 1 s so clocks are observed under load
        n_updates = args.steps  # updates behind the filter counters below
        while time.perf_counter() - t_clock0 < args.clock_window_s:
            step_device(args.warmup + (args.steps - 1))
            torch.cuda.synchronize()
            n_updates += 1
    if up is not None:
        up.check()  # device-side errors of the stream-ordered updates
    step_ms = [a.elapsed_time(b) for a, b in ev]
    # the fp32 filters' undecided pairs (re-tested exactly) over the timed steps plus the clock window
    fstats = eng.filter_stats(reset=True)
    # phase split (untimed): the same last steps again with per-kernel events
    eng.set_phase_timing(True)
    for k in range(min(5, args.steps)):
        with torch.cuda.stream(tstream):
            flush.zero_()
        step_device(args.warmup + args.steps - 1 - k)
        st = eng.last_stats()
        classify_ms.append(st["classify_ms"])
        stats.append(st)
    eng.set_phase_timing(False)
    total_ms = float(sum(step_ms))
    if dist is not None:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    launches_per_step = 5  # pose, bin, touch, narrow, apply (one CUDA graph); gray ids are compacted on demand
    # one more (untimed) update of the last step's moves with the byte census on, then the flop census
    eng.update_device(ids_d[args.warmup + args.steps - 1].data_ptr(), rts_d[args.warmup + args.steps - 1].data_ptr(),
                      m_step, per_move=True, census=True)
    census = eng.census()
    flops = census["sat_flops"] + 21 * census["seg_sphere_tests"]
    byts = census["bytes_components"] + m_step * 768
    mean_classify = statistics.mean(classify_ms)

    # ---- e2e through the public API with host buffers (rank 0 drives; N>1 via torch collectives)
    eng_e2e = E.GpuEngine(lv, device=local)
    up_e2e = None
    if dist is not None:
        from paper_2603_28674_b200.dist import DistributedUpdater

        up_e2e = DistributedUpdater(eng_e2e, dev)
    e2e_s = []
    for it in range(iterations):
        if it >= args.warmup:
            with torch.cuda.stream(stream):
                flush.zero_()
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        if dist is None:
            reps = eng_e2e.batch_update((ids_h[it], rts_h[it]), per_move=True)
        else:
            ids_t = torch.from_numpy(ids_h[it]).pin_memory().to(dev, non_blocking=True)
            rts_t = torch.from_numpy(rts_h[it]).pin_memory().to(dev, non_blocking=True)
            reps = up_e2e.update(ids_t, rts_t, per_move=True).cpu()
        t1 = time.perf_counter()
        if it >= args.warmup:
            e2e_s.append(t1 - t0)
    e2e_total = sum(e2e_s)
    if dist is not None:
        t = torch.tensor([e2e_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    # e2e and device engines must agree on the final labels
    agree = bool(np.array_equal(eng.states(), eng_e2e.states()))

    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return 0

    n_total = N * world
    value = n_total * args.steps / (total_ms * 1e-3)
    e2e_value = n_total * args.steps / e2e_total
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    fp64 = E.fp64_peak_gflops(local)
    t_fl = flops / (fp64 * 1e9)
    t_by = byts / (hbm * 1e9)
    if t_fl >= t_by:
        roof = {"bound": "fp64", "achieved": flops / (mean_classify * 1e-3) / 1e12, "peak": fp64 / 1e3,
                "unit": "TFLOP/s", "peak_source": "measured live: non-FMA DADD/DMUL issue rate (rgg_gpu_fp64_peak)"}
    else:
        roof = {"bound": "hbm", "achieved": byts / (mean_classify * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback B200_PROFILING.md"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    # dram__bytes_read.sum + dram__bytes_write.sum of the classify kernel from the committed
    # `ncu --set full` capture (profiles/r1f_classify_ncu.json); null when absent
    roof["traffic"] = None
    pf = os.path.join(ROOT, "profiles", "r1f_classify_ncu.json")
    if os.path.exists(pf):
        try:
            p = json.load(open(pf))
            unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd, wr = p["dram__bytes_read.sum"], p["dram__bytes_write.sum"]
            roof["traffic"] = float(rd[0]) * unit[rd[1]] + float(wr[0]) * unit[wr[1]]
            roof["traffic_source"] = "profiles/r1f_classify_ncu.json (ncu --set full, one c2 update, 3 kernels)"
        except (KeyError, ValueError):
            pass
    roof["kernel"] = ("classify stage = touch_warp_kernel + narrow_kernel + apply_warp_kernel "
                      "(paper_2603_28674_b200/csrc/rgg_kernels.cu), timed together by the phase events")
    roof["algorithmic"] = {"flops_per_launch": flops, "bytes_per_launch": byts, "classify_ms_mean": mean_classify,
                           "roof_ms": 1e3 * max(t_fl, t_by), "census": census}
    line = {
        "metric": BASE_METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(args, N, world),
        "per_update_ms": total_ms / args.steps, "per_move_us": 1e3 * total_ms / args.steps / m_step,
        "e2e": {"value": e2e_value, "unit": "edges/s", "ms_per_step": 1e3 * e2e_total / args.steps,
                "h2d_bytes_per_step": m_step * (4 + 96 + 4 + 1), "d2h_bytes_per_step": m_step * 16 + 32,
                "path": "GpuEngine.batch_update -> rgg_gpu_update (host numpy moves, per-move reports)",
                "labels_equal_device_path": agree},
        "gpu_launches": launches_per_step * args.steps,
        "phase_ms_mean": {k: statistics.mean(s[k] for s in stats) for k in
                          ("pose_ms", "bin_ms", "classify_ms", "compact_ms", "total_ms")},
        "dirty_cells_mean": statistics.mean(s["dirty_cells"] for s in stats),
        "roofline": roof, "clocks": clk.summary(),
        "parity": {"mismatches_vs_reference": None, "eps_band": "none: fp32-filter-undecided pairs are re-tested with the "
                   "reference's fp64 sequence", "filter_rechecks_per_update": {k: v / n_updates for k, v in fstats.items()},
                   "over_pairs_per_update": census["over_pairs"],
                   "seg_sphere_tests_per_update": census["seg_sphere_tests"]},
    }
    if world == 1 and args.extra_configs and args.config == "c2":
        line["extra"] = {}
        for cfg in [c for c in args.extra_configs.split(",") if c and c != args.config]:
            try:
                line["extra"][cfg] = measure_extra(cfg, args.seed, local)
            except Exception as ex:  # keep the headline line even if an extra config fails
                line["extra"][cfg] = {"error": str(ex)[:200]}
    if world == 1 and args.config == "c2" and not args.no_resolve:
        try:
            line["resolve"] = measure_resolve(args.config, args.seed, local, cpu=not args.no_cpu_baseline)
        except Exception as ex:
            line["resolve"] = {"error": str(ex)[:200]}
    if world == 1 and args.config == "c2" and not args.no_resolve:
        try:
            line["prm"] = measure_prm(cpu=not args.no_cpu_baseline)
        except Exception as ex:
            line["prm"] = {"error": str(ex)[:200]}
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        n, done, spent, per_step, ref_eng = cpu_reference_run(args.config, args.seed, iterations,
                                                              args.cpu_sample_s, threads)
        cpu_v = n * done / spent
        # label parity on the full c2 tile: a fresh engine, the same `done` updates, every label compared
        eng_chk = E.GpuEngine(lv, device=local)
        for it in range(done):
            eng_chk.batch_update((ids_h[it], rts_h[it]), per_move=False)
        line["parity"]["mismatches_vs_reference"] = int(np.sum(eng_chk.states() != ref_eng.states()))
        line["parity"]["checked"] = f"{n} labels after {done} updates against rgg::BatchEngine"
        del eng_chk
        line["cpu_baseline"] = {"value": cpu_v, "unit": "edges/s", "cores": threads, "kind": "reference",
                                "sample": f"rgg::BatchEngine (AVX2, {threads} threads) on the same tile-0 roadmap "
                                          f"and moves: {done} updates x 64 moves in {spent:.1f} s",
                                "ms_per_step": 1e3 * spent / done}
    print(json.dumps(line), flush=True)
    if args.json_out:
        json.dump(line, open(args.json_out, "w"), indent=1)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
