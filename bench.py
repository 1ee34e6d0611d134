#!/usr/bin/env python
"""bench.py — SerRGG edge classification on B200: edges classified/s and per-update latency.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Workload (the north star's target, BASELINE.json configs[4], "c5"): SE(2) roadmap,
87,000 nodes / 988,896 edges (N = 1,075,896 components incl. nodes), 1024 moving
yaw-rotated box obstacles.  One STEP = one update of the obstacle set = all 1024
obstacles re-posed through ``batch_update`` with per-move UpdateReports (the
reference's 1024 calls to BatchEngine::update_obstacle, proj/src/engine_batch.cpp:
145-215, with the GRAY-id list compacted on the device, :193-200).  After each step
every one of the N labels is the reference's, so

    value = N_components x steps / device time          ("edges/s")
    per-update latency = ms_per_step

* ``value``: moves already resident in HBM, CUDA events on the engine's stream, L2
  flushed (512 MB write) between steps; the update includes the gray-list compaction.
* ``e2e``: the same steps through the public API with HOST buffers
  (GpuEngine.batch_update -> rgg_gpu_update: H2D of the moves, D2H of the per-move
  reports, then the GRAY ids D2H), wall clock around the calls.
* ``--impl reference``: the reference's own CPU SerRGG path on the same roadmap and
  moves (oracle/_ref, built from /root/reference's sources): ceil(1024/64) = 16
  grouped SequentialEngines (the reference refuses > 64 obstacles per engine,
  engine_batch.cpp:27; SequentialEngine is its fastest CPU path at c5).
* N > 1 (torchrun, one rank per GPU, NCCL): strong scaling of the same c5 roadmap.
  Rank r owns the Morton-ordered cells c with c % N == r; per step the moves are
  broadcast from rank 0, the per-move report counters all-reduced and the GRAY-id
  lists gathered to rank 0 (paper_2603_28674_b200/dist.py).
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
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="c5")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--seed", type=int, default=12345)
    p.add_argument("--cpu-sample-s", type=float, default=8.0, help="CPU seconds per reference-engine sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip the other configs, resolve and PRM")
    p.add_argument("--json-out", default="")
    p.add_argument("--clock-window-s", type=float, default=1.0)
    p.add_argument("--extra-configs", default="c2,c3,c4,c1")
    return p.parse_args()


# ------------------------------------------------------------------ workloads

def tile_workload(config, rank, seed, iterations):
    """The config's roadmap and obstacle set (rank kept for the tools' call signature:
    tile r is the roadmap shifted by r tiles in x)."""
    from paper_2603_28674_b200 import synth

    kind, nodes, k, half, m, ohalf = synth.CONFIGS[config]
    rm = synth.make_roadmap(kind, nodes, k, half, seed + 1000 * rank)
    obs = synth.make_obstacles(kind, m, seed + 1)
    shift = 2.0 * (ohalf + 5.0) * rank
    rm.nodes[:, 0] += shift
    rm.env[[0, 3]] += shift
    return rm, obs, shift


def world_moves(config, world, seed, iterations):
    """The move script [iteration][move]: every obstacle once per iteration, or the
    rotating subset of MOVES_PER_STEP (c4's ~5 % dirty cells)."""
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
    return np.ascontiguousarray(ids), np.ascontiguousarray(rts)


def workload_name(config, n_components):
    from paper_2603_28674_b200 import synth

    kind, nodes, k, half, m, ohalf = synth.CONFIGS[config]
    mv = synth.MOVES_PER_STEP.get(config)
    step = (f"1 step = 1 update = {mv} of the {m} obstacles re-posed (rotating subset, ~5 % of cells dirty: "
            f"see dirty_fraction)"
            if mv else f"1 step = 1 update = all {m} obstacles re-posed")
    return (f"{config}: {'SE(2)' if kind == 'se2' else '3D'} roadmap {nodes} nodes k={k} ({n_components} components "
            f"incl. nodes) x {m} moving OBB obstacles; {step} (per-move reports, gray-id list compacted on device)")


def config_dict(config, n_components, world=1):
    from paper_2603_28674_b200 import synth

    m = synth.CONFIGS[config][4]
    return {"workload": workload_name(config, n_components), "components": n_components, "obstacles": m,
            "moves_per_step": synth.MOVES_PER_STEP.get(config) or m,
            "l2": "flushed (512 MB write) between timed steps",
            "parallelism": (f"{world} shards of one roadmap (interleaved Morton cells), obstacles replicated, "
                            f"moves broadcast, counters all-reduced, gray ids gathered" if world > 1 else "1 GPU"),
            "precision": "verdicts exact: fp32 filters with proven error bounds, fp64 reference op order otherwise"}


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


def host_info():
    model = ""
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model}


# ------------------------------------------------------------ reference (CPU)

def ref_world(rm, obs):
    from oracle import ref

    w = ref.World.from_roadmap(rm.robot_he, rm.env, rm.nodes, rm.edges, rm.eps, rm.max_segments)
    for he, ns in zip(obs.he, obs.spheres):
        w.add_obstacle(he, int(ns))
    return w


def ref_engine_kind(m, threads):
    """The reference engine a CPU arm runs: SequentialEngine, the reference's fastest
    CPU path wherever we probed it, grouped by 64 obstacles; the
    groups' independent engines run concurrently on the host threads."""
    groups = (m + 63) // 64
    return 1, (f"rgg::SequentialEngine x {groups} obstacle groups of <= 64 (engine_batch.cpp:27 caps an engine "
               f"at 64), the groups' engines on {min(threads, groups)} host threads" if groups > 1
               else "rgg::SequentialEngine, 1 thread (single-threaded by design)")


def run_reference(args):
    """--impl reference: the reference's own CPU path (oracle/_ref) on this arm's
    workload, metric and unit; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import ref

    iterations = args.warmup + args.steps
    rm, obs, _ = tile_workload(args.config, 0, args.seed, iterations)
    t0 = time.time()
    w = ref_world(rm, obs)
    threads = os.cpu_count() or 1
    kind, what = ref_engine_kind(len(obs.he), threads)
    eng = ref.Engine(w, kind=kind, threads=1, group_size=64)
    build_s = time.time() - t0
    ids, rts = world_moves(args.config, 1, args.seed, iterations)
    n = w.counts()["N"]
    cores = min(threads, eng.groups)
    per = [eng.run_parallel(ids[it], rts[it], cores, lazy=True) * 1e-6 for it in range(iterations)]
    timed = per[args.warmup:]
    t = sum(timed)
    value = n * len(timed) / t
    line = {
        "impl": "reference", "metric": BASE_METRIC, "value": value, "unit": "edges/s", "n_gpus": args.gpus,
        "steps": len(timed), "warmup": args.warmup, "ms_per_step": 1e3 * t / len(timed), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config, n),
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": cores, "kind": "reference",
                         "sample": f"{what}, oracle/_ref/librgg_ref.so: {len(timed)} full updates of "
                                   f"{ids.shape[1]} moves each (+{args.warmup} untimed); engines built in "
                                   f"{build_s:.0f} s", "host": host_info()},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baselines(config, rm, obs, ids, rts, sample_s, parity_updates=2):
    """The reference's CPU engines on the headline workload:
    grouped SequentialEngine (1 thread), BatchEngine with 1 thread and with all host
    threads.  Returns (baselines, sequential engine after its updates, updates run)."""
    from oracle import ref

    m = len(obs.he)
    groups = (m + 63) // 64
    nproc = os.cpu_count() or 1
    out = {"host": host_info()}
    t0 = time.time()
    w = ref_world(rm, obs)
    out["world_build_s"] = round(time.time() - t0, 1)
    n = w.counts()["N"]
    # grouped SequentialEngines over whole updates (also the parity reference): the
    # first updates on one thread, the next with the groups' engines on all host threads
    t0 = time.time()
    seq = ref.Engine(w, kind=1, threads=1, group_size=64)
    build = time.time() - t0
    per1, per_n, spent, done = [], [], 0.0, 0
    for it in range(len(ids)):
        par = len(per1) >= parity_updates // 2 + 1 and spent >= sample_s / 2 and groups > 1
        s = (seq.run_parallel(ids[it], rts[it], nproc) if par else seq.run(ids[it], rts[it], lazy=True)) * 1e-6
        (per_n if par else per1).append(s)
        spent += s
        done += 1
        if done >= parity_updates and spent >= sample_s and (per_n or groups == 1):
            break
    out["sequential_1t"] = {"ms_per_update": 1e3 * statistics.mean(per1), "edges_per_s": n / statistics.mean(per1),
                            "cores": 1, "build_s": round(build, 1),
                            "sample": f"{len(per1)} full updates x {ids.shape[1]} moves, {groups} grouped engines "
                                      f"run one after the other"}
    if per_n:
        out[f"sequential_{nproc}t"] = {"ms_per_update": 1e3 * statistics.mean(per_n),
                                       "edges_per_s": n / statistics.mean(per_n), "cores": min(nproc, groups),
                                       "sample": f"{len(per_n)} full updates x {ids.shape[1]} moves, the {groups} "
                                                 f"grouped engines on {min(nproc, groups)} host threads"}
    # BatchEngine: a bounded sample, the first obstacle group's moves of each update
    # (its engine holds the whole roadmap, ~64 B/comp per group of layout); the per-update
    # figure scales the per-move time by the moves per update
    for threads in (1, nproc):
        t0 = time.time()
        bat = ref.Engine(w, kind=0, threads=threads, group_size=64, max_groups=1)
        build = time.time() - t0
        mv_s, nmv, spent = [], 0, 0.0
        for it in range(len(ids)):
            sel = ids[it] < 64
            if not sel.any():
                continue
            s = bat.run(np.ascontiguousarray(ids[it][sel]), np.ascontiguousarray(rts[it][sel]), lazy=True) * 1e-6
            nmv += int(sel.sum())
            spent += s
            if spent >= sample_s / 2:
                break
        per_move = spent / max(1, nmv)
        ms = 1e3 * per_move * ids.shape[1]
        out[f"batch_{threads}t"] = {"ms_per_update": ms, "edges_per_s": n / (ms * 1e-3), "cores": threads,
                                    "build_s_one_group": round(build, 1),
                                    "sample": f"{nmv} moves of obstacle group 0 (one BatchEngine over all {n} "
                                              f"components), {1e3 * per_move:.2f} ms/move x {ids.shape[1]} moves"}
        del bat
    best = min((k for k in out if k.startswith(("sequential_", "batch_"))), key=lambda k: out[k]["ms_per_update"])
    out["fastest"] = best
    return out, seq, done, n


def cpu_reference_run(config, seed, iterations, sample_s, out_path):
    """cpu_baselines on the headline workload, rebuilt from its seed (run_isolated's child);
    the grouped SequentialEngines' labels and bits after the updates they ran go to out_path."""
    rm, obs, _ = tile_workload(config, 0, seed, iterations)
    ids, rts = world_moves(config, 1, seed, iterations)
    base, seq, done, _ = cpu_baselines(config, rm, obs, ids, rts, sample_s)
    np.savez(out_path, states=np.asarray(seq.states()), bits=np.asarray(seq.bits()))
    return {"baselines": base, "done": done}


# --------------------------------------------------------------- GPU helpers

def measure_extra(config, seed, device, steps=10, warmup=3, cell_capacity=64, parity=False):
    """A further BASELINE config on one GPU (device-resident moves, L2 flushed between
    updates): per-update latency and edges/s, the census of one update; parity
    against the pinned C oracle's pure-function labels and bits when asked."""
    import torch

    from paper_2603_28674_b200 import engine as E
    from paper_2603_28674_b200 import producer, synth

    t0 = time.time()
    rm, obs, _ = tile_workload(config, 0, seed, warmup + steps)
    lv = producer.layout_for(rm, obs)
    build_s = time.time() - t0
    eng = E.GpuEngine(lv, device=device, cell_capacity=cell_capacity)
    ids_h, rts_h = world_moves(config, 1, seed, warmup + steps)
    dev = torch.device("cuda", device)
    ids_d = torch.from_numpy(ids_h).to(dev)
    rts_d = torch.from_numpy(rts_h).to(dev)
    m = ids_h.shape[1]
    stream = torch.cuda.ExternalStream(eng.stream(), device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for it in range(warmup):
        eng.update_device(ids_d[it].data_ptr(), rts_d[it].data_ptr(), m, per_move=True, gray_list=True)
    torch.cuda.synchronize()
    ms = []
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.update_device(ids_d[warmup + k].data_ptr(), rts_d[warmup + k].data_ptr(), m, per_move=True,
                          gray_list=True)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    eng.sync()
    st = eng.last_stats()
    last = warmup + steps - 1
    eng.update_device(ids_d[last].data_ptr(), rts_d[last].data_ptr(), m, per_move=True, census=True)
    cen = eng.census()
    per = statistics.mean(ms)
    ncells = (lv.N + 127) // 128
    out = {"workload": workload_name(config, lv.N), "components": lv.N, "moves_per_update": m,
           "per_update_ms": per,
           # incremental configs: the components of the dirty cells are the ones relabelled
           "value": (min(lv.N, st["dirty_cells"] * 128) if synth.MOVES_PER_STEP.get(config) else lv.N) / (per * 1e-3),
           "value_all_components": lv.N / (per * 1e-3), "unit": "edges/s", "steps": steps,
           "build_s": round(build_s, 1), "cell_capacity": cell_capacity, "dirty_cells": st["dirty_cells"],
           "dirty_fraction": st["dirty_cells"] / max(1, ncells), "overflow_cells": st["overflow_cells"],
           "census": {k: cen[k] for k in ("over_pairs", "sat_flops", "under_pairs", "seg_sphere_tests",
                                           "bytes_components", "bytes_fp32", "gray")}}
    if parity:
        from oracle import oracle as O

        ora = O.Engine(lv)
        t0 = time.time()
        for it in range(last + 1):
            for o, rt in zip(ids_h[it], rts_h[it]):
                ora.update(int(o), rt)
        sts, bits = ora.pure()
        got_bits = eng.obstacle_bits().reshape(lv.N, -1)
        out["parity"] = {"mismatches_vs_oracle": int(np.sum(eng.states() != sts)),
                         "bit_word_mismatches": int(np.sum(got_bits != bits.reshape(got_bits.shape))),
                         "checked": f"{lv.N} labels and {got_bits.size} bit words after {last + 1} updates against "
                                    f"the pinned C oracle's pure-function labels (oracle/rgg_oracle.c ro_engine_pure)",
                         "oracle_s": round(time.time() - t0, 1)}
    return out


def measure_c1(device, reps=20):
    """C1 (BASELINE configs[0]): table4_obstacles_1000_5x as shipped.
    Replay iteration 1 (activates all 5 obstacles), then time ONE update_obstacle,
    the first move of iteration 2, through the host API; the reference engines time
    the same single move on the same state."""
    from oracle import ref
    from paper_2603_28674_b200 import engine as E

    scn = os.path.join(ROOT, "tests", "golden", "scenarios", "table4_obstacles_1000_5x.scn")
    w = ref.World.from_scn(open(scn).read())
    k = w.counts()
    lay = w.layout()
    ids, rts = w.moves()
    m = k["M"]
    lv = E.LayoutView.from_any(lay)
    out = {"workload": f"c1: table4_obstacles_1000_5x ({k['N']} components, {m} obstacles); one update_obstacle "
                       f"(the first move of iteration 2) after replaying iteration 1"}
    gpu = []
    for _ in range(reps):
        eng = E.GpuEngine(lv, device=device)
        for o, rt in zip(ids[:m], rts[:m]):  # iteration 1, one move at a time (the single-move graph is built here)
            eng.update_obstacle(int(o), rt)
        t0 = time.perf_counter()
        eng.update_obstacle(int(ids[m]), rts[m])
        gpu.append(1e6 * (time.perf_counter() - t0))
        last = eng
    out["gpu_us"] = statistics.median(gpu)
    cpu = {}
    for name, kind, threads in (("sequential_1t", 1, 1), ("batch_1t", 0, 1), (f"batch_{os.cpu_count()}t", 0,
                                                                                 os.cpu_count() or 1)):
        us = []
        for _ in range(reps):
            e = ref.Engine(w, kind=kind, threads=threads)
            e.run(ids[:m], rts[:m])
            us.append(e.run(ids[m:m + 1], rts[m:m + 1]))
        cpu[name] = statistics.median(us)
        if name == "batch_1t":
            out["labels_equal_reference"] = bool(np.array_equal(last.states(), e.states()))
    out["cpu_us"] = cpu
    out["speedup_vs_fastest_cpu"] = min(cpu.values()) / out["gpu_us"]
    return out


def measure_resolve(config, seed, device, rounds=4, cpu=True):
    """The exact resolve on the GPU: resolve_all_unknown after
    each lazy update, and one eager update, through the host API; the reference's
    own resolve_all_unknown / eager update_obstacle on the same roadmap and moves."""
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
    out = {"what": f"{config}: resolve_all_unknown after each lazy update ({ids.shape[1]} moves), then one eager "
                   f"update (each move's gray over-hits resolved before the next); host API wall time",
           "configs": int(lv.resolver[0][-1]), "pose_upload_s": round(upload_s, 3),
           "resolve_all": {"gray_per_call": grays, "gpu_ms": gpu_ms,
                           "gpu_components_per_s": sum(grays) / (1e-3 * sum(gpu_ms))},
           "eager_update": {"moves": int(len(ids[rounds])), "resolve_checks": checks, "gpu_ms": eager_ms}}
    if cpu:
        from oracle import ref

        w = ref_world(rm, obs)
        re = ref.Engine(w, kind=0, threads=os.cpu_count() or 1)
        cpu_ms = []
        for r in range(min(rounds, 2)):  # bounded sample
            re.run(ids[r], rts[r], lazy=True)
            t0 = time.perf_counter()
            re.resolve_all_unknown()
            cpu_ms.append(1e3 * (time.perf_counter() - t0))
        out["resolve_all"]["cpu_ref_ms"] = cpu_ms
        out["resolve_all"]["speedup"] = statistics.mean(cpu_ms) / statistics.mean(gpu_ms[: len(cpu_ms)])
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
    nodes (timed beside the reference) and at the 1M-edge configs' 87,000 nodes."""
    from paper_2603_28674_b200 import prm

    out = {"what": "rgg_prm_knn_edges: k nearest nodes under dof_distance2, (min, max) pairs sorted + unique; "
                   "host API wall time (H2D nodes, D2H edges) and device time"}
    scn = os.path.join(ROOT, "tests", "golden", "scenarios", "table3_roadmap_10000.scn")
    for name, n, k, half, seed in (("table3_roadmap_10000", 10000, 8, 10.0, 105),
                                   ("n87000_k20", 87000, 20, 71.0, 12345)):
        lo, hi = prm.dof_bounds_free_flying([-half] * 3 + [half] * 3)
        nodes = prm.sample_nodes(seed, n, lo, hi)
        prm.knn_edges(nodes, k)
        wall, dev = [], []
        for _ in range(reps):
            t0 = time.perf_counter()
            edges, ms = prm.knn_edges(nodes, k, return_ms=True)
            wall.append(1e3 * (time.perf_counter() - t0))
            dev.append(ms)
        r = {"nodes": n, "k": k, "dof": 6, "edges": int(len(edges)), "gpu_wall_ms": statistics.median(wall),
             "gpu_device_ms": statistics.median(dev)}
        if cpu and name.startswith("table3") and os.path.exists(scn):
            from oracle import ref

            rn, re_, _, _, sec = ref.build_prm(open(scn).read())
            r["cpu_ref_ms"] = 1e3 * sec
            r["speedup_wall"] = 1e3 * sec / r["gpu_wall_ms"]
            r["edges_equal_reference"] = bool(np.array_equal(rn.view(np.uint64), nodes.view(np.uint64)) and
                                              np.array_equal(re_, edges))
        out[name] = r
    return out


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def roofline(census, kernel_ms, world, profile_json=None):
    """HBM roofline of the update (the slower of the FP32 test rate and HBM for the
    census bytes): achieved = algorithmic bytes (fp32 model) / time."""
    from paper_2603_28674_b200 import engine as E

    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6550.0))
    fp32 = E.fp32_peak_gflops(0)
    flops = census["sat_flops"] + 21 * census["seg_sphere_tests"]
    byts = census["bytes_fp32"]
    t_fl, t_by = flops / (fp32 * 1e9), byts / (hbm * 1e9)
    roof = {"bound": "hbm" if t_by >= t_fl else "fp32",
            "achieved": byts / (kernel_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk else "fallback B200_PROFILING.md",
            "kernel": "the whole update (pose, bin scatter + cell lists, touch, narrow over + under, apply, gray compaction: "
                      "paper_2603_28674_b200/csrc/rgg_kernels.cu), timed with CUDA events per update",
            "algorithmic": {"bytes_per_update": byts, "bytes_model": "SURVEY.md §8(d) fp32 model (DESIGN.md §4)",
                            "bytes_fp64_records": census["bytes_components"], "flops_per_update": flops,
                            "fp32_peak_gflops_measured": fp32, "t_bytes_ms": 1e3 * t_by, "t_flops_ms": 1e3 * t_fl,
                            "per_shard": world > 1}}
    if roof["bound"] == "fp32":
        roof.update(achieved=flops / (kernel_ms * 1e-3) / 1e12, peak=fp32 / 1e3, unit="TFLOP/s",
                    peak_source="measured live: FFMA issue rate (rgg_gpu_fp32_peak)")
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = None
    if profile_json and os.path.exists(profile_json):
        try:
            p = json.load(open(profile_json))
            roof["traffic"] = p["dram_bytes_per_update"]
            roof["traffic_source"] = os.path.relpath(profile_json, ROOT)
        except (KeyError, ValueError):
            pass
    return roof


# ---------------------------------------------------------------------- main

def run_isolated(fn: str, *args, **kwargs) -> dict:
    """bench.<fn>(*args, **kwargs) in a child process (its JSON result), or {"error": ...}."""
    code = ("import json, sys; sys.path.insert(0, %r); import bench; "
            "a = json.loads(sys.argv[1]); print(json.dumps(getattr(bench, %r)(*a['args'], **a['kwargs'])))"
            % (ROOT, fn))
    try:
        r = subprocess.run([sys.executable, "-X", "faulthandler", "-c", code,
                            json.dumps({"args": list(args), "kwargs": kwargs})],
                           capture_output=True, text=True, timeout=1800, cwd=ROOT)
    except subprocess.TimeoutExpired:
        return {"error": f"{fn}: timed out"}
    if r.returncode != 0:
        return {"error": f"{fn}: exit {r.returncode}: " + (r.stderr or "")[-400:]}
    try:
        return json.loads(r.stdout.strip().splitlines()[-1])
    except (ValueError, IndexError):
        return {"error": f"{fn}: no JSON result: " + (r.stdout or "")[-200:]}


def main():
    import faulthandler

    faulthandler.enable()  # a native crash prints the Python stacks to stderr
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    # RGG_BENCH_DIST=1 (tests, under torchrun): the N > 1 path (NCCL collectives) at any N
    if world > 1 or os.environ.get("RGG_BENCH_DIST") == "1":
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2603_28674_b200 import engine as E
    from paper_2603_28674_b200 import producer

    iterations = args.warmup + args.steps
    rm, obs, _ = tile_workload(args.config, 0, args.seed, iterations)
    lv = producer.layout_for(rm, obs)
    N = lv.N
    eng = E.GpuEngine(lv, device=local, shard_rank=rank, shard_count=world)
    ids_h, rts_h = world_moves(args.config, 1, args.seed, iterations)
    m_step = ids_h.shape[1]
    dev = torch.device("cuda", local)
    stream = torch.cuda.ExternalStream(eng.stream(), device=dev)
    if rank == 0:
        ids_d, rts_d = torch.from_numpy(ids_h).to(dev), torch.from_numpy(rts_h).to(dev)
    else:  # filled by the broadcast inside each step
        ids_d = torch.zeros((iterations, m_step), dtype=torch.int32, device=dev)
        rts_d = torch.zeros((iterations, m_step, 12), dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    up = None
    if dist is not None:
        from paper_2603_28674_b200.dist import DistributedUpdater

        np_max = torch.tensor([eng.n_owned], dtype=torch.int64, device=dev)
        dist.all_reduce(np_max, op=dist.ReduceOp.MAX)
        up = DistributedUpdater(eng, dev, gray_cap=int(np_max.item()))

    def step_device(it):
        if up is None:
            eng.update_device(ids_d[it].data_ptr(), rts_d[it].data_ptr(), m_step, per_move=True, gray_list=True)
        else:  # move broadcast, shard update, counter all-reduce, gray-list gather: all stream-ordered
            up.update(ids_d[it], rts_d[it], per_move=True, check=False, gather_gray=True)

    # N = 1: the engine's stream carries everything; N > 1: the collectives run on torch's
    # current stream and DistributedUpdater orders the engine stream against it
    tstream = stream if dist is None else torch.cuda.current_stream(dev)
    eng.set_phase_timing(False)
    for it in range(args.warmup):
        step_device(it)
    torch.cuda.synchronize()
    if up is not None:
        up.check()
    eng.filter_stats(reset=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        t_clock0 = time.perf_counter()
        for k in range(args.steps):
            with torch.cuda.stream(tstream):
                flush.zero_()
            ev[k][0].record(tstream)
            step_device(args.warmup + k)
            ev[k][1].record(tstream)
        torch.cuda.synchronize()
        n_updates = args.steps
        while time.perf_counter() - t_clock0 < args.clock_window_s:  # >= 1 s of the same load under the sampler
            step_device(args.warmup + args.steps - 1)
            torch.cuda.synchronize()
            n_updates += 1
    if up is not None:
        up.check()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(step_ms))
    if dist is not None:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    fstats = eng.filter_stats(reset=True)
    # kernel-only time of one update on this shard (no collectives), then the phase split
    # (untimed: per-kernel events serialise the programmatic launches) and the census
    kern_ms = []
    for k in range(min(10, args.steps)):
        it = args.warmup + k
        with torch.cuda.stream(stream):
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.update_device(ids_d[it].data_ptr(), rts_d[it].data_ptr(), m_step, per_move=True, gray_list=True)
        b.record(stream)
        torch.cuda.synchronize()
        kern_ms.append(a.elapsed_time(b))
    eng.set_phase_timing(True)
    stats = []
    for k in range(3):
        with torch.cuda.stream(stream):
            flush.zero_()
        it = args.warmup + args.steps - 1 - k
        eng.update_device(ids_d[it].data_ptr(), rts_d[it].data_ptr(), m_step, per_move=True, gray_list=True)
        stats.append(eng.last_stats())
    eng.set_phase_timing(False)
    last = args.warmup + args.steps - 1
    eng.update_device(ids_d[last].data_ptr(), rts_d[last].data_ptr(), m_step, per_move=True, census=True)
    census = eng.census()
    eng.close()

    # ---- e2e through the public API with host buffers
    eng_e2e = E.GpuEngine(lv, device=local, shard_rank=rank, shard_count=world)
    stream = torch.cuda.ExternalStream(eng_e2e.stream(), device=dev)  # the first engine's stream is gone
    up_e2e = None
    if dist is not None:
        from paper_2603_28674_b200.dist import DistributedUpdater

        up_e2e = DistributedUpdater(eng_e2e, dev, gray_cap=up.gray_cap)
    e2e_s, d2h, ngray = [], [], 0
    # each step's moves sit in pinned host memory when the step starts (the engine's staging
    # buffers, rgg_gpu_stage, at N = 1); the host-to-device copy is inside the timed region
    if dist is not None:
        pin_ids_t = torch.empty((m_step,), dtype=torch.int32, pin_memory=True)
        pin_rts_t = torch.empty((m_step, 12), dtype=torch.float64, pin_memory=True)
        pin_ids, pin_rts = pin_ids_t.numpy(), pin_rts_t.numpy()
    else:
        pin_ids, pin_rts = eng_e2e.staging(m_step)
    for it in range(iterations):
        if it >= args.warmup:
            with torch.cuda.stream(stream):
                flush.zero_()
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
        pin_ids[:] = ids_h[it]
        pin_rts[:] = rts_h[it]
        t0 = time.perf_counter()
        if dist is None:
            reps = eng_e2e.batch_update((pin_ids, pin_rts), per_move=True, gray_list=True)
            gray = eng_e2e.gray_ids_view()  # written into mapped host memory by the update
        else:
            ids_t = pin_ids_t.to(dev, non_blocking=True)
            rts_t = pin_rts_t.to(dev, non_blocking=True)
            reps = up_e2e.update(ids_t, rts_t, per_move=True, gather_gray=True).cpu()
            gray = up_e2e.gathered_gray()
        t1 = time.perf_counter()
        if it >= args.warmup:
            e2e_s.append(t1 - t0)
            ngray = 0 if gray is None else len(gray)
            d2h.append(m_step * 16 + 96 + 4 * ngray)
    e2e_total = sum(e2e_s)
    if dist is not None:
        t = torch.tensor([e2e_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    labels_e2e = eng_e2e.states() if dist is None else up_e2e.states(N)
    eng_e2e.close()

    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return 0

    value = N * args.steps / (total_ms * 1e-3)
    e2e_value = N * args.steps / e2e_total
    per_update = total_ms / args.steps
    import glob

    prof = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r2*_{args.config}_ncu.json")))
    roof = roofline(census, statistics.mean(kern_ms), world, prof[-1] if prof else None)
    line = {
        "metric": BASE_METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_update, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded roadmap, obstacles and poses of the named shape)",
        "config": config_dict(args.config, N, world),
        "per_update_ms": per_update, "per_move_us": 1e3 * per_update / m_step,
        "kernel_ms_per_update": statistics.mean(kern_ms),
        "e2e": {"value": e2e_value, "unit": "edges/s", "ms_per_step": 1e3 * e2e_total / args.steps,
                "h2d_bytes_per_step": m_step * (4 + 96), "d2h_bytes_per_step": int(statistics.mean(d2h)),
                "path": "moves in the engine's pinned staging buffers (rgg_gpu_stage) -> GpuEngine.batch_update "
                        "(per-move reports, gray list) -> rgg_gpu_update: H2D copy, update, reports and gray ids "
                        "written into mapped host memory; then gray_ids_view()" + (" ; N>1: pinned H2D on every rank, DistributedUpdater (broadcast, "
                                            "all-reduce, gray gather), reports + gray ids D2H on rank 0"
                                            if world > 1 else "")},
        "gpu_launches": 9 * args.steps,
        "gpu_launches_note": "per update: pose, bin scatter, bin cells, touch, narrow over, narrow under, apply, gray "
                             "count, gray write "
                             "(one CUDA graph)",
        "phase_ms_mean": {k: statistics.mean(s[k] for s in stats) for k in
                          ("pose_ms", "bin_ms", "classify_ms", "compact_ms", "total_ms")},
        "dirty_cells": stats[0]["dirty_cells"], "overflow_cells": stats[0]["overflow_cells"],
        "gray_after_update": census["gray"],
        "roofline": roof, "clocks": clk.summary(),
        "parity": {"mismatches_vs_reference": None,
                   "eps_band": "none: fp32-filter-undecided pairs are re-tested with the reference's fp64 sequence",
                   "filter_rechecks_per_update": {k: v / n_updates for k, v in fstats.items()},
                   "over_pairs_per_update": census["over_pairs"],
                   "seg_sphere_tests_per_update": census["seg_sphere_tests"]},
    }
    if world == 1 and not args.no_cpu_baseline:
        # the reference's CPU engines in a child process (it saves its labels and bits after
        # `done` updates), so a failure there cannot take the headline line with it
        import tempfile

        with tempfile.TemporaryDirectory() as tmp:
            res = run_isolated("cpu_reference_run", args.config, args.seed, iterations, args.cpu_sample_s,
                               os.path.join(tmp, "ref.npz"))
            if "error" in res:
                raise RuntimeError("reference CPU run failed: " + res["error"])
            with np.load(os.path.join(tmp, "ref.npz")) as z:
                ref_states, ref_bits = z["states"], z["bits"]
        base, done = res["baselines"], res["done"]
        # label and bit parity on the full roadmap: a fresh engine, the same `done` updates
        eng_chk = E.GpuEngine(lv, device=local)
        reps_chk = []
        for it in range(done):
            reps_chk.append(eng_chk.batch_update((ids_h[it], rts_h[it]), per_move=True).counts())
        gst = eng_chk.states()
        gbits = eng_chk.obstacle_bits().reshape(N, -1)
        rbits = ref_bits
        line["parity"]["mismatches_vs_reference"] = int(np.sum(gst != ref_states))
        line["parity"]["bit_word_mismatches_vs_reference"] = int(np.sum(gbits != rbits.reshape(gbits.shape)))
        line["parity"]["checked"] = (f"{N} labels and {gbits.size} obstacle-bit words after {done} updates against "
                                     f"the reference's grouped SequentialEngines ({rbits.shape[1]} x 64 obstacles)")
        line["parity"]["labels_equal_e2e_path"] = bool(np.array_equal(labels_e2e, gst)) if done == iterations else None
        # per-move reports: the pinned C oracle (one ungrouped engine; the reference caps an
        # engine at 64 obstacles, so it has no per-move reports for M > 64)
        from oracle import oracle as O

        t0 = time.time()
        ora = O.Engine(lv)
        bad = 0
        n_rep = min(done, 2)
        for it in range(n_rep):
            exp = np.array([ora.update(int(o), rt) for o, rt in zip(ids_h[it], rts_h[it])])
            bad += int(np.sum(np.any(exp[:, :4] != reps_chk[it], 1)))
        line["parity"]["report_mismatches_vs_oracle"] = bad
        line["parity"]["reports_checked"] = (f"{n_rep * m_step} per-move reports (new_green, new_red, new_gray, "
                                             f"unknown_after_heuristic) of updates 0..{n_rep - 1} against the pinned C "
                                             f"oracle's engine (oracle/rgg_oracle.c ro_engine_update), "
                                             f"{time.time() - t0:.0f} s")
        del eng_chk
        fast = base[base["fastest"]]
        line["cpu_baseline"] = {"value": fast["edges_per_s"], "unit": "edges/s", "cores": fast["cores"],
                                "kind": "reference", "ms_per_step": fast["ms_per_update"],
                                "sample": f"the fastest of the reference's CPU engines on this workload "
                                          f"({base['fastest']}): {fast['sample']}",
                                "all": base}
    if world == 1 and not args.no_extras:
        # each extra measurement in its own process: a failure there (even a native one)
        # cannot take the headline line with it
        line["extra"] = {}
        for cfg in [c for c in args.extra_configs.split(",") if c and c != args.config]:
            if cfg == "c1":
                line["extra"][cfg] = run_isolated("measure_c1", local)
            elif cfg == "c3":  # fixed-capacity overflow: 16 inline slots per cell
                line["extra"][cfg] = run_isolated("measure_extra", cfg, args.seed, local, cell_capacity=16, parity=True)
            else:  # c2, c4: parity against the oracle too
                line["extra"][cfg] = run_isolated("measure_extra", cfg, args.seed, local, parity=True)
        line["resolve"] = run_isolated("measure_resolve", "c2", args.seed, local, cpu=not args.no_cpu_baseline)
        line["prm"] = run_isolated("measure_prm", cpu=not args.no_cpu_baseline)
    print(json.dumps(line), flush=True)
    if args.json_out:
        json.dump(line, open(args.json_out, "w"), indent=1)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
