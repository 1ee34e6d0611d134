"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/librgg_ref.so).

ORACLE / TEST INFRASTRUCTURE.  Run in the build container (needs /root/reference
to build oracle/_ref):

    make -C oracle && python -m oracle.gen_golden

Every fixture records what the reference computes on a seeded input:
  kat_sat.npz        proj/tests/test_kernels.cpp:46-87 (seed 2025) — SAT bytes
  kat_seg.npz        proj/tests/test_kernels.cpp:89-121 (seed 777) — seg-sphere bytes
  kat_pairs.npz      random_obb pairs (proj/tests/oracles.hpp:98-109) + sat_margin (:62-84)
  kat_obstacle.npz   BatchLayout::update_transforms (proj/src/batch_layout.cpp:148-172)
  prm.npz            build_prm (proj/src/roadmap.cpp:56-102) nodes + edges per scenario
  scn_*.npz          engine replays: layout + move script + BatchEngine reports after
                     every move + states/bits snapshots (proj/src/engine_batch.cpp:145-205),
                     plus batch_over/batch_under masks (:55-112)
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import ref  # noqa: E402
from paper_2603_28674_b200 import synth  # noqa: E402

REF_SCN = "/root/reference/proj/scenarios"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def layout_arrays(L: ref.Layout, with_corners=False):
    d = dict(N=L.N, B=L.B, S=L.S, K=L.K, M=L.M, C=L.C, n_nodes=L.n_nodes, n_edges=L.n_edges,
             edge_sat=L.edge_sat, comp_aabb=L.comp_aabb, row_off=L.row_off, segs=L.segs,
             spline_r=L.spline_r, obst_he=L.obst_he, obst_sph_local=L.obst_sph_local,
             obst_sph_r=L.obst_sph_r, obst_sph_n=L.obst_sph_n)
    if with_corners:
        d["e_plus"] = L.e_plus
        d["seg_pts"] = L.seg_pts
    return d


def replay(world: ref.World, ids, rts, name, snap_every=1, snap_first=None, with_corners=False, lazy=True):
    L = world.layout()
    eng = ref.Engine(world, kind=0, threads=1)
    reports, snaps_at, snap_states, snap_bits = [], [], [], []
    for i in range(len(ids)):
        rep = eng.update(ids[i], rts[i], lazy=lazy)
        reports.append(rep[[1, 2, 3, 8, 9]])
        take = (snap_first is not None and i < snap_first) or ((i + 1) % snap_every == 0) or i == len(ids) - 1
        if take:
            snaps_at.append(i)
            snap_states.append(eng.states())
            snap_bits.append(eng.bits())
    # pair masks after the last move, for the last moved obstacle and obstacle 0
    allc = np.arange(L.N, dtype=np.int32)
    last = int(ids[-1])
    masks = np.stack([eng.mask(0, allc, last), eng.mask(1, allc, last)])
    d = layout_arrays(L, with_corners)
    d.update(ids=np.asarray(ids, np.int32), rts=np.asarray(rts), reports=np.asarray(reports, np.int64),
             snap_at=np.asarray(snaps_at, np.int32), snap_states=np.asarray(snap_states, np.uint8),
             snap_bits=np.asarray(snap_bits, np.uint64), mask_obstacle=last, masks=masks,
             groups=eng.groups, lazy=int(lazy))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    st = snap_states[-1]
    print(f"{name}: N={L.N} B={L.B} S={L.S} M={L.M} segs={len(L.segs)} moves={len(ids)} "
          f"labels={np.bincount(st, minlength=3).tolist()} groups={eng.groups}")


def scn(name, **kw):
    w = ref.World.from_scn(open(os.path.join(REF_SCN, name + ".scn")).read())
    ids, rts = w.moves()
    replay(w, ids, rts, "scn_" + name, **kw)


def synthetic(name, kind, n_nodes, k, half, m, iterations, seed, snap_every):
    rm = synth.make_roadmap(kind, n_nodes, k, half, seed)
    w = ref.World.from_roadmap(rm.robot_he, rm.env, rm.nodes, rm.edges, rm.eps, rm.max_segments)
    obs = synth.make_obstacles(kind, m, seed + 1)
    for he, ns in zip(obs.he, obs.spheres):
        w.add_obstacle(he, int(ns))
    ids, rts = synth.make_moves(kind, m, iterations, half + 1.0, seed + 2)
    replay(w, ids, rts, name, snap_every=snap_every)


def kats():
    boxes, obst, idx, out, pose, he = ref.kat_sat(2025, 5000, 10000)
    np.savez_compressed(os.path.join(OUT, "kat_sat.npz"), boxes=boxes, obstacle=obst, idx=idx, out=out,
                        obstacle_pose=pose, obstacle_he=he)
    segs, idx, out = ref.kat_seg(777, 4000, 50, 9001)
    np.savez_compressed(os.path.join(OUT, "kat_seg.npz"), segs=segs, idx=idx, out=out,
                        center=np.array([0.3, -0.2, 0.1]), r_total=1.1)
    a, b, out, margin = ref.kat_sat_pairs(4242, 1000, 4.0, 2.0)
    np.savez_compressed(os.path.join(OUT, "kat_pairs.npz"), a=a, b=b, out=out, margin=margin)
    # obstacle operands under random rotations (exercises cross axes and fmin/fmax)
    w = ref.World.from_scn(open(os.path.join(REF_SCN, "quick_smoke.scn")).read())
    w.add_obstacle([1.3, 0.4, 0.7], 3)
    L = w.layout()
    rng = np.random.default_rng(99)
    rows = []
    for i in range(60):
        o = i % L.M
        axis = rng.normal(size=3)
        rt = ref.tf_axis_angle(axis / np.linalg.norm(axis), rng.uniform(-np.pi, np.pi))
        rt[9:] = rng.uniform(-5, 5, 3)
        if i % 7 == 0:
            rt = ref.tf_euler(0.0, 0.0, rng.uniform(-np.pi, np.pi))
            rt[9:] = rng.uniform(-5, 5, 3)
        sat, aabb, cen, saabb = w.obstacle_operands(o, rt)
        cpad = np.zeros((L.C, 3))
        cpad[: len(cen)] = cen
        rows.append((o, rt, sat, aabb, cpad, saabb))
    np.savez_compressed(os.path.join(OUT, "kat_obstacle.npz"), o=np.array([r[0] for r in rows], np.int32),
                        rt=np.array([r[1] for r in rows]), sat=np.array([r[2] for r in rows]),
                        aabb=np.array([r[3] for r in rows]), centres=np.array([r[4] for r in rows]),
                        saabb=np.array([r[5] for r in rows]), obst_he=L.obst_he, obst_sph_local=L.obst_sph_local,
                        obst_sph_r=L.obst_sph_r, obst_sph_n=L.obst_sph_n)
    print("kats written")


def kat_boxes(n=1200, seed=31):
    """Near-contact box pairs for the exact resolve (polytopes_intersect, geometry.cpp:278-303):
    random rotations (axis-angle and yaw-only, the latter with parallel edges whose cross
    products vanish), ~half intersecting, plus exactly touching axis-aligned pairs."""
    rng = np.random.default_rng(seed)
    rt_a, rt_b, he_a, he_b, out = [], [], [], [], []
    for c in range(n):
        # box a plays the robot body (one half-extent triple for all pairs), box b the obstacle
        ha, hb = np.array([0.5, 0.3, 0.25]), rng.uniform(0.2, 1.5, 3)
        kind = c % 10
        if kind == 0:  # touching faces along x: the reference counts touching as intersecting
            a = ref.tf_euler(0.0, 0.0, 0.0)
            b = ref.tf_euler(0.0, 0.0, 0.0)
            a[9:] = [50.0 * c, 0.25, -0.5]
            b[9:] = [50.0 * c + ha[0] + hb[0], 0.25 + rng.uniform(-0.1, 0.1), -0.5]
        else:
            if kind < 4:
                a = ref.tf_euler(0.0, 0.0, rng.uniform(-np.pi, np.pi))
                b = ref.tf_euler(0.0, 0.0, rng.uniform(-np.pi, np.pi))
            else:
                ax, bx = rng.normal(size=3), rng.normal(size=3)
                a = ref.tf_axis_angle(ax / np.linalg.norm(ax), rng.uniform(-np.pi, np.pi))
                b = ref.tf_axis_angle(bx / np.linalg.norm(bx), rng.uniform(-np.pi, np.pi))
            a[9:] = [50.0 * c + rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1)]
            u = rng.normal(size=3)
            u /= np.linalg.norm(u)
            d = rng.uniform(0.35, 1.05) * (np.linalg.norm(ha) + np.linalg.norm(hb))
            b[9:] = a[9:] + d * u
        rt_a.append(a), rt_b.append(b), he_a.append(ha), he_b.append(hb)
        out.append(1 if ref.box_intersect(a, ha, b, hb) else 0)
    out = np.array(out, np.uint8)
    np.savez_compressed(os.path.join(OUT, "kat_boxes.npz"), rt_a=np.array(rt_a), he_a=np.array(he_a),
                        rt_b=np.array(rt_b), he_b=np.array(he_b), out=out)
    print("kat_boxes written:", int(out.sum()), "of", n, "intersect")


def prm():
    """build_prm (proj/src/roadmap.cpp:56-102) of every shipped scenario's build scene,
    proj/tests/test_roadmap.cpp:34-60's free-cube cases, and a digest of table3's
    10,000-node roadmap (too large to store)."""
    import glob
    import hashlib
    import re

    d = {}
    names = []

    def put(name, text, n=-1, k=-1, seed=-1, digest=False):
        nodes, edges, lo, hi, sec = ref.build_prm(text, n, k, seed)
        kk = k if k >= 0 else int(re.search(r"k_neighbors\s*=\s*(\d+)", text).group(1))
        sd = seed if seed >= 0 else int(re.search(r"roadmap_seed\s*=\s*(\d+)", text).group(1))
        names.append(name)
        d[f"{name}__meta"] = np.array([len(nodes), kk, sd, nodes.shape[1], len(edges)], np.int64)
        d[f"{name}__lo"], d[f"{name}__hi"] = lo, hi
        if digest:
            d[f"{name}__sha_nodes"] = np.frombuffer(hashlib.sha256(nodes.tobytes()).digest(), np.uint8)
            d[f"{name}__sha_edges"] = np.frombuffer(hashlib.sha256(edges.tobytes()).digest(), np.uint8)
        else:
            d[f"{name}__nodes"], d[f"{name}__edges"] = nodes, edges
        print(f"prm {name}: {len(nodes)} nodes, {len(edges)} edges, reference {sec * 1e3:.1f} ms")

    for f in sorted(glob.glob(os.path.join(REF_SCN, "*.scn"))):
        base = os.path.basename(f)[:-4]
        put(base, open(f).read(), digest=base.startswith("table3"))
    cube = open(os.path.join(REF_SCN, "table2_density_10_10x2x2.scn")).read()  # env +-10, free-flying 0.5 cube
    for n, k, seed in ((10, 16, 42), (1, 4, 7), (60, 8, 1234), (60, 8, 1235), (2, 5, 3), (300, 40, 5)):
        put(f"cube_{n}_{k}_{seed}", cube, n, k, seed)
    d["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "prm.npz"), **d)


def main():
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1:  # regenerate selected fixtures only, e.g. `gen_golden.py kat_boxes`
        for name in sys.argv[1:]:
            globals()[name]()
        return
    kats()
    kat_boxes()
    scn("quick_smoke", with_corners=True)
    scn("table2_density_100_10x2x2")
    scn("table4_obstacles_1000_5x", snap_every=25, snap_first=10)
    scn("table5_manipulator_100", lazy=True)
    synthetic("syn_se2_m80", "se2", 800, 12, 20.0, 80, 3, 11, snap_every=40)
    synthetic("syn_3d_m20", "3d", 300, 10, 4.5, 20, 4, 21, snap_every=1)
    prm()


if __name__ == "__main__":
    main()
