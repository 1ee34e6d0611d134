"""Multi-rank host logic on CPU (gloo, world_size 2): move broadcast, per-move
counter all-reduce and gray-id gather, checked against the reference's golden
reports and labels.  Shards are oracle-backed (the CUDA engine needs a GPU) and
split the roadmap either into tiles (contiguous id ranges) or, as bench.py's
strong-scaling run does with GpuEngine shards, into interleaved 128-component
cells (rank r owns cells c with c % world == r); the same DistributedUpdater
drives both."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, load_golden


class InterleavedShard:
    """The DistributedUpdater engine interface over the C oracle on the whole
    roadmap, owning the components of cells c (128 consecutive ids) with
    c % world == rank: counters, labels and gray ids are reported for those only
    (ids are global, labels 0xFF elsewhere), like a sharded GpuEngine."""

    def __init__(self, g, rank, world, cell=128):
        from oracle import oracle

        self.eng = oracle.Engine(g_layout(g))
        n = int(g["N"])
        self.own = (np.arange(n) // cell) % world == rank
        self.last = None

    def update_tensors(self, ids, rts, per_move=True, gray_list=False):
        rows = []
        for o, rt in zip(ids.numpy(), rts.numpy()):
            prev = self.eng.states()
            self.eng.update(int(o), rt)
            cur = self.eng.states()
            ch = (prev != cur) & self.own
            rows.append([np.sum(ch & (cur == 0)), np.sum(ch & (cur == 1)), np.sum(ch & (cur == 2)),
                         np.sum(ch & (prev == 2))])
        self.last = np.asarray(rows, np.int32)

    def counters_into(self, out, n, check=True):
        out.copy_(torch.from_numpy(self.last[:n]))

    def sync(self):
        pass

    def gray_ids(self):
        return np.nonzero((self.eng.states() == 2) & self.own)[0]

    def gray_count_into(self, out):
        out[0] = len(self.gray_ids())

    def gray_ids_into(self, out, cap):
        g = torch.from_numpy(self.gray_ids().astype(np.int32))[:cap]
        out[: len(g)] = g

    def states(self):
        s = self.eng.states().copy()
        s[~self.own] = 0xFF
        return s


def g_layout(g):
    class L:
        pass

    sub = L()
    for k in ("N", "B", "S", "M", "C"):
        setattr(sub, k, int(g[k]))
    for k in ("edge_sat", "comp_aabb", "row_off", "segs", "spline_r", "obst_he", "obst_sph_local", "obst_sph_r",
              "obst_sph_n"):
        setattr(sub, k, g[k])
    return sub


class OracleShard:
    """The DistributedUpdater engine interface over the C oracle, owning the
    components [lo, hi) of a layout (a tile)."""

    def __init__(self, g, lo, hi):
        from oracle import oracle

        B, S = int(g["B"]), int(g["S"])
        r0, r1 = g["row_off"][lo * B * S], g["row_off"][hi * B * S]

        class L:
            pass

        sub = L()
        sub.N, sub.B, sub.S, sub.M, sub.C = hi - lo, B, S, int(g["M"]), int(g["C"])
        sub.edge_sat = g["edge_sat"][lo * B:hi * B]
        sub.comp_aabb = g["comp_aabb"][lo:hi]
        sub.row_off = (g["row_off"][lo * B * S:hi * B * S + 1] - r0).astype(np.int32)
        sub.segs = g["segs"][r0:r1]
        for k in ("spline_r", "obst_he", "obst_sph_local", "obst_sph_r", "obst_sph_n"):
            setattr(sub, k, g[k])
        self.eng = oracle.Engine(sub)
        self.last = None

    def update_tensors(self, ids, rts, per_move=True, gray_list=False):
        rows = []
        for o, rt in zip(ids.numpy(), rts.numpy()):
            prev = self.eng.states()
            self.eng.update(int(o), rt)
            cur = self.eng.states()
            ch = prev != cur
            rows.append([np.sum(ch & (cur == 0)), np.sum(ch & (cur == 1)), np.sum(ch & (cur == 2)),
                         np.sum(ch & (prev == 2))])
        self.last = np.asarray(rows, np.int32)

    def counters_into(self, out, n, check=True):
        out.copy_(torch.from_numpy(self.last[:n]))

    def sync(self):
        pass

    def gray_ids(self):
        return np.nonzero(self.eng.states() == 2)[0]

    def gray_count_into(self, out):
        out[0] = len(self.gray_ids())

    def gray_ids_into(self, out, cap):
        g = torch.from_numpy(self.gray_ids().astype(np.int32))[:cap]
        out[: len(g)] = g

    def states(self):
        return self.eng.states()


def _worker(rank, world, port, name, out, mode="tiles"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, ROOT)
    from paper_2603_28674_b200.dist import DistributedUpdater

    g = load_golden(name)
    N = int(g["N"])
    if mode == "tiles":
        cut = [0, N // 2, N][rank:rank + 2] if world == 2 else [0, N]
        shard = OracleShard(g, cut[0], cut[1])
        up = DistributedUpdater(shard, torch.device("cpu"), id_offset=cut[0], gray_cap=N)
    else:
        shard = InterleavedShard(g, rank, world)
        up = DistributedUpdater(shard, torch.device("cpu"), gray_cap=N)
    ids = torch.from_numpy(g["ids"].astype(np.int32)) if rank == 0 else torch.zeros(len(g["ids"]), dtype=torch.int32)
    rts = torch.from_numpy(g["rts"]) if rank == 0 else torch.zeros(len(g["ids"]), 12, dtype=torch.float64)
    reports, unknown, step_gray = [], 0, None
    for a in range(0, len(g["ids"]), 16):  # batches of 16 moves, the gray list gathered inside each
        c = up.update(ids[a:a + 16].contiguous(), rts[a:a + 16].contiguous(), check=False, gather_gray=True)
        reps = up.reports(c, unknown)
        unknown = reps[-1]["unknown_after_heuristic"]
        reports += reps
        step_gray = up.gathered_gray()
    up.check()
    gray = up.gray_ids()
    labels = up.states(N)
    if rank == 0:
        out.put((reports, gray, labels, step_gray))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", ["tiles", "interleaved"])
@pytest.mark.parametrize("name", ["scn_table4_obstacles_1000_5x", "syn_3d_m20"])
def test_two_rank_shards_reproduce_reference_reports(name, mode):
    g = load_golden(name)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    reports, gray, labels, step_gray = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.array([[r["new_green"], r["new_red"], r["new_gray"], r["unknown_after_heuristic"]] for r in reports])
    assert np.array_equal(got, g["reports"][:, :4]), "sharded per-move reports differ from the reference"
    assert np.array_equal(gray, np.nonzero(g["snap_states"][-1] == 2)[0]), "gathered gray list differs"
    assert np.array_equal(step_gray, gray), "gray list gathered inside the last update differs"
    assert np.array_equal(labels, g["snap_states"][-1]), "merged labels differ"
