"""Multi-GPU driver: one process per GPU, components sharded, obstacles replicated.

SURVEY.md §8(e): a component's label depends only on its own geometry and the
(replicated) obstacle set, so components shard with no data-path exchange.  One
roadmap is split by the engine's interleaved cell sharding
(``rgg_gpu_options.shard_rank / shard_count``: rank r owns the Morton-ordered cells
c with c % world == r, so the cells an obstacle dirties spread over every rank).
Per update (torch.distributed over NCCL on B200, gloo in the CPU tests):

1. ``broadcast`` of the move batch (ids int32[n], poses float64[n, 12]) from
   rank 0 — the host that receives the obstacle updates;
2. ``all_reduce`` (sum) of the per-move report counters
   (n x {to_green, to_red, to_gray, from_gray}); shards own disjoint components,
   so the sums are the reference's UpdateReport counts for the whole roadmap;
3. with ``gather_gray``, the per-shard GRAY id lists (compacted inside each
   shard's update) are gathered to rank 0: an all_gather of the counts and a
   fixed-capacity all_gather of the lists (capacity = the largest shard, so no
   host round trip is needed to size it).

Everything is stream-ordered: the engine stream waits on the broadcast, torch's
stream waits on the engine's counters and gray list; nothing blocks the host
unless ``check`` asks for the update's device-side status.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


class DistributedUpdater:
    """Drive a per-rank engine shard.

    ``engine`` needs ``update_tensors(ids, rts, per_move, gray_list)``,
    ``counters_into(t, n, check)``, ``sync()``, ``states()``, ``gray_ids()`` and, for
    ``gather_gray``, ``gray_count_into(t)`` / ``gray_ids_into(t, cap)`` (GpuEngine
    provides them; the CPU tests use an oracle-backed shard).  ``id_offset`` maps a
    shard's local component ids to global ids (0 for interleaved cell shards, whose
    ids are global already).  ``gray_cap``: capacity per rank of the gathered gray
    lists (the largest shard's component count).
    """

    def __init__(self, engine, device: torch.device, group=None, id_offset: int = 0, gray_cap: int = 0):
        self.engine = engine
        self.device = device
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.id_offset = id_offset
        self.gray_cap = int(gray_cap)
        self._gray = None
        self._pin = None  # pinned host buffer of gathered_gray

    def update(self, ids: torch.Tensor, rts: torch.Tensor, per_move: bool = True, check: bool = True,
               gather_gray: bool = False) -> torch.Tensor:
        """Apply one batch of moves on every shard; returns the summed per-move
        counters (n x 4 int32) on every rank.  ``ids``/``rts`` are only read on rank 0.
        check=False leaves the update's status to a later ``check()`` (no host wait)."""
        n = int(ids.numel())
        if self.world > 1:
            dist.broadcast(ids, 0, group=self.group)
            dist.broadcast(rts, 0, group=self.group)
        # allocated before the update is enqueued: the engine stream waits on this
        # allocation's stream, and the copy below writes every entry
        counters = torch.empty((n, 4), dtype=torch.int32, device=self.device)
        self.engine.update_tensors(ids, rts, per_move, gray_list=gather_gray)
        self.engine.counters_into(counters, n, check=check)
        if self.world > 1:
            dist.all_reduce(counters, group=self.group)
        if gather_gray:
            self._gather_gray()
        return counters

    def check(self):
        """Wait for the enqueued updates and raise their device-side errors."""
        self.engine.sync()

    def _gather_gray(self):
        cap = max(1, self.gray_cap)
        cnt = torch.empty(1, dtype=torch.int32, device=self.device)
        ids = torch.empty(cap, dtype=torch.int32, device=self.device)
        self.engine.gray_count_into(cnt)
        self.engine.gray_ids_into(ids, cap)
        if self.id_offset:
            ids += self.id_offset
        if self.world > 1:
            counts = torch.empty(self.world, dtype=torch.int32, device=self.device)
            lists = torch.empty(self.world * cap, dtype=torch.int32, device=self.device)
            dist.all_gather_into_tensor(counts, cnt, group=self.group)
            dist.all_gather_into_tensor(lists, ids, group=self.group)
        else:
            counts, lists = cnt, ids
        self._gray = (counts, lists, cap)

    def gathered_gray(self) -> np.ndarray | None:
        """The GRAY ids (ascending, global, int32) gathered by the last
        ``update(gather_gray=True)``, on rank 0 (None elsewhere): one copy into a pinned
        host buffer, returned as a view that the next call overwrites."""
        if self._gray is None:
            raise RuntimeError("no gray list gathered: call update(..., gather_gray=True)")
        if self.rank != 0:
            return None
        counts, lists, cap = self._gray
        c = counts.cpu().numpy()
        if int(c.max(initial=0)) > cap:
            raise RuntimeError("a shard's gray list exceeds the gather capacity")
        # merge on the device (each shard's list is ascending; interleaved shards interleave
        # their ids), then one copy of just the ids into a reused pinned buffer
        total = int(c.sum())
        if total == 0:
            return np.zeros(0, np.int32)
        if len(c) == 1:
            merged = lists[:total]
        else:
            keep = torch.arange(cap, device=lists.device)[None, :] < counts.to(torch.int64)[:, None]
            merged = torch.sort(lists.view(len(c), cap)[keep]).values
        if not merged.is_cuda:
            return merged.numpy().copy()
        if self._pin is None or self._pin.numel() < total:
            self._pin = torch.empty(max(total, 1 << 16), dtype=torch.int32, pin_memory=True)
        out = self._pin[:total]
        out.copy_(merged)
        return out.numpy()  # int32 view of the pinned buffer: valid until the next call

    @staticmethod
    def reports(counters: torch.Tensor, unknown_before: int) -> list[dict]:
        """Per-move UpdateReport counts from summed counters (update_report.hpp:11-25)."""
        c = counters.cpu().numpy().astype(np.int64)
        unknown = unknown_before + np.cumsum(c[:, 2] - c[:, 3])
        return [dict(new_green=int(g), new_red=int(r), new_gray=int(y), unknown_after_heuristic=int(u),
                     residual_unknown=int(u)) for (g, r, y, _), u in zip(c, unknown)]

    def states(self, n_global: int) -> np.ndarray:
        """All labels (component-id order) on every rank: each shard's labels placed at
        its id offset (tiles) or already in global order with 0xFF for other shards'
        components (interleaved cells), merged with one MIN all-reduce."""
        local = np.asarray(self.engine.states(), np.uint8)
        full = np.full(n_global, 0xFF, np.uint8)
        full[self.id_offset:self.id_offset + len(local)] = local
        if self.world == 1:
            return full
        t = torch.from_numpy(full).to(self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return t.cpu().numpy()

    def resolve_all_unknown(self) -> int:
        """resolve_all_unknown on every shard (the exact check is per component, so
        shard-local); the total count on every rank."""
        n = int(self.engine.resolve_all_unknown())
        if self.world == 1:
            return n
        t = torch.tensor([n], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, group=self.group)
        return int(t.item())

    def gray_ids(self) -> np.ndarray | None:
        """All GRAY component ids (ascending) on rank 0, None elsewhere (host lists,
        outside the update)."""
        local = np.asarray(self.engine.gray_ids(), np.int64) + self.id_offset
        if self.world == 1:
            return np.sort(local)
        cnt = torch.tensor([len(local)], dtype=torch.int64, device=self.device)
        counts = [torch.zeros_like(cnt) for _ in range(self.world)]
        dist.all_gather(counts, cnt, group=self.group)
        width = max(1, int(max(int(c.item()) for c in counts)))
        buf = torch.full((width,), -1, dtype=torch.int64, device=self.device)
        buf[: len(local)] = torch.from_numpy(local).to(self.device)
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(parts, buf, group=self.group)
        if self.rank != 0:
            return None
        allids = torch.cat([p[: int(c.item())] for p, c in zip(parts, counts)]).cpu().numpy()
        return np.sort(allids)
