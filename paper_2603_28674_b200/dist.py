"""Multi-GPU driver: one process per GPU, components sharded, obstacles replicated.

SURVEY.md §8(e): a component's label depends only on its own geometry and the
(replicated) obstacle set, so components shard with no data-path exchange.  Per
update there are exactly two collectives (torch.distributed over NCCL on B200,
gloo in the CPU tests):

1. ``broadcast`` of the move batch (ids int32[n], poses float64[n, 12]) from
   rank 0 — the host that receives the obstacle updates;
2. ``all_reduce`` (sum) of the per-move report counters
   (n x {to_green, to_red, to_gray, from_gray}); shards own disjoint components,
   so the sums are the reference's UpdateReport counts for the whole roadmap.

The gray list is gathered to rank 0 on request (``gray_ids``): per-shard counts
with one all_gather, then the id lists padded to the largest count.

Sharding itself is either spatial tiles (each rank's engine holds its own part
of the roadmap, bench.py's weak-scaling world) or the engine's interleaved cell
sharding of one roadmap (``rgg_gpu_options.shard_rank / shard_count``).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


class DistributedUpdater:
    """Drive a per-rank engine shard.

    ``engine`` needs ``update_tensors(ids, rts, per_move)``, ``counters_into(t, n)``
    and ``gray_ids()`` (GpuEngine provides them; tests use an oracle-backed shard).
    ``id_offset`` maps the shard's local component ids to global ids for gray_ids.
    """

    def __init__(self, engine, device: torch.device, group=None, id_offset: int = 0):
        self.engine = engine
        self.device = device
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.id_offset = id_offset

    def update(self, ids: torch.Tensor, rts: torch.Tensor, per_move: bool = True) -> torch.Tensor:
        """Apply one batch of moves on every shard; returns the summed per-move
        counters (n x 4 int32) on every rank.  ``ids``/``rts`` are only read on rank 0."""
        n = int(ids.numel())
        if self.world > 1:
            dist.broadcast(ids, 0, group=self.group)
            dist.broadcast(rts, 0, group=self.group)
        self.engine.update_tensors(ids, rts, per_move)
        counters = torch.zeros((n, 4), dtype=torch.int32, device=self.device)
        self.engine.counters_into(counters, n)
        if self.world > 1:
            dist.all_reduce(counters, group=self.group)
        return counters

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
        """All GRAY component ids (ascending) on rank 0, None elsewhere."""
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
