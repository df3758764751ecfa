"""Multi-GPU driver (SURVEY row e): one process per GPU, replicated graph,
walkers sharded by global id, update batches broadcast, PPR visit counts
combined with one all-reduce.

The walk path shards naturally over walkers: walker i's walk
depends only on the graph and its own Philox stream keyed by its global id
(R-1), so giving rank r the id range [first_r, first_r + count_r) reproduces the
single-GPU run bit for bit.  Every rank applies every update batch (replicas
stay identical because bingo_apply_updates is deterministic); replica equality
is checkable with `replica_digest`.  The paper's own multi-GPU design (1-D
partitioning with walker transfer) was never evaluated; it is the
NEXT item f3 in DESIGN.md.

Collectives go through torch.distributed (NCCL over NVLink on B200; gloo for
the CPU tests of this module's logic).  The engine is a `bingo.Graph` (or any
object with the same methods -- the gloo tests inject a CPU stand-in; the
product path always uses the CUDA library).
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist

MASK64 = (1 << 64) - 1


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced split of [0, total): returns (first, count) of `rank`."""
    base, rem = divmod(total, world)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


class ReplicatedBingo:
    def __init__(self, engine, device: Optional[torch.device] = None, group=None):
        self.g = engine
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device if device is not None else getattr(engine, "device", torch.device("cpu"))

    # ------------------------------------------------------------ updates
    def broadcast_batch(self, batch: Optional[torch.Tensor], n: Optional[int] = None) -> torch.Tensor:
        """Rank 0's (n, 4) int32 batch reaches every rank.  When every rank already knows
        the record count (`n`, e.g. a fixed batch size) only the payload is broadcast and
        nothing waits on the host; otherwise the size goes first (one host read).  At world
        size 1 the batch is returned as is (moved to the device if needed)."""
        if self.world == 1:
            return batch.to(self.device, dtype=torch.int32).contiguous()
        if n is None:
            nt = torch.zeros(1, dtype=torch.int64, device=self.device)
            if self.rank == 0:
                nt[0] = batch.shape[0]
            dist.broadcast(nt, 0, group=self.group)
            n = int(nt.item())
        if self.rank == 0:
            buf = batch.to(self.device, dtype=torch.int32).contiguous()
            assert buf.shape[0] == n, (buf.shape, n)
        else:
            buf = torch.empty((n, 4), dtype=torch.int32, device=self.device)
        if n:
            dist.broadcast(buf, 0, group=self.group)
        return buf

    def apply_updates(self, batch: Optional[torch.Tensor], n: Optional[int] = None) -> dict:
        buf = self.broadcast_batch(batch, n)
        return self.g.apply_updates(buf)

    # ------------------------------------------------------------ walks
    def walk(self, num_walkers: int, first_walker: int = 0, **kw) -> dict:
        """Walk this rank's shard of walker ids [first_walker, first_walker + num_walkers).
        One walker per vertex by default (starts = id mod V).  Per-walker inputs and
        outputs given for ALL walkers are sliced to this rank's shard: `starts` and
        `lengths` ([num_walkers]) and walker-major `paths` ([num_walkers, L + 1]);
        step-major paths must already be this shard's ([L + 1, count]).  Returns the
        engine's outputs plus this rank's (first, count)."""
        first, count = shard_range(num_walkers, self.rank, self.world)
        if kw.get("starts") is not None:
            st = kw["starts"]
            if len(st) != num_walkers:
                raise ValueError(f"starts has {len(st)} entries for {num_walkers} walkers")
            kw["starts"] = st[first:first + count]
        ln = kw.get("lengths")
        if isinstance(ln, torch.Tensor) and ln.shape[0] == num_walkers and count != num_walkers:
            kw["lengths"] = ln[first:first + count]
        pa = kw.get("paths")
        if isinstance(pa, torch.Tensor):
            if kw.get("walker_major"):
                if pa.shape[0] == num_walkers and count != num_walkers:
                    kw["paths"] = pa[first:first + count]
            elif pa.dim() == 2 and pa.shape[1] != count:
                raise ValueError("step-major paths must hold this rank's shard: shape (L + 1, count)")
        out = self.g.walk(first_walker=first_walker + first, num_walkers=count, **kw)
        out["shard"] = (first_walker + first, count)
        return out

    def visit_counts(self, reset: bool = False) -> torch.Tensor:
        """PPR visit frequencies summed over ranks: one all-reduce (north_star)."""
        c = self.g.visit_counts(reset=reset)
        if self.world > 1:
            dist.all_reduce(c, op=dist.ReduceOp.SUM, group=self.group)
        return c

    def replica_digest(self) -> int:
        """A 64-bit digest of this rank's replica (sum of per-vertex digests mod 2^64)."""
        d = self.g.digests()
        return int(d.to(torch.int64).sum().item()) & MASK64

    def replicas_identical(self) -> bool:
        mine = self.replica_digest()
        t = torch.tensor([mine - (1 << 64) if mine >= (1 << 63) else mine], dtype=torch.int64, device=self.device)
        if self.world == 1:
            return True
        allv = [torch.zeros_like(t) for _ in range(self.world)]
        dist.all_gather(allv, t, group=self.group)
        return all(int(x.item()) == int(t.item()) for x in allv)
