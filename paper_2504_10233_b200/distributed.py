"""Multi-GPU driver (SURVEY row e): one process per GPU, replicated graph,
walkers sharded by global id, update batches broadcast, PPR visit counts
combined with one all-reduce.

The walk path shards naturally over walkers: walker i's walk
depends only on the graph and its own Philox stream keyed by its global id
(R-1), so giving rank r the id range [first_r, first_r + count_r) reproduces the
single-GPU run bit for bit.  Every rank applies every update batch (replicas
stay identical because bingo_apply_updates is deterministic); replica equality
is checkable with `replica_digest`.

For graphs larger than one GPU, `PartitionedBingo` is the paper's own multi-GPU
design (1-D partitioning with walker transfer): each rank
holds only its vertex range's arcs and walkers move, over NCCL all-to-all, to the
rank that owns their current vertex; the walks are still the single-GPU walks.

Collectives go through torch.distributed (NCCL over NVLink on B200; gloo for
the CPU tests of this module's logic).  The engine is a `bingo.Graph` (or any
object with the same methods -- the gloo tests inject a CPU stand-in; the
product path always uses the CUDA library).
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np
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

    def apply_updates(self, batch: Optional[torch.Tensor], n: Optional[int] = None, sharded: bool = False) -> dict:
        """Every replica applies rank 0's batch.  sharded=True: each rank applies
        only the records whose source it owns (src mod P, after validating the whole batch)
        and the replicas exchange the post-batch state of their touched vertices
        (bingo_export_vertices -> variable-size all-gather -> bingo_import_vertices), so every
        replica ends with the same canonical state while each applies ~1/P of the records.
        Statistics are summed over the ranks."""
        buf = self.broadcast_batch(batch, n)
        if not sharded or self.world == 1:
            return self.g.apply_updates(buf)
        V = self.g.V
        mine = owned_records(buf, None, self.rank, V, world=self.world)
        st = self.g.apply_updates(mine)
        ids = torch.unique(mine[:, 1].to(torch.int64)) if mine.shape[0] else mine.new_zeros(0, dtype=torch.int64)
        rbuf, roff = self.g.export_vertices(ids.to(self.device))
        self._exchange_state(rbuf, roff)
        keys = ("inserted", "deleted", "missing_deletes", "touched_vertices")
        t = torch.tensor([int(st[k]) for k in keys], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, group=self.group)
        kt = torch.as_tensor(np.asarray(st["kind_transitions"], dtype=np.int64), device=self.device)
        dist.all_reduce(kt, group=self.group)
        out = dict(st)
        out.update({k: int(v) for k, v in zip(keys, t.tolist())})
        out["kind_transitions"] = kt.cpu().numpy().astype(np.uint64)
        return out

    def _exchange_state(self, rbuf: torch.Tensor, roff: torch.Tensor) -> None:
        """All-gather every rank's vertex records (padded to the largest) and install the
        other ranks' into this replica."""
        sizes = torch.tensor([rbuf.numel(), roff.numel()], dtype=torch.int64, device=self.device)
        alls = [torch.zeros_like(sizes) for _ in range(self.world)]
        dist.all_gather(alls, sizes, group=self.group)
        wmax = max(int(x[0]) for x in alls)
        omax = max(int(x[1]) for x in alls)
        pb = torch.zeros(max(wmax, 1), dtype=torch.int32, device=self.device)
        pb[:rbuf.numel()] = rbuf
        po = torch.zeros(omax, dtype=torch.int64, device=self.device)
        po[:roff.numel()] = roff
        gb = [torch.empty_like(pb) for _ in range(self.world)]
        go = [torch.empty_like(po) for _ in range(self.world)]
        dist.all_gather(gb, pb, group=self.group)
        dist.all_gather(go, po, group=self.group)
        for r in range(self.world):
            if r == self.rank:
                continue
            nw, no = int(alls[r][0]), int(alls[r][1])
            if no > 1:
                self.g.import_vertices(gb[r][:nw], go[r][:no])

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


# ---------------------------------------------------------------- 1-D partitioning
def partition_bounds(row_offsets, parts: int) -> list:
    """Contiguous external-id ranges [b_r, b_{r+1}) holding about the same number of arcs
    (1-D partitioning; KnightKing balances by edges too)."""
    import numpy as np
    ro = np.asarray(row_offsets.cpu() if isinstance(row_offsets, torch.Tensor) else row_offsets).astype(np.int64)
    V = len(ro) - 1
    A = int(ro[-1])
    b = [0]
    for r in range(1, parts):
        b.append(int(min(max(np.searchsorted(ro, A * r // parts, side="left"), b[-1]), V)))
    b.append(V)
    return b


def partition_csr(row_offsets, dst, bias, v0: int, v1: int):
    """This rank's partition graph: the full vertex-id space, arcs only for rows [v0, v1)."""
    is_t = isinstance(row_offsets, torch.Tensor)
    if is_t:
        ro = row_offsets.to(torch.int64)
        a0, a1 = int(ro[v0]), int(ro[v1])
        lro = torch.clamp(ro - a0, min=0, max=a1 - a0)
        return lro, dst[a0:a1], bias[a0:a1]
    import numpy as np
    ro = np.asarray(row_offsets, dtype=np.int64)
    a0, a1 = int(ro[v0]), int(ro[v1])
    lro = np.clip(ro - a0, 0, a1 - a0).astype(np.uint64)
    return lro, np.asarray(dst)[a0:a1], np.asarray(bias)[a0:a1]


def fresh_inbox(bounds, me: int, num_walkers: int, first_walker: int, V: int, device) -> torch.Tensor:
    """The walkers whose start vertex ((first + i) mod V) this rank owns: {id, start, 0, fresh}."""
    ids = torch.arange(num_walkers, dtype=torch.int64, device=device) + first_walker
    st = ids % V
    mine = (st >= bounds[me]) & (st < bounds[me + 1])
    ids, st = ids[mine], st[mine]
    out = torch.zeros((ids.numel(), 4), dtype=torch.int32, device=device)
    out[:, 0] = ids.to(torch.int32)
    out[:, 1] = st.to(torch.int32)
    out[:, 3] = 1
    return out


class PartitionedBingo:
    """One rank of the 1-D partitioned walk with walker transfer.

    `engine` is this rank's partition graph (a bingo.Graph built from partition_csr, or any
    object with walk_partition / visit_counts); `bounds` the P + 1 range boundaries.  A walk
    runs in rounds: every rank advances the walkers on its vertices until they leave
    (bingo_walk_partition), then the leaving walkers are exchanged with ONE all-to-all per
    round; rounds repeat until no walker is left anywhere (an all-reduce of the count).
    Every draw is keyed by (walker, step), so paths, lengths and visit counts equal the
    single-GPU walk's: paths / lengths are assembled by a sum over ranks (each entry is
    written by exactly one rank), PPR counts by the usual all-reduce."""

    def __init__(self, engine, bounds, device=None, group=None):
        self.g = engine
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        assert len(bounds) == self.world + 1
        self.bounds_list = list(bounds)
        self.device = device if device is not None else getattr(engine, "device", torch.device("cpu"))
        self.bounds = torch.tensor(bounds, dtype=torch.int32, device=self.device)
        self.rounds = 0

    # ------------------------------------------------------------ sharded updates
    def apply_updates(self, batch: Optional[torch.Tensor], n: Optional[int] = None) -> dict:
        """Sharded update application: rank 0's batch is broadcast, validated whole on every
        rank (EINVAL before anything is applied, bingo.h), and each rank applies only the
        records whose SOURCE vertex it owns -- its partition holds the only copy of that
        vertex's sampling structure (adjacency, groups, alias), so the update work is split P
        ways and no vertex state has to be exchanged.  Every rank applies every batch (an
        empty share still advances the epoch, R-9), so arc epochs match the single-graph run.
        The statistics are summed over ranks."""
        V = self.bounds_list[-1]
        if self.world > 1:
            if n is None:
                nt = torch.zeros(1, dtype=torch.int64, device=self.device)
                if self.rank == 0:
                    nt[0] = batch.shape[0]
                dist.broadcast(nt, 0, group=self.group)
                n = int(nt.item())
            buf = batch.to(self.device, dtype=torch.int32).contiguous() if self.rank == 0 else \
                torch.empty((n, 4), dtype=torch.int32, device=self.device)
            if n:
                dist.broadcast(buf, 0, group=self.group)
        else:
            buf = batch.to(self.device, dtype=torch.int32).contiguous()
        mine = owned_records(buf, self.bounds_list, self.rank, V)
        st = self.g.apply_updates(mine)
        if self.world > 1:
            vec = torch.tensor([st["inserted"], st["deleted"], st["missing_deletes"], st["touched_vertices"]]
                               + [int(x) for x in np.asarray(st["kind_transitions"]).reshape(-1)],
                               dtype=torch.int64, device=self.device)
            dist.all_reduce(vec, group=self.group)
            v = vec.tolist()
            st = dict(st, inserted=v[0], deleted=v[1], missing_deletes=v[2], touched_vertices=v[3],
                      kind_transitions=np.array(v[4:29], dtype=np.uint64).reshape(5, 5))
        return st

    def _exchange(self, outbox: torch.Tensor, counts: torch.Tensor) -> torch.Tensor:
        send_counts = counts.to(torch.int64)
        recv_counts = torch.zeros_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc, rc = send_counts.tolist(), recv_counts.tolist()
        send = torch.cat([outbox[d, :sc[d]] for d in range(self.world)]) if sum(sc) else \
            torch.zeros((0, 4), dtype=torch.int32, device=self.device)
        recv = torch.empty((sum(rc), 4), dtype=torch.int32, device=self.device)
        dist.all_to_all_single(recv, send, rc, sc, group=self.group)
        return recv

    def walk(self, num_walkers: int, app: int = 0, length: int = 80, seed: int = 0, first_walker: int = 0,
             stop=(1, 80), paths: bool = True, max_rounds: int = 1 << 20) -> dict:
        V = self.bounds_list[-1]
        W = num_walkers
        no_cap = length == 0xFFFFFFFF
        pa = torch.zeros((length + 1, W), dtype=torch.int32, device=self.device) if (paths and not no_cap) else None
        ln = torch.zeros(W, dtype=torch.int32, device=self.device)
        inbox = fresh_inbox(self.bounds_list, self.rank, W, first_walker, V, self.device)
        finished = 0
        self.rounds = 0
        for _ in range(max_rounds):
            n = inbox.shape[0]
            outbox = torch.empty((self.world, max(n, 1), 4), dtype=torch.int32, device=self.device)
            cnt = torch.zeros(self.world, dtype=torch.int32, device=self.device)
            finished += self.g.walk_partition(self.bounds, self.rank, inbox, outbox, cnt, app=app, length=length,
                                              seed=seed, first_walker=first_walker, num_walkers=W, stop=stop,
                                              paths=pa, lengths=ln)
            self.rounds += 1
            inbox = self._exchange(outbox, cnt) if self.world > 1 else outbox[0, :int(cnt[0])]
            left = torch.tensor([inbox.shape[0]], dtype=torch.int64, device=self.device)
            if self.world > 1:
                dist.all_reduce(left, group=self.group)
            if int(left) == 0:
                break
        if self.world > 1:
            dist.all_reduce(ln, group=self.group)
            if pa is not None:
                dist.all_reduce(pa, group=self.group)
        return {"paths": pa, "lengths": ln, "rounds": self.rounds}

    def visit_counts(self, reset: bool = False) -> torch.Tensor:
        c = self.g.visit_counts(reset=reset)
        if self.world > 1:
            dist.all_reduce(c, op=dist.ReduceOp.SUM, group=self.group)
        return c


def owned_records(batch: torch.Tensor, bounds, me: int, V: int, world: int = 0) -> torch.Tensor:
    """The records of a (n, 4) {op, src, dst, bias} batch whose source vertex this rank owns
    (bounds: [bounds[me], bounds[me + 1]); bounds None: src mod world == me), in batch order,
    after validating the WHOLE batch (the ABI's whole-batch rule: one bad record anywhere
    rejects the batch before any rank applies anything)."""
    b = batch.to(torch.int64) & 0xFFFFFFFF
    op, src, dst, w = b[:, 0], b[:, 1], b[:, 2], b[:, 3]
    bad = (op > 1) | (src >= V) | (dst >= V) | ((op == 0) & (w == 0))
    if bool(bad.any()):
        from . import bingo
        raise bingo.BingoError(bingo.E_INVAL, "partitioned apply_updates")
    mine = (src % world == me) if bounds is None else (src >= bounds[me]) & (src < bounds[me + 1])
    return batch[mine].contiguous()


def apply_updates_partitions_local(engines, bounds, batch) -> list:
    """Sharded update application with every partition in THIS process: partition r applies
    the records whose source it owns (PartitionedBingo.apply_updates without the broadcast)."""
    V = bounds[-1]
    return [e.apply_updates(owned_records(batch, bounds, r, V)) for r, e in enumerate(engines)]


def walk_partitions_local(engines, bounds, num_walkers: int, app: int = 0, length: int = 80, seed: int = 0,
                          first_walker: int = 0, stop=(1, 80), paths: bool = True, device=None) -> dict:
    """The same rounds with every partition in THIS process (e.g. several partition graphs on
    one GPU): the all-to-all becomes a regrouping of the outboxes; paths and lengths are
    shared buffers (each entry written by exactly one partition)."""
    P = len(engines)
    device = device if device is not None else engines[0].device
    bt = torch.tensor(bounds, dtype=torch.int32, device=device)
    V = bounds[-1]
    W = num_walkers
    no_cap = length == 0xFFFFFFFF
    pa = torch.zeros((length + 1, W), dtype=torch.int32, device=device) if (paths and not no_cap) else None
    ln = torch.zeros(W, dtype=torch.int32, device=device)
    inbox = [fresh_inbox(bounds, r, W, first_walker, V, device) for r in range(P)]
    rounds = 0
    while any(x.shape[0] for x in inbox):
        nxt = [[] for _ in range(P)]
        for r in range(P):
            n = inbox[r].shape[0]
            outbox = torch.empty((P, max(n, 1), 4), dtype=torch.int32, device=device)
            cnt = torch.zeros(P, dtype=torch.int32, device=device)
            engines[r].walk_partition(bt, r, inbox[r], outbox, cnt, app=app, length=length, seed=seed,
                                      first_walker=first_walker, num_walkers=W, stop=stop, paths=pa, lengths=ln)
            for d, c in enumerate(cnt.tolist()):
                if c:
                    nxt[d].append(outbox[d, :c])
        inbox = [torch.cat(x) if x else torch.zeros((0, 4), dtype=torch.int32, device=device) for x in nxt]
        rounds += 1
    return {"paths": pa, "lengths": ln, "rounds": rounds}
