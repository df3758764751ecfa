"""-m "not gpu": the 1-D partitioned walk's driver (paper_2504_10233_b200.distributed.
PartitionedBingo) and its sharded update application (f1) on world_size 2
with gloo on CPU.  Each rank's engine
is the CPU oracle built from its partition (partition_csr: only its rows' arcs) wrapped in a
test-only stepper with bingo_walk_partition's contract (walk while on owned vertices, leave
for the owner otherwise).  Walker transfer by all-to-all must reproduce the unpartitioned
oracle walk exactly: paths, lengths and PPR visit counts."""
from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NONE = 0xFFFFFFFF


class OraclePartEngine:
    """bingo_walk_partition emulated step by step with the oracle's sampler (tests only)."""

    def __init__(self, ro, dst, bias):
        import oracle
        self.o = oracle.OracleGraph(ro, dst, bias)
        self.V = len(ro) - 1
        self.device = torch.device("cpu")
        self.counts = np.zeros(self.V, dtype=np.int64)

    def walk_partition(self, bounds, me, inbox, outbox, out_count, app=0, length=80, seed=0, first_walker=0,
                       num_walkers=None, stop=(1, 80), paths=None, lengths=None):
        import oracle
        b = bounds.tolist()
        thr, always = oracle.stop_threshold(*stop)
        fin = 0

        def owner(x):
            r = 0
            while r + 1 < len(b) - 1 and x >= b[r + 1]:
                r += 1
            return r
        for w, u, t, fresh in inbox.tolist():
            i = w - first_walker
            if fresh:
                if paths is not None:
                    paths[0, i] = u
                if app == oracle.APP_PPR:
                    self.counts[u] += 1
            finished = False
            while True:
                if length != NONE and t >= length:
                    finished = True
                    break
                if oracle.lib().ora_degree(self.o._h, u) == 0:
                    finished = True
                    break
                nxt = self.o.sample(u, seed, w, t, 0)
                if paths is not None:
                    paths[t + 1, i] = nxt
                stopped = False
                if app == oracle.APP_PPR:
                    self.counts[nxt] += 1
                    if always:
                        stopped = True
                    else:
                        r = oracle.philox([w, t, 0, 3], [seed & 0xFFFFFFFF, seed >> 32])
                        stopped = ((int(r[0]) << 32) | int(r[1])) < thr
                t += 1
                if stopped:
                    finished = True
                    break
                o = owner(nxt)
                if o != me:
                    k = int(out_count[o])
                    outbox[o, k] = torch.tensor([w, nxt, t, 0], dtype=torch.int32)
                    out_count[o] += 1
                    break
                u = nxt
            if finished:
                fin += 1
                lengths[i] = t
                if paths is not None and length != NONE:
                    paths[t + 1:, i] = -1
        return fin

    def apply_updates(self, batch):
        return self.o.apply_updates(batch.numpy().view(np.uint32))

    def visit_counts(self, reset=False):
        c = torch.from_numpy(self.counts.copy())
        if reset:
            self.counts[:] = 0
        return c


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_2504_10233_b200.distributed import PartitionedBingo, partition_bounds, partition_csr
    w = synth.make_workload("c1", rounds=2)
    bounds = partition_bounds(w.row_offsets, world)
    ro, dst, bias = partition_csr(w.row_offsets, w.dst, w.bias, bounds[rank], bounds[rank + 1])
    pb = PartitionedBingo(OraclePartEngine(ro, dst, bias), bounds)
    out = pb.walk(num_walkers=700, length=15, seed=3, first_walker=40)
    np.save(os.path.join(outdir, f"paths{rank}.npy"), out["paths"].numpy())
    np.save(os.path.join(outdir, f"len{rank}.npy"), out["lengths"].numpy())
    out = pb.walk(num_walkers=600, app=oracle.APP_PPR, length=NONE, seed=4, paths=False)
    np.save(os.path.join(outdir, f"plen{rank}.npy"), out["lengths"].numpy())
    np.save(os.path.join(outdir, f"counts{rank}.npy"), pb.visit_counts().numpy())
    np.save(os.path.join(outdir, f"rounds{rank}.npy"), np.array([out["rounds"]]))
    # sharded update application: each rank applies the records its vertices own
    for b in w.batches:
        st = pb.apply_updates(torch.from_numpy(b.view(np.int32)) if rank == 0 else None, n=b.shape[0])
        np.save(os.path.join(outdir, f"st{rank}_{st['epoch']}.npy"),
                np.array([st["inserted"], st["deleted"], st["missing_deletes"], st["touched_vertices"]]))
    dig = pb.g.o.digests()[bounds[rank]:bounds[rank + 1]]
    np.save(os.path.join(outdir, f"dig{rank}.npy"), dig)
    out = pb.walk(num_walkers=500, length=12, seed=8)
    np.save(os.path.join(outdir, f"upaths{rank}.npy"), out["paths"].numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_partition_bounds_and_csr():
    import synth
    from paper_2504_10233_b200.distributed import partition_bounds, partition_csr
    w = synth.make_workload("c1")
    for P in (1, 2, 3, 5):
        b = partition_bounds(w.row_offsets, P)
        assert b[0] == 0 and b[-1] == w.V and all(x <= y for x, y in zip(b, b[1:]))
        arcs = 0
        for r in range(P):
            ro, dst, bias = partition_csr(w.row_offsets, w.dst, w.bias, b[r], b[r + 1])
            deg = np.diff(ro.astype(np.int64))
            assert deg[:b[r]].sum() == 0 and deg[b[r + 1]:].sum() == 0
            full = np.diff(w.row_offsets.astype(np.int64))[b[r]:b[r + 1]]
            assert np.array_equal(deg[b[r]:b[r + 1]], full)
            arcs += len(dst)
        assert arcs == w.num_arcs


def test_two_rank_partitioned_walk_gloo(tmp_path):
    import oracle
    import synth
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    w = synth.make_workload("c1", rounds=2)
    o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    ref = o.walk(length=15, seed=3, first_walker=40, num_walkers=700)
    for r in range(world):     # assembled on every rank
        assert np.array_equal(np.load(tmp_path / f"paths{r}.npy").view(np.uint32), ref["paths"])
        assert np.array_equal(np.load(tmp_path / f"len{r}.npy").view(np.uint32), ref["lengths"])
    refp = o.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=4, num_walkers=600, paths=False, counts=True)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"plen{r}.npy").view(np.uint32), refp["lengths"])
        assert np.array_equal(np.load(tmp_path / f"counts{r}.npy").view(np.uint64), refp["counts"])
        assert int(np.load(tmp_path / f"rounds{r}.npy")[0]) > 2     # walkers really moved between ranks
    # after sharded updates: owned vertices' canonical state, statistics and walks equal the
    # single graph that applied every record
    o2 = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    for b in w.batches:
        so = o2.apply_updates(b)
        for r in range(world):
            got = np.load(tmp_path / f"st{r}_{so['epoch']}.npy")
            assert got.tolist() == [so["inserted"], so["deleted"], so["missing_deletes"], so["touched_vertices"]]
    from paper_2504_10233_b200.distributed import partition_bounds
    bounds = partition_bounds(w.row_offsets, world)
    full = o2.digests()
    assert np.array_equal(np.concatenate([np.load(tmp_path / f"dig{r}.npy") for r in range(world)]), full)
    ref = o2.walk(length=12, seed=8, num_walkers=500)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"upaths{r}.npy").view(np.uint32), ref["paths"])
