"""-m "not gpu": the multi-GPU driver's host logic (paper_2504_10233_b200.distributed) on
world_size 2 with the gloo backend on CPU.  The engine under the driver is the CPU
oracle wrapped in the Graph interface (test infrastructure only): sharded walks must
reproduce the unsharded run, replicas must stay identical after broadcast batches,
and all-reduced PPR counts must equal the single-process counts."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleEngine:
    """Graph-like adapter over the oracle (tests only)."""

    def __init__(self, w):
        import oracle
        self.o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
        self.V = w.V
        self.device = torch.device("cpu")
        self._counts = np.zeros(self.V, dtype=np.uint64)

    def apply_updates(self, batch):
        return self.o.apply_updates(batch.numpy().view(np.uint32))

    def walk(self, app=0, length=80, seed=0, first_walker=0, num_walkers=None, stop=(1, 80), starts=None, **kw):
        import oracle
        counts = app == oracle.APP_PPR
        if starts is not None:
            assert len(starts) == num_walkers
            starts = np.asarray(starts, dtype=np.uint32)
        r = self.o.walk(app=app, length=length, seed=seed, first_walker=first_walker, num_walkers=num_walkers,
                        starts=starts, stop=stop, paths=length != oracle.NONE, counts=counts, threads=1)
        if counts:
            self._counts += r["counts"]
        out = {"lengths": torch.from_numpy(r["lengths"].view(np.int32).copy())}
        out["paths"] = torch.from_numpy(r["paths"].view(np.int32).copy()) if r["paths"] is not None else None
        return out

    def visit_counts(self, reset=False):
        c = torch.from_numpy(self._counts.view(np.int64).copy())
        if reset:
            self._counts[:] = 0
        return c

    def digests(self):
        return torch.from_numpy(self.o.digests().view(np.int64).copy())


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
    from paper_2504_10233_b200.distributed import ReplicatedBingo, shard_range
    w = synth.make_workload("c1", rounds=3)
    rb = ReplicatedBingo(OracleEngine(w))
    for b in w.batches:
        st = rb.apply_updates(torch.from_numpy(b.view(np.int32)) if rank == 0 else None)
        assert st["epoch"] >= 1
    assert rb.replicas_identical()
    out = rb.walk(num_walkers=w.V, length=20, seed=3)
    first, count = out["shard"]
    assert (first, count) == shard_range(w.V, rank, world)
    rb.walk(num_walkers=3 * w.V, length=oracle.NONE, app=oracle.APP_PPR, seed=4)
    counts = rb.visit_counts()
    # explicit per-walker starts given for ALL walkers: each rank must walk its own slice
    starts = np.random.default_rng(17).integers(0, w.V, size=2 * w.V + 3).astype(np.uint32)
    sout = rb.walk(num_walkers=len(starts), length=12, seed=9, starts=starts)
    np.save(os.path.join(outdir, f"spaths{rank}.npy"), sout["paths"].numpy())
    np.save(os.path.join(outdir, f"paths{rank}.npy"), out["paths"].numpy())
    np.save(os.path.join(outdir, f"counts{rank}.npy"), counts.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    from paper_2504_10233_b200.distributed import shard_range
    for total in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and sum(c for _, c in spans) == total
            for (f0, c0), (f1, _) in zip(spans, spans[1:]):
                assert f0 + c0 == f1
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def test_two_rank_gloo_driver(tmp_path):
    import oracle
    import synth
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    # single-process reference on the same stream
    w = synth.make_workload("c1", rounds=3)
    o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    for b in w.batches:
        o.apply_updates(b)
    full = o.walk(length=20, seed=3, num_walkers=w.V)["paths"]
    parts = [np.load(tmp_path / f"paths{r}.npy").view(np.uint32) for r in range(world)]
    assert np.array_equal(np.concatenate(parts, axis=1), full)
    starts = np.random.default_rng(17).integers(0, w.V, size=2 * w.V + 3).astype(np.uint32)
    sfull = o.walk(length=12, seed=9, starts=starts, num_walkers=len(starts))["paths"]
    sparts = [np.load(tmp_path / f"spaths{r}.npy").view(np.uint32) for r in range(world)]
    assert np.array_equal(np.concatenate(sparts, axis=1), sfull), "explicit starts must be sliced per rank"
    ref = o.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=4, num_walkers=3 * w.V, paths=False, counts=True)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"counts{r}.npy").view(np.uint64), ref["counts"])


class ListEngine:
    """A plain adjacency-list engine (tests only) with the state-exchange interface, to test
    ReplicatedBingo's sharded update application on gloo: inserts append, a
    delete removes the first live instance; export / import move whole vertex states."""

    def __init__(self, w):
        self.V = w.V
        self.device = torch.device("cpu")
        self.adj = [[(int(w.dst[a]), int(w.bias[a])) for a in range(int(w.row_offsets[u]), int(w.row_offsets[u + 1]))]
                    for u in range(w.V)]
        self.epoch = 0

    def apply_updates(self, batch):
        b = np.asarray(batch.numpy() if isinstance(batch, torch.Tensor) else batch).view(np.uint32).reshape(-1, 4)
        st = {"inserted": 0, "deleted": 0, "missing_deletes": 0,
              "touched_vertices": len(set(b[:, 1].tolist())), "kind_transitions": np.zeros((5, 5), np.uint64)}
        for op, s, d, w in b.tolist():
            if op == 0:
                self.adj[s].append((d, w))
                st["inserted"] += 1
            else:
                for i, e in enumerate(self.adj[s]):
                    if e[0] == d:
                        del self.adj[s][i]
                        st["deleted"] += 1
                        break
                else:
                    st["missing_deletes"] += 1
        self.epoch += 1
        st["epoch"] = self.epoch
        return st

    def export_vertices(self, ids):
        words, off = [], [0]
        for u in ids.tolist():
            words += [u, len(self.adj[u])] + [x for e in self.adj[u] for x in e]
            off.append(len(words))
        return torch.tensor(words, dtype=torch.int64).to(torch.int32), torch.tensor(off, dtype=torch.int64)

    def import_vertices(self, buf, off):
        b, o = buf.to(torch.int64).tolist(), off.tolist()
        for i in range(len(o) - 1):
            r = b[o[i]:o[i + 1]]
            self.adj[r[0]] = [(r[2 + 2 * j], r[3 + 2 * j]) for j in range(r[1])]

    def digests(self):
        return torch.tensor([hash(tuple(a)) & 0x7FFFFFFFFFFF for a in self.adj], dtype=torch.int64)


def _sharded_worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_2504_10233_b200.distributed import ReplicatedBingo
    w = synth.make_workload("c1", rounds=4)
    e = ListEngine(w)
    rb = ReplicatedBingo(e)
    tot = []
    for b in w.batches:
        st = rb.apply_updates(torch.from_numpy(b.view(np.int32)) if rank == 0 else None, sharded=True)
        assert rb.replicas_identical()
        tot.append([st["inserted"], st["deleted"], st["missing_deletes"], st["touched_vertices"], st["epoch"]])
    np.save(os.path.join(outdir, f"dig{rank}.npy"), e.digests().numpy())
    np.save(os.path.join(outdir, f"st{rank}.npy"), np.array(tot))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_updates(tmp_path):
    """sharded=True: each rank applies the records it owns and the ranks exchange the touched
    vertices' states; every replica must equal the single-process application of each whole
    batch, and the summed statistics must match."""
    import synth
    world = 2
    mp.spawn(_sharded_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    w = synth.make_workload("c1", rounds=4)
    ref = ListEngine(w)
    sts = [ref.apply_updates(b) for b in w.batches]
    want = ref.digests().numpy()
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"dig{r}.npy"), want)
        got = np.load(tmp_path / f"st{r}.npy")
        for k, s in enumerate(sts):
            assert got[k].tolist() == [s["inserted"], s["deleted"], s["missing_deletes"], s["touched_vertices"],
                                       s["epoch"]]
