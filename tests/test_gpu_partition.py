"""-m gpu: the 1-D partitioned walk with walker transfer through the
C-ABI (bingo_walk_partition): P partition graphs on one GPU, each built from its rows only
(distributed.partition_csr), walkers regrouped between rounds (walk_partitions_local, the
single-process stand-in for the all-to-all).  Paths, lengths and PPR visit counts must equal
the oracle's unpartitioned walk bit for bit, under both pool layouts."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("layout", ["hot", "relabel"])
@pytest.mark.parametrize("P", [2, 3, 5])
def test_partitioned_walk_equals_oracle(layout, P, monkeypatch):
    import paper_2504_10233_b200 as pb
    from paper_2504_10233_b200.distributed import partition_bounds, partition_csr, walk_partitions_local
    monkeypatch.setenv("BINGO_LAYOUT", layout)
    w = synth.Workload(15, 300_000, compact=True, batch=1000, rounds=1)
    o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    bounds = partition_bounds(w.row_offsets, P)
    engines = [pb.Graph(*partition_csr(w.row_offsets, w.dst, w.bias, bounds[r], bounds[r + 1])) for r in range(P)]
    W = 70_001
    out = walk_partitions_local(engines, bounds, W, length=40, seed=11, first_walker=5)
    ref = o.walk(length=40, seed=11, first_walker=5, num_walkers=W)
    assert np.array_equal(u32(out["lengths"]), ref["lengths"])
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    assert out["rounds"] > 5
    for e in engines:
        e.reset_visit_counts()
    out = walk_partitions_local(engines, bounds, W, app=pb.PPR, length=pb.NO_CAP, seed=12, paths=False)
    refp = o.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=12, num_walkers=W, paths=False, counts=True)
    assert np.array_equal(u32(out["lengths"]), refp["lengths"])
    counts = sum(e.visit_counts().cpu().numpy().view(np.uint64) for e in engines)
    assert np.array_equal(counts, refp["counts"])


def test_partitioned_equals_replicated_gpu_walk():
    """The same launch unpartitioned (bingo_walk) and partitioned 4 ways: identical outputs."""
    import paper_2504_10233_b200 as pb
    from paper_2504_10233_b200.distributed import partition_bounds, partition_csr, walk_partitions_local
    w = synth.Workload(16, 600_000, compact=True, batch=1000, rounds=1)
    g = pb.Graph(w.row_offsets, w.dst, w.bias)
    full = g.walk(length=80, seed=21, num_walkers=w.V)
    bounds = partition_bounds(w.row_offsets, 4)
    engines = [pb.Graph(*partition_csr(w.row_offsets, w.dst, w.bias, bounds[r], bounds[r + 1])) for r in range(4)]
    out = walk_partitions_local(engines, bounds, w.V, length=80, seed=21)
    assert np.array_equal(u32(out["paths"]), u32(full["paths"]))
    assert np.array_equal(u32(out["lengths"]), u32(full["lengths"]))


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_updates_on_partitions(P):
    """f1 in the partitioned regime: every partition applies only the batch records whose
    source vertex it owns (the only copy of that vertex's sampling structure).  After each
    batch the owned vertices' canonical digests equal the oracle graph that applied every
    record, the summed statistics equal its statistics, and the partitioned walk equals its
    walk."""
    import paper_2504_10233_b200 as pb
    from paper_2504_10233_b200.distributed import (apply_updates_partitions_local, partition_bounds, partition_csr,
                                                   walk_partitions_local)
    w = synth.Workload(14, 150_000, compact=True, batch=4000, rounds=3)
    o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    bounds = partition_bounds(w.row_offsets, P)
    engines = [pb.Graph(*partition_csr(w.row_offsets, w.dst, w.bias, bounds[r], bounds[r + 1])) for r in range(P)]
    import torch
    for b in w.batches:
        sts = apply_updates_partitions_local(engines, bounds, torch.from_numpy(b.view(np.int32)).cuda())
        so = o.apply_updates(b)
        for k in ("inserted", "deleted", "missing_deletes", "touched_vertices"):
            assert sum(st[k] for st in sts) == so[k], k
        assert all(st["epoch"] == so["epoch"] for st in sts)
        full = o.digests()
        for r, e in enumerate(engines):
            dg = e.digests().cpu().numpy().view(np.uint64)
            assert np.array_equal(dg[bounds[r]:bounds[r + 1]], full[bounds[r]:bounds[r + 1]]), r
    out = walk_partitions_local(engines, bounds, 40_000, length=50, seed=4)
    ref = o.walk(length=50, seed=4, num_walkers=40_000)
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    with pytest.raises(pb.bingo.BingoError):
        apply_updates_partitions_local(engines, bounds, torch.tensor([[0, 1, w.V, 3]], dtype=torch.int32).cuda())
