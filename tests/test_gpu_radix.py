"""-m gpu: Bingo with an arbitrary radix base B = 2^b (reading R-17)
through the C-ABI (bingo_build with BINGO_BUILD_RADIX_LOG2(b)): the structure (radix dump
R-18: groups, subgroups, both integer-Vose tables, member order), DeepWalk paths and PPR
visit counts equal the oracle's RadixGraph bit for bit for b = 1..5, also after batches of
updates (reading R-19)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def _check(ro, dst, bias, b, V, walkers=None, L=40):
    import paper_2504_10233_b200 as pb
    g = pb.Graph(ro, dst, bias, radix_log2=b)
    o = oracle.RadixGraph(ro, dst, bias, b)
    a, r = g.export(), o.dump()
    if a != r:
        pa, pr = oracle.parse_radix_dump(a, V), oracle.parse_radix_dump(r, V)
        for u in range(V):
            assert pa[u] == pr[u], f"b={b} vertex {u}:\n gpu    {pa[u]}\n oracle {pr[u]}"
    assert a == r
    W = walkers or V
    out = g.walk(length=L, seed=7 + b, num_walkers=W, first_walker=3)
    ref = o.walk(length=L, seed=7 + b, num_walkers=W, first_walker=3)
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    assert np.array_equal(u32(out["lengths"]), ref["lengths"])
    g.reset_visit_counts()
    out = g.walk(app=pb.PPR, length=pb.NO_CAP, seed=9 + b, num_walkers=W, paths=None)
    ref = o.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=9 + b, num_walkers=W, paths=False, counts=True)
    assert np.array_equal(u32(out["lengths"]), ref["lengths"])
    assert np.array_equal(g.visit_counts().cpu().numpy().view(np.uint64), ref["counts"])
    return g


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5])
def test_radix_c1_and_random_multigraphs(b):
    w = synth.make_workload("c1")
    _check(w.row_offsets, w.dst, w.bias, b, w.V)
    rng = np.random.default_rng(b)
    for trial in range(3):
        V = int(rng.integers(1, 400))
        ro, dst, bias = synth.random_small_graph(rng, V, int(rng.integers(0, 300)),
                                                 int(rng.choice([1, 7, 255, 1 << 20, (1 << 32) - 1])))
        _check(ro, dst, bias, b, V, walkers=5000)


@pytest.mark.parametrize("b", [2, 4])
def test_radix_larger_graph_many_walkers(b):
    w = synth.Workload(16, 600_000, compact=True, batch=1000, rounds=1)
    _check(w.row_offsets, w.dst, w.bias, b, w.V, walkers=400_000, L=80)


def _dump_eq(g, o, V, tag):
    a, r = g.export(), o.dump()
    if a != r:
        pa, pr = oracle.parse_radix_dump(a, V), oracle.parse_radix_dump(r, V)
        for u in range(V):
            assert pa[u] == pr[u], f"{tag} vertex {u}:\n gpu    {pa[u]}\n oracle {pr[u]}"
    assert a == r, tag


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5])
def test_radix_updates_match_the_oracle(b):
    """R-19 through bingo_apply_updates: after every batch (duplicates, deletes of arcs inserted
    in the same batch, missing deletes, a hub of thousands of arcs, delete-all-then-regrow) the
    radix dump, the statistics, DeepWalk paths and PPR counts equal the oracle's; host and
    device batches; pool growth."""
    import paper_2504_10233_b200 as pb
    rng = np.random.default_rng(40 + b)
    V = 300
    ro, dst, bias = synth.random_small_graph(rng, V, 60, int(rng.choice([255, 1 << 20, (1 << 32) - 1])))
    # hubs: vertex 7 crosses the block-per-vertex threshold (4096 arcs) downwards when it loses
    # 2500 arcs, vertex 11 stays above it
    deg = np.diff(ro.astype(np.int64))
    deg[7] = 6000
    deg[11] = 9000
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    dst = rng.integers(0, V, size=int(ro[-1])).astype(np.uint32)
    bias = rng.integers(1, 1 << 16, size=int(ro[-1])).astype(np.uint32)
    g = pb.Graph(ro, dst, bias, radix_log2=b, arc_slack=0.0)
    o = oracle.RadixGraph(ro, dst, bias, b)
    existing = [(u, int(dst[a])) for u in range(V) for a in range(int(ro[u]), int(ro[u + 1]))]
    import torch
    for r in range(8):
        recs = synth.random_batch(rng, V, int(rng.integers(1, 3000)), 1 << 16, existing=existing, p_delete=0.5)
        if r == 2:   # the hub loses many arcs, some twice (missing), and regrows
            hub = [(synth.DELETE, 7, e[0], 0) for e in o.adjacency(7)[:2500]]
            recs = np.concatenate([recs, np.array(hub, dtype=np.uint32), np.array(hub[:40], dtype=np.uint32),
                                   np.array([(synth.INSERT, 7, 3, 9)] * 5, dtype=np.uint32)])
        if r == 5:   # vertex 0: delete everything, then regrow in the next batch
            recs = np.concatenate([recs, np.array([(synth.DELETE, 0, e[0], 0) for e in o.adjacency(0)],
                                                  dtype=np.uint32).reshape(-1, 4)])
        so = o.apply_updates(recs)
        if r % 2:
            sg = g.apply_updates(torch.from_numpy(recs.view(np.int32)).cuda())
        else:
            sg = g.apply_updates(recs)
        for k in ("inserted", "deleted", "missing_deletes", "touched_vertices", "epoch"):
            assert sg[k] == so[k], (r, k, sg[k], so[k])
        _dump_eq(g, o, V, f"b={b} batch {r}")
        existing = [(u, int(e[0])) for u in range(V) for e in o.adjacency(u)]
    out = g.walk(length=40, seed=3, num_walkers=4000)
    ref = o.walk(length=40, seed=3, num_walkers=4000)
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    g.reset_visit_counts()
    out = g.walk(app=pb.PPR, length=pb.NO_CAP, seed=5, num_walkers=20000, paths=None)
    ref = o.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=5, num_walkers=20000, paths=False, counts=True)
    assert np.array_equal(g.visit_counts().cpu().numpy().view(np.uint64), ref["counts"])


def test_radix_update_errors_leave_the_graph_untouched():
    import paper_2504_10233_b200 as pb
    w = synth.make_workload("c1")
    g = pb.Graph(w.row_offsets, w.dst, w.bias, radix_log2=2)
    before = g.export()
    bad = np.array([[0, 1, 2, 0]], dtype=np.uint32)                    # insert with bias 0
    assert g.try_apply_updates(bad) == pb.bingo.E_INVAL
    bad = np.array([[0, 1, 2, 5], [1, w.V, 2, 0]], dtype=np.uint32)    # src >= V
    assert g.try_apply_updates(bad) == pb.bingo.E_INVAL
    assert g.export() == before
    with pytest.raises(pb.bingo.BingoError):
        g.walk(app=pb.NODE2VEC, length=10, p=2.0, q=0.5)
    with pytest.raises(pb.bingo.BingoError):
        pb.Graph(w.row_offsets, w.dst, w.bias, radix_log2=6)
