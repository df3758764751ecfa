"""-m gpu: Bingo with an arbitrary radix base B = 2^b (reading R-17)
through the C-ABI (bingo_build with BINGO_BUILD_RADIX_LOG2(b)): the structure (radix dump
R-18: groups, subgroups, both integer-Vose tables, member order), DeepWalk paths and PPR
visit counts equal the oracle's RadixGraph bit for bit for b = 1..5; the static structure
refuses updates."""
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


def test_radix_graph_is_static():
    import paper_2504_10233_b200 as pb
    w = synth.make_workload("c1")
    g = pb.Graph(w.row_offsets, w.dst, w.bias, radix_log2=2)
    assert g.try_apply_updates(w.batches[0]) == pb.bingo.E_INVAL
    with pytest.raises(pb.bingo.BingoError):
        g.walk(app=pb.NODE2VEC, length=10, p=2.0, q=0.5)
    with pytest.raises(pb.bingo.BingoError):
        pb.Graph(w.row_offsets, w.dst, w.bias, radix_log2=6)
