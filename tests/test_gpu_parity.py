"""-m gpu: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Integer biases -> bit-exact: canonical dumps (R-11), per-vertex digests, walk
paths, lengths and PPR visit counts.  Inputs come from synth (seeded)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _pb():
    import paper_2504_10233_b200 as pb
    return pb


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def _graphs(ro, dst, bias, **kw):
    pb = _pb()
    flags = oracle.FLAG_BS_MODE if kw.get("bs_mode") else 0
    g = pb.Graph(ro, dst, bias, alpha=kw.get("alpha", 40), beta=kw.get("beta", 10), bs_mode=kw.get("bs_mode", False))
    o = oracle.OracleGraph(ro, dst, bias, alpha=kw.get("alpha", 40), beta=kw.get("beta", 10), flags=flags)
    return g, o


def _assert_same_dump(g, o, V):
    a, b = g.export(), o.dump()
    if a != b:
        pa, pb_ = oracle.parse_dump(a, V), oracle.parse_dump(b, V)
        for u in range(V):
            assert pa[u] == pb_[u], f"vertex {u}: gpu {pa[u]} != oracle {pb_[u]}"
    assert a == b
    dg = g.digests().cpu().numpy().view(np.uint64)
    assert np.array_equal(dg, o.digests())


@pytest.mark.parametrize("bias_kind", ["degree", "uniform", "loguniform"])
def test_build_parity_c1(bias_kind):
    w = synth.make_workload("c1", bias=bias_kind)
    g, o = _graphs(w.row_offsets, w.dst, w.bias)
    _assert_same_dump(g, o, w.V)


@pytest.mark.parametrize("bs_mode", [False, True])
def test_build_parity_random_multigraphs(bs_mode):
    rng = np.random.default_rng(3)
    for trial in range(6):
        V = int(rng.integers(1, 300))
        ro, dst, bias = synth.random_small_graph(rng, V, max_deg=int(rng.integers(0, 200)),
                                                 max_bias=int(rng.choice([1, 3, 255, 1 << 20, (1 << 32) - 1])))
        g, o = _graphs(ro, dst, bias, bs_mode=bs_mode)
        _assert_same_dump(g, o, V)


def test_build_parity_hub_and_many_groups():
    """A hub spanning many 32-arc chunks with all 32 radix bits in use (ragged tail)."""
    rng = np.random.default_rng(9)
    d = 50_003
    V = 5
    ro = np.array([0, d, d, d + 7, d + 7, d + 7], dtype=np.uint64)
    dst = rng.integers(0, V, size=d + 7).astype(np.uint32)
    bias = (rng.integers(1, 1 << 31, size=d + 7) | (1 << rng.integers(0, 32, size=d + 7))).astype(np.uint32)
    bias[:100] = 1 << 31
    g, o = _graphs(ro, dst, bias)
    _assert_same_dump(g, o, V)


def test_build_rejects_invalid():
    pb = _pb()
    with pytest.raises(pb.BingoError):
        pb.Graph([0, 1], [5], [1])            # dst >= V
    with pytest.raises(pb.BingoError):
        pb.Graph([0, 1], [0], [0])            # zero bias
    g = pb.Graph([0, 2, 2], [0, 1], [(1 << 32) - 1] * 2)   # max biases: T * n < 2^64 is fine
    assert g.info()["num_vertices"] == 2


@pytest.mark.parametrize("seed", [1, 2, 0xDEADBEEFCAFEF00D])
def test_deepwalk_parity_c1(seed):
    pb = _pb()
    w = synth.make_workload("c1")
    g, o = _graphs(w.row_offsets, w.dst, w.bias)
    out = g.walk(app=pb.DEEPWALK, length=80, seed=seed)
    ref = o.walk(length=80, seed=seed)
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    assert np.array_equal(u32(out["lengths"]), ref["lengths"])


def test_deepwalk_parity_starts_shards_and_host_path():
    pb = _pb()
    w = synth.make_workload("c1", bias="loguniform")
    g, o = _graphs(w.row_offsets, w.dst, w.bias)
    rng = np.random.default_rng(4)
    starts = rng.integers(0, w.V, size=5000).astype(np.uint32)
    ref = o.walk(length=33, seed=77, first_walker=1000, starts=starts)
    out = g.walk(length=33, seed=77, first_walker=1000, starts=starts)
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    # host buffers through the same C-ABI call
    import torch
    hp = torch.empty((34, 5000), dtype=torch.int32).pin_memory()
    hl = torch.empty(5000, dtype=torch.int32).pin_memory()
    g.walk_host(length=33, seed=77, first_walker=1000, starts=starts, paths=hp, lengths=hl)
    assert np.array_equal(hp.numpy().view(np.uint32), ref["paths"])
    assert np.array_equal(hl.numpy().view(np.uint32), ref["lengths"])
    # chunked host-output pipeline (several chunks: > 2^18 walkers), step- and walker-major
    big = rng.integers(0, w.V, size=700_001).astype(np.uint32)
    refb = o.walk(length=12, seed=5, first_walker=3, starts=big)
    hp2 = torch.empty((13, len(big)), dtype=torch.int32).pin_memory()
    hl2 = torch.empty(len(big), dtype=torch.int32).pin_memory()
    g.walk_host(length=12, seed=5, first_walker=3, starts=big, paths=hp2, lengths=hl2)
    assert np.array_equal(hp2.numpy().view(np.uint32), refb["paths"])
    assert np.array_equal(hl2.numpy().view(np.uint32), refb["lengths"])
    hp3 = torch.empty((len(big), 13), dtype=torch.int32).pin_memory()
    g.walk_host(length=12, seed=5, first_walker=3, starts=big, paths=hp3, lengths=hl2, walker_major=True)
    assert np.array_equal(hp3.numpy().view(np.uint32).T, refb["paths"])
    # sharding by first_walker_id reproduces the unsharded run (P-invariance)
    a = g.walk(length=33, seed=77, first_walker=1000, starts=starts[:1234])
    b = g.walk(length=33, seed=77, first_walker=1000 + 1234, starts=starts[1234:])
    assert np.array_equal(np.concatenate([u32(a["paths"]), u32(b["paths"])], axis=1), ref["paths"])


def test_walk_edge_cases():
    pb = _pb()
    # isolated vertices, a self loop, length 0, a single huge-bias arc
    ro = np.array([0, 0, 1, 3, 3], dtype=np.uint64)
    dst = np.array([1, 0, 2], dtype=np.uint32)
    bias = np.array([7, (1 << 32) - 1, 1], dtype=np.uint32)
    g, o = _graphs(ro, dst, bias)
    _assert_same_dump(g, o, 4)
    for L in (0, 1, 5):
        out = g.walk(length=L, seed=3)
        ref = o.walk(length=L, seed=3)
        assert np.array_equal(u32(out["paths"]), ref["paths"])
        assert np.array_equal(u32(out["lengths"]), ref["lengths"])


@pytest.mark.parametrize("p,q,index", [(2.0, 0.5, True), (0.5, 2.0, True), (1.0, 1.0, True), (2.0, 0.5, False),
                                        (1.0, 2.0, True), (0.25, 4.0, False), (3.0, 0.7, True)])
def test_node2vec_parity(p, q, index):
    pb = _pb()
    w = synth.make_workload("c1")
    g = pb.Graph(w.row_offsets, w.dst, w.bias, neighbor_index=index)
    o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    out = g.walk(app=pb.NODE2VEC, length=40, p=p, q=q, seed=21)
    ref = o.walk(app=oracle.APP_NODE2VEC, length=40, p=p, q=q, seed=21)
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    # the neighbour index follows updates
    for b in synth.make_workload("c1", rounds=2).batches:
        g.apply_updates(b)
        o.apply_updates(b)
    out = g.walk(app=pb.NODE2VEC, length=40, p=p, q=q, seed=22)
    ref = o.walk(app=oracle.APP_NODE2VEC, length=40, p=p, q=q, seed=22)
    assert np.array_equal(u32(out["paths"]), ref["paths"])


def test_ppr_parity_counts():
    pb = _pb()
    w = synth.make_workload("c1")
    g, o = _graphs(w.row_offsets, w.dst, w.bias)
    starts = np.arange(20_000, dtype=np.uint32) % w.V
    g.walk(app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), seed=8, starts=starts, paths=None)
    ref = o.walk(app=oracle.APP_PPR, length=oracle.NONE, stop=(1, 80), seed=8, starts=starts, paths=False, counts=True)
    assert np.array_equal(g.visit_counts(reset=True).cpu().numpy().view(np.uint64), ref["counts"])
    out = g.walk(app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), seed=8, starts=starts, paths=None)
    assert np.array_equal(u32(out["lengths"]), ref["lengths"])
    # capped PPR with paths
    out = g.walk(app=pb.PPR, length=50, stop=(1, 10), seed=9, starts=starts)
    ref = o.walk(app=oracle.APP_PPR, length=50, stop=(1, 10), seed=9, starts=starts)
    assert np.array_equal(u32(out["paths"]), ref["paths"])


def test_walk_parity_larger_graph():
    """A scale-16 R-MAT with unclamped degree biases (big T): spans many warps, tiles and a
    ragged tail of walkers; sampled outputs compared element by element."""
    pb = _pb()
    w = synth.Workload(16, 600_000, compact=True, batch=1000, rounds=1)
    g, o = _graphs(w.row_offsets, w.dst, w.bias)
    dg = g.digests().cpu().numpy().view(np.uint64)
    assert np.array_equal(dg, o.digests())
    W = 100_003
    starts = (np.arange(W, dtype=np.uint64) * 2654435761 % w.V).astype(np.uint32)
    out = g.walk(length=80, seed=1234, starts=starts)
    ref = o.walk(length=80, seed=1234, starts=starts)
    assert np.array_equal(u32(out["paths"]), ref["paths"])


def test_walker_major_layout_and_profile():
    """BINGO_WALK_WALKER_MAJOR is the transpose of the step-major paths; the profiling variant
    returns the same walks and load counts consistent with the steps taken."""
    pb = _pb()
    w = synth.make_workload("c1")
    g, o = _graphs(w.row_offsets, w.dst, w.bias)
    ref = o.walk(length=80, seed=31)
    wm = g.walk(length=80, seed=31, walker_major=True)
    assert np.array_equal(u32(wm["paths"]).T, ref["paths"])
    assert np.array_equal(u32(wm["lengths"]), ref["lengths"])
    pr = g.walk_profile(length=80, seed=31)
    assert np.array_equal(u32(pr["paths"]), ref["paths"])
    assert pr["steps"] == int(ref["lengths"].astype(np.int64).sum())
    assert pr["bkt"] == pr["steps"] and pr["walkers"] == w.V
    assert pr["hdr"] >= pr["steps"] and pr["arc"] + pr["mem"] <= pr["steps"] + pr["arc"]
    ppr = g.walk(app=pb.PPR, length=40, stop=(1, 7), seed=4, walker_major=True)
    rp = o.walk(app=oracle.APP_PPR, length=40, stop=(1, 7), seed=4)
    assert np.array_equal(u32(ppr["paths"]).T, rp["paths"])


def test_walk_on_a_side_stream():
    """temporaries (starts copied from host, auto-allocated paths/lengths) are made on
    the current stream; a launch on another stream must be ordered after them and must keep
    them alive until it completes."""
    import torch
    pb = _pb()
    w = synth.make_workload("c1")
    g, o = _graphs(w.row_offsets, w.dst, w.bias)
    s = torch.cuda.Stream()
    starts = (np.arange(50_000, dtype=np.uint64) * 7919 % w.V).astype(np.uint32)
    outs = [g.walk(length=40, seed=100 + i, starts=starts, stream=s) for i in range(4)]
    torch.cuda.synchronize()
    for i, out in enumerate(outs):
        ref = o.walk(length=40, seed=100 + i, starts=starts)
        assert np.array_equal(u32(out["paths"]), ref["paths"])
    g.walk(app=pb.PPR, length=pb.NO_CAP, seed=5, starts=starts, paths=None, stream=s)
    c = g.visit_counts(reset=True, stream=s)
    s.synchronize()
    ref = o.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=5, starts=starts, paths=False, counts=True)
    assert np.array_equal(c.cpu().numpy().view(np.uint64), ref["counts"])
