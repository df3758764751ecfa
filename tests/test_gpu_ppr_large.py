"""-m gpu: PPR visit counts (row a6) and long walks compared element by element with the
oracle at sizes that exercise every code path of the walker kernel:

* V >= 65,536, so almost every vertex lives in the PACKED part of the visit-counter array
  (only the 4,096 hottest internal ids get padded 256 B slots, visit_slot in
  csrc/bingo_internal.cuh), under both pool layouts the build picks between ("hot":
  external ids, "relabel": internal id = hot rank, counts translated back at the boundary);
* more walkers than the persistent grid holds (148 SMs x resident blocks x 256 lanes, about
  227K), so lanes claim new walker ids while others still walk (the refill in k_walk) --
  PPR's geometric lengths make the claims staggered;
* after update batches, so the counts are taken on a mutated structure.

The oracle is the plain CPU definition (P:93 visit frequency, P:536 stop w.p. 1/80 after
each step, start counted -- R-13); the two share only the seeded inputs of synth/."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

W_PPR = 600_000          # > 2.6x the resident grid
W_CAP = 300_000
FIRST = 123_457          # a walker-id offset (sharded runs start anywhere)


def u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.fixture(scope="module")
def big():
    w = synth.Workload(17, 1_300_000, compact=True, batch=3000, rounds=2)
    assert w.V >= 65_536 and w.V > 4096 * 8
    o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    for b in w.batches:
        o.apply_updates(b)
    return w, o


def _gpu_graph(w, layout, monkeypatch):
    import paper_2504_10233_b200 as pb
    monkeypatch.setenv("BINGO_LAYOUT", layout)
    g = pb.Graph(w.row_offsets, w.dst, w.bias)
    for b in w.batches:
        g.apply_updates(b)
    return g


@pytest.mark.parametrize("layout", ["hot", "relabel"])
def test_ppr_counts_large_graph_many_walkers(big, layout, monkeypatch):
    import paper_2504_10233_b200 as pb
    w, o = big
    g = _gpu_graph(w, layout, monkeypatch)
    assert g.digests().cpu().numpy().view(np.uint64).tolist() == o.digests().tolist()
    g.reset_visit_counts()
    out = g.walk(app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), seed=77, first_walker=FIRST, num_walkers=W_PPR,
                 paths=None)
    ref = o.walk(app=oracle.APP_PPR, length=oracle.NONE, stop=(1, 80), seed=77, first_walker=FIRST,
                 num_walkers=W_PPR, paths=False, counts=True)
    assert np.array_equal(u32(out["lengths"]), ref["lengths"])
    got = g.visit_counts().cpu().numpy().view(np.uint64)
    bad = np.nonzero(got != ref["counts"])[0]
    assert bad.size == 0, f"{bad.size} count mismatches, first at vertices {bad[:8].tolist()}"
    # the packed part of the counter array carried real traffic
    assert int(ref["counts"].sum()) == int(ref["lengths"].astype(np.int64).sum()) + W_PPR
    assert np.count_nonzero(ref["counts"]) > 4096 * 4
    # the host copy path and the reset
    assert np.array_equal(g.visit_counts_host(reset=True), ref["counts"])
    assert int(g.visit_counts().sum()) == 0
    # a second launch accumulates on top of the first (no reset in between)
    g.walk(app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), seed=78, num_walkers=W_PPR // 3, paths=None)
    g.walk(app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), seed=79, first_walker=W_PPR // 3, num_walkers=W_PPR // 3,
           paths=None)
    r1 = o.walk(app=oracle.APP_PPR, length=oracle.NONE, stop=(1, 80), seed=78, num_walkers=W_PPR // 3,
                paths=False, counts=True)
    r2 = o.walk(app=oracle.APP_PPR, length=oracle.NONE, stop=(1, 80), seed=79, first_walker=W_PPR // 3,
                num_walkers=W_PPR // 3, paths=False, counts=True)
    assert np.array_equal(g.visit_counts(reset=True).cpu().numpy().view(np.uint64), r1["counts"] + r2["counts"])


@pytest.mark.parametrize("layout", ["hot", "relabel"])
def test_capped_ppr_paths_large_graph(big, layout, monkeypatch):
    """PPR with a length cap of 400 (paths returned): every path entry, every length and the
    counts of the same launch."""
    import paper_2504_10233_b200 as pb
    w, o = big
    g = _gpu_graph(w, layout, monkeypatch)
    g.reset_visit_counts()
    starts = (np.arange(W_CAP, dtype=np.uint64) * 40503 % w.V).astype(np.uint32)
    out = g.walk(app=pb.PPR, length=400, stop=(1, 80), seed=91, starts=starts, first_walker=FIRST)
    ref = o.walk(app=oracle.APP_PPR, length=400, stop=(1, 80), seed=91, starts=starts, first_walker=FIRST,
                 counts=True)
    assert np.array_equal(u32(out["lengths"]), ref["lengths"])
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    assert (ref["lengths"] == 400).any() and (ref["lengths"] < 400).any()
    assert np.array_equal(g.visit_counts(reset=True).cpu().numpy().view(np.uint64), ref["counts"])


@pytest.mark.parametrize("layout", ["hot", "relabel"])
def test_deepwalk_many_walkers_and_profile(big, layout, monkeypatch):
    """DeepWalk with more walkers than the grid holds (refill in groups of 32), and the
    profiling launch's dense-attempt count (the roofline numerator's arc term) pinned to the
    oracle's own count of sequential dense attempts."""
    import paper_2504_10233_b200 as pb
    w, o = big
    g = _gpu_graph(w, layout, monkeypatch)
    W = 500_000
    out = g.walk(length=80, seed=33, first_walker=FIRST, num_walkers=W)
    ref = o.walk(length=80, seed=33, first_walker=FIRST, num_walkers=W)
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    pr = g.walk_profile(length=80, seed=33, first_walker=FIRST, num_walkers=W)
    assert np.array_equal(u32(pr["paths"]), ref["paths"])
    steps = int(ref["lengths"].astype(np.int64).sum())
    assert pr["steps"] == steps and pr["bkt"] == steps and pr["walkers"] == W
    assert pr["arc"] == ref["dense_attempts"], (pr["arc"], ref["dense_attempts"])
    assert pr["mem"] + (pr["arc"] > 0) <= steps + 1


def test_node2vec_profile_dense_attempts(big, monkeypatch):
    import paper_2504_10233_b200 as pb
    w, o = big
    g = _gpu_graph(w, "hot", monkeypatch)
    pr = g.walk_profile(app=pb.NODE2VEC, length=20, p=2.0, q=0.5, seed=44, num_walkers=50_000)
    ref = o.walk(app=oracle.APP_NODE2VEC, length=20, p=2.0, q=0.5, seed=44, num_walkers=50_000)
    assert np.array_equal(u32(pr["paths"]), ref["paths"])
    assert pr["arc"] == ref["dense_attempts"]


@pytest.mark.parametrize("app", ["deepwalk", "ppr"])
def test_trace_replay_counts(big, app, monkeypatch):
    """Measurement path (bench.py's gather ceiling): bingo_walk_trace runs the same walks as
    bingo_walk and records one entry per step; bingo_walk_replay re-issues exactly the loads the
    profile counted (headers = buckets = steps, members = profile members, dense attempts =
    the first two of every dense step)."""
    import torch
    import paper_2504_10233_b200 as pb
    w, o = big
    g = _gpu_graph(w, "relabel", monkeypatch)
    kw = dict(app=pb.PPR, length=pb.NO_CAP, stop=(1, 80)) if app == "ppr" else dict(app=pb.DEEPWALK, length=80)
    W = 200_000
    pr = g.walk_profile(seed=55, first_walker=FIRST, num_walkers=W, paths=False, **kw)
    lens = pr["lengths"].to(torch.int64)
    off = torch.zeros(W + 1, dtype=torch.int64, device=lens.device)
    off[1:] = torch.cumsum(lens, 0)
    n = int(off[-1])
    trace = torch.empty((n, 4), dtype=torch.int32, device=lens.device)
    tp = g.walk_trace(off, trace, seed=55, first_walker=FIRST, num_walkers=W, **kw)
    for k in ("steps", "hdr", "bkt", "mem", "arc"):
        assert tp[k] == pr[k], (k, tp[k], pr[k])
    assert n == pr["steps"]
    rep = g.walk_replay(trace, off)
    assert rep["hdr"] == rep["bkt"] == n
    assert rep["mem"] == pr["mem"]
    assert 0 < rep["arc"] <= pr["arc"]
    ref = o.walk(app=oracle.APP_PPR if app == "ppr" else oracle.APP_DEEPWALK,
                 length=oracle.NONE if app == "ppr" else 80, stop=(1, 80), seed=55, first_walker=FIRST,
                 num_walkers=W, paths=False)
    assert np.array_equal(lens.cpu().numpy().astype(np.uint32), ref["lengths"])
