"""-m gpu: parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

c2 (LiveJournal-shaped, 4.7M vertices / 69M arcs, DeepWalk: one walker per vertex x 80 steps in
ONE launch, 100K-record update batches) and c3 (Orkut-shaped, 2.7M vertices / 230M arcs, node2vec
p=2 q=0.5 with the neighbour index, 2M-record batches).  The CUDA path runs exactly as bench.py
runs it; the lazy oracle (builds only the vertices a comparison touches) replays the same batches
and recomputes sampled outputs one by one: canonical digests of touched and random vertices, and
walker-id ranges sliced out of the full launch.  (c4/c5 run the same comparison in
tools/fullsize.py / tools/streaming_sweep.py: minutes of generation, results in profiles/.)"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
import synth
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.mark.parametrize("config", ["c2", "c3"])
def test_fullsize_sampled_parity(config):
    import torch
    import paper_2504_10233_b200 as pb
    app = synth.CONFIGS[config]["app"]
    w = synth.make_workload(config, rounds=2, device="cuda")
    torch.cuda.empty_cache()
    g = pb.Graph(w.row_offsets, w.dst, w.bias, neighbor_index=(app == "node2vec"))
    o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias, lazy=True)
    touched = set()
    for b in w.batches:
        sg = g.apply_updates(torch.from_numpy(b.view(np.int32)).cuda())
        so = o.apply_updates(b)
        for k in ("inserted", "deleted", "missing_deletes", "touched_vertices"):
            assert sg[k] == so[k], (k, sg[k], so[k])
        assert np.array_equal(sg["kind_transitions"], so["kind_transitions"])
        touched.update(np.unique(b[:, 1]).tolist())
    rng = np.random.default_rng(5)
    tv = np.array(sorted(touched), dtype=np.int64)
    sample = np.unique(np.concatenate([rng.choice(tv, size=min(len(tv), 1500), replace=False),
                                       rng.integers(0, w.V, size=1500)]))
    dg = g.digests().cpu().numpy().view(np.uint64)
    bad = [int(u) for u in sample if int(dg[u]) != o.vertex_digest(int(u))]
    assert not bad, f"digest mismatch at vertices {bad[:10]}"
    # the full launch: one walker per vertex x 80 steps (bench.py's configuration)
    kw = dict(app=pb.NODE2VEC if app == "node2vec" else pb.DEEPWALK, length=80, seed=77, num_walkers=w.V)
    okw = dict(app=oracle.APP_NODE2VEC if app == "node2vec" else oracle.APP_DEEPWALK, length=80, seed=77)
    if app == "node2vec":
        kw.update(p=2.0, q=0.5)
        okw.update(p=2.0, q=0.5)
    out = g.walk(**kw)
    P = out["paths"]
    lens = out["lengths"].cpu().numpy().view(np.uint32)
    for s0 in rng.integers(0, w.V - 256, size=4).tolist():
        ref = o.walk(first_walker=s0, num_walkers=256, **okw)
        assert np.array_equal(P[:, s0:s0 + 256].cpu().numpy().view(np.uint32), ref["paths"]), s0
        assert np.array_equal(lens[s0:s0 + 256], ref["lengths"])


def test_c4_ppr_fullsize_parity():
    """c4 (Twitter-shaped, 46M vertices / 1.47B arcs) at full size on the default layout for
    V >= 2^23 (hot-first relabelling, packed visit counters beyond the 4,096 hottest ids):
    two 100K-record update batches with digest parity, the full bench launch (one PPR walker
    per vertex, stop 1/80) with lengths compared on sampled walker ranges, then the counts of a
    2^18-walker id range (more walkers than the resident grid) compared on ALL 46M vertices,
    and capped PPR paths on a sampled range.  The graph is generated in HBM (synth.DeviceWorkload)."""
    import torch
    import paper_2504_10233_b200 as pb
    w = synth.make_workload("c4", rounds=2, hold_rounds=10, device="cuda", resident=True)
    g = pb.Graph(w.row_offsets, w.dst, w.bias)
    assert w.V >= (1 << 23)
    ro, dst, bias = w.host_csr()
    o = oracle.OracleGraph(ro, dst, bias, lazy=True)
    touched = set()
    for b in w.batches:
        sg = g.apply_updates(torch.from_numpy(b.view(np.int32)).cuda())
        so = o.apply_updates(b)
        for k in ("inserted", "deleted", "missing_deletes", "touched_vertices"):
            assert sg[k] == so[k], (k, sg[k], so[k])
        assert np.array_equal(sg["kind_transitions"], so["kind_transitions"])
        touched.update(np.unique(b[:, 1]).tolist())
    rng = np.random.default_rng(9)
    tv = np.array(sorted(touched), dtype=np.int64)
    sample = np.unique(np.concatenate([rng.choice(tv, size=800, replace=False), rng.integers(0, w.V, size=800)]))
    dg = g.digests().cpu().numpy().view(np.uint64)
    bad = [int(u) for u in sample if int(dg[u]) != o.vertex_digest(int(u))]
    assert not bad, f"digest mismatch at vertices {bad[:10]}"
    # the bench launch: every vertex's walker, no paths
    g.reset_visit_counts()
    out = g.walk(app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), seed=4242, num_walkers=w.V, paths=None)
    lens = out["lengths"].cpu().numpy().view(np.uint32)
    tot = g.visit_counts(reset=True)
    assert int(tot.sum()) == int(lens.astype(np.int64).sum()) + w.V
    for s0 in rng.integers(0, w.V - 512, size=3).tolist():
        ref = o.walk(app=oracle.APP_PPR, length=oracle.NONE, stop=(1, 80), seed=4242, first_walker=s0,
                     num_walkers=512, paths=False)
        assert np.array_equal(lens[s0:s0 + 512], ref["lengths"]), s0
    # counts of a 2^18-walker range, compared on every vertex
    W, s0 = 1 << 18, int(rng.integers(0, w.V - (1 << 18)))
    g.walk(app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), seed=4243, first_walker=s0, num_walkers=W, paths=None)
    got = g.visit_counts_host(reset=True)
    ref = o.walk(app=oracle.APP_PPR, length=oracle.NONE, stop=(1, 80), seed=4243, first_walker=s0, num_walkers=W,
                 paths=False, counts=True, threads=os.cpu_count())
    badv = np.nonzero(got != ref["counts"])[0]
    assert badv.size == 0, f"{badv.size} count mismatches, first at {badv[:8].tolist()}"
    assert np.count_nonzero(ref["counts"]) > 100_000
    # capped PPR paths (cap 400) on a sampled range
    s1 = int(rng.integers(0, w.V - 4096))
    outc = g.walk(app=pb.PPR, length=400, stop=(1, 80), seed=4244, first_walker=s1, num_walkers=4096)
    refc = o.walk(app=oracle.APP_PPR, length=400, stop=(1, 80), seed=4244, first_walker=s1, num_walkers=4096,
                  threads=os.cpu_count())
    assert np.array_equal(outc["paths"].cpu().numpy().view(np.uint32), refc["paths"])
