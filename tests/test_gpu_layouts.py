"""-m gpu: the pool layouts / vertex relabelling are performance choices only:
under each of them (vertex-id order, hot-first pools, hot-first relabelling) builds, walks,
PPR counts, node2vec with the neighbour index, batched / streaming / float updates must equal
the oracle bit for bit (exports and digests are in external ids)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

LAYOUTS = ["id", "hot", "relabel"]


def u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("route", [{}, {"BINGO_UPD_LEGACY": "1"}])
def test_layout_build_walks_updates(layout, route, monkeypatch):
    import paper_2504_10233_b200 as pb
    monkeypatch.setenv("BINGO_LAYOUT", layout)
    for k, v in route.items():
        monkeypatch.setenv(k, v)
    w = synth.make_workload("c1", rounds=3)
    g = pb.Graph(w.row_offsets, w.dst, w.bias, neighbor_index=True)
    o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    assert g.export() == o.dump()
    for i, b in enumerate(w.batches):
        if i == 1:   # streaming: one record per call (single-launch fast path)
            for r in b[:40]:
                g.apply_updates(r[None, :])
                o.apply_updates(r[None, :])
            b = b[40:]
        sg, so = g.apply_updates(b), o.apply_updates(b)
        assert (sg["deleted"], sg["missing_deletes"], sg["touched_vertices"]) == \
               (so["deleted"], so["missing_deletes"], so["touched_vertices"])
        assert g.export() == o.dump(), f"{layout} batch {i}"
        assert np.array_equal(g.digests().cpu().numpy().view(np.uint64), o.digests())
    starts = (np.arange(3000, dtype=np.uint64) * 2654435761 % w.V).astype(np.uint32)
    out = g.walk(length=60, seed=5, starts=starts)
    ref = o.walk(length=60, seed=5, starts=starts)
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    out = g.walk(app=pb.NODE2VEC, length=30, p=2.0, q=0.5, seed=6)
    ref = o.walk(app=oracle.APP_NODE2VEC, length=30, p=2.0, q=0.5, seed=6)
    assert np.array_equal(u32(out["paths"]), ref["paths"])
    g.walk(app=pb.PPR, length=pb.NO_CAP, seed=7, starts=starts, paths=None)
    refp = o.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=7, starts=starts, paths=False, counts=True)
    assert np.array_equal(g.visit_counts().cpu().numpy().view(np.uint64), refp["counts"])
    assert np.array_equal(g.visit_counts_host(), refp["counts"])


@pytest.mark.parametrize("layout", LAYOUTS)
def test_layout_float_updates(layout, monkeypatch):
    import paper_2504_10233_b200 as pb
    monkeypatch.setenv("BINGO_LAYOUT", layout)
    rng = np.random.default_rng(3)
    w = synth.make_workload("c1")
    wf = rng.random(len(w.dst)) * 8 + 1e-3
    g = pb.Graph(w.row_offsets, w.dst, wf, float_bias=True, arc_slack=0.0, member_slack=0.0, pool_reserve=0.0)
    o = oracle.OracleGraph(w.row_offsets, w.dst, wf, float_bias=True)
    for e in range(3):
        recs = synth.random_batch(rng, w.V, 300, 100)
        ws = rng.random(300) * 6 + 1e-3
        g.apply_updates(recs, bias_f64=ws)
        o.apply_updates(recs, bias_f64=ws)
        assert g.export() == o.dump()
    out = g.walk(length=20, seed=9)
    ref = o.walk(length=20, seed=9)
    assert np.array_equal(u32(out["paths"]), ref["paths"])
