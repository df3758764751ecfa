"""-m gpu: sharded update application in the replicated regime (updates are
independent per source vertex) through the C-ABI.  Two replicas of one graph each apply only
the records whose source they own (src mod 2), export the post-batch state of those vertices
(bingo_export_vertices) and install the other replica's export (bingo_import_vertices); after
every batch both replicas' canonical dumps equal the oracle that applied the whole batch, the
statistics add up to the oracle's, and walks after the batches are bit-exact -- under the
vertex-id, hot-first and relabelled layouts, with hubs, duplicate arcs, missing deletes and
pool growth."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def _owned(recs, r, P):
    return np.ascontiguousarray(recs[recs[:, 1] % P == r])


@pytest.mark.parametrize("layout", ["id", "hot", "relabel"])
def test_sharded_updates_keep_replicas_identical(layout, monkeypatch):
    import paper_2504_10233_b200 as pb
    monkeypatch.setenv("BINGO_LAYOUT", layout)
    if layout == "relabel":   # hub delete / group indices on (imports drop them, later batches rebuild)
        monkeypatch.setenv("BINGO_INDEX_MIN", "1024")
    rng = np.random.default_rng({"id": 1, "hot": 2, "relabel": 3}[layout])
    V = 500
    ro, dst, bias = synth.random_small_graph(rng, V, 50, 1 << 20)
    deg = np.diff(ro.astype(np.int64))
    deg[3], deg[8] = 4000, 1500   # hubs (the bulk route's large-vertex chain)
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    dst = rng.integers(0, V, size=int(ro[-1])).astype(np.uint32)
    bias = rng.integers(1, 1 << 20, size=int(ro[-1])).astype(np.uint32)
    P = 2
    reps = [pb.Graph(ro, dst, bias, arc_slack=0.0, member_slack=0.0, pool_reserve=0.0) for _ in range(P)]
    o = oracle.OracleGraph(ro, dst, bias)
    existing = [(u, int(dst[a])) for u in range(V) for a in range(int(ro[u]), int(ro[u + 1]))]
    for r in range(6):
        recs = synth.random_batch(rng, V, int(rng.integers(50, 2500)), 1 << 20, existing=existing, p_delete=0.5)
        if r == 2:   # hub 3 loses most of its arcs
            hub = [(synth.DELETE, 3, int(dst[a]), 0) for a in range(int(ro[3]), int(ro[3]) + 3500)]
            recs = np.concatenate([recs, np.array(hub, dtype=np.uint32)])
        so = o.apply_updates(recs)
        st = [g.apply_updates(_owned(recs, k, P)) for k, g in enumerate(reps)]
        for key in ("inserted", "deleted", "missing_deletes", "touched_vertices"):
            assert sum(s[key] for s in st) == so[key], (r, key)
        assert np.array_equal(sum(s["kind_transitions"] for s in st), so["kind_transitions"])
        assert all(s["epoch"] == so["epoch"] for s in st)
        exports = []
        for k, g in enumerate(reps):
            ids = torch.unique(torch.from_numpy(_owned(recs, k, P)[:, 1].astype(np.int64)))
            exports.append(g.export_vertices(ids.cuda()))
        for k, g in enumerate(reps):
            for j, (buf, off) in enumerate(exports):
                if j != k:
                    g.import_vertices(buf, off)
        want = o.dump()
        for k, g in enumerate(reps):
            assert g.export() == want, (layout, r, k)
        existing = [(u, e[0]) for u, v in enumerate(oracle.parse_dump(want, V)) for e in v["adj"]]
    ref = o.walk(length=40, seed=9, num_walkers=3000)
    for g in reps:
        out = g.walk(length=40, seed=9, num_walkers=3000)
        assert np.array_equal(u32(out["paths"]), ref["paths"])
    # the replicas keep updating normally after imports (their pools and indices stay consistent)
    recs = synth.random_batch(rng, V, 800, 1 << 20, existing=existing, p_delete=0.5)
    o.apply_updates(recs)
    for g in reps:
        g.apply_updates(recs)
        assert g.export() == o.dump()


def test_export_import_errors():
    import paper_2504_10233_b200 as pb
    w = synth.make_workload("c1")
    g = pb.Graph(w.row_offsets, w.dst, w.bias)
    with pytest.raises(pb.bingo.BingoError):
        g.export_vertices(torch.tensor([w.V], dtype=torch.int32).cuda())
    buf, off = g.export_vertices(torch.tensor([], dtype=torch.int32).cuda())
    assert off.numel() == 1 and int(off[0]) == 0
    before = g.export()
    g.import_vertices(*g.export_vertices(torch.arange(w.V, dtype=torch.int32).cuda()))   # a no-op round trip
    assert g.export() == before
    # records that do not parse are rejected before anything is written
    buf, off = g.export_vertices(torch.arange(4, dtype=torch.int32).cuda())
    for bad in ("vertex", "length", "member"):
        b2 = buf.clone()
        if bad == "vertex":
            b2[0] = w.V
        elif bad == "length":
            b2[1] += 1
        else:   # a list member index beyond the adjacency, or (no list groups) the group count
            b2[2] = 33
        with pytest.raises(pb.bingo.BingoError):
            g.import_vertices(b2, off)
        assert g.export() == before
    gn = pb.Graph(w.row_offsets, w.dst, w.bias, neighbor_index=True)
    with pytest.raises(pb.bingo.BingoError):
        gn.export_vertices(torch.tensor([0], dtype=torch.int32).cuda())
