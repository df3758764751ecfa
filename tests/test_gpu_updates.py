"""-m gpu: batched insert/delete on the device vs the CPU oracle, bit-exact after every batch
(canonical dumps, digests, statistics), plus walks on the updated structures."""
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


def _pair(ro, dst, bias, bs_mode=False, **kw):
    pb = _pb()
    g = pb.Graph(ro, dst, bias, bs_mode=bs_mode, **kw)
    o = oracle.OracleGraph(ro, dst, bias, flags=oracle.FLAG_BS_MODE if bs_mode else 0)
    return g, o


def _same(g, o, V, ctx=""):
    a, b = g.export(), o.dump()
    if a != b:
        pa, pb_ = oracle.parse_dump(a, V), oracle.parse_dump(b, V)
        for u in range(V):
            assert pa[u] == pb_[u], f"{ctx} vertex {u}:\n gpu    {pa[u]}\n oracle {pb_[u]}"
    assert a == b
    assert np.array_equal(g.digests().cpu().numpy().view(np.uint64), o.digests())


def _same_stats(sg, so):
    for k in ("inserted", "deleted", "missing_deletes", "touched_vertices", "epoch"):
        assert sg[k] == so[k], (k, sg[k], so[k])
    assert np.array_equal(sg["kind_transitions"], so["kind_transitions"])


def test_paper_examples_bs_mode():
    """P:317 insertion then P:336 deletion on the running example, explicit lists (BS mode)."""
    ro = np.array([0, 0, 0, 3, 3, 3, 3], dtype=np.uint64)
    g, o = _pair(ro, [1, 4, 5], [5, 4, 3], bs_mode=True)
    for batch in ([[0, 2, 3, 3]], [[1, 2, 1, 0]]):
        _same_stats(g.apply_updates(np.array(batch, dtype=np.uint32)), o.apply_updates(batch))
        _same(g, o, 6)


def test_c1_stream_batches():
    w = synth.make_workload("c1", rounds=4)
    g, o = _pair(w.row_offsets, w.dst, w.bias)
    for i, b in enumerate(w.batches):
        _same_stats(g.apply_updates(b), o.apply_updates(b))
        _same(g, o, w.V, f"batch {i}")
        out = g.walk(length=80, seed=100 + i)
        ref = o.walk(length=80, seed=100 + i)
        assert np.array_equal(u32(out["paths"]), ref["paths"])


def _bias_of(u, v, e, hi):
    return 1 + ((u * 2654435761 + v * 40503 + e * 97) % hi)


ROUTES = {
    "bsp": {},                                                  # bulk-synchronous pipeline (default)
    "bsp-sub": {"BINGO_BSP_MAXT": "7"},                         # ... in sub-batches of 7 touched vertices
    "bsp-hix": {"BINGO_HUB_INDEX": "1", "BINGO_INDEX_MIN": "1024"},   # ... with both update indices from 1K arcs
    "bsp-noidx": {"BINGO_HUB_INDEX": "0", "BINGO_GROUP_INDEX": "0"},  # ... without any update index
    "bsp-fused": {"BINGO_BSP_FUSED": "1"},                      # ... small vertices by one fused kernel
    "bsp-sync": {"BINGO_UPD_SYNC": "1"},                        # ... host round trips after front end / plan
    "bsp-radix": {"BINGO_UPD_RADIX_FRONT": "1"},                # ... segmented by the radix sort
    "bsp-nogix": {"BINGO_GROUP_INDEX": "0", "BINGO_INDEX_MIN": "1024"},  # ... hub delete index, group scans
    "legacy": {"BINGO_UPD_LEGACY": "1"},                        # per-vertex mutate kernels (warp / block)
    "legacy-block": {"BINGO_UPD_LEGACY": "1", "BINGO_UPD_SMALL_L": "0"},   # ... every vertex on a block
}


@pytest.mark.parametrize("seed,bs_mode,hi,route,hub", [
    (0, False, 200, "bsp", 700), (1, False, 1 << 20, "bsp", 700), (2, True, 200, "bsp", 700),
    (3, False, 7, "bsp", 700), (4, False, 255, "bsp", 700), (5, True, 1 << 31, "bsp", 700),
    (7, False, 200, "bsp", 3500), (8, False, 7, "bsp", 5000), (9, True, 255, "bsp", 3000),
    (0, False, 200, "bsp-sub", 700), (8, False, 7, "bsp-sub", 5000),
    (7, False, 200, "bsp-hix", 3500), (8, False, 7, "bsp-hix", 5000), (9, True, 255, "bsp-hix", 3000),
    (0, False, 200, "bsp-sync", 700), (8, False, 7, "bsp-sync", 5000), (9, True, 255, "bsp-sync", 3000),
    (1, False, 1 << 20, "bsp-radix", 700), (8, False, 7, "bsp-radix", 5000),
    (7, False, 200, "bsp-nogix", 3500), (9, True, 255, "bsp-nogix", 3000),
    (7, False, 200, "bsp-noidx", 3500), (8, False, 7, "bsp-noidx", 5000),
    (0, False, 200, "bsp-fused", 700), (5, True, 1 << 31, "bsp-fused", 700),
    (0, False, 200, "legacy", 700), (3, False, 7, "legacy", 700), (7, False, 200, "legacy", 3500),
    (0, False, 200, "legacy-block", 700), (3, False, 7, "legacy-block", 700),
    (6, False, 1 << 20, "legacy-block", 700)])
def test_random_multigraph_batches(seed, bs_mode, hi, route, hub, monkeypatch):
    """Random multigraphs with duplicates, hubs (multi-chunk scans: 32-arc warp chunks and
    1024-position chunk items), missing deletes, repeated deletes of one pair, mixed biases
    forcing kind transitions in every direction -- through every update route."""
    for k, v in ROUTES[route].items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(1000 + seed)
    V = int(rng.integers(5, 60))
    deg = rng.integers(0, 30, size=V)
    deg[0] = hub                               # a hub spanning many chunks
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    A = int(ro[-1])
    dst = rng.integers(0, V, size=A).astype(np.uint32)
    src = np.repeat(np.arange(V), deg)
    bias = np.array([_bias_of(int(s), int(d), 0, hi) for s, d in zip(src, dst)], dtype=np.uint32)
    g, o = _pair(ro, dst, bias, bs_mode=bs_mode, arc_slack=0.0, member_slack=0.0, pool_reserve=0.0)
    live = {u: list(dst[int(ro[u]):int(ro[u + 1])]) for u in range(V)}
    for e in range(1, 13):
        n = int(rng.integers(0, 400))
        recs = np.zeros((n, 4), dtype=np.uint32)
        for i in range(n):
            u = 0 if rng.random() < 0.3 else int(rng.integers(0, V))
            if rng.random() < 0.5:
                if live[u] and rng.random() < 0.85:
                    v = int(live[u][int(rng.integers(0, len(live[u])))])
                else:
                    v = int(rng.integers(0, V))
                recs[i] = (1, u, v, 0)
            else:
                v = int(rng.integers(0, V))
                recs[i] = (0, u, v, _bias_of(u, v, e, hi) if rng.random() < 0.7 else int(rng.integers(1, hi + 1)))
                live[u].append(v)
        _same_stats(g.apply_updates(recs), o.apply_updates(recs))
        _same(g, o, V, f"seed {seed} batch {e}")
        d = oracle.parse_dump(o.dump(), V)
        live = {u: [a[0] for a in d[u]["adj"]] for u in range(V)}
    out = g.walk(length=30, seed=5)
    ref = o.walk(length=30, seed=5)
    assert np.array_equal(u32(out["paths"]), ref["paths"])


def test_delete_everything_and_regrow():
    rng = np.random.default_rng(7)
    ro, dst, bias = synth.random_small_graph(rng, 20, 40, 1000)
    g, o = _pair(ro, dst, bias)
    recs = []
    for u in range(20):
        for i in range(int(ro[u]), int(ro[u + 1])):
            recs.append((1, u, int(dst[i]), 0))
    recs = np.array(recs, dtype=np.uint32)
    _same_stats(g.apply_updates(recs), o.apply_updates(recs))
    _same(g, o, 20, "all deleted")
    ins = np.array([(0, u, (u * 7 + j) % 20, 1 + (u * 31 + j) % 900) for u in range(20) for j in range(25)], dtype=np.uint32)
    _same_stats(g.apply_updates(ins), o.apply_updates(ins))
    _same(g, o, 20, "regrown")


def test_invalid_batch_and_empty_batch():
    pb = _pb()
    w = synth.make_workload("c1")
    g, o = _pair(w.row_offsets, w.dst, w.bias)
    before = g.export()
    for bad in ([[0, 0, w.V, 1]], [[0, w.V, 0, 1]], [[0, 1, 2, 0]], [[3, 1, 2, 3]]):
        assert g.try_apply_updates(np.array(bad, dtype=np.uint32)) == pb.bingo.E_INVAL
        assert g.export() == before
    st = g.apply_updates(np.zeros((0, 4), dtype=np.uint32))
    assert st["epoch"] == 1 and st["touched_vertices"] == 0
    o.apply_updates(np.zeros((0, 4), dtype=np.uint32))
    b = w.batches[0]
    _same_stats(g.apply_updates(b), o.apply_updates(b))
    _same(g, o, w.V)


def test_device_batch_equals_host_batch():
    import torch
    w = synth.make_workload("c1", rounds=2)
    g1, o = _pair(w.row_offsets, w.dst, w.bias)
    g2, _ = _pair(w.row_offsets, w.dst, w.bias)
    for b in w.batches:
        g1.apply_updates(b)
        g2.apply_updates(torch.from_numpy(b.view(np.int32)).cuda())
        o.apply_updates(b)
    assert g1.export() == g2.export() == o.dump()


def test_streaming_single_records():
    """a11: the same stream applied one record per call (streaming updates, S4.2)."""
    w = synth.make_workload("c1")
    g, o = _pair(w.row_offsets, w.dst, w.bias)
    for r in w.batches[0][:300]:
        _same_stats(g.apply_updates(r[None, :]), o.apply_updates(r[None, :]))
    _same(g, o, w.V)


def test_larger_graph_batches_digests():
    """scale-16 R-MAT, unclamped degree biases, 3 batches of 20K arc records: per-vertex
    digests after each batch, then sampled walks."""
    w = synth.Workload(16, 600_000, compact=True, batch=10_000, rounds=3)
    g, o = _pair(w.row_offsets, w.dst, w.bias)
    for b in w.batches:
        _same_stats(g.apply_updates(b), o.apply_updates(b))
        assert np.array_equal(g.digests().cpu().numpy().view(np.uint64), o.digests())
    starts = (np.arange(50_000, dtype=np.uint64) * 2654435761 % w.V).astype(np.uint32)
    out = g.walk(length=80, seed=3, starts=starts)
    ref = o.walk(length=80, seed=3, starts=starts)
    assert np.array_equal(u32(out["paths"]), ref["paths"])


def test_small_batches_fast_path():
    """a11: batches of 1..256 records take the single-launch path (up to 64 inline, larger ones
    through one H2D copy); the state after each equals
    the oracle's, including when a batch needs pool growth (the fast path hands over to the
    general pipeline without mutating)."""
    rng = np.random.default_rng(17)
    w = synth.make_workload("c1", rounds=3)
    g, o = _pair(w.row_offsets, w.dst, w.bias, arc_slack=0.0, member_slack=0.0, pool_reserve=0.0)
    stream = np.concatenate(w.batches)
    pos = 0
    while pos < len(stream):
        k = int(rng.integers(1, 65)) if rng.random() < 0.6 else int(rng.integers(65, 257))
        b = stream[pos:pos + k]
        pos += k
        if k > 64 and rng.random() < 0.5:   # a device batch (no staging copy)
            import torch
            _same_stats(g.apply_updates(torch.from_numpy(np.ascontiguousarray(b).view(np.int32)).cuda()),
                        o.apply_updates(b))
        else:
            _same_stats(g.apply_updates(b), o.apply_updates(b))
    _same(g, o, w.V, "after the small-batch stream")
    # a hub gaining many arcs in small batches forces relocations (SLOW -> general path)
    for i in range(20):
        b = np.array([(0, 5, (7 * i + j) % w.V, 1 + (i * 64 + j) % 300) for j in range(64)], dtype=np.uint32)
        _same_stats(g.apply_updates(b), o.apply_updates(b))
    _same(g, o, w.V, "after hub growth")


@pytest.mark.parametrize("route", ["bsp", "bsp-sub", "bsp-sync", "bsp-fused", "legacy"])
def test_node2vec_neighbour_index_across_batches(route, monkeypatch):
    """The node2vec distance test (Eq.1, A-17) reads per-vertex neighbour sets that updates
    maintain in place (inserted destinations added, a destination whose last live instance
    is deleted tombstoned, rebuilt on relocation / size change / too many tombstones).
    Multigraph with duplicate arcs and a hub; batches delete every copy of some
    destinations, some copies of others, and re-insert removed ones.  Walks with the index
    must equal the oracle's (which scans the adjacency) after every batch."""
    for k, v in ROUTES[route].items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(77)
    V = 300
    deg = rng.integers(1, 12, size=V)
    deg[0] = 900                               # hub: duplicates of ~300 destinations
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    A = int(ro[-1])
    dst = rng.integers(0, V, size=A).astype(np.uint32)
    bias = rng.integers(1, 300, size=A).astype(np.uint32)
    g, o = _pair(ro, dst, bias, neighbor_index=True)
    live = {u: list(dst[int(ro[u]):int(ro[u + 1])]) for u in range(V)}
    removed = {u: [] for u in range(V)}
    for e in range(1, 25):
        recs = []
        for _ in range(int(rng.integers(5, 40))):
            u = 0 if rng.random() < 0.5 else int(rng.integers(0, V))
            r = rng.random()
            if r < 0.4 and live[u]:            # delete every copy of one destination
                v = int(live[u][int(rng.integers(0, len(live[u])))])
                recs += [(1, u, v, 0)] * live[u].count(v)
                removed[u].append(v)
            elif r < 0.6 and live[u]:          # delete one copy
                recs.append((1, u, int(live[u][int(rng.integers(0, len(live[u])))]), 0))
            elif r < 0.8 and removed[u]:       # re-insert a removed destination
                recs.append((0, u, int(removed[u][int(rng.integers(0, len(removed[u])))]), int(rng.integers(1, 300))))
            else:
                recs.append((0, u, int(rng.integers(0, V)), int(rng.integers(1, 300))))
        recs = np.array(recs, dtype=np.uint32)
        _same_stats(g.apply_updates(recs), o.apply_updates(recs))
        d = oracle.parse_dump(o.dump(), V)
        live = {u: [a[0] for a in d[u]["adj"]] for u in range(V)}
        if e % 4 == 0:
            _same(g, o, V, f"batch {e}")
        for p, q in ((2.0, 0.5), (0.5, 2.0)):
            out = g.walk(app=_pb().NODE2VEC, length=20, p=p, q=q, seed=e)
            ref = o.walk(app=oracle.APP_NODE2VEC, length=20, p=p, q=q, seed=e)
            assert np.array_equal(u32(out["paths"]), ref["paths"]), f"{route} batch {e} p={p} q={q}"


@pytest.mark.parametrize("hix", ["1", "0"])
def test_hub_delete_index_maintained_across_batches(hix, monkeypatch):
    """Hub delete index (hub_index.cuh): large vertices locate their deleted arcs through a
    destination -> position multimap kept exact across batches (deletes, tail moves, inserts),
    dropped on repeated deletes of one pair, on other routes (single-record fast path) and on
    load, and rebuilt (opt-in: BINGO_HUB_INDEX=1).  Dumps must equal the oracle's after every
    batch, index on and off."""
    monkeypatch.setenv("BINGO_HUB_INDEX", hix)
    monkeypatch.setenv("BINGO_INDEX_MIN", "1024")
    rng = np.random.default_rng(2024)
    V = 3000
    deg = rng.integers(0, 6, size=V)
    deg[0], deg[1] = 5000, 2500                 # two hubs (> 1024 arcs: the large-vertex route)
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    A = int(ro[-1])
    dst = rng.integers(0, V, size=A).astype(np.uint32)
    bias = rng.integers(1, 1 << 12, size=A).astype(np.uint32)
    g, o = _pair(ro, dst, bias)
    live = {u: list(dst[int(ro[u]):int(ro[u + 1])]) for u in range(V)}
    for e in range(1, 15):
        recs = []
        for hub in (0, 1):
            if hub == 1 and e % 3 == 0:          # hub 1: insert-only batches now and then
                recs += [(0, 1, int(rng.integers(0, V)), int(rng.integers(1, 4096))) for _ in range(40)]
                continue
            k = int(rng.integers(10, 80))
            for v in rng.choice(np.unique(np.array(live[hub])), size=min(k, len(set(live[hub]))), replace=False):
                recs.append((1, hub, int(v), 0))   # distinct destinations: the index route
            recs += [(0, hub, int(rng.integers(0, V)), int(rng.integers(1, 4096))) for _ in range(k)]
            if e % 5 == 0:                         # a repeated delete of one pair: the scan route
                recs += [(1, hub, int(live[hub][0]), 0)] * 2
        for _ in range(100):
            u = int(rng.integers(2, V))
            recs.append((0, u, int(rng.integers(0, V)), int(rng.integers(1, 4096))))
        recs = np.array(recs, dtype=np.uint32)
        recs = recs[rng.permutation(len(recs))]
        if e % 4 == 2:                             # single-record calls touch hub 0 (fast path drops its index)
            one = np.array([[1, 0, int(live[0][3]), 0], [0, 0, 7, 9]], dtype=np.uint32)
            for r in one:
                _same_stats(g.apply_updates(r[None, :]), o.apply_updates(r[None, :]))
        _same_stats(g.apply_updates(recs), o.apply_updates(recs))
        _same(g, o, V, f"batch {e}")
        d = oracle.parse_dump(o.dump(), V)
        live = {u: [a[0] for a in d[u]["adj"]] for u in range(V)}
    out = g.walk(length=40, seed=11)
    ref = o.walk(length=40, seed=11)
    assert np.array_equal(u32(out["paths"]), ref["paths"])


def test_fast_path_rejects_out_of_range_ids_without_reading_them():
    """a single-launch (<= 256 records) batch with src = V must come back EINVAL
    with nothing touched, also when the graph's memory does not come from the caching
    allocator (an out-of-bounds header read would then fault instead of landing in a
    neighbouring allocation)."""
    pb = _pb()
    w = synth.make_workload("c1")
    for torch_alloc in (False, True):
        g = pb.Graph(w.row_offsets, w.dst, w.bias, torch_alloc=torch_alloc)
        before = g.export()
        for bad in ([[0, w.V, 0, 1]], [[1, w.V, 3, 0]], [[0, 1, 2, 3], [1, w.V + 7, 1, 0]],
                    [[0, 0xFFFFFFFF, 1, 1]]):
            assert g.try_apply_updates(np.array(bad, dtype=np.uint32)) == pb.bingo.E_INVAL
            assert g.export() == before
        o = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
        b = w.batches[0][:100]
        _same_stats(g.apply_updates(b), o.apply_updates(b))
        _same(g, o, w.V)
        g.close()


def test_single_records_on_a_vertex_above_the_fast_path_handoff():
    """Single-record updates touching a vertex with more than 8192 arcs (FAST_HANDOFF_L in
    csrc/update.cu): the single-launch path hands the call to the bulk-synchronous pipeline;
    inserts, deletes (duplicates, the newest and oldest instance) and misses stay exact."""
    rng = np.random.default_rng(12)
    V = 64
    deg = rng.integers(0, 30, size=V)
    deg[5] = 9000
    deg[9] = 8190
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    A = int(ro[-1])
    dst = rng.integers(0, V, size=A).astype(np.uint32)
    bias = rng.integers(1, 5000, size=A).astype(np.uint32)
    g, o = _pair(ro, dst, bias)
    hub = [int(x) for x in dst[int(ro[5]):int(ro[6])]]
    recs = []
    for i in range(60):
        r = rng.random()
        if r < 0.35:
            recs.append((0, 5, int(rng.integers(0, V)), int(rng.integers(1, 1 << 20))))
        elif r < 0.75:
            recs.append((1, 5, hub[int(rng.integers(0, len(hub)))], 0))
        elif r < 0.85:
            recs.append((1, 5, int(rng.integers(0, V)), 0))
        elif r < 0.95:
            recs.append((0, 9, int(rng.integers(0, V)), int(rng.integers(1, 300))))
        else:
            recs.append((1, 9, int(rng.integers(0, V)), 0))
    for r in recs:
        one = np.array([r], dtype=np.uint32)
        _same_stats(g.apply_updates(one), o.apply_updates(one))
    _same(g, o, V)
    out = g.walk(length=30, seed=3, num_walkers=2000)
    ref = o.walk(length=30, seed=3, num_walkers=2000)
    assert np.array_equal(u32(out["paths"]), ref["paths"])


def test_streaming_queue_single_records():
    """f2: records applied one at a time through the persistent device-side queue
    (bingo_stream_update) equal the oracle after every record -- statistics each time, full
    dumps at checkpoints -- with walks, batched updates, stream synchronisation (idle exit),
    invalid records and records that need the batched pipeline interleaved."""
    import time
    import torch
    pb = _pb()
    w = synth.make_workload("c1", rounds=3)
    g, o = _pair(w.row_offsets, w.dst, w.bias)
    recs = np.concatenate([w.batches[0][:300], w.batches[1][:100]])
    for i, r in enumerate(recs):
        sg = g.stream_update(r)
        so = o.apply_updates(r[None, :])
        _same_stats(sg, so)
        if i in (50, 149, 250):
            _same(g, o, w.V, f"after streaming record {i}")
            out = g.walk(length=20, seed=i, num_walkers=500)          # quiesces the queue
            ref = o.walk(length=20, seed=i, num_walkers=500)
            assert np.array_equal(u32(out["paths"]), ref["paths"])
        if i == 100:
            torch.cuda.synchronize()                                  # waits for the idle exit
            time.sleep(0.005)
        if i == 200:
            b = w.batches[2][:400]                                    # a batched update in between
            _same_stats(g.apply_updates(b), o.apply_updates(b))
        if i == 300:
            with pytest.raises(pb.bingo.BingoError):
                g.stream_update(np.array([0, w.V, 1, 1], dtype=np.uint32))
            with pytest.raises(pb.bingo.BingoError):
                g.stream_update(np.array([0, 1, 2, 0], dtype=np.uint32))
    _same(g, o, w.V, "end")
    assert g.info()["epoch"] == o.epoch


def test_streaming_queue_hub_handoff_and_pool_growth():
    """Records the single-warp path cannot take (a vertex above 8192 arcs, pool growth) leave
    the queue for the batched pipeline and come back."""
    rng = np.random.default_rng(21)
    V = 64
    deg = rng.integers(0, 20, size=V)
    deg[7] = 9000
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    dst = rng.integers(0, V, size=int(ro[-1])).astype(np.uint32)
    bias = rng.integers(1, 3000, size=int(ro[-1])).astype(np.uint32)
    pb = _pb()
    g = pb.Graph(ro, dst, bias, arc_slack=0.0, member_slack=0.0, pool_reserve=0.0)
    o = oracle.OracleGraph(ro, dst, bias)
    hub = [int(x) for x in dst[int(ro[7]):int(ro[8])]]
    for i in range(200):
        u = 7 if i % 5 == 0 else int(rng.integers(0, V))
        if rng.random() < 0.6:
            r = np.array([0, u, int(rng.integers(0, V)), int(rng.integers(1, 1 << 16))], dtype=np.uint32)
        else:
            v = hub[int(rng.integers(0, len(hub)))] if u == 7 else int(rng.integers(0, V))
            r = np.array([1, u, v, 0], dtype=np.uint32)
        _same_stats(g.stream_update(r), o.apply_updates(r[None, :]))
    _same(g, o, V)


@pytest.mark.parametrize("hix,gix", [("0", "1"), ("1", "1"), ("1", "0")])
def test_one_sync_route_reruns_only_when_short(hix, gix, monkeypatch):
    """The one-sync route (apply_bsp_async) enqueues the whole batch before the host knows
    the touched-vertex count; a batch that finds a pool or its scratch short mutates nothing
    and is re-applied on the synchronous route.  Bulk batches (> 256 records, so not the
    single-launch fast path) on a graph with hubs: every batch equals the oracle, the first
    batch(es) re-run while scratch is sized, later ones complete in one host round trip."""
    monkeypatch.setenv("BINGO_HUB_INDEX", hix)
    monkeypatch.setenv("BINGO_GROUP_INDEX", gix)
    monkeypatch.setenv("BINGO_INDEX_MIN", "1024")
    rng = np.random.default_rng(99)
    V = 4000
    deg = rng.integers(0, 12, size=V)
    deg[:3] = (6000, 3000, 1500)
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    A = int(ro[-1])
    dst = rng.integers(0, V, size=A).astype(np.uint32)
    bias = rng.integers(1, 1 << 10, size=A).astype(np.uint32)
    g, o = _pair(ro, dst, bias)
    live = {u: list(dst[int(ro[u]):int(ro[u + 1])]) for u in range(V)}
    for e in range(1, 13):
        recs = []
        for _ in range(int(rng.integers(300, 1500))):
            u = int(rng.integers(0, 3)) if rng.random() < 0.4 else int(rng.integers(0, V))
            if live[u] and rng.random() < 0.5:
                recs.append((1, u, int(live[u][int(rng.integers(0, len(live[u])))]), 0))
            else:
                recs.append((0, u, int(rng.integers(0, V)), int(rng.integers(1, 1 << 10))))
        recs = np.array(recs, dtype=np.uint32)
        _same_stats(g.apply_updates(recs), o.apply_updates(recs))
        if e % 3 == 0:
            _same(g, o, V, f"batch {e}")
        d = oracle.parse_dump(o.dump(), V)
        live = {u: [a[0] for a in d[u]["adj"]] for u in range(V)}
        if e == 6:
            mid = g.info()["update_reruns"]
    reruns = g.info()["update_reruns"]
    assert 1 <= mid and reruns - mid <= 2, (mid, reruns)   # scratch settles: later batches take one sync
    out = g.walk(length=40, seed=3)
    ref = o.walk(length=40, seed=3)
    assert np.array_equal(u32(out["paths"]), ref["paths"])


@pytest.mark.parametrize("hub_records", [40, 3000, 9000])
def test_segment_order_short_long_and_radix_fallback(hub_records):
    """Segmentation (a7) without a sort: records are placed per touched vertex in any order,
    then put back in batch order inside each segment -- one thread for <= 32 records, a
    block bitonic sort for <= 8192, and above that the batch is re-segmented by the radix
    sort.  One hub receives hub_records interleaved inserts and deletes (order matters: a
    delete takes the earliest live instance, R-8, and inserts append in batch order,
    P:500); the rest of the batch touches other vertices.  Dumps must equal the oracle's."""
    rng = np.random.default_rng(hub_records)
    V = 600
    deg = rng.integers(1, 8, size=V)
    deg[0] = 2000
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    A = int(ro[-1])
    dst = rng.integers(0, 50, size=A).astype(np.uint32)     # many duplicates of few destinations
    bias = rng.integers(1, 1 << 12, size=A).astype(np.uint32)
    g, o = _pair(ro, dst, bias)
    for e in range(3):
        recs = []
        for j in range(hub_records):
            v = int(rng.integers(0, 50))
            recs.append((1, 0, v, 0) if rng.random() < 0.45 else (0, 0, v, int(rng.integers(1, 1 << 12))))
        for _ in range(400):
            u = int(rng.integers(1, V))
            recs.append((0, u, int(rng.integers(0, V)), int(rng.integers(1, 1 << 12))))
        recs = np.array(recs, dtype=np.uint32)
        recs = recs[rng.permutation(len(recs))]
        _same_stats(g.apply_updates(recs), o.apply_updates(recs))
        _same(g, o, V, f"hub_records {hub_records} batch {e}")


@pytest.mark.parametrize("ndel,gix", [(20, "1"), (300, "1"), (5000, "1"), (300, "0")])
def test_hub_delete_routes_by_pick_count(ndel, gix, monkeypatch):
    """A hub's holes come from its sorted picks (one warp for <= 32, a block sort for
    <= 4096) and its group holes from one pass over each group front plus a sort; a batch
    deleting more than 4096 arcs of one hub takes the counted-rank passes instead.  Each
    route must leave the oracle's structure (R-6 pairing on the adjacency and on every
    member list).  With the group index (default) the group holes and renames of the sorted
    routes come from its lookups, and the index persists across the batches."""
    monkeypatch.setenv("BINGO_GROUP_INDEX", gix)
    monkeypatch.setenv("BINGO_INDEX_MIN", "1024")
    rng = np.random.default_rng(ndel)
    V = 2000
    deg = rng.integers(0, 5, size=V)
    deg[0] = 12000
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    A = int(ro[-1])
    dst = rng.integers(0, V, size=A).astype(np.uint32)
    bias = rng.integers(1, 1 << 14, size=A).astype(np.uint32)
    g, o = _pair(ro, dst, bias)
    for e in range(5):
        d = oracle.parse_dump(o.dump(), V)
        hub = [a[0] for a in d[0]["adj"]]
        pick = rng.choice(len(hub), size=min(ndel, len(hub)), replace=False)
        recs = [(1, 0, int(hub[j]), 0) for j in pick]
        recs += [(0, 0, int(rng.integers(0, V)), int(rng.integers(1, 1 << 14))) for _ in range(300)]
        recs += [(0, int(rng.integers(1, V)), int(rng.integers(0, V)), int(rng.integers(1, 1 << 14)))
                 for _ in range(300)]
        recs = np.array(recs, dtype=np.uint32)[rng.permutation(len(recs))]
        _same_stats(g.apply_updates(recs), o.apply_updates(recs))
        _same(g, o, V, f"ndel {ndel} batch {e}")
