"""-m gpu: the floating-point-bias extension (a12, S4.3-4.4; R-15) on the device vs the oracle:
bit-exact structures (incl. the decimal trailer of the dump), digests and walks."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _pair(ro, dst, wf, **kw):
    import paper_2504_10233_b200 as pb
    g = pb.Graph(ro, dst, wf, float_bias=True, **kw)
    o = oracle.OracleGraph(ro, dst, wf, float_bias=True)
    return g, o


def _same(g, o, V):
    a, b = g.export(), o.dump()
    if a != b:
        pa, pb_ = oracle.parse_dump(a, V, True), oracle.parse_dump(b, V, True)
        for u in range(V):
            assert pa[u] == pb_[u], f"vertex {u}:\n gpu    {pa[u]}\n oracle {pb_[u]}"
    assert a == b
    assert np.array_equal(g.digests().cpu().numpy().view(np.uint64), o.digests())


def _float_biases(rng, n, kind):
    if kind == "uniform":
        return rng.random(n) * 10 + 1e-3
    if kind == "logspread":
        return np.exp(rng.uniform(np.log(1e-5), np.log(1e5), size=n))
    return rng.integers(1, 400, size=n) / 7.0


@pytest.mark.parametrize("kind", ["uniform", "logspread", "sevenths"])
def test_float_build_and_walk_parity(kind):
    import paper_2504_10233_b200 as pb
    rng = np.random.default_rng(5)
    w = synth.make_workload("c1")
    wf = _float_biases(rng, len(w.dst), kind)
    g, o = _pair(w.row_offsets, w.dst, wf)
    _same(g, o, w.V)
    out = g.walk(length=40, seed=3)
    ref = o.walk(length=40, seed=3)
    assert np.array_equal(out["paths"].cpu().numpy().view(np.uint32), ref["paths"])
    starts = np.arange(5000, dtype=np.uint32) % w.V
    g.walk(app=pb.PPR, length=pb.NO_CAP, seed=4, starts=starts, paths=None)
    refp = o.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=4, starts=starts, paths=False, counts=True)
    assert np.array_equal(g.visit_counts().cpu().numpy().view(np.uint64), refp["counts"])


def test_float_paper_example_and_edge_cases():
    # paper example, an all-decimal vertex, an integral vertex, an isolated vertex
    ro = np.array([0, 3, 5, 7, 7], dtype=np.uint64)
    dst = np.array([1, 2, 3, 0, 2, 0, 1], dtype=np.uint32)
    wf = np.array([0.554, 0.726, 0.320, 1e-7, 3e-7, 2.0, 3.0])
    g, o = _pair(ro, dst, wf)
    _same(g, o, 4)
    for L in (1, 7):
        out = g.walk(length=L, seed=9, starts=np.zeros(20000, dtype=np.uint32) + np.arange(20000, dtype=np.uint32) % 4)
        ref = o.walk(length=L, seed=9, starts=np.zeros(20000, dtype=np.uint32) + np.arange(20000, dtype=np.uint32) % 4)
        assert np.array_equal(out["paths"].cpu().numpy().view(np.uint32), ref["paths"])


ROUTES = {"bsp": {}, "bsp-sub": {"BINGO_BSP_MAXT": "5"}, "legacy": {"BINGO_UPD_LEGACY": "1"}}


@pytest.mark.parametrize("route", ["bsp", "bsp-sub", "legacy"])
@pytest.mark.parametrize("kind", ["uniform", "logspread"])
def test_float_updates_parity(route, kind, monkeypatch):
    """R-16 on the device vs the oracle: batches of float-bias inserts (incl. integer part 0,
    duplicates, hub growth forcing arc and decimal-member relocations) and deletes; bit-exact
    dumps with the decimal trailer and digests after every batch, walks and PPR counts after."""
    import paper_2504_10233_b200 as pb
    for k, v in ROUTES[route].items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(31)
    w = synth.make_workload("c1")
    wf = _float_biases(rng, len(w.dst), kind)
    g = pb.Graph(w.row_offsets, w.dst, wf, float_bias=True, arc_slack=0.0, member_slack=0.0, pool_reserve=0.0)
    o = oracle.OracleGraph(w.row_offsets, w.dst, wf, float_bias=True)
    V = w.V
    assert g.try_apply_updates(np.array([[0, 1, 2, 5]], dtype=np.uint32)) == pb.bingo.E_INVAL   # needs bias_f64
    d0 = oracle.parse_dump(o.dump(), V, True)
    live = {u: [a[0] for a in d0[u]["adj"]] for u in range(V)}
    for e in range(1, 9):
        n = int(rng.integers(50, 400))
        recs = np.zeros((n, 4), dtype=np.uint32)
        ws = np.zeros(n)
        for i in range(n):
            u = 3 if rng.random() < 0.2 else int(rng.integers(0, V))
            if live[u] and rng.random() < 0.4:
                recs[i] = (1, u, int(live[u][int(rng.integers(0, len(live[u])))]), 0)
            else:
                recs[i] = (0, u, int(rng.integers(0, V)), 0)
                r = rng.random()
                ws[i] = (_float_biases(rng, 1, kind)[0] if r < 0.7 else
                         float(rng.uniform(1e-4, 0.05)) if r < 0.9 else float(rng.integers(1, 50)))
        sg = g.apply_updates(recs, bias_f64=ws)
        so = o.apply_updates(recs, bias_f64=ws)
        for k in ("inserted", "deleted", "missing_deletes", "touched_vertices", "epoch"):
            assert sg[k] == so[k], (k, sg[k], so[k])
        _same(g, o, V)
        d = oracle.parse_dump(o.dump(), V, True)
        live = {u: [a[0] for a in d[u]["adj"]] for u in range(V)}
        if e % 3 == 0:
            out = g.walk(length=30, seed=e)
            ref = o.walk(length=30, seed=e)
            assert np.array_equal(out["paths"].cpu().numpy().view(np.uint32), ref["paths"])
    # a batch whose scaled bias reaches 2^32 is refused whole, nothing mutated
    before = g.export()
    lam = 10 ** d[7]["lam"]
    bad = np.array([[0, 5, 1, 0], [0, 7, 2, 0]], dtype=np.uint32)
    assert g.try_apply_updates(bad, bias_f64=np.array([1.0, 2.0 ** 33 / lam])) == pb.bingo.E_OVERFLOW
    assert g.try_apply_updates(bad, bias_f64=np.array([1.0, -2.0])) == pb.bingo.E_INVAL
    assert g.export() == before
    starts = np.arange(4000, dtype=np.uint32) % V
    g.walk(app=pb.PPR, length=pb.NO_CAP, seed=4, starts=starts, paths=None)
    refp = o.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=4, starts=starts, paths=False, counts=True)
    assert np.array_equal(g.visit_counts().cpu().numpy().view(np.uint64), refp["counts"])


def test_float_updates_device_batch():
    """The device-pointer path of bingo_apply_updates_f64 equals the host path."""
    import torch
    import paper_2504_10233_b200 as pb
    rng = np.random.default_rng(8)
    ro, dst, _ = synth.random_small_graph(rng, 40, 20, 100)
    wf = rng.random(len(dst)) * 5 + 1e-3
    g1 = pb.Graph(ro, dst, wf, float_bias=True)
    g2 = pb.Graph(ro, dst, wf, float_bias=True)
    o = oracle.OracleGraph(ro, dst, wf, float_bias=True)
    recs = synth.random_batch(rng, 40, 300, 100, existing=None)
    ws = rng.random(300) * 3 + 1e-3
    g1.apply_updates(recs, bias_f64=ws)
    g2.apply_updates(torch.from_numpy(recs.view(np.int32)).cuda(), bias_f64=torch.from_numpy(ws).cuda())
    o.apply_updates(recs, bias_f64=ws)
    assert g1.export() == g2.export() == o.dump()
