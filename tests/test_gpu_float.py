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


def test_float_updates_refused():
    import paper_2504_10233_b200 as pb
    ro = np.array([0, 1, 1], dtype=np.uint64)
    g, _ = _pair(ro, np.array([1], dtype=np.uint32), np.array([0.5]))
    assert g.try_apply_updates(np.array([[0, 0, 1, 3]], dtype=np.uint32)) == pb.bingo.E_INVAL
