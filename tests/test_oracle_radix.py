"""Pins of the oracle's arbitrary-radix-base structure (reading R-17)
against what the paper and mathematics fix (-m "not gpu"): the running example worked by
hand in base 4, Theorem 1 generalised to base B checked in exact rationals on random
multigraphs for every b, the b = 1 case reducing to the paper's all-regular baseline (BS
mode) table for table, chi-square of sampled steps against w / sum w, and PPR /
DeepWalk length laws."""
from __future__ import annotations

from collections import Counter
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import chi2_crit, chi2_stat


def radix_distribution(v):
    """Exact induced next-vertex distribution of a dumped radix vertex: sum over groups of
    P(group) * P(subgroup | group) * (multiplicity of v in the subgroup) / c."""
    T = v["T"]
    n = len(v["groups"])
    pg = [Fraction(0)] * n
    for b, g in enumerate(v["groups"]):
        pg[b] += Fraction(g["thr"], n * T)
        pg[g["alias"]] += Fraction(T - g["thr"], n * T)
    out = Counter()
    for b, g in enumerate(v["groups"]):
        subs = g["subs"]
        S = sum(s["j"] * s["c"] for s in subs)
        m = len(subs)
        ps = [Fraction(0)] * m
        for k, s in enumerate(subs):
            ps[k] += Fraction(s["thr"], m * S)
            ps[s["alias"]] += Fraction(S - s["thr"], m * S)
        for k, s in enumerate(subs):
            for dv in s["mem"]:
                out[dv] += pg[b] * ps[k] / s["c"]
    return out


def test_base4_running_example(golden):
    ex = golden["radix4_running_example"]
    ro = np.array([0, 0, 0, 3, 3, 3, 3], dtype=np.uint64)
    e = golden["running_example"]["edges"]
    g = oracle.RadixGraph(ro, [x[1] for x in e], [x[2] for x in e], ex["b"])
    v = oracle.parse_radix_dump(g.dump(), 6)[ex["vertex"]]
    assert v["groups"] == ex["groups"] and v["T"] == ex["T"]
    assert radix_distribution(v) == {1: Fraction(5, 12), 4: Fraction(4, 12), 5: Fraction(3, 12)}


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5])
def test_theorem1_any_base(b):
    """P(v) = sum_{arcs u->v} w / T exactly, for every vertex, every base; groups in
    ascending i, subgroups ascending j, members in ascending adjacency order."""
    rng = np.random.default_rng(40 + b)
    for trial in range(4):
        V = int(rng.integers(2, 60))
        ro, dst, bias = synth.random_small_graph(rng, V, int(rng.integers(1, 70)),
                                                 int(rng.choice([3, 255, 1 << 16, (1 << 32) - 1])))
        g = oracle.RadixGraph(ro, dst, bias, b)
        for u, v in enumerate(oracle.parse_radix_dump(g.dump(), V)):
            lo, hi = int(ro[u]), int(ro[u + 1])
            assert v["d"] == hi - lo and v["T"] == int(bias[lo:hi].astype(np.int64).sum())
            exp = Counter()
            for a in range(lo, hi):
                exp[int(dst[a])] += Fraction(int(bias[a]), v["T"])
            if v["d"]:
                assert radix_distribution(v) == exp
            ii = [gr["i"] for gr in v["groups"]]
            assert ii == sorted(ii) and all(i < -(-32 // b) for i in ii)
            for gr in v["groups"]:
                jj = [s["j"] for s in gr["subs"]]
                assert jj == sorted(jj) and all(1 <= j < (1 << b) for j in jj)
                for s in gr["subs"]:
                    idx = [a - lo for a in range(lo, hi) if ((int(bias[a]) >> (gr["i"] * b)) & ((1 << b) - 1)) == s["j"]]
                    assert s["mem"] == [int(dst[lo + k]) for k in idx]


def test_base2_reduces_to_the_all_regular_baseline():
    """b = 1: every group has the single subgroup j = 1, and the group tables are exactly the
    BS-mode (all-regular) Bingo tables: W_k = c_k 2^k, the same integer Vose."""
    rng = np.random.default_rng(9)
    ro, dst, bias = synth.random_small_graph(rng, 40, 50, 1 << 20)
    r = oracle.parse_radix_dump(oracle.RadixGraph(ro, dst, bias, 1).dump(), 40)
    bs = oracle.parse_dump(oracle.OracleGraph(ro, dst, bias, flags=oracle.FLAG_BS_MODE).dump(), 40)
    for u in range(40):
        assert [g["i"] for g in r[u]["groups"]] == [g["k"] for g in bs[u]["groups"]]
        assert [(g["thr"], g["alias"]) for g in r[u]["groups"]] == [(g["thr"], g["alias"]) for g in bs[u]["groups"]]
        for gr, gb in zip(r[u]["groups"], bs[u]["groups"]):
            assert len(gr["subs"]) == 1 and gr["subs"][0]["j"] == 1
            assert gr["subs"][0]["mem"] == [bs[u]["adj"][k][0] for k in gb["mem"]]


@pytest.mark.parametrize("b", [2, 4])
def test_radix_single_step_chi_square(b):
    rng = np.random.default_rng(3)
    V = 8
    deg = [1, 5, 40, 3, 17, 9, 2, 60]
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    dst = rng.integers(0, V, size=int(ro[-1])).astype(np.uint32)
    bias = rng.integers(1, 5000, size=int(ro[-1])).astype(np.uint32)
    g = oracle.RadixGraph(ro, dst, bias, b)
    for u in (2, 4, 7):
        lo, hi = int(ro[u]), int(ro[u + 1])
        T = int(bias[lo:hi].astype(np.int64).sum())
        p = Counter()
        for a in range(lo, hi):
            p[int(dst[a])] += bias[a] / T
        N = 120_000
        obs = Counter(g.sample(u, 77, w, 5) for w in range(N))
        keys = sorted(p)
        assert set(obs) <= set(keys)
        assert chi2_stat([obs[k] for k in keys], [p[k] for k in keys], N) < chi2_crit(len(keys) - 1)


def test_radix_walk_laws():
    w = synth.make_workload("c1")
    g = oracle.RadixGraph(w.row_offsets, w.dst, w.bias, 2)
    r = g.walk(length=80, seed=1)
    pa = r["paths"]
    ro = w.row_offsets.astype(np.int64)
    deg = np.diff(ro)
    L = r["lengths"].astype(np.int64)
    last = pa[L, np.arange(w.V)]
    assert np.all((L == 80) | (deg[last] == 0)), "a walk stops early only at a dead end (R-13)"
    for i in range(0, w.V, 97):          # every transition is a live arc
        for t in range(80):
            if pa[t + 1, i] == oracle.NONE:
                break
            u = int(pa[t, i])
            assert int(pa[t + 1, i]) in set(w.dst[ro[u]:ro[u + 1]].tolist())
    wc = synth.Workload(12, 30_000, compact=True, batch=100, rounds=1)     # min out-degree >= 1
    gc = oracle.RadixGraph(wc.row_offsets, wc.dst, wc.bias, 3)
    rp = gc.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=2, num_walkers=200_000, paths=False, counts=True)
    assert abs(rp["lengths"].mean() - 80) < 0.5
    assert int(rp["counts"].sum()) == int(rp["lengths"].astype(np.int64).sum()) + 200_000


# ---------------------------------------------------------------- radix updates (reading R-19)
def _csr_of(adj_lists):
    """CSR (row offsets, dst, bias) of per-vertex [(dst, bias, epoch)] lists."""
    deg = [len(a) for a in adj_lists]
    ro = np.zeros(len(adj_lists) + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    dst = np.array([e[0] for a in adj_lists for e in a], dtype=np.uint32)
    bias = np.array([e[1] for a in adj_lists for e in a], dtype=np.uint32)
    return ro, dst, bias


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5])
def test_radix_updates_follow_the_base2_adjacency_readings(b):
    """R-19: the adjacency of an updated radix graph is, arc for arc and epoch for epoch, the
    adjacency the base-2 oracle's independently written update path (R-6..R-9, pinned by the
    paper's insertion / deletion examples) produces for the same batches; statistics agree;
    and the nested structure equals a fresh build of that adjacency (whose tables are pinned
    by Theorem 1 above)."""
    rng = np.random.default_rng(100 + b)
    V = 30
    ro, dst, bias = synth.random_small_graph(rng, V, 40, 1 << 12)
    base = oracle.OracleGraph(ro, dst, bias)
    rad = oracle.RadixGraph(ro, dst, bias, b)
    existing = [(u, int(dst[a])) for u in range(V) for a in range(int(ro[u]), int(ro[u + 1]))]
    for r in range(6):
        # hubs: some vertices get many records (duplicates, deletes of arcs inserted earlier
        # in the same batch, missing deletes, delete-all-then-regrow on vertex 0)
        recs = synth.random_batch(rng, V, 120, 1 << 12, existing=existing, p_delete=0.45)
        if r == 3:
            dels = [(synth.DELETE, 0, e[0], 0) for e in rad.adjacency(0)]
            recs = np.concatenate([recs, np.array(dels, dtype=np.uint32).reshape(-1, 4),
                                   np.array([(synth.INSERT, 0, 5, 7), (synth.INSERT, 0, 5, 9)], dtype=np.uint32)])
        sb = base.apply_updates(recs)
        sr = rad.apply_updates(recs)
        for k in ("inserted", "deleted", "missing_deletes", "touched_vertices", "epoch"):
            assert sr[k] == sb[k], (k, sr[k], sb[k])
        pb = oracle.parse_dump(base.dump(), V)
        adj = []
        for u in range(V):
            a = [tuple(int(x) for x in e) for e in rad.adjacency(u)]
            assert a == [tuple(e) for e in pb[u]["adj"]], (r, u)
            adj.append(a)
        existing = [(u, e[0]) for u in range(V) for e in adj[u]]
        fresh = oracle.RadixGraph(*_csr_of(adj), b)
        assert rad.dump() == fresh.dump(), r
        rv = oracle.parse_radix_dump(rad.dump(), V)
        for u in range(V):
            if not adj[u]:
                continue
            T = sum(e[1] for e in adj[u])
            want = Counter()
            for e in adj[u]:
                want[e[0]] += Fraction(e[1], T)
            assert radix_distribution(rv[u]) == want, (r, u)


def test_radix_update_validation_and_overflow_leave_the_graph_untouched():
    rng = np.random.default_rng(7)
    ro, dst, bias = synth.random_small_graph(rng, 12, 10, 100)
    rad = oracle.RadixGraph(ro, dst, bias, 3)
    before = rad.dump()
    bad = [np.array([[0, 3, 4, 0]], dtype=np.uint32),            # insert with bias 0
           np.array([[2, 3, 4, 5]], dtype=np.uint32),            # unknown op
           np.array([[0, 3, 12, 5]], dtype=np.uint32),           # dst >= V
           np.array([[1, 2, 4, 0], [0, 12, 4, 5]], dtype=np.uint32)]   # src >= V after a valid record
    for recs in bad:
        assert rad.try_apply_updates(recs) == 1
        assert rad.dump() == before
    st = rad.apply_updates(np.zeros((0, 4), dtype=np.uint32))      # an empty batch is a successful call
    assert st["epoch"] == 1 and rad.dump() == before
    st = rad.apply_updates(np.array([[0, 1, 2, 3]], dtype=np.uint32))
    assert st["epoch"] == 2 and rad.adjacency(1)[-1].tolist() == [2, 3, 2]
