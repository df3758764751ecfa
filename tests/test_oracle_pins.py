"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it pins.  Nothing here compares the oracle with
itself: expected values are paper-printed (tests/golden/paper_examples.json),
closed forms (Theorem 1, alias exactness), brute force on tiny inputs, or
statistical tests against the Eq.2 / Eq.1 definitions.
"""
from __future__ import annotations

from collections import Counter
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import (check_vertex_invariants, chi2_crit, chi2_stat, exact_distribution,
                           live_multiset)

KIND = {"ONE": oracle.ONE, "DENSE": oracle.DENSE, "SPARSE": oracle.SPARSE, "REGULAR": oracle.REGULAR}


def running_example_graph(golden, flags=0):
    ex = golden["running_example"]
    V = 6
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[3:] = 3
    dst = [e[1] for e in ex["edges"]]
    bias = [e[2] for e in ex["edges"]]
    return oracle.OracleGraph(ro, dst, bias, flags=flags), V


# ---------------------------------------------------------------- RNG (R-1)
def test_philox_known_answers(golden):
    for ctr, key, out in golden["philox_kat"]["cases"]:
        got = oracle.philox([int(x, 16) for x in ctr], [int(x, 16) for x in key])
        assert [f"{int(x):08x}" for x in got] == out


# ---------------------------------------------------------------- Eq.3/4, Fig. SAMPLING
def test_running_example_groups(golden):
    """groups 2^0={1,5}, 2^1={5}, 2^2={1,4}, sums 2, 2, 8."""
    ex = golden["running_example"]
    g, V = running_example_graph(golden, flags=oracle.FLAG_BS_MODE)
    v = oracle.parse_dump(g.dump(), V)[2]
    adj_dst = [a[0] for a in v["adj"]]
    for grp in v["groups"]:
        ids = sorted(adj_dst[i] for i in grp["mem"])
        assert ids == sorted(ex["groups_by_dst"][str(grp["k"])])
    assert [grp["c"] << grp["k"] for grp in v["groups"]] == ex["group_sums"]
    assert v["T"] == sum(ex["group_sums"])
    check_vertex_invariants(v, bs_mode=True)


def test_running_example_adaptive_kinds(golden):
    """Eq.9 with alpha=40, beta=10 on d=3: c=2 -> 67% > 40% dense; c=1 -> one-element."""
    g, V = running_example_graph(golden)
    v = oracle.parse_dump(g.dump(), V)[2]
    assert [grp["kind"] for grp in v["groups"]] == [oracle.DENSE, oracle.ONE, oracle.DENSE]
    check_vertex_invariants(v)
    assert exact_distribution(v) == [Fraction(5, 12), Fraction(4, 12), Fraction(3, 12)]


def test_classify_examples(golden):
    c = golden["classify"]
    for cnt, d, kind in c["cases"]:
        assert oracle.classify(cnt, d, c["alpha"], c["beta"]) == KIND[kind]


def test_classify_boundaries():
    """Eq.9 uses strict > alpha% and < beta%: exactly 40% / 10% is regular (R-3)."""
    assert oracle.classify(4, 10) == oracle.REGULAR          # 40% is not > 40%
    assert oracle.classify(5, 10) == oracle.DENSE
    assert oracle.classify(10, 100) == oracle.REGULAR        # 10% is not < 10%
    assert oracle.classify(9, 100) == oracle.SPARSE
    assert oracle.classify(0, 10) == oracle.EMPTY
    assert oracle.classify(1, 1) == oracle.ONE               # one-element before dense (R-3)
    assert oracle.classify(1, 5, flags=oracle.FLAG_BS_MODE) == oracle.REGULAR


# ---------------------------------------------------------------- alias
def test_alias_running_example():
    thr, al = oracle.alias_build([2, 2, 8])
    n, T = 3, 12
    p = [Fraction(0)] * 3
    for b in range(3):
        p[b] += Fraction(int(thr[b]), n * T)
        p[al[b]] += Fraction(T - int(thr[b]), n * T)
    assert p == [Fraction(1, 6), Fraction(1, 6), Fraction(2, 3)]     # S:39, Eq.5


@pytest.mark.parametrize("seed", range(5))
def test_alias_exact_identity(seed):
    """Closed form: the alias method's induced distribution is exactly W_j / T
    ("volume of each bucket ... equal"): thr[j] + sum_{alias[b]=j, b!=j} (T - thr[b]) = n W_j."""
    rng = np.random.default_rng(seed)
    for _ in range(400):
        n = int(rng.integers(1, 33))
        W = rng.integers(0, 1 << int(rng.integers(1, 41)), size=n, dtype=np.uint64)
        W[rng.integers(0, n)] |= np.uint64(1)
        thr, al = oracle.alias_build(W)
        T = int(W.sum())
        acc = [0] * n
        for b in range(n):
            assert 0 <= int(thr[b]) <= T and al[b] < n
            acc[b] += int(thr[b])
            if al[b] != b:
                acc[al[b]] += T - int(thr[b])
        assert acc == [n * int(w) for w in W]
        # each bucket holds at most two candidates (P:191 (i))
        assert all(int(thr[b]) == T or al[b] != b for b in range(n))


# ---------------------------------------------------------------- S4.2 insertion / deletion
def test_insertion_example(golden):
    """inserting (2,3,3) appends index 3 to groups 2^0 and 2^1; sums become 3, 4, 8."""
    g, V = running_example_graph(golden, flags=oracle.FLAG_BS_MODE)
    e = golden["insertion"]["edge"]
    g.apply_updates([[0, e[0], e[1], e[2]]])
    v = oracle.parse_dump(g.dump(), V)[2]
    by_k = {grp["k"]: grp for grp in v["groups"]}
    for k in golden["insertion"]["bits"]:
        assert by_k[k]["mem"][-1] == 3           # appended at the end
    assert [grp["c"] << grp["k"] for grp in v["groups"]] == [3, 4, 8]
    assert exact_distribution(v) == [Fraction(5, 15), Fraction(4, 15), Fraction(3, 15), Fraction(3, 15)]
    check_vertex_invariants(v, bs_mode=True)


def test_deletion_example(golden):
    """deleting (2,1,5) (index 0) from groups 2^0 and 2^2; in group 2^0 index 0
    swaps with the tail index 3 -- then the adjacency swap renames 3 -> 0."""
    g, V = running_example_graph(golden, flags=oracle.FLAG_BS_MODE)
    g.apply_updates([[0, 2, 3, 3]])
    before = oracle.parse_dump(g.dump(), V)[2]
    g0 = [grp for grp in before["groups"] if grp["k"] == 0][0]["mem"]
    assert g0 == [0, 2, 3]
    dl = golden["deletion"]
    g.apply_updates([[1, dl["edge"][0], dl["edge"][1], 0]])
    v = oracle.parse_dump(g.dump(), V)[2]
    by_k = {grp["k"]: grp for grp in v["groups"]}
    # slot 0 of group 2^0 now holds the former tail entry (index 3, renamed to 0 because
    # arc 3 moved into adjacency hole 0)
    assert by_k[0]["mem"][0] == 0 and v["adj"][0][:2] == (3, 3)
    assert [a[:2] for a in v["adj"]] == [(3, 3), (4, 4), (5, 3)]
    assert exact_distribution(v) == [Fraction(3, 10), Fraction(4, 10), Fraction(3, 10)]
    check_vertex_invariants(v, bs_mode=True)


def test_two_phase_paper_example(golden):
    tp = golden["two_phase"]
    assert oracle.two_phase(list(range(tp["length"])), tp["delete"]) == tp["expect"]


def test_two_phase_single_is_swap_with_tail():
    """N = 1 reduces to the streaming swap-with-tail of P:333-336."""
    for L in range(1, 12):
        for j in range(L):
            arr = list(range(L))
            exp = arr[:]
            exp[j] = exp[L - 1]
            exp.pop()
            assert oracle.two_phase(arr, [j]) == exp


def test_two_phase_brute_force():
    """Brute force over every deletion set of small arrays: result is compact, the multiset
    is the original minus the deleted entries, untouched front entries stay in place, and
    no deleted entry survives (the hazard P:514 warns about)."""
    import itertools
    for L in range(0, 9):
        for N in range(0, L + 1):
            for S in itertools.combinations(range(L), N):
                out = oracle.two_phase(list(range(L)), list(S))
                assert len(out) == L - N
                assert sorted(out) == sorted(set(range(L)) - set(S))
                for i in range(L - N):
                    if i not in S:
                        assert out[i] == i


def test_dense_rejection_rule(golden):
    """a neighbour of bias 4 is rejected for group 2^0 -- the dense sampler's
    accepted arcs are exactly those with the group's bit set."""
    dr = golden["dense_rejection"]
    assert bool((dr["bias"] >> dr["k"]) & 1) == dr["accept"]
    # a vertex whose 2^0 group is dense: every sample drawn through it has an odd bias
    V = 8
    ro = np.array([0, 8, 8, 8, 8, 8, 8, 8, 8], dtype=np.uint64)
    bias = np.array([1, 3, 5, 4, 7, 9, 2, 11], dtype=np.uint32)      # 6/8 odd -> dense
    g = oracle.OracleGraph(ro, np.arange(8, dtype=np.uint32), bias)
    v = oracle.parse_dump(g.dump(), V)[0]
    assert [grp for grp in v["groups"] if grp["k"] == 0][0]["kind"] == oracle.DENSE
    check_vertex_invariants(v)


# ---------------------------------------------------------------- batches (S5.2)
def _bias_of(u, v, e):
    return 1 + ((u * 2654435761 + v * 40503 + e * 97) % 200)


def _random_graph(rng, V, max_deg):
    deg = rng.integers(0, max_deg + 1, size=V)
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    dst = rng.integers(0, V, size=int(ro[-1])).astype(np.uint32)
    src = np.repeat(np.arange(V), deg)
    bias = np.array([_bias_of(int(s), int(d), 0) for s, d in zip(src, dst)], dtype=np.uint32)
    return ro, dst, bias


def _replay(model, recs, e):
    """Reference semantics of P:497 on multisets: per vertex all inserts (batch order),
    then each delete removes the earliest-epoch live instance of (u, v)."""
    missing = 0
    by_src = {}
    for r in recs:
        by_src.setdefault(int(r[1]), []).append(r)
    for u, lst in by_src.items():
        for r in lst:
            if r[0] == 0:
                model[u].append((int(r[2]), int(r[3]), e))
        for r in lst:
            if r[0] == 1:
                cands = [x for x in model[u] if x[0] == int(r[2])]
                if not cands:
                    missing += 1
                    continue
                model[u].remove(min(cands, key=lambda x: x[2]))
    return missing


@pytest.mark.parametrize("seed,bs_mode", [(s, b) for s in range(6) for b in (False, True)])
def test_batches_vs_replay_and_invariants(seed, bs_mode):
    """Incremental vs definition: after each random batch the live multiset
    equals the P:497 replay, and every vertex satisfies Eq.3/4/9, alias exactness and
    Theorem 1 exactly; epochs and stats match the batch."""
    rng = np.random.default_rng(100 + seed)
    V = int(rng.integers(3, 24))
    ro, dst, bias = _random_graph(rng, V, 40)
    flags = oracle.FLAG_BS_MODE if bs_mode else 0
    g = oracle.OracleGraph(ro, dst, bias, flags=flags)
    model = {u: [(int(dst[i]), int(bias[i]), 0) for i in range(int(ro[u]), int(ro[u + 1]))] for u in range(V)}
    for e in range(1, 9):
        n = int(rng.integers(0, 60))
        recs = np.zeros((n, 4), dtype=np.uint32)
        for i in range(n):
            u = int(rng.integers(0, V))
            if rng.random() < 0.5:
                if model[u] and rng.random() < 0.85:
                    v_ = model[u][int(rng.integers(0, len(model[u])))][0]
                else:
                    v_ = int(rng.integers(0, V))
                recs[i] = (1, u, v_, 0)
            else:
                v_ = int(rng.integers(0, V))
                recs[i] = (0, u, v_, _bias_of(u, v_, e))
        st = g.apply_updates(recs)
        missing = _replay(model, recs, e)
        assert st["epoch"] == e and g.epoch == e
        assert st["inserted"] == int((recs[:, 0] == 0).sum())
        assert st["missing_deletes"] == missing
        assert st["deleted"] == int((recs[:, 0] == 1).sum()) - missing
        assert st["touched_vertices"] == len(set(recs[:, 1].tolist()))
        dump = oracle.parse_dump(g.dump(), V)
        for u in range(V):
            assert live_multiset(dump[u]) == Counter((x[0], x[1]) for x in model[u]), (seed, e, u)
            assert sorted(a[2] for a in dump[u]["adj"]) == sorted(x[2] for x in model[u])
            check_vertex_invariants(dump[u], bs_mode=bs_mode)


def test_invalid_batch_rejected_without_mutation():
    rng = np.random.default_rng(5)
    ro, dst, bias = _random_graph(rng, 10, 10)
    g = oracle.OracleGraph(ro, dst, bias)
    before = g.dump()
    for bad in ([[0, 0, 10, 1]], [[0, 10, 0, 1]], [[0, 1, 2, 0]], [[2, 1, 2, 3]],
                [[0, 1, 2, 3], [1, 99, 0, 0]]):
        assert g.try_apply_updates(bad) == 1          # BINGO_E_INVAL
        assert g.dump() == before and g.epoch == 0


def test_duplicate_edges_delete_earliest_first():
    """duplicated insertions carry a time stamp; deletion removes the earlier version."""
    V = 4
    ro = np.array([0, 1, 1, 1, 1], dtype=np.uint64)
    g = oracle.OracleGraph(ro, [1], [5])                      # (0,1,5) at epoch 0
    g.apply_updates([[0, 0, 1, 6]])                           # duplicate (0,1,6) at epoch 1
    g.apply_updates([[1, 0, 1, 0]])                           # deletes the epoch-0 instance
    v = oracle.parse_dump(g.dump(), V)[0]
    assert v["adj"] == [(1, 6, 1)]
    # same-batch insert + delete of a fresh pair: insert-then-delete per vertex
    g.apply_updates([[1, 0, 2, 0], [0, 0, 2, 3]])
    v = oracle.parse_dump(g.dump(), V)[0]
    assert v["adj"] == [(1, 6, 1)]


def test_batch_vs_stream_on_paper_stream():
    """applying a S6.1-style batch at once or record by record gives the same live
    multiset and the same exact distributions (layouts may differ, distributions may not)."""
    w = synth.make_workload("c1", rounds=2)
    a = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    b = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    for recs in w.batches:
        a.apply_updates(recs)
        for r in recs:
            b.apply_updates(r[None, :])
    da, db = oracle.parse_dump(a.dump(), w.V), oracle.parse_dump(b.dump(), w.V)
    for u in range(w.V):
        assert live_multiset(da[u]) == live_multiset(db[u])
        T = da[u]["T"]
        assert T == db[u]["T"]
        pa = Counter()
        pb = Counter()
        for x, p in zip(da[u]["adj"], exact_distribution(da[u])):
            pa[x[:2]] += p
        for x, p in zip(db[u]["adj"], exact_distribution(db[u])):
            pb[x[:2]] += p
        assert pa == pb


# ---------------------------------------------------------------- sampling statistics
def _star_graph(biases):
    d = len(biases)
    V = d + 1
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = d
    return oracle.OracleGraph(ro, np.arange(1, d + 1, dtype=np.uint32), np.array(biases, dtype=np.uint32)), V


@pytest.mark.parametrize("biases", [
    [5, 4, 3],                                                     # running example
    [1, 3, 5, 4, 7, 9, 2, 11, 200, 1 << 20],                       # dense + one + regular
    list(range(1, 61)) + [1 << 30],                                # sparse groups at high bits
])
def test_single_step_chi_square(biases):
    """Eq.2: 10^6 single steps from one vertex match w_i / sum w under a chi-square
    test at the 99.9% quantile and TV < 0.005."""
    g, V = _star_graph(biases)
    n = 1_000_000
    out = g.walk(length=1, seed=12345, starts=np.zeros(n, dtype=np.uint32))
    nxt = out["paths"][1]
    counts = np.bincount(nxt, minlength=V)[1:]
    p = np.array(biases, dtype=np.float64) / sum(biases)
    tv = 0.5 * np.abs(counts / n - p).sum()
    assert tv < 0.005
    big = p * n >= 5
    obs = list(counts[big]) + [counts[~big].sum()] if (~big).any() else list(counts[big])
    exp = list(p[big]) + [p[~big].sum()] if (~big).any() else list(p[big])
    assert chi2_stat(obs, exp, n) < chi2_crit(len(obs) - 1)


def test_dense_rejection_efficiency():
    """S5.1 / S:209: a dense group's acceptance is > alpha% so < 2.5 expected attempts."""
    biases = [1, 3, 5, 4, 7, 9, 2, 11, 6, 13, 15, 17]
    g, V = _star_graph(biases)
    v = oracle.parse_dump(g.dump(), V)[0]
    dense = [grp for grp in v["groups"] if grp["kind"] == oracle.DENSE]
    assert dense
    n = 200_000
    out = g.walk(length=1, seed=7, starts=np.zeros(n, dtype=np.uint32))
    pg = {grp["k"]: p for grp, p in zip(v["groups"], __import__("tests.helpers", fromlist=["x"]).induced_group_probs(v["groups"], v["T"]))}
    p_dense = float(sum(pg[grp["k"]] for grp in dense))
    # expected attempts per dense pick = d / c
    exp_att = float(sum(pg[grp["k"]] * Fraction(v["d"], grp["c"]) for grp in dense)) / p_dense
    got = out["dense_attempts"] / (p_dense * n)
    assert got < 2.5 and abs(got - exp_att) < 0.05


# ---------------------------------------------------------------- applications (S6.1)
def test_deepwalk_lengths_and_edges():
    """P:536 + S:385: length 80 -> 81 vertices on a graph with min out-degree >= 1; every
    transition is a live arc; length 0 -> [start]."""
    w = synth.make_workload("c1")
    ro, dst = w.row_offsets, w.dst
    g = oracle.OracleGraph(ro, dst, w.bias)
    out = g.walk(length=80, seed=3)
    P, Ln = out["paths"], out["lengths"]
    deg = np.diff(ro.astype(np.int64))
    arcs = set(zip(np.repeat(np.arange(w.V), deg).tolist(), dst.tolist()))
    for i in range(w.V):
        if deg[i] == 0:
            assert Ln[i] == 0 and (P[1:, i] == oracle.NONE).all()
            continue
        assert Ln[i] == 80          # symmetric graph: no dead ends after the first step
        for t in range(80):
            assert (int(P[t, i]), int(P[t + 1, i])) in arcs
    out0 = g.walk(length=0, seed=3)
    assert (out0["paths"][0] == np.arange(w.V)).all() and (out0["lengths"] == 0).all()


def test_deepwalk_determinism_and_sharding():
    """Counter-based keying (R-1): identical seed -> identical walks; a walker's path depends
    only on its global id, so shards with first_walker_id reproduce the unsharded run."""
    w = synth.make_workload("c1")
    g = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    full = g.walk(length=20, seed=9)["paths"]
    assert (g.walk(length=20, seed=9, threads=1)["paths"] == full).all()
    h = w.V // 2
    a = g.walk(length=20, seed=9, first_walker=0, num_walkers=h)["paths"]
    b = g.walk(length=20, seed=9, first_walker=h, num_walkers=w.V - h)["paths"]
    assert (np.concatenate([a, b], axis=1) == full).all()
    assert not (g.walk(length=20, seed=10)["paths"] == full).all()


def _n2v_brute(adj, w, prev, cur, p, q):
    """Eq.1 x Eq.2 normalised, by enumeration."""
    f = []
    for v, wt in zip(adj[cur], w[cur]):
        if v == prev:
            fa = 1.0 / p
        elif v in adj[prev]:
            fa = 1.0
        else:
            fa = 1.0 / q
        f.append(fa * wt)
    s = sum(f)
    out = {}
    for v, x in zip(adj[cur], f):
        out[v] = out.get(v, 0.0) + x / s
    return out


@pytest.mark.parametrize("p,q", [(0.5, 2.0), (2.0, 0.5), (1.0, 1.0)])
def test_node2vec_paper_cases(p, q):
    """S:403-404/S:512-513 + Eq.1: path 0-1-2 and triangle, prev=0, cur=1, unit biases."""
    for edges, V in ((((0, 1), (1, 2)), 3), (((0, 1), (1, 2), (0, 2)), 3)):
        adj = {u: [] for u in range(V)}
        for a, b in edges:
            adj[a].append(b)
            adj[b].append(a)
        ro = np.zeros(V + 1, dtype=np.uint64)
        ro[1:] = np.cumsum([len(adj[u]) for u in range(V)])
        dst = np.array([v for u in range(V) for v in sorted(adj[u])], dtype=np.uint32)
        for u in adj:
            adj[u] = sorted(adj[u])
        g = oracle.OracleGraph(ro, dst, np.ones(len(dst), dtype=np.uint32))
        n = 400_000
        out = g.walk(app=oracle.APP_NODE2VEC, length=2, p=p, q=q, seed=11, starts=np.zeros(n, dtype=np.uint32))
        P = out["paths"]
        sel = P[1] == 1
        exp = _n2v_brute(adj, {u: [1] * len(adj[u]) for u in adj}, 0, 1, p, q)
        m = int(sel.sum())
        obs = [int((P[2][sel] == v).sum()) for v in sorted(exp)]
        assert chi2_stat(obs, [exp[v] for v in sorted(exp)], m) < chi2_crit(len(obs) - 1)
    if (p, q) == (2.0, 0.5):
        assert abs(exp[0] - 1 / 3) < 1e-12 and abs(exp[2] - 2 / 3) < 1e-12


@pytest.mark.parametrize("seed", range(4))
def test_node2vec_random_graphs(seed):
    """S criterion 9: random small graphs, second-order step distribution vs brute force."""
    rng = np.random.default_rng(seed)
    V = 7
    pairs = set()
    while len(pairs) < 12:
        a, b = sorted(rng.integers(0, V, size=2).tolist())
        if a != b:
            pairs.add((a, b))
    adj = {u: [] for u in range(V)}
    wt = {}
    for a, b in sorted(pairs):
        adj[a].append(b)
        adj[b].append(a)
    for u in range(V):
        adj[u] = sorted(adj[u])
    wt = {u: [1 + (u * 7 + v * 3) % 9 for v in adj[u]] for u in range(V)}
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum([len(adj[u]) for u in range(V)])
    g = oracle.OracleGraph(ro, np.array([v for u in range(V) for v in adj[u]], dtype=np.uint32),
                           np.array([x for u in range(V) for x in wt[u]], dtype=np.uint32))
    prev = [u for u in range(V) if adj[u]][0]
    cur = adj[prev][0]
    n = 300_000
    for p, q in ((0.5, 2.0), (2.0, 0.5)):
        out = g.walk(app=oracle.APP_NODE2VEC, length=2, p=p, q=q, seed=seed, starts=np.full(n, prev, dtype=np.uint32))
        P = out["paths"]
        sel = P[1] == cur
        m = int(sel.sum())
        exp = _n2v_brute(adj, wt, prev, cur, p, q)
        obs = np.array([(P[2][sel] == v).sum() for v in sorted(exp)], dtype=np.float64)
        tv = 0.5 * np.abs(obs / m - np.array([exp[v] for v in sorted(exp)])).sum()
        assert tv < 0.01


def test_ppr_lengths_and_counts():
    """P:536 + S:408-413: stop = 1 -> exactly one step; stop 1/80 -> mean 80 +- 0.5 over
    10^6 walks; visit counts include the start, so sum(counts) = sum(lengths + 1)."""
    w = synth.make_workload("c1")
    g = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    deg = np.diff(w.row_offsets.astype(np.int64))
    live = np.nonzero(deg > 0)[0].astype(np.uint32)
    one = g.walk(app=oracle.APP_PPR, length=oracle.NONE, stop=(1, 1), starts=live, counts=True, seed=1)
    assert (one["lengths"] == 1).all()
    n = 1_000_000
    starts = live[np.arange(n) % len(live)]
    out = g.walk(app=oracle.APP_PPR, length=oracle.NONE, stop=(1, 80), starts=starts, counts=True, seed=2)
    assert abs(out["lengths"].mean() - 80.0) < 0.5
    assert int(out["counts"].sum()) == int(out["lengths"].astype(np.int64).sum()) + n
    assert oracle.stop_threshold(1, 80)[0] == 230584300921369395       # floor(2^64 / 80)


def test_lazy_oracle_equals_eager():
    """The lazy oracle (used for BASELINE-scale parity) is the eager oracle, vertex for vertex."""
    w = synth.make_workload("c1", rounds=3)
    a = oracle.OracleGraph(w.row_offsets, w.dst, w.bias)
    b = oracle.OracleGraph(w.row_offsets, w.dst, w.bias, lazy=True)
    for bt in w.batches:
        assert a.apply_updates(bt)["deleted"] == b.apply_updates(bt)["deleted"]
    assert np.array_equal(a.walk(length=30, seed=3)["paths"], b.walk(length=30, seed=3)["paths"])
    assert a.dump() == b.dump()
    d = a.digests()
    for u in range(0, w.V, 37):
        assert b.vertex_digest(u) == int(d[u])


def test_alias_exact_tables_worked_by_hand(golden):
    """R-4's canonical order pinned on exact tables (worked by hand from
    the rule): a lowest->highest index slip made on both sides would change thr/alias here
    although every distribution identity still holds."""
    cases = {c["stage"]: c for c in golden["alias_worked"]["cases"]}
    for c in cases.values():
        thr, al = oracle.alias_build(c["W"])
        assert [int(x) for x in thr] == c["thr"] and [int(x) for x in al] == c["alias"], c["stage"]

    def tables(g, V):
        v = oracle.parse_dump(g.dump(), V)[2]
        return v, [grp["thr"] for grp in v["groups"]], [grp["alias"] for grp in v["groups"]]

    g, V = running_example_graph(golden, flags=oracle.FLAG_BS_MODE)
    v, thr, al = tables(g, V)
    assert v["T"] == cases["running_example"]["T"]
    assert thr == cases["running_example"]["thr"] and al == cases["running_example"]["alias"]
    e = golden["insertion"]["edge"]
    g.apply_updates([[0, e[0], e[1], e[2]]])
    v, thr, al = tables(g, V)
    assert v["T"] == cases["after_insertion"]["T"]
    assert thr == cases["after_insertion"]["thr"] and al == cases["after_insertion"]["alias"]
    dl = golden["deletion"]["edge"]
    g.apply_updates([[1, dl[0], dl[1], 0]])
    v, thr, al = tables(g, V)
    c = cases["after_deletion"]
    assert v["T"] == c["T"] and thr == c["thr"] and al == c["alias"]
    assert {str(grp["k"]): grp["mem"] for grp in v["groups"]} == c["groups_by_index"]
    # the same state built adaptively (alpha = 40, beta = 10)
    ga, _ = running_example_graph(golden)
    ga.apply_updates([[0, e[0], e[1], e[2]]])
    ga.apply_updates([[1, dl[0], dl[1], 0]])
    va = oracle.parse_dump(ga.dump(), V)[2]
    assert [oracle.KIND_NAMES[grp["kind"]] for grp in va["groups"]] == c["kinds_adaptive"]
    assert [grp["thr"] for grp in va["groups"]] == c["thr"] and [grp["alias"] for grp in va["groups"]] == c["alias"]


def test_node2vec_outer_attempts_never_repeat_counters():
    """R-1 (draw_oi): node2vec outer attempts >= 65536 carry their high bits into the tag
    word, so attempt 65536 + x does not replay attempt x (the old 16-bit field cycled and a
    walker that kept rejecting would loop forever).  Attempts < 65536 are unchanged: their
    draw is the plain counter (w, t, (outer << 16) + inner, tag)."""
    rng = np.random.default_rng(5)
    ro, dst, bias = synth.random_small_graph(rng, 8, 40, 1000)
    o = oracle.OracleGraph(ro, dst, bias)
    u = int(np.argmax(np.diff(ro.astype(np.int64))))
    same = sum(o.sample(u, 99, w, 3, x) == o.sample(u, 99, w, 3, x + 65536) for w in range(200) for x in (0, 7))
    assert same < 200, "attempt 65536 + x must not replay attempt x"
    # attempt < 65536: the bucket draw is Philox(w, t, outer << 16, 0) -- the first step of Eq.5
    r = oracle.philox([3, 1, 5 << 16, 0], [99, 0])
    v = oracle.parse_dump(o.dump(), 8)[u]
    b = (int(r[0]) * len(v["groups"])) >> 32
    coin = (((int(r[1]) << 32) | int(r[2])) * v["T"]) >> 64
    g = v["groups"][b] if coin < v["groups"][b]["thr"] else v["groups"][v["groups"][b]["alias"]]
    s = o.sample(u, 99, 3, 1, 5)
    assert any(v["adj"][i][0] == s and (v["adj"][i][1] >> g["k"]) & 1 for i in range(v["d"])), \
        "the sampled arc must belong to the group the (outer << 16) counter selects"


def test_node2vec_unacceptable_ratio_rejected():
    with pytest.raises(ValueError):
        oracle.n2v_thresholds(1e-30, 1.0)
