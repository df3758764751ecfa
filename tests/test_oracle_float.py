"""Pins of the oracle's floating-point-bias extension (S4.3-4.4; reading R-15)."""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests.helpers import chi2_crit, chi2_stat, induced_group_probs


def _star(biases):
    d = len(biases)
    V = d + 1
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = d
    g = oracle.OracleGraph(ro, np.arange(1, d + 1, dtype=np.uint32), np.array(biases, dtype=np.float64),
                           float_bias=True)
    return g, V


def _vertex(g, V):
    return oracle.parse_dump(g.dump(), V, float_mode=True)[0]


def induced_float(v):
    """Exact induced distribution of a float-mode vertex (structure -> probabilities):
    P(decimal) = thrD / 2^64 (or 1 when the integer part is empty), then the integer alias
    (Theorem 1 over I_i) or rejection over the decimal members (prop. to D_i)."""
    d = v["d"]
    out = [Fraction(0)] * d
    if v["fflags"] & 2:
        pdec = Fraction(1)
    else:
        pdec = Fraction(v["thrD"], 1 << 64)
    if v["dec"]:
        tot = sum(D for _, D in v["dec"])
        for i, D in v["dec"]:
            out[i] += pdec * Fraction(D, tot)
    if v["groups"]:
        pg = induced_group_probs(v["groups"], v["T"])
        for b, grp in enumerate(v["groups"]):
            k = grp["k"]
            members = [i for i in range(d) if (v["adj"][i][1] >> k) & 1]
            for i in members:
                out[i] += (1 - pdec) * pg[b] / len(members)
    return out


def test_paper_float_example(golden):
    """P:362-363 / P:377: lambda = 10; groups 2^0 {1,4,5}, 2^1 {4,5}, 2^2 {1,4}; decimal group
    {1,4,5}; W_D/(W_I+W_D) = 1/16 < 1/3 (A-22: 1e-12 tolerance for the IEEE residuals)."""
    ex = golden["float_example"]
    V = 6
    ro = np.array([0, 0, 0, 3, 3, 3, 3], dtype=np.uint64)
    g = oracle.OracleGraph(ro, [e[1] for e in ex["edges"]], [e[2] for e in ex["edges"]], float_bias=True)
    v = oracle.parse_dump(g.dump(), V, float_mode=True)[2]
    assert 10 ** v["lam"] == ex["lambda"] and v["fflags"] == 0
    ids = [a[0] for a in v["adj"]]
    groups = {grp["k"]: sorted(ids[i] for i in range(3) if (v["adj"][i][1] >> grp["k"]) & 1) for grp in v["groups"]}
    assert groups == {0: [1, 4, 5], 1: [4, 5], 2: [1, 4]}
    assert sorted(ids[i] for i, _ in v["dec"]) == [1, 4, 5]
    assert abs(v["thrD"] / 2 ** 64 - ex["ratio"]) < 1e-12
    dist = induced_float(v)
    exp = [5.54 / 16, 7.26 / 16, 3.20 / 16]
    assert max(abs(float(p) - e) / e for p, e in zip(dist, exp)) < 1e-6


def test_spec_lambda_examples():
    """({0.554,0.726,0.320}, d=3) -> 10; ({2.0, 3.0}) -> 1; ({0.01,0.02,0.03}) -> 100."""
    for biases, lam in (([0.554, 0.726, 0.320], 10), ([2.0, 3.0], 1), ([0.01, 0.02, 0.03], 100)):
        g, V = _star(biases)
        assert 10 ** _vertex(g, V)["lam"] == lam


@pytest.mark.parametrize("seed", range(4))
def test_float_induced_distribution_within_1e6(seed):
    """BASELINE north_star: deviation in sampled probability <= 1e-6 relative to w/sum w, and the
    lambda constraint: decimal probability < 1/d unless flagged."""
    rng = np.random.default_rng(seed)
    for _ in range(30):
        d = int(rng.integers(1, 60))
        kind = rng.integers(0, 3)
        if kind == 0:
            w = rng.random(d) * 10
        elif kind == 1:
            w = np.exp(rng.uniform(np.log(1e-6), np.log(1e6), size=d))
        else:
            w = rng.integers(1, 1000, size=d) / 7.0
        w = np.maximum(w, 1e-9)
        g, V = _star(w.tolist())
        v = _vertex(g, V)
        dist = induced_float(v)
        tot = sum(Fraction(float(x)) for x in w)
        for i in range(d):
            ref = Fraction(float(w[i])) / tot
            assert abs(dist[i] - ref) / ref <= Fraction(1, 10 ** 6), (i, float(dist[i]), float(ref))
        if not (v["fflags"] & 1) and not (v["fflags"] & 2):
            assert Fraction(v["thrD"], 1 << 64) < Fraction(1, d) + Fraction(1, 1 << 60)


def test_float_sampling_chi_square():
    w = [0.554, 0.726, 0.320, 3.3e-3, 12.5, 0.75]
    g, V = _star(w)
    n = 600_000
    out = g.walk(length=1, seed=77, starts=np.zeros(n, dtype=np.uint32))
    counts = np.bincount(out["paths"][1], minlength=V)[1:]
    p = np.array(w) / sum(w)
    assert (p * n >= 5).all()
    assert chi2_stat(list(counts), list(p), n) < chi2_crit(len(p) - 1)


def test_float_updates_need_real_biases():
    """Float-mode graphs take inserted biases as doubles (R-16); an integer-only batch is refused."""
    g, V = _star([0.5, 1.5])
    assert g.try_apply_updates([[0, 0, 1, 3]]) == 1
    assert g.try_apply_updates([[0, 0, 1, 3]], bias_f64=[0.25]) == 0
    assert g.try_apply_updates([[0, 0, 1, 0]], bias_f64=[-1.0]) == 1          # w <= 0: EINVAL
    assert g.try_apply_updates([[0, 0, 1, 0]], bias_f64=[float("nan")]) == 1
    lam = 10 ** _vertex(g, V)["lam"]
    before = g.dump()
    assert g.try_apply_updates([[0, 0, 2, 0], [0, 0, 1, 0]], bias_f64=[1.0, 2.0 ** 33 / lam]) == 4   # I >= 2^32
    assert g.dump() == before                                                      # whole batch refused


def _real_dist(ws):
    tot = sum(Fraction(float(x)) for x in ws)
    return [Fraction(float(x)) / tot for x in ws]


@pytest.mark.parametrize("seed", range(3))
def test_float_updates_keep_distribution_within_1e6(seed):
    """R-16: with each vertex's lambda fixed at build, inserts split the real bias into
    I = floor(fl(w lambda)) (radix groups, Eq.3-9) and D (decimal group); after every batch the
    structure's exact induced distribution is within 1e-6 relative of w / sum w over the live arcs
    (BASELINE north_star), the integer part satisfies every invariant (Eq.4, Eq.9, exact alias),
    lambda never changes and flag bit 0 is exactly the P:377 constraint check."""
    from tests.helpers import check_vertex_invariants
    rng = np.random.default_rng(100 + seed)
    V = 12
    live = {u: {} for u in range(V)}                     # u -> {dst: real bias}; unique dst per vertex
    ro = np.zeros(V + 1, dtype=np.uint64)
    dst, wf = [], []
    for u in range(V):
        d = int(rng.integers(0, 9)) if u else 0         # vertex 0 starts isolated (lambda = 1)
        ds = rng.choice(np.arange(V, 4 * V), size=d, replace=False) % (4 * V)
        for v in ds:
            w = float(rng.uniform(0.05, 20.0))
            live[u][int(v) % V + 0] = live[u].get(int(v) % V, 0) or w
        ro[u + 1] = ro[u] + len(live[u])
        for v, w in live[u].items():
            dst.append(v)
            wf.append(w)
    g = oracle.OracleGraph(ro, np.array(dst, dtype=np.uint32), np.array(wf), float_bias=True)
    lam0 = [v["lam"] for v in oracle.parse_dump(g.dump(), V, float_mode=True)]
    for e in range(1, 15):
        recs, ws = [], []
        for _ in range(int(rng.integers(1, 12))):
            u = int(rng.integers(0, V))
            if live[u] and rng.random() < 0.45:
                v = int(rng.choice(list(live[u])))
                recs.append((1, u, v, 0))
                ws.append(0.0)
                del live[u][v]
            else:
                free = [v for v in range(V) if v not in live[u]]
                if not free:
                    continue
                v = int(rng.choice(free))
                w = float(rng.uniform(0.05, 20.0)) if rng.random() < 0.8 else float(rng.uniform(0.001, 0.05))
                recs.append((0, u, v, 0))
                ws.append(w)
                live[u][v] = w
        st = g.apply_updates(np.array(recs, dtype=np.uint32).reshape(-1, 4), bias_f64=np.array(ws))
        assert st["epoch"] == e
        dump = oracle.parse_dump(g.dump(), V, float_mode=True)
        for u in range(V):
            v = dump[u]
            assert v["lam"] == lam0[u]
            assert sorted(a[0] for a in v["adj"]) == sorted(live[u])
            if not v["d"]:
                continue
            if v["T"]:                                   # integer part nonempty (else flag bit 1)
                check_vertex_invariants(v)
            dist = induced_float(v)
            ref = _real_dist([live[u][a[0]] for a in v["adj"]])
            for i in range(v["d"]):
                assert abs(dist[i] - ref[i]) / ref[i] <= Fraction(1, 10 ** 6), (u, i, float(dist[i]), float(ref[i]))
            WI = sum(a[1] for a in v["adj"])
            WD = sum(D for _, D in v["dec"])
            assert bool(v["fflags"] & 1) == (not ((v["d"] - 1) * WD < (WI << 52)))
            assert bool(v["fflags"] & 2) == (WI == 0)
            assert [i for i, _ in v["dec"]] == sorted(i for i, _ in v["dec"])
