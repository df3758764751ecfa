"""Test-side analytic helpers (exact rationals).  These compute what a sampling
structure *induces* -- they never sample -- so they pin the oracle (and the CUDA
path's dumps) against the paper's definitions rather than against themselves."""
from __future__ import annotations

from collections import Counter
from fractions import Fraction

EMPTY, ONE, DENSE, SPARSE, REGULAR = 0, 1, 2, 3, 4


def induced_group_probs(groups, T):
    """Alias table -> P(group b) = sum over buckets of (1/n)(thr/T or (T-thr)/T)."""
    n = len(groups)
    p = [Fraction(0)] * n
    for b, g in enumerate(groups):
        p[b] += Fraction(g["thr"], n * T)
        p[g["alias"]] += Fraction(T - g["thr"], n * T)
    return p


def exact_distribution(v):
    """Theorem 1 evaluated on a dumped vertex: P(i) = sum_k P(p_k) P(i|p_k),
    P(p_k) from the alias table, P(i|p_k) from the group's Eq.9 layout.  Returns
    a list of Fractions indexed by adjacency position."""
    d = v["d"]
    if d == 0:
        return []
    pg = induced_group_probs(v["groups"], v["T"])
    out = [Fraction(0)] * d
    for b, g in enumerate(v["groups"]):
        k = g["k"]
        if g["kind"] == ONE:
            out[g["one"]] += pg[b]
        elif g["kind"] in (REGULAR, SPARSE):
            for i in g["mem"]:
                out[i] += pg[b] / len(g["mem"])
        elif g["kind"] == DENSE:
            members = [i for i in range(d) if (v["adj"][i][1] >> k) & 1]
            for i in members:
                out[i] += pg[b] / len(members)
        else:
            raise AssertionError("EMPTY group in the list")
    return out


def check_vertex_invariants(v, alpha=40, beta=10, bs_mode=False):
    """BASELINE.json invariants + SPEC S:85-95/S:206-207 on a dumped vertex."""
    d = v["d"]
    adj = v["adj"]
    T = sum(a[1] for a in adj)
    assert v["T"] == T, "group weights must sum to the vertex weight (Eq.4, Theorem 1)"
    ks = [g["k"] for g in v["groups"]]
    assert ks == sorted(ks) and len(set(ks)) == len(ks)
    mask = 0
    for a in adj:
        mask |= a[1]
    assert set(ks) == {k for k in range(32) if (mask >> k) & 1}, "nonempty groups = set bits"
    n = len(v["groups"])
    for g in v["groups"]:
        k = g["k"]
        members = [i for i in range(d) if (adj[i][1] >> k) & 1]
        assert g["c"] == len(members), "c_k = #{i : w_i AND 2^k != 0} (Eq.3/4)"
        c = g["c"]
        if bs_mode:
            exp = REGULAR
        elif c == 1:
            exp = ONE
        elif 100 * c > alpha * d:
            exp = DENSE
        elif 100 * c < beta * d:
            exp = SPARSE
        else:
            exp = REGULAR
        assert g["kind"] == exp, (g, d)
        if g["kind"] in (REGULAR, SPARSE):
            assert sorted(g["mem"]) == members, "each arc appears exactly once in each of its groups"
        elif g["kind"] == ONE:
            assert [g["one"]] == members
        assert 0 <= g["thr"] <= T and 0 <= g["alias"] < n
    # alias exactness: thr[j] + sum_{b != j, alias[b] = j} (T - thr[b]) = n W_j
    acc = [0] * n
    for b, g in enumerate(v["groups"]):
        acc[b] += g["thr"]
        if g["alias"] != b:
            acc[g["alias"]] += T - g["thr"]
    for b, g in enumerate(v["groups"]):
        assert acc[b] == n * (g["c"] << g["k"]), "alias table must be exact"
    # Theorem 1
    if d:
        dist = exact_distribution(v)
        for i in range(d):
            assert dist[i] == Fraction(adj[i][1], T), "Theorem 1: P(v_i) = w_i / sum w"


def live_multiset(v):
    return Counter((a[0], a[1]) for a in v["adj"])


def chi2_stat(observed, expected_probs, n):
    s = 0.0
    for o, p in zip(observed, expected_probs):
        e = float(p) * n
        s += (o - e) ** 2 / e
    return s


# upper 0.1% quantiles of chi-square, dof 1..40 (from scipy.stats.chi2.ppf(0.999, dof))
def chi2_crit(dof, q=0.999):
    from scipy.stats import chi2
    return float(chi2.ppf(q, dof))
