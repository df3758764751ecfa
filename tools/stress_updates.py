"""Randomised update stress (test infrastructure): many seeds of random multigraph batches
through every update route, canonical dumps compared with the oracle after every batch."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2504_10233_b200 as pb  # noqa: E402

ROUTES = [{}, {"BINGO_UPD_LEGACY": "1"}, {"BINGO_HUB_INDEX": "1"}, {"BINGO_BSP_MAXT": "5"}]


def run(seed, route):
    for k in ("BINGO_UPD_LEGACY", "BINGO_HUB_INDEX", "BINGO_BSP_MAXT"):
        os.environ.pop(k, None)
    os.environ.update(route)
    rng = np.random.default_rng(seed)
    V = int(rng.integers(5, 400))
    deg = rng.integers(0, 40, size=V)
    deg[0] = int(rng.integers(500, 6000))
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    dst = rng.integers(0, V, size=int(ro[-1])).astype(np.uint32)
    hi = int(rng.choice([7, 255, 1 << 12, 1 << 20]))
    bias = rng.integers(1, hi + 1, size=len(dst)).astype(np.uint32)
    bs = bool(rng.random() < 0.2)
    g = pb.Graph(ro, dst, bias, bs_mode=bs, arc_slack=float(rng.choice([0.0, 0.25])), member_slack=0.0,
                 pool_reserve=0.0, neighbor_index=bool(rng.random() < 0.3))
    o = oracle.OracleGraph(ro, dst, bias, flags=oracle.FLAG_BS_MODE if bs else 0)
    live = {u: list(dst[int(ro[u]):int(ro[u + 1])]) for u in range(V)}
    for e in range(8):
        n = int(rng.integers(1, 600))
        recs = np.zeros((n, 4), dtype=np.uint32)
        for i in range(n):
            u = 0 if rng.random() < 0.3 else int(rng.integers(0, V))
            if rng.random() < 0.5 and live[u]:
                recs[i] = (1, u, int(live[u][int(rng.integers(0, len(live[u])))]), 0)
            else:
                recs[i] = (0, u, int(rng.integers(0, V)), int(rng.integers(1, hi + 1)))
        g.apply_updates(recs)
        o.apply_updates(recs)
        if g.export() != o.dump():
            return f"seed {seed} route {route} batch {e}: dump mismatch"
        d = oracle.parse_dump(o.dump(), V)
        live = {u: [a[0] for a in d[u]["adj"]] for u in range(V)}
    out = g.walk(length=20, seed=seed)
    ref = o.walk(length=20, seed=seed)
    if not np.array_equal(out["paths"].cpu().numpy().view(np.uint32), ref["paths"]):
        return f"seed {seed} route {route}: walk mismatch"
    return None


def run_float(seed, route):
    for k in ("BINGO_UPD_LEGACY", "BINGO_HUB_INDEX", "BINGO_BSP_MAXT"):
        os.environ.pop(k, None)
    os.environ.update(route)
    rng = np.random.default_rng(seed)
    V = int(rng.integers(5, 300))
    deg = rng.integers(0, 30, size=V)
    deg[0] = int(rng.integers(300, 3000))
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    dst = rng.integers(0, V, size=int(ro[-1])).astype(np.uint32)
    scale = float(rng.choice([1e-3, 1.0, 1e3]))
    wf = rng.random(len(dst)) * scale + 1e-6
    g = pb.Graph(ro, dst, wf, float_bias=True, arc_slack=float(rng.choice([0.0, 0.25])), member_slack=0.0,
                 pool_reserve=0.0)
    o = oracle.OracleGraph(ro, dst, wf, float_bias=True)
    live = {u: list(dst[int(ro[u]):int(ro[u + 1])]) for u in range(V)}
    for e in range(6):
        n = int(rng.integers(1, 400))
        recs = np.zeros((n, 4), dtype=np.uint32)
        ws = np.zeros(n)
        for i in range(n):
            u = 0 if rng.random() < 0.3 else int(rng.integers(0, V))
            if rng.random() < 0.5 and live[u]:
                recs[i] = (1, u, int(live[u][int(rng.integers(0, len(live[u])))]), 0)
            else:
                recs[i] = (0, u, int(rng.integers(0, V)), 0)
                ws[i] = rng.random() * scale + 1e-6
        rg, ro_ = g.try_apply_updates(recs, bias_f64=ws), o.try_apply_updates(recs, bias_f64=ws)
        if rg != ro_:
            return f"float seed {seed} route {route} batch {e}: status {rg} vs {ro_}"
        if g.export() != o.dump():
            return f"float seed {seed} route {route} batch {e}: dump mismatch"
        d = oracle.parse_dump(o.dump(), V, True)
        live = {u: [a[0] for a in d[u]["adj"]] for u in range(V)}
    out = g.walk(length=20, seed=seed)
    ref = o.walk(length=20, seed=seed)
    if not np.array_equal(out["paths"].cpu().numpy().view(np.uint32), ref["paths"]):
        return f"float seed {seed} route {route}: walk mismatch"
    return None


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    fl = "--float" in sys.argv
    bad = 0
    for s in range(n):
        for r in ROUTES:
            err = (run_float if fl else run)(10_000 + s, r)
            if err:
                bad += 1
                print(err, flush=True)
    print(f"{'float ' if fl else ''}{n} seeds x {len(ROUTES)} routes: {bad} failures", flush=True)
