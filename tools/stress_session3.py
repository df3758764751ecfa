"""Randomised stress of session 3's update paths against the oracle (test infrastructure):
  * radix-base graphs (R-19): random b, random multigraphs with hubs, random batches;
  * replicated-regime sharded updates (f1): P replicas apply their owned records and exchange
    vertex states; every replica's dump must equal the oracle after every batch.
usage: python tools/stress_session3.py [--seeds 30]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2504_10233_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seeds", type=int, default=30)
a = ap.parse_args()


def graph(rng):
    V = int(rng.integers(2, 700))
    ro, dst, bias = synth.random_small_graph(rng, V, int(rng.integers(1, 60)),
                                             int(rng.choice([3, 255, 1 << 20, (1 << 32) - 1])))
    deg = np.diff(ro.astype(np.int64))
    for h in rng.integers(0, V, size=int(rng.integers(0, 3))):
        deg[h] = int(rng.integers(1000, 7000))
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    dst = rng.integers(0, V, size=int(ro[-1])).astype(np.uint32)
    bias = rng.integers(1, int(rng.choice([3, 255, 1 << 20])) + 1, size=int(ro[-1])).astype(np.uint32)
    return V, ro, dst, bias


res = {"radix": 0, "exchange": 0}
for seed in range(a.seeds):
    rng = np.random.default_rng(1000 + seed)
    V, ro, dst, bias = graph(rng)
    b = int(rng.integers(1, 6))
    g = pb.Graph(ro, dst, bias, radix_log2=b, arc_slack=float(rng.choice([0.0, 0.25])))
    o = oracle.RadixGraph(ro, dst, bias, b)
    existing = [(u, int(dst[x])) for u in range(V) for x in range(int(ro[u]), int(ro[u + 1]))]
    for r in range(5):
        recs = synth.random_batch(rng, V, int(rng.integers(1, 3000)), 1 << 16, existing=existing,
                                  p_delete=float(rng.uniform(0.2, 0.8)))
        sg, so = g.apply_updates(recs), o.apply_updates(recs)
        assert all(sg[k] == so[k] for k in ("inserted", "deleted", "missing_deletes", "touched_vertices")), seed
        assert g.export() == o.dump(), ("radix", seed, b, r)
        existing = [(u, int(e[0])) for u in range(V) for e in o.adjacency(u)]
    res["radix"] += 1
    # sharded updates with P replicas
    V, ro, dst, bias = graph(rng)
    P = int(rng.integers(2, 5))
    os.environ["BINGO_LAYOUT"] = str(rng.choice(["id", "hot", "relabel"]))
    if rng.random() < 0.5:
        os.environ["BINGO_INDEX_MIN"] = "1024"
    else:
        os.environ.pop("BINGO_INDEX_MIN", None)
    reps = [pb.Graph(ro, dst, bias, arc_slack=0.0, member_slack=0.0, pool_reserve=0.0) for _ in range(P)]
    o = oracle.OracleGraph(ro, dst, bias)
    existing = [(u, int(dst[x])) for u in range(V) for x in range(int(ro[u]), int(ro[u + 1]))]
    for r in range(5):
        recs = synth.random_batch(rng, V, int(rng.integers(1, 3000)), 1 << 16, existing=existing,
                                  p_delete=float(rng.uniform(0.2, 0.8)))
        o.apply_updates(recs)
        ex = []
        for k, gk in enumerate(reps):
            mine = np.ascontiguousarray(recs[recs[:, 1] % P == k])
            gk.apply_updates(mine)
            ex.append(gk.export_vertices(torch.unique(torch.from_numpy(mine[:, 1].astype(np.int64))).cuda()))
        for k, gk in enumerate(reps):
            for j, (buf, off) in enumerate(ex):
                if j != k:
                    gk.import_vertices(buf, off)
        want = o.dump()
        for k, gk in enumerate(reps):
            assert gk.export() == want, ("exchange", seed, P, r, k)
        existing = [(u, e[0]) for u, v in enumerate(oracle.parse_dump(want, V)) for e in v["adj"]]
    res["exchange"] += 1
    os.environ.pop("BINGO_LAYOUT", None)
    os.environ.pop("BINGO_INDEX_MIN", None)
print(json.dumps({"seeds_passed": res}), flush=True)
