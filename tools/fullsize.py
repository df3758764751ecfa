"""Full-size parity + throughput on a BASELINE config (c2 .. c5).

The CUDA path runs exactly as bench.py runs it (full graph, all walkers of the
config in one launch, update batches through the C-ABI); the CPU oracle (lazy:
builds only the vertices the comparison touches) replays the same batches and
recomputes sampled outputs one by one:
  * per-vertex canonical digests of every touched vertex of the last batch plus a
    random sample of vertices,
  * walks of contiguous walker-id ranges sliced out of the full launch.
Prints one JSON line.  Test infrastructure (imports the oracle)."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2504_10233_b200 as pb  # noqa: E402

APP = {"deepwalk": pb.DEEPWALK, "node2vec": pb.NODE2VEC, "ppr": pb.PPR}
OAPP = {"deepwalk": oracle.APP_DEEPWALK, "node2vec": oracle.APP_NODE2VEC, "ppr": oracle.APP_PPR}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--ranges", type=int, default=6, help="walker-id ranges compared")
    ap.add_argument("--range-len", type=int, default=512)
    ap.add_argument("--vertices", type=int, default=3000, help="random vertices whose digests are compared")
    ap.add_argument("--walkers", type=int, default=0, help="walkers in the launch (default: one per vertex)")
    ap.add_argument("--ppr-cap", type=int, default=400)
    ap.add_argument("--count-walkers", type=int, default=1 << 20,
                    help="PPR: walker-id range whose visit counts are compared on EVERY vertex")
    ap.add_argument("--slack", type=float, default=0.25)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    app = cfg["app"]
    t0 = time.time()
    if a.config == "c5":   # too big for the in-HBM generator's temporaries: generated on the GPU, kept on the host
        w = synth.make_workload(a.config, rounds=a.rounds, device="cuda")
        w.host_csr = lambda: (w.row_offsets, w.dst, w.bias)
    else:
        w = synth.make_workload(a.config, rounds=a.rounds, hold_rounds=10, device="cuda", resident=True)
    torch.cuda.empty_cache()
    t_gen = time.time() - t0
    rec = {"config": a.config, "V": int(w.V), "arcs": int(w.num_arcs), "app": app, "gen_s": round(t_gen, 1)}
    t0 = time.time()
    g = pb.Graph(w.row_offsets, w.dst, w.bias, neighbor_index=(app == "node2vec"), arc_slack=a.slack,
                 member_slack=a.slack)
    torch.cuda.synchronize()
    rec["gpu_build_s"] = round(time.time() - t0, 2)
    o = oracle.OracleGraph(*w.host_csr(), lazy=True)
    # ---- updates, timed on the device, replayed by the oracle
    upd_ms = []
    touched = set()
    for b in w.batches:
        db = torch.from_numpy(b.view(np.int32)).cuda()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sg = g.apply_updates(db)
        e1.record()
        torch.cuda.synchronize()
        upd_ms.append(e0.elapsed_time(e1))
        so = o.apply_updates(b)
        for k in ("inserted", "deleted", "missing_deletes", "touched_vertices"):
            assert sg[k] == so[k], (k, sg[k], so[k])
        assert np.array_equal(sg["kind_transitions"], so["kind_transitions"])
        touched.update(np.unique(b[:, 1]).tolist())
    rec["update_ms"] = [round(x, 3) for x in upd_ms]
    rec["update_arcs_per_s"] = float(len(w.batches[0]) / (np.mean(upd_ms) / 1e3))
    # ---- digests: touched vertices + a random sample
    rng = np.random.default_rng(11)
    tv = np.array(sorted(touched), dtype=np.int64)
    sample = np.unique(np.concatenate([rng.choice(tv, size=min(len(tv), a.vertices), replace=False),
                                       rng.integers(0, w.V, size=a.vertices)]))
    dg = g.digests().cpu().numpy().view(np.uint64)
    bad = [int(u) for u in sample if int(dg[u]) != o.vertex_digest(int(u))]
    assert not bad, f"digest mismatch at vertices {bad[:10]}"
    rec["digests_compared"] = int(len(sample))
    # ---- the full launch, as bench.py runs it
    W = a.walkers or w.V
    L = 80 if app != "ppr" else pb.NO_CAP       # PPR: geometric lengths, visit counts, no paths
    kw = dict(app=APP[app], length=L, seed=4242, num_walkers=W)
    if app == "node2vec":
        kw.update(p=2.0, q=0.5)
    if app == "ppr":
        kw.update(stop=(1, 80), paths=None)
        g.reset_visit_counts()
    else:   # outputs allocated outside the timed region
        kw.update(paths=torch.empty((L + 1, W), dtype=torch.int32, device="cuda"))
    kw.update(lengths=torch.empty(W, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = g.walk(**kw)
    e1.record()
    torch.cuda.synchronize()
    walk_ms = e0.elapsed_time(e1)
    lens = out["lengths"].cpu().numpy().view(np.uint32)
    steps = int(lens.astype(np.int64).sum())
    rec["walk_ms"] = round(walk_ms, 2)
    rec["walk_steps_per_s"] = steps / (walk_ms / 1e3)
    rec["steps"] = steps
    P = out["paths"]
    if app == "ppr":
        counts = g.visit_counts().cpu().numpy().view(np.uint64)
        assert int(counts.astype(np.uint64).sum()) == steps + W, "PPR: sum of visit counts = sum(lengths + 1)"
        rec["ppr_mean_length"] = steps / W
    # ---- sampled walker ranges vs the oracle
    starts = rng.integers(0, max(1, W - a.range_len), size=a.ranges)
    okw = dict(app=OAPP[app], length=L, seed=4242, stop=(1, 80), threads=os.cpu_count())
    if app == "node2vec":
        okw.update(p=2.0, q=0.5)
    t0 = time.time()
    for s0 in starts.tolist():
        ref = o.walk(first_walker=s0, num_walkers=a.range_len, paths=(app != "ppr"), **okw)
        if P is not None:
            gp = P[:, s0:s0 + a.range_len].cpu().numpy().view(np.uint32)
            assert np.array_equal(gp, ref["paths"]), f"walk mismatch in walker range [{s0}, {s0 + a.range_len})"
        assert np.array_equal(lens[s0:s0 + a.range_len], ref["lengths"])
    rec["walkers_compared"] = int(a.ranges * a.range_len)
    rec["oracle_walk_s"] = round(time.time() - t0, 2)
    if app == "ppr":
        # the visit counts of a contiguous walker-id range, compared on every vertex, and
        # capped PPR paths (cap --ppr-cap) on sampled ranges
        g.reset_visit_counts()
        Wc = min(a.count_walkers, W)
        c0 = int(rng.integers(0, max(1, W - Wc)))
        g.walk(app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), seed=5151, first_walker=c0, num_walkers=Wc, paths=None)
        got = g.visit_counts_host(reset=True)
        t0 = time.time()
        ref = o.walk(app=oracle.APP_PPR, length=oracle.NONE, stop=(1, 80), seed=5151, first_walker=c0,
                     num_walkers=Wc, paths=False, counts=True, threads=os.cpu_count())
        rec["oracle_count_walk_s"] = round(time.time() - t0, 2)
        bad = np.nonzero(got != ref["counts"])[0]
        assert bad.size == 0, f"{bad.size} visit-count mismatches, first at {bad[:8].tolist()}"
        rec["count_vector"] = {"walkers": Wc, "first_walker": c0, "vertices_compared": int(w.V),
                               "nonzero": int(np.count_nonzero(ref["counts"])), "sum": int(ref["counts"].sum())}
        for s0 in rng.integers(0, max(1, W - a.range_len), size=a.ranges).tolist():
            outc = g.walk(app=pb.PPR, length=a.ppr_cap, stop=(1, 80), seed=5152, first_walker=s0,
                          num_walkers=a.range_len)
            refc = o.walk(app=oracle.APP_PPR, length=a.ppr_cap, stop=(1, 80), seed=5152, first_walker=s0,
                          num_walkers=a.range_len, threads=os.cpu_count())
            assert np.array_equal(outc["paths"].cpu().numpy().view(np.uint32), refc["paths"]), s0
        g.reset_visit_counts()
        rec["capped_paths_compared"] = int(a.ranges * a.range_len)
    rec["parity"] = "bit-exact"
    print(json.dumps(rec), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
