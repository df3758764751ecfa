"""BASELINE configs[4]: streaming single-edge insert/delete latency sweep on the
Friendster-shaped graph, interleaved with DeepWalk batches of 1M walkers (the
ABI is one-writer-or-many-readers, so "mixed" = update batch, then walk batch on
the same stream; P:523 (ii)).  Batch sizes 1, 16, 256, 4K, 64K, 1M arc records
(undirected edge events expand to 2 records); per size the device latency of
each bingo_apply_updates call (p50/p99) and the walk throughput.  Parity: the lazy
oracle replays every batch; touched-vertex digests and walker ranges compared.
Prints one JSON line."""
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--sizes", default="1,16,256,4096,65536,1048576")
    ap.add_argument("--calls", type=int, default=64, help="batches per size (fewer for the big sizes)")
    ap.add_argument("--walkers", type=int, default=1 << 20)
    ap.add_argument("--slack", type=float, default=0.1)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    sizes = [int(x) for x in a.sizes.split(",")]
    # one stream long enough for the whole sweep (undirected events -> 2 records each)
    need = sum(s * (a.calls if s <= 4096 else 4 if s <= 65536 else 2) for s in sizes)
    t0 = time.time()
    w = synth.make_workload(a.config, rounds=1, device="cuda", batch=(need + 1) // 2 + 1)
    torch.cuda.empty_cache()
    stream = w.batches[0]
    rec = {"config": a.config, "V": int(w.V), "arcs": int(w.num_arcs), "gen_s": round(time.time() - t0, 1)}
    t0 = time.time()
    g = pb.Graph(w.row_offsets, w.dst, w.bias, arc_slack=a.slack, member_slack=a.slack, pool_reserve=0.05)
    torch.cuda.synchronize()
    rec["gpu_build_s"] = round(time.time() - t0, 2)
    info = g.info()
    rec["device_bytes"] = int(info["device_bytes"])
    o = None if a.no_oracle else oracle.OracleGraph(w.row_offsets, w.dst, w.bias, lazy=True)
    paths = torch.empty((81, a.walkers), dtype=torch.int32, device="cuda")
    lens = torch.empty(a.walkers, dtype=torch.int32, device="cuda")
    pos = 0
    sweep = {}
    touched = set()
    walk_ms = []
    first = 0
    for s in sizes:
        ncalls = a.calls if s <= 4096 else (4 if s <= 65536 else 2)
        lat = []
        for c in range(ncalls):
            b = stream[pos:pos + s]
            pos += s
            db = torch.from_numpy(np.ascontiguousarray(b).view(np.int32)).cuda()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sg = g.apply_updates(db)
            e1.record()
            torch.cuda.synchronize()
            lat.append(1e3 * e0.elapsed_time(e1))
            if o is not None:
                so = o.apply_updates(b)
                assert sg["deleted"] == so["deleted"] and sg["touched_vertices"] == so["touched_vertices"]
                touched.update(np.unique(b[:, 1]).tolist())
            if c == ncalls - 1:
                # a DeepWalk batch of 1M walkers between update batches
                e0.record()
                g.walk(length=80, seed=99 + len(walk_ms), first_walker=first, num_walkers=a.walkers, paths=paths,
                       lengths=lens)
                e1.record()
                torch.cuda.synchronize()
                walk_ms.append(e0.elapsed_time(e1))
                first = (first + a.walkers) % w.V
        lat = np.array(lat)
        sweep[str(s)] = {"calls": ncalls, "p50_us": float(np.percentile(lat, 50)),
                         "p99_us": float(np.percentile(lat, 99)),
                         "arcs_per_s": float(s / (np.median(lat) / 1e6))}
    rec["sweep"] = sweep
    steps = int(lens.to(torch.int64).sum())
    rec["walk_ms"] = [round(x, 2) for x in walk_ms]
    rec["walk_steps_per_s_last"] = steps / (walk_ms[-1] / 1e3)
    if o is not None:
        rng = np.random.default_rng(5)
        tv = np.array(sorted(touched), dtype=np.int64)
        sample = np.unique(np.concatenate([rng.choice(tv, size=min(len(tv), 3000), replace=False),
                                           rng.integers(0, w.V, size=2000)]))
        dg = g.digests().cpu().numpy().view(np.uint64)
        bad = [int(u) for u in sample if int(dg[u]) != o.vertex_digest(int(u))]
        assert not bad, f"digest mismatch at {bad[:10]}"
        last_first = (first - a.walkers) % w.V
        for s0 in rng.integers(0, a.walkers - 512, size=4).tolist():
            ref = o.walk(length=80, seed=99 + len(walk_ms) - 1, first_walker=last_first + s0, num_walkers=512,
                         threads=os.cpu_count())
            assert np.array_equal(paths[:, s0:s0 + 512].cpu().numpy().view(np.uint32), ref["paths"])
        rec["digests_compared"] = int(len(sample))
        rec["walkers_compared"] = 4 * 512
        rec["parity"] = "bit-exact"
    print(json.dumps(rec), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
