"""Sharded update application in the replicated regime, measured on one GPU
(measurement only).  For P ranks, rank r applies the records whose source it owns
(src mod P), exports its touched vertices' states, and imports every other rank's.  On one
graph the sub-batches are applied one after another (disjoint vertex sets, so the graph ends
in the same state as after the whole batch) and each rank's phases are timed separately:
  apply(owned_r) + export(owned_r) + import(records of the other ranks)
the slowest rank is the step's update time (plus an all-gather of the records, estimated at
the given bus bandwidth).  Against: the replicated apply of the whole batch.
usage: python tools/sharded_update.py [--config c2] [--batches 4] [--parts 2,4,8]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2504_10233_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--batches", type=int, default=4)
ap.add_argument("--parts", default="2,4,8")
ap.add_argument("--bus-gbs", type=float, default=400.0, help="all-gather bus bandwidth for the estimate")
a = ap.parse_args()
w = synth.make_workload(a.config, rounds=2 + a.batches * (len(a.parts.split(",")) + 1), hold_rounds=10,
                        device="cuda", resident=True)
torch.cuda.empty_cache()
g = pb.Graph(w.row_offsets, w.dst, w.bias)
ev = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))  # noqa: E731


def timed(fn):
    e0, e1 = ev()
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), r


db = [torch.from_numpy(b.view(np.int32)).cuda() for b in w.batches]
g.apply_updates(db[0])
g.apply_updates(db[1])
parts = [int(x) for x in a.parts.split(",")]
rec = {"config": a.config, "V": w.V, "arcs": w.num_arcs, "records": int(db[0].shape[0]), "replicated_ms": [],
       "parts": {P: [] for P in parts}}
idx = 2
for rep in range(a.batches):
    for P in parts:   # each measurement on its own batch, so the graph sees every batch once
        b = db[idx]
        idx += 1
        src = b[:, 1].to(torch.int64) & 0xFFFFFFFF
        owned = [b[src % P == r].contiguous() for r in range(P)]
        ids = [torch.unique(o[:, 1].to(torch.int64)) for o in owned]
        t_apply = [timed(lambda o=o: g.apply_updates(o))[0] for o in owned]
        ex = [timed(lambda i=i: g.export_vertices(i.cuda())) for i in ids]
        t_export = [t for t, _ in ex]
        bufs = [r for _, r in ex]
        t_import = []
        for r in range(P):   # the other ranks' records (re-installing the state they already hold)
            t_import.append(sum(timed(lambda j=j: g.import_vertices(*bufs[j]))[0] for j in range(P) if j != r))
        words = sum(int(bb.numel()) for bb, _ in bufs)
        ag_ms = 4.0 * words / (a.bus_gbs * 1e9) * 1e3
        per = [t_apply[r] + t_export[r] + t_import[r] for r in range(P)]
        rec["parts"][P].append({"apply_ms": t_apply, "export_ms": t_export, "import_ms": t_import,
                                "record_words": words, "allgather_ms_est": ag_ms,
                                "slowest_rank_ms": max(per) + ag_ms})
for rep in range(a.batches):   # the replicated reference: whole batches on the same graph
    rec["replicated_ms"].append(timed(lambda b=db[idx]: g.apply_updates(b))[0])
    idx += 1
med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
rec["summary_ms"] = {"replicated": med(rec["replicated_ms"]),
                     **{f"sharded_P{P}": med([r["slowest_rank_ms"] for r in rec["parts"][P]]) for P in parts}}
print(json.dumps(rec), flush=True)
