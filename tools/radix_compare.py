"""f4 at a BASELINE config: the base-2^b structure (b = 1..4) against the paper's base-2 Bingo
with adaptive groups -- memory (buckets, member entries, bytes), the DeepWalk / PPR walk time of
one launch over every vertex, and (session 3, reading R-19) the time of the config's update
batches (the radix graphs rebuild every touched vertex from its adjacency)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2504_10233_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--bases", default="0,1,2,3,4")
a = ap.parse_args()
w = synth.make_workload(a.config, rounds=6, hold_rounds=10, device="cuda", resident=True)
rec = {"config": a.config, "V": w.V, "arcs": w.num_arcs, "structures": {}}
for b in [int(x) for x in a.bases.split(",")]:
    g = pb.Graph(w.row_offsets, w.dst, w.bias, radix_log2=b) if b else pb.Graph(w.row_offsets, w.dst, w.bias)
    info = g.info()
    thdr_n = None
    r = {"device_gb": info["device_bytes"] / 1e9, "buckets": info["bucket_pool_used"],
         "member_entries": info["member_pool_used"], "arcs_stored": info["arc_pool_used"],
         "sampling_bytes": 32 * info["bucket_pool_used"] + 4 * info["member_pool_used"]
                           + (0 if b else 8 * info["arc_pool_used"]) + 8 * w.V,
         "sampling_bytes_def": "32 B buckets + 4 B member dsts + 8 B {dst, bias} arcs (base 2 only: its dense "
                               "groups sample them) + 8 B thin header per vertex: what a walk reads"}
    ums = []
    for k, bt in enumerate(w.batches):
        db = torch.from_numpy(bt.view("int32")).cuda()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.apply_updates(db)
        e1.record()
        torch.cuda.synchronize()
        if k >= 2:
            ums.append(e0.elapsed_time(e1))
    ums.sort()
    r["update_ms_median"] = ums[len(ums) // 2]
    r["update_records"] = int(w.batches[0].shape[0])
    for app, name in ((pb.DEEPWALK, "deepwalk"), (pb.PPR, "ppr")):
        kw = dict(app=app, seed=5)
        if app == pb.PPR:
            kw.update(length=pb.NO_CAP, paths=None)
            g.reset_visit_counts()
        else:
            kw.update(length=80)
        ms = []
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = g.walk(num_walkers=w.V, **kw)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        steps = int(out["lengths"].to(torch.int64).sum())
        r[name + "_ms"] = min(ms)
        r[name + "_gsteps"] = steps / (min(ms) / 1e3) / 1e9
    rec["structures"]["base2_adaptive" if b == 0 else f"radix_b{b}"] = r
    del g, out
    torch.cuda.empty_cache()
print(json.dumps(rec), flush=True)
