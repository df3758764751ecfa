"""Sampled parity of an updated radix graph at a BASELINE config (measurement support): the
GPU radix graph and the oracle's RadixGraph apply the same update batches; then DeepWalk paths
and PPR lengths of a walker sample must agree, and walk times are taken before and after.
usage: python tools/radix_check.py [--config c2] [--b 4] [--batches 4] [--walkers 200000]"""
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
ap.add_argument("--config", default="c2")
ap.add_argument("--b", type=int, default=4)
ap.add_argument("--batches", type=int, default=4)
ap.add_argument("--walkers", type=int, default=200000)
a = ap.parse_args()
w = synth.make_workload(a.config, rounds=a.batches, hold_rounds=10, device="cuda", resident=True)
ro, dst, bias = w.host_csr()
g = pb.Graph(w.row_offsets, w.dst, w.bias, radix_log2=a.b)
o = oracle.RadixGraph(ro, dst, bias, a.b)


def tw():
    ms = []
    for _ in range(3):
        paths = torch.empty((81, w.V), dtype=torch.int32, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.walk(length=80, seed=1, paths=paths)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return min(ms)


rec = {"config": a.config, "b": a.b, "walk_ms_before": tw()}
for bt in w.batches:
    sg = g.apply_updates(bt)
    so = o.apply_updates(bt)
    assert all(sg[k] == so[k] for k in ("inserted", "deleted", "missing_deletes", "touched_vertices")), (sg, so)
rec["walk_ms_after"] = tw()
W = a.walkers
out = g.walk(length=40, seed=11, num_walkers=W, first_walker=12345)
ref = o.walk(length=40, seed=11, num_walkers=W, first_walker=12345)
rec["deepwalk_paths_equal"] = bool(np.array_equal(out["paths"].cpu().numpy().view(np.uint32), ref["paths"]))
out = g.walk(app=pb.PPR, length=pb.NO_CAP, seed=12, num_walkers=W, paths=None)
ref = o.walk(app=oracle.APP_PPR, length=oracle.NONE, seed=12, num_walkers=W, paths=False)
rec["ppr_lengths_equal"] = bool(np.array_equal(out["lengths"].cpu().numpy().view(np.uint32), ref["lengths"]))
rec["walkers"] = W
print(json.dumps(rec), flush=True)
assert rec["deepwalk_paths_equal"] and rec["ppr_lengths_equal"]
