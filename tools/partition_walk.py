"""1-D partitioned walk at a BASELINE config on one GPU: P partition graphs in
this process, walkers regrouped between rounds (the single-process stand-in for the NCCL
all-to-all of PartitionedBingo).  Reports rounds, time per round and the memory per partition
against the replicated single-graph walk, and checks the outputs are identical."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2504_10233_b200 as pb  # noqa: E402
from paper_2504_10233_b200.distributed import (owned_records, partition_bounds, partition_csr,  # noqa: E402
                                               walk_partitions_local)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--parts", default="2,4,8")
ap.add_argument("--app", default="deepwalk")
a = ap.parse_args()
w = synth.make_workload(a.config, rounds=3, hold_rounds=10, device="cuda", resident=True)
dbs = [torch.from_numpy(b.view(np.int32)).cuda() for b in w.batches]


def timed_apply(g, b):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.apply_updates(b)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)
app = pb.PPR if a.app == "ppr" else pb.DEEPWALK
L = pb.NO_CAP if app == pb.PPR else 80
kw = dict(app=app, length=L, seed=77)
g = pb.Graph(w.row_offsets, w.dst, w.bias)
full_bytes = g.info()["device_bytes"]
upd_full = [timed_apply(g, b) for b in dbs]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ref = g.walk(num_walkers=w.V, paths=(app != pb.PPR), **kw)
e1.record()
torch.cuda.synchronize()
rec = {"config": a.config, "V": w.V, "arcs": w.num_arcs, "app": a.app, "replicated_ms": e0.elapsed_time(e1),
       "replicated_update_ms": upd_full,
       "replicated_graph_gb": full_bytes / 1e9, "parts": {}}
refl = ref["lengths"].clone()
refp = ref["paths"].clone() if ref["paths"] is not None else None
del g, ref
torch.cuda.empty_cache()
for P in [int(x) for x in a.parts.split(",")]:
    bounds = partition_bounds(w.row_offsets, P)
    engines = [pb.Graph(*partition_csr(w.row_offsets, w.dst, w.bias, bounds[r], bounds[r + 1])) for r in range(P)]
    gb = [e.info()["device_bytes"] / 1e9 for e in engines]
    # sharded update application: partition r applies the records whose source it owns
    upd = [[timed_apply(e, owned_records(b, bounds, r, w.V)) for r, e in enumerate(engines)] for b in dbs]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = walk_partitions_local(engines, bounds, w.V, paths=(app != pb.PPR), **kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    same = bool(torch.equal(out["lengths"], refl)) and (refp is None or bool(torch.equal(out["paths"], refp)))
    rec["parts"][P] = {"rounds": out["rounds"], "wall_ms_all_partitions_serial": 1e3 * dt,
                       "sharded_update_ms_per_partition": upd,
                       "sharded_update_ms_max": [max(x) for x in upd],
                       "partition_graph_gb": gb, "identical_to_replicated": same}
    del engines, out
    torch.cuda.empty_cache()
print(json.dumps(rec), flush=True)
