"""Update-pipeline timing on the bench workload: per-batch device time (CUDA events) and,
under ncu, the per-kernel launch list.  usage: python tools/profile_update.py [--batches 5]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2504_10233_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--batches", type=int, default=5)
ap.add_argument("--single", type=int, default=0, help="also time this many single-record updates")
ap.add_argument("--gen", default="resident", help="cpu | cuda | resident (generated and kept in HBM, as bench.py)")
a = ap.parse_args()
if a.gen == "resident":
    w = synth.make_workload(a.config, rounds=a.batches + 1, hold_rounds=10, device="cuda", resident=True)
else:
    w = synth.make_workload(a.config, rounds=a.batches + 1, device=a.gen)
torch.cuda.empty_cache()
g = pb.Graph(w.row_offsets, w.dst, w.bias)
db = [torch.from_numpy(b.view(np.int32)).cuda() for b in w.batches]
g.apply_updates(db[0])
torch.cuda.synchronize()
for i in range(1, a.batches + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    st = g.apply_updates(db[i])
    e1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"batch {i}: {e0.elapsed_time(e1):.3f} ms device, {1e3 * (t1 - t0):.3f} ms host, "
          f"touched {st['touched_vertices']}, deleted {st['deleted']}, missing {st['missing_deletes']}")
print(f"update_reruns {g.info()['update_reruns']}")
if a.single:
    recs = w.batches[0][: a.single]
    lat = []
    for r in recs:
        t0 = time.perf_counter()
        g.apply_updates(r[None, :])
        lat.append(time.perf_counter() - t0)
    lat = np.array(lat) * 1e6
    print(f"single-record updates: p50 {np.percentile(lat, 50):.1f} us, p99 {np.percentile(lat, 99):.1f} us")
