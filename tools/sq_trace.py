"""Where a streamed record's time goes (measurement only): runs records through the
persistent streaming queue (bingo_stream_update) with a -DBINGO_SQ_TRACE build
(BINGO_LIB_OVERRIDE=build/variants/sqtrace/libbingo.so) and prints, per phase, the median
of the kernel's globaltimer deltas:
  valid   record seen -> validated        plan   -> plan + capacity decision
  mutate  -> mutation done                out    -> status / statistics written
  fence   -> __threadfence_system         host   the host call, post to completion
host - (seen -> fence) is the PCIe part: detection by the poll and the write-back.
usage: BINGO_LIB_OVERRIDE=... python tools/sq_trace.py [--config c2] [--records 3000]"""
import argparse
import ctypes
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
from paper_2504_10233_b200 import bingo as bb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--records", type=int, default=3000)
ap.add_argument("--invalid", action="store_true", help="post records with src = V (rejected by validation)")
a = ap.parse_args()
w = synth.make_workload(a.config, rounds=2, hold_rounds=10, device="cuda", resident=True)
g = pb.Graph(w.row_offsets, w.dst, w.bias)
recs = np.ascontiguousarray(np.concatenate(w.batches)[: a.records], dtype=np.uint32)
if a.invalid:
    recs[:, 1] = w.V
lib, h = bb._lib(), g.handle
lib.bingo_sq_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
sp = torch.cuda.current_stream().cuda_stream
st = bb.UpdateStats()
lat = []
for i in range(len(recs)):
    t0 = time.perf_counter()
    rc = lib.bingo_stream_update(h, recs.ctypes.data + 16 * i, ctypes.byref(st), sp)
    lat.append(1e6 * (time.perf_counter() - t0))
    assert rc == (bb.E_INVAL if a.invalid else 0), rc
torch.cuda.synchronize()
tr = np.zeros((8192, 8), dtype=np.uint64)
assert lib.bingo_sq_trace_read(tr.ctypes.data, 8192) == 0
# record k of a fresh graph's queue is traced at row k
tr = tr[: len(recs)].astype(np.int64)
lat = np.array(lat)
ok = tr[:, 0] > 0
d = {"valid": tr[:, 1] - tr[:, 0], "plan": tr[:, 2] - tr[:, 1], "mutate": tr[:, 3] - tr[:, 2],
     "out": tr[:, 4] - tr[:, 3], "fence": tr[:, 5] - tr[:, 4], "seen_to_fence": tr[:, 5] - tr[:, 0]}
res = {"config": a.config, "records": len(recs), "invalid": a.invalid,
       "host_us": {"p50": float(np.percentile(lat, 50)), "p90": float(np.percentile(lat, 90)),
                   "p99": float(np.percentile(lat, 99))}}
for k, v in d.items():
    v = v[ok & (v >= 0) & (v < 10_000_000)] / 1e3
    if len(v):
        res[k + "_us"] = {"p50": float(np.percentile(v, 50)), "p90": float(np.percentile(v, 90))}
print(json.dumps(res), flush=True)
