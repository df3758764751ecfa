"""Single-record update latency (a11 / f2) on a BASELINE graph: the same records applied one
per call through (a) the persistent streaming queue (bingo_stream_update) and (b) one launch
per record (bingo_apply_updates), both via ctypes, host call to host-visible completion.
Latencies are broken down by the degree of the record's source vertex.  With --check the lazy
oracle replays every record (statistics compared per record, touched digests at the end).
Prints one JSON line."""
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
ap.add_argument("--records", type=int, default=4000)
ap.add_argument("--check", action="store_true")
a = ap.parse_args()
if a.config in ("c1", "c2", "c3", "c4"):
    w = synth.make_workload(a.config, rounds=3, hold_rounds=10, device="cuda", resident=True)
    host = w.host_csr() if a.check else None
    deg = torch.diff(w.row_offsets).cpu().numpy()
else:   # c5: too big for the in-HBM generator's temporaries next to the graph
    w = synth.make_workload(a.config, rounds=1, device="cuda", batch=a.records)
    host = (w.row_offsets, w.dst, w.bias) if a.check else None
    deg = np.diff(w.row_offsets.astype(np.int64))
    torch.cuda.empty_cache()
if a.config == "c5":   # 139 GB of pools: the slack of tools/streaming_sweep.py
    g = pb.Graph(w.row_offsets, w.dst, w.bias, arc_slack=0.1, member_slack=0.1, pool_reserve=0.05)
else:
    g = pb.Graph(w.row_offsets, w.dst, w.bias)
recs = np.ascontiguousarray(np.concatenate(w.batches)[: 2 * a.records], dtype=np.uint32)
qrec, lrec = recs[: a.records], recs[a.records: 2 * a.records]
lib, h = bb._lib(), g.handle
sp = torch.cuda.current_stream().cuda_stream
o = None
if a.check:
    import oracle
    o = oracle.OracleGraph(*host, lazy=True)
st = bb.UpdateStats()


def run(fn, arr):
    lat = []
    for i in range(len(arr)):
        t0 = time.perf_counter()
        rc = fn(h, arr.ctypes.data + 16 * i, ctypes.byref(st), sp)
        lat.append(1e6 * (time.perf_counter() - t0))
        assert rc == 0, rc
        if o is not None:
            so = o.apply_updates(arr[i:i + 1])
            assert (st.inserted, st.deleted, st.missing_deletes) == (so["inserted"], so["deleted"],
                                                                       so["missing_deletes"]), i
    return np.array(lat)


lq = run(lambda h_, p, s_, sp_: lib.bingo_stream_update(h_, p, s_, sp_), qrec)
ll = run(lambda h_, p, s_, sp_: lib.bingo_apply_updates(h_, p, 1, bb.UPD_HOST_BATCH, s_, sp_), lrec)
torch.cuda.synchronize()


def summary(lat, arr):
    d = deg[arr[:, 1].astype(np.int64)]
    out = {"p50_us": float(np.percentile(lat, 50)), "p90_us": float(np.percentile(lat, 90)),
           "p99_us": float(np.percentile(lat, 99)), "updates_per_s": float(len(lat) / (1e-6 * lat.sum()))}
    bins = [(0, 64), (64, 512), (512, 8192), (8192, 1 << 40)]
    out["by_src_degree"] = {f"[{lo},{hi})": {"n": int(((d >= lo) & (d < hi)).sum()),
                                           "p50_us": float(np.percentile(lat[(d >= lo) & (d < hi)], 50))
                                           if ((d >= lo) & (d < hi)).any() else None}
                            for lo, hi in bins}
    return out


rec = {"config": a.config, "V": int(w.V), "arcs": int(w.num_arcs), "records": a.records,
       "queue": summary(lq, qrec), "launch_per_record": summary(ll, lrec), "oracle_checked": bool(a.check)}
if o is not None:
    touched = np.unique(recs[:, 1])
    dg = g.digests().cpu().numpy().view(np.uint64)
    bad = [int(u) for u in touched[:3000] if int(dg[u]) != o.vertex_digest(int(u))]
    assert not bad, bad[:5]
    rec["digests_compared"] = int(min(len(touched), 3000))
print(json.dumps(rec), flush=True)
