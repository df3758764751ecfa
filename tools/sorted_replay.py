"""Locality experiment for the PPR walk: does processing steps in VERTEX order (instead of
walker order) raise the gather rate of the walk's own loads?

Traces the loads of a prefix of the bench's c4 PPR walkers (bingo_walk_trace), then replays the
same records (bingo_walk_replay, no dependency between loads) three ways:
  walker   -- walker by walker (the bench's gather ceiling)
  chunk    -- the trace cut into fixed chunks of C records, trace order
  sorted   -- the records sorted by their vertex (internal id = hot rank), same chunks
  bins<k>  -- the records grouped by vertex >> k (a counting-sort bin), same chunks
Measurement only.  usage: python tools/sorted_replay.py [--config c4] [--records 6e8]"""
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
ap.add_argument("--config", default="c4")
ap.add_argument("--records", type=float, default=6e8)
ap.add_argument("--chunk", type=int, default=8)
ap.add_argument("--variants", default="")
ap.add_argument("--window", type=float, default=0, help="sort within windows of this many records")
a = ap.parse_args()

w = synth.make_workload(a.config, rounds=1, hold_rounds=10, device="cuda", resident=True)
torch.cuda.empty_cache()
g = pb.Graph(w.row_offsets, w.dst, w.bias)
for b in w.batches:
    g.apply_updates(b)
V = w.V
lens = torch.empty(V, dtype=torch.int32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g.walk(app=pb.PPR, length=pb.NO_CAP, seed=3, paths=None, lengths=lens)
e0.record()
g.walk(app=pb.PPR, length=pb.NO_CAP, seed=3, paths=None, lengths=lens)
e1.record()
torch.cuda.synchronize()
walk_ms = e0.elapsed_time(e1)
steps = int(lens.to(torch.int64).sum())
out = {"config": a.config, "V": V, "walk_ms": walk_ms, "steps": steps,
       "walk_gsteps": steps / walk_ms / 1e6}
cum = torch.cumsum(lens.to(torch.int64), 0)
Wt = int(torch.searchsorted(cum, torch.tensor([int(a.records)], device="cuda"), right=True)[0])
n = int(cum[Wt - 1])
rec_off = torch.zeros(Wt + 1, dtype=torch.int64, device="cuda")
rec_off[1:] = cum[:Wt]
trace = torch.empty((n, 4), dtype=torch.int32, device="cuda")
g.walk_trace(rec_off, trace, app=pb.PPR, length=pb.NO_CAP, stop=(1, 80), seed=3, num_walkers=Wt)
del lens, cum
out.update(walkers_traced=Wt, records=n)


def replay(tr, off, tag):
    best = None
    sw = {}
    for ahead in (1, 2, 4, 8):
        for bps in (2, 4, 6, 8):
            ts = []
            for _ in range(2):
                e0.record()
                g.walk_replay(tr, off, ahead=ahead, blocks_per_sm=bps)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = min(ts)
            sw[f"a{ahead}b{bps}"] = round(t, 3)
            if best is None or t < best[0]:
                best = (t, ahead, bps)
    out[tag] = {"ms": best[0], "ahead": best[1], "bps": best[2], "g_records_s": n / best[0] / 1e6, "sweep": sw}
    print(tag, out[tag], flush=True)


replay(trace, rec_off, "walker")
C = a.chunk
coff = torch.arange(0, n + C, C, dtype=torch.int64, device="cuda").clamp_(max=n)
coff = torch.unique_consecutive(coff)
replay(trace, coff, "chunk")
key = trace[:, 0].to(torch.int64)
win = int(a.window) if a.window else 0


def hybrid(k, hot_bits, cold_shift):
    # hubs (internal id = hot rank < 2^hot_bits) keep their own bin, the rest are binned by id >> cold_shift
    h = 1 << hot_bits
    return torch.where(k < h, k, h + (k >> cold_shift))


variants = [("sorted", lambda k: k), ("bins10", lambda k: k >> 10), ("bins6", lambda k: k >> 6),
            ("hyb15_s11", lambda k: hybrid(k, 15, 11)), ("hyb15_s8", lambda k: hybrid(k, 15, 8)),
            ("hyb12_s11", lambda k: hybrid(k, 12, 11)), ("hyb17_s6", lambda k: hybrid(k, 17, 6))]
if a.variants:
    variants = [v for v in variants if v[0] in a.variants.split(",")]
for tag, f in variants:
    kk = f(key)
    if win:   # sort within windows of `win` records (one super-step's worth of walkers)
        kk = kk + (torch.arange(n, device="cuda", dtype=torch.int64) // win) * (1 << 40)
        tag = tag + "_win"
    idx = torch.sort(kk, stable=True).indices
    del kk
    st = trace.index_select(0, idx)
    del idx
    replay(st, coff, tag)
    del st
    torch.cuda.empty_cache()
print(json.dumps(out))
