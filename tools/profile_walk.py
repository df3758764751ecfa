"""One update batch + one DeepWalk on the bench workload (c2), for ncu captures.
usage: python tools/profile_walk.py [--config c2] [--walks 2]"""
import argparse
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
ap.add_argument("--walks", type=int, default=2)
ap.add_argument("--app", default="deepwalk")
ap.add_argument("--gen", default="resident", help="cpu | cuda | resident (generated and kept in HBM, as bench.py)")
a = ap.parse_args()
if a.gen == "resident":
    w = synth.make_workload(a.config, rounds=2, hold_rounds=10, device="cuda", resident=True)
else:
    w = synth.make_workload(a.config, rounds=2, device=a.gen)
torch.cuda.empty_cache()
g = pb.Graph(w.row_offsets, w.dst, w.bias, neighbor_index=("node2vec" in a.app))
for b in w.batches:
    g.apply_updates(b)
lens = torch.empty(w.V, dtype=torch.int32, device="cuda")
paths = None
for name in a.app.split(","):
    app = {"deepwalk": pb.DEEPWALK, "node2vec": pb.NODE2VEC, "ppr": pb.PPR}[name]
    if app != pb.PPR and paths is None:
        paths = torch.empty((81, w.V), dtype=torch.int32, device="cuda")
    for i in range(a.walks):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if app == pb.PPR:
            g.walk(app=app, length=pb.NO_CAP, seed=i, paths=None, lengths=lens)
        else:
            g.walk(app=app, length=80, seed=i, paths=paths, lengths=lens, p=2.0, q=0.5)
        e1.record()
        torch.cuda.synchronize()
        steps = int(lens.to(torch.int64).sum())
        ms = e0.elapsed_time(e1)
        print(f"{name} walk {i}: {ms:.2f} ms, {steps} steps, {steps / ms / 1e6:.2f} G steps/s", flush=True)
print("done", w.V, w.num_arcs)
