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
a = ap.parse_args()
w = synth.make_workload(a.config, rounds=2)
g = pb.Graph(w.row_offsets, w.dst, w.bias)
for b in w.batches:
    g.apply_updates(b)
app = {"deepwalk": pb.DEEPWALK, "node2vec": pb.NODE2VEC, "ppr": pb.PPR}[a.app]
paths = torch.empty((81, w.V), dtype=torch.int32, device="cuda")
for i in range(a.walks):
    if app == pb.PPR:
        g.walk(app=app, length=pb.NO_CAP, seed=i, paths=None)
    else:
        g.walk(app=app, length=80, seed=i, paths=paths, p=2.0, q=0.5)
torch.cuda.synchronize()
print("done", w.V, w.num_arcs)
