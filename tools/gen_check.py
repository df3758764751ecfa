"""Time the HBM-resident generator (synth.DeviceWorkload) at a config and build the graph from it."""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2504_10233_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--rounds", type=int, default=13)
a = ap.parse_args()
t0 = time.time()
w = synth.make_workload(a.config, rounds=a.rounds, hold_rounds=10, device="cuda", resident=True)
torch.cuda.synchronize()
t1 = time.time()
g = pb.Graph(w.row_offsets, w.dst, w.bias)
torch.cuda.synchronize()
t2 = time.time()
info = g.info()
rec = {"config": a.config, "V": w.V, "arcs": w.num_arcs, "gen_s": t1 - t0, "build_s": t2 - t1,
       "graph_gb": info["device_bytes"] / 1e9, "max_alloc_gb": torch.cuda.max_memory_allocated() / 1e9,
       "batches": len(w.batches), "batch_records": int(w.batches[0].shape[0])}
print(json.dumps(rec), flush=True)
