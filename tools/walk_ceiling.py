"""Walk throughput with the graph L2-resident (scale-14/16 R-MAT) vs the c2 graph, same
launch shape (4.71M walkers x 80 steps): separates the memory bound from the
instruction/latency bound of the walk kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2504_10233_b200 as pb  # noqa: E402

W = 4_710_158
for scale, edges in ((12, 60_000), (16, 600_000), (20, 8_000_000)):
    w = synth.Workload(scale, edges, compact=True, batch=10, rounds=1, device="cuda")
    g = pb.Graph(w.row_offsets, w.dst, w.bias)
    paths = torch.empty((81, W), dtype=torch.int32, device="cuda")
    lens = torch.empty(W, dtype=torch.int32, device="cuda")
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.walk(length=80, seed=rep, num_walkers=W, paths=paths, lengths=lens)
        e1.record()
        torch.cuda.synchronize()
    steps = int(lens.to(torch.int64).sum())
    ms = e0.elapsed_time(e1)
    info = g.info()
    print(f"scale {scale}: V {w.V} arcs {w.num_arcs} device MB {info['device_bytes'] / 1e6:.0f}: "
          f"{ms:.2f} ms, {steps / ms / 1e6:.2f} G steps/s", flush=True)
