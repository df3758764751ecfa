"""Print (V, arcs) of the R-MAT recipe for candidate (scale, raw edges) on the GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402

for arg in sys.argv[1:]:
    sc, e = arg.split(":")
    t = time.time()
    V, a, b = synth.simple_undirected(int(sc), int(float(e)), 1, True, device="cuda")
    print(f"scale {sc} raw {float(e):.3g}: V {V:,} arcs {2 * len(a):,} ({time.time() - t:.1f} s)", flush=True)
    del a, b
    torch.cuda.empty_cache()
