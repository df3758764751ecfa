"""TLB-reach experiment (measurement infrastructure): a dependent random chase over a
FIXED set of 128 B lines scattered over a growing address range (tools/gather_bench.cu
gather_spread).  If random-access throughput falls while the touched-line set (and so
the L2 footprint) is unchanged, the limit is address translation, not DRAM or L2."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2504_10233_b200 import _build  # noqa: E402

L = ctypes.CDLL(_build.TOOLS_LIB)
L.gather_spread.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                            ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float),
                            ctypes.c_void_p]
scratch = torch.zeros(16, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
res = []
blocks, threads, iters = 148 * 8, 256, 64
for log_slots in (18, 19, 21, 23, 25):
    for spread in (1, 4, 16, 64, 256, 1024, 4096):
        nbytes = (1 << log_slots) * spread * 128
        if nbytes > (48 << 30) or nbytes < (1 << 20):
            continue
        buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        best = 1e9
        for rep in range(3):
            ms = ctypes.c_float()
            L.gather_spread(buf.data_ptr(), 1 << log_slots, spread, blocks, threads, iters, 7 + rep,
                            scratch.data_ptr(), ctypes.byref(ms), s)
            best = min(best, ms.value)
        gls = blocks * threads * iters / (best / 1e3) / 1e9
        r = {"lines": 1 << log_slots, "line_mb": (1 << log_slots) * 128 >> 20, "spread": spread,
             "range_mb": nbytes >> 20, "pages_2mb": max(1, nbytes >> 21), "G_loads_per_s": round(gls, 2)}
        res.append(r)
        print(r, flush=True)
        del buf
        torch.cuda.empty_cache()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "tlb_sweep.json"), "w"), indent=1)
