"""Random-gather roofline sweep over footprints (measurement infrastructure)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2504_10233_b200 import _build  # noqa: E402

L = ctypes.CDLL(_build.TOOLS_LIB)
L.gather_fill.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
L.gather_run.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                         ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float),
                         ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]
res = {}
scratch = torch.zeros(16, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for mb in [64, 256, 1024, 2048, 8192, 32768]:
    nbytes = mb << 20
    buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    nslots = nbytes // 32
    L.gather_fill(buf.data_ptr(), nslots, 12345, s)
    torch.cuda.synchronize()
    row = {}
    for mode, name, blocks, threads, iters in ((0, "indep8", 148 * 8, 256, 64), (1, "chase1", 148 * 8, 256, 64),
                                               (2, "chase2", 148 * 8, 256, 32), (3, "chase4", 148 * 8, 256, 16),
                                               (1, "chase1_half_occ", 148 * 4, 256, 64)):
        best = 0
        for rep in range(3):
            ms, loads = ctypes.c_float(), ctypes.c_double()
            L.gather_run(buf.data_ptr(), nslots, mode, blocks, threads, iters, 7 + rep, scratch.data_ptr(),
                         ctypes.byref(ms), ctypes.byref(loads), s)
            best = max(best, 32 * loads.value / (ms.value / 1e3) / 1e9)
        row[name] = round(best, 1)
    res[mb] = row
    print(mb, "MiB", row, flush=True)
    del buf
    torch.cuda.empty_cache()
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "gather_sweep.json"), "w"), indent=1)
