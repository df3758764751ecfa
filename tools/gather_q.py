"""Load-qualifier experiment: 16 B dependent chases over 2 GiB with ldg / cg / ca / nc.no_allocate."""
import ctypes
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
nbytes = int(sys.argv[1]) << 20 if len(sys.argv) > 1 else 2 << 30
modes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [10, 11, 12, 13, 1]
torch.zeros(1, device="cuda")
L.gather_set_l2_fetch.argtypes = [ctypes.c_int]
gran = int(sys.argv[3]) if len(sys.argv) > 3 else -1
print("l2 fetch granularity", L.gather_set_l2_fetch(gran))
buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
scratch = torch.zeros(16, dtype=torch.int32, device="cuda")
nslots = nbytes // 32
s = torch.cuda.current_stream().cuda_stream
L.gather_fill(buf.data_ptr(), nslots, 12345, s)
torch.cuda.synchronize()
for mode in modes:
    ms, loads = ctypes.c_float(), ctypes.c_double()
    L.gather_run(buf.data_ptr(), nslots, mode, 148 * 8, 256, 64, 7, scratch.data_ptr(), ctypes.byref(ms),
                 ctypes.byref(loads), s)
    print(mode, f"{loads.value / (ms.value / 1e3) / 1e9:.2f} G loads/s")
