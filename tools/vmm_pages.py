"""Does the GPU map a large physical allocation with bigger pages than 2 MB when the VA range
is reserved with a large alignment (cuMemCreate + cuMemAddressReserve(align) + cuMemMap)?
Runs the TLB-reach chase of tools/tlb_sweep.py (gather_spread: a FIXED set of lines scattered
over a growing range) on (a) a torch (cudaMalloc) buffer and (b) VMM buffers reserved at
2 MB / 1 GB / 4 GB alignment.  If (b) keeps its rate at ranges where (a) falls, the walk's
pools could live in such a mapping.  Measurement only."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402
from paper_2504_10233_b200 import _build  # noqa: E402


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) == 2 else r


torch.cuda.init()
torch.zeros(1, device="cuda")
L = ctypes.CDLL(_build.TOOLS_LIB)
L.gather_spread.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                            ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float),
                            ctypes.c_void_p]
scratch = torch.zeros(16, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream

prop = cu.CUmemAllocationProp()
prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
prop.location.id = 0
gmin = ck(cu.cuMemGetAllocationGranularity(prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))
grec = ck(cu.cuMemGetAllocationGranularity(prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
print("granularity min", gmin, "recommended", grec, flush=True)

SIZE = 16 << 30


def vmm_buffer(size, align):
    h = ck(cu.cuMemCreate(size, prop, 0))
    ptr = ck(cu.cuMemAddressReserve(size, align, 0, 0))
    ck(cu.cuMemMap(ptr, size, 0, h, 0))
    acc = cu.CUmemAccessDesc()
    acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = 0
    acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    ck(cu.cuMemSetAccess(ptr, size, [acc], 1))
    return int(ptr), h


def free_vmm(ptr, h, size):
    ck(cu.cuMemUnmap(ptr, size))
    ck(cu.cuMemAddressFree(ptr, size))
    ck(cu.cuMemRelease(h))


def sweep(ptr, tag):
    out = []
    blocks, threads, iters = 148 * 8, 256, 64
    log_slots = 18   # 32 MB of lines
    for spread in (4, 16, 64, 256, 512):
        nbytes = (1 << log_slots) * spread * 128
        if nbytes > SIZE:
            continue
        best = 1e9
        for rep in range(3):
            ms = ctypes.c_float()
            rc = L.gather_spread(ptr, 1 << log_slots, spread, blocks, threads, iters, 7 + rep, scratch.data_ptr(),
                                 ctypes.byref(ms), s)
            assert rc == 0, rc
            best = min(best, ms.value)
        r = {"alloc": tag, "range_mb": nbytes >> 20, "G_loads_per_s": round(blocks * threads * iters / (best / 1e3) / 1e9, 2)}
        print(r, flush=True)
        out.append(r)
    return out


res = []
buf = torch.empty(SIZE, dtype=torch.uint8, device="cuda")
res += sweep(buf.data_ptr(), "torch")
del buf
torch.cuda.empty_cache()
for align in (2 << 20, 1 << 30, 4 << 30):
    p, h = vmm_buffer(SIZE, align)
    res += sweep(p, f"vmm_align_{align >> 20}MB")
    free_vmm(p, h, SIZE)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump({"granularity_min": int(gmin), "granularity_rec": int(grec), "sweep": res},
          open(os.path.join(ROOT, "gpurun_out", "vmm_pages.json"), "w"), indent=1)
