"""PCIe D2H probe (measurement infrastructure): contiguous vs step-major 2-D (strided rows)
copies of walk-path chunks into pinned host memory, as bingo_walk(HOST_OUTPUT) issues them."""
import ctypes
import time

import torch

cudart = ctypes.CDLL("libcudart.so") if False else None
try:
    cudart = ctypes.CDLL("libcudart.so.12")
except OSError:
    import glob
    cudart = ctypes.CDLL(sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))[0])
cudart.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
cudart.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
W, R = 4_710_158, 81
host = torch.empty((R, W), dtype=torch.int32).pin_memory()
dev = torch.empty((R, W), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
for nch in (1, 4, 8, 16):
    wc = (W + nch - 1) // nch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for c in range(nch):
        c0, wn = c * wc, min(wc, W - c * wc)
        cudart.cudaMemcpy2DAsync(host.data_ptr() + 4 * c0, 4 * W, dev.data_ptr() + 4 * c0, 4 * W, 4 * wn, R, 2,
                                 ctypes.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"2-D rows, {nch} chunks: {4 * W * R / dt / 1e9:.1f} GB/s")
torch.cuda.synchronize()
t0 = time.perf_counter()
cudart.cudaMemcpyAsync(host.data_ptr(), dev.data_ptr(), 4 * W * R, 2, ctypes.c_void_p(s.cuda_stream))
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"contiguous: {4 * W * R / dt / 1e9:.1f} GB/s")
