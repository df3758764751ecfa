// unit_kernels.cu -- device-function unit probes for the tests (libbingo_tools.so):
// runs a libbingo device helper on host-supplied inputs so a test can compare it
// with exact integer arithmetic in Python.  Test infrastructure, not product code.
#include <cstdint>
#include <cuda_runtime.h>

#include "bingo_internal.cuh"
#include "build_common.cuh"

namespace {
__global__ void k_alias_lim(const uint64_t *thr, const uint64_t *T, uint64_t *out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = bingo::alias_lim(thr[i], T[i]);
}
}  // namespace

// out[i] = alias_lim(thr[i], T[i]) computed on the device; host arrays; 0 on success
extern "C" int bt_alias_lim(const uint64_t *thr, const uint64_t *T, uint64_t *out, uint64_t n) {
    uint64_t *d = nullptr;
    if (cudaMalloc(&d, 24 * n + 8) != cudaSuccess) return 1;
    int rc = 0;
    if (cudaMemcpy(d, thr, 8 * n, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(d + n, T, 8 * n, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = 2;
    if (!rc) {
        k_alias_lim<<<148, 256>>>(d, d + n, d + 2 * n, n);
        if (cudaMemcpy(out, d + 2 * n, 8 * n, cudaMemcpyDeviceToHost) != cudaSuccess) rc = 3;
    }
    cudaFree(d);
    return rc;
}
