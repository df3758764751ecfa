// scan.cuh -- device exclusive prefix sums (u64) used by build and updates.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bingo {

// Exclusive scan of in[0..n) into out[0..n); out[n] receives the total.
// `tmp` must hold scan_tmp_words(n) u64.  Asynchronous on `s`.
size_t scan_tmp_words(uint64_t n);
cudaError_t exclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t *tmp, cudaStream_t s);
// `count` (<= SCAN_MULTI_MAX) independent scans of length n in one launch; tmp must hold
// count * scan_tmp_words(n) u64
#define SCAN_MULTI_MAX 8
cudaError_t exclusive_scan_u64_multi(const uint64_t *const *in, uint64_t *const *out, int count, uint64_t n,
                                     uint64_t *tmp, cudaStream_t s);
// the same with the length read on the device from *pn (<= nmax; tmp sized for nmax):
// for launches enqueued before the length is known on the host
cudaError_t exclusive_scan_u64_multi_dn(const uint64_t *const *in, uint64_t *const *out, int count,
                                        const unsigned long long *pn, uint64_t nmax, uint64_t *tmp, cudaStream_t s);

}  // namespace bingo
