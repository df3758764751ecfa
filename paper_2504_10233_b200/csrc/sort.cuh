// sort.cuh -- stable LSD radix sort of (u32 key, u32 value) pairs.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bingo {

size_t radix_tmp_words(uint64_t n);
// Sorts the lowest key_bits bits of k0 stably, carrying v0.  Ping-pongs with
// (k1, v1); *result_in_1 tells which buffer holds the result.
cudaError_t radix_sort_pairs(uint32_t *k0, uint32_t *v0, uint32_t *k1, uint32_t *v1, uint64_t n, int key_bits,
                             uint64_t *tmp, cudaStream_t s, bool *result_in_1);

}  // namespace bingo
