// nbr_index.cuh -- per-vertex neighbour hash sets for the node2vec distance
// test (Eq.1: is there a live arc prev -> v?).  Derived, not canonical state
// (only the boolean answer is defined; A-17): open addressing with linear
// probing over u32 destination ids, load factor <= 1/2, one table per vertex
// of size next_pow2(2d) at entry offset 4 * adj_off of a pool 4x the arc pool
// (so it moves with the adjacency and never needs its own allocator).
// nbo[u] = table base | log2(size) << 48.
#pragma once
#include <cstdint>

namespace bingo {

static constexpr uint32_t NB_EMPTY = 0xFFFFFFFFu;

__host__ __device__ inline uint32_t nb_log2size(uint32_t d) {
    uint32_t lg = 0;
    while ((1ull << lg) < 2ull * d) lg++;
    return lg;   // d = 0 -> size 1
}

__device__ __forceinline__ uint32_t nb_hash(uint32_t v) {
    v ^= v >> 16;
    v *= 0x45d9f3bu;
    v ^= v >> 16;
    return v;
}

__device__ __forceinline__ void nb_insert(uint32_t *tbl, uint32_t mask, uint32_t v) {
    uint32_t h = nb_hash(v) & mask;
    for (;;) {
        const uint32_t old = atomicCAS(&tbl[h], NB_EMPTY, v);
        if (old == NB_EMPTY || old == v) return;
        h = (h + 1) & mask;
    }
}

__device__ __forceinline__ bool nb_contains(const uint32_t *tbl, uint32_t mask, uint32_t v) {
    uint32_t h = nb_hash(v) & mask;
    for (;;) {
        const uint32_t x = __ldg(tbl + h);
        if (x == v) return true;
        if (x == NB_EMPTY) return false;
        h = (h + 1) & mask;
    }
}

__host__ __device__ inline uint64_t nb_pack(uint64_t base, uint32_t lg) { return base | ((uint64_t)lg << 48); }
__host__ __device__ inline uint64_t nb_base(uint64_t p) { return p & ((1ull << 48) - 1); }
__host__ __device__ inline uint32_t nb_mask(uint64_t p) { return (uint32_t)((1ull << (p >> 48)) - 1); }

}  // namespace bingo
