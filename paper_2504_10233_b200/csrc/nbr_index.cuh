// nbr_index.cuh -- per-vertex neighbour hash sets for the node2vec distance
// test (Eq.1: is there a live arc prev -> v?).  Derived, not canonical state
// (only the boolean answer is defined; A-17): open addressing with linear
// probing over u32 destination ids, load factor <= 1/2, one table per vertex
// of size next_pow2(2d) at entry offset 4 * adj_off of a pool 4x the arc pool
// (so it moves with the adjacency and never needs its own allocator).
// nbo[u] = table base | log2(size) << 48.
// Updates maintain a table in place while its base and size stay the same:
// inserted destinations are added, a destination whose last live arc the batch
// deletes is overwritten by a tombstone (probes walk past tombstones; they are
// never reused), nbtomb[u] counts them, and the table is rebuilt from the
// adjacency once tombstones would pass a quarter of it (so >= 1/4 stays EMPTY).
#pragma once
#include <cstdint>

namespace bingo {

static constexpr uint32_t NB_EMPTY = 0xFFFFFFFFu;
static constexpr uint32_t NB_TOMB = 0xFFFFFFFEu;   // vertex ids are < 2^31 - 1

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

// overwrite v by a tombstone; returns whether v was present
__device__ __forceinline__ bool nb_remove(uint32_t *tbl, uint32_t mask, uint32_t v) {
    uint32_t h = nb_hash(v) & mask;
    for (;;) {
        const uint32_t x = tbl[h];
        if (x == v) {
            tbl[h] = NB_TOMB;
            return true;
        }
        if (x == NB_EMPTY) return false;
        h = (h + 1) & mask;
    }
}

__host__ __device__ inline uint64_t nb_pack(uint64_t base, uint32_t lg) { return base | ((uint64_t)lg << 48); }
__host__ __device__ inline uint64_t nb_base(uint64_t p) { return p & ((1ull << 48) - 1); }
__host__ __device__ inline uint32_t nb_mask(uint64_t p) { return (uint32_t)((1ull << (p >> 48)) - 1); }

}  // namespace bingo
