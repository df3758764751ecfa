// gix_table.cuh -- table primitives of the group inverted index (group_index.cuh), included
// before update_bsp.cuh (the insert and group-tail phases maintain the tables).
#pragma once

namespace bingo {

static constexpr uint32_t GIX_TOMB = 0xFFFFFFFFu;
static constexpr uint32_t GIX_MAXL = (1u << 27) - 2;   // key = p << 5 | k, + 1 must fit 32 bits

struct GixT {
    uint32_t *t;
    uint32_t mask;
};
__device__ __forceinline__ GixT gix_table(const uint32_t *pool, uint64_t o) {
    GixT h;
    h.t = const_cast<uint32_t *>(pool) + (o & ((1ull << 48) - 1));
    h.mask = (uint32_t)((1ull << (o >> 48)) - 1);
    return h;
}
__device__ __forceinline__ uint32_t gix_key(uint32_t p, uint32_t k) { return (p << 5) | k; }

// entries hold keys known to be absent: the first empty or removed word along the probe path
// is taken; false when the table is full (the caller drops the index)
__device__ __forceinline__ bool gix_insert(const GixT &h, uint32_t key, uint32_t slot) {
    uint32_t s = nb_hash(key) & h.mask;
    for (uint32_t n = 0; n <= h.mask; n++) {
        const uint32_t w = h.t[2 * s];
        if (w == 0u || w == GIX_TOMB) {
            if (atomicCAS(&h.t[2 * s], w, key + 1) == w) {
                h.t[2 * s + 1] = slot;
                return true;
            }
            continue;   // taken by another lane: look at the same word again
        }
        s = (s + 1) & h.mask;
    }
    return false;
}
// entry index of key, or 0xFFFFFFFF
__device__ __forceinline__ uint32_t gix_find(const GixT &h, uint32_t key) {
    uint32_t s = nb_hash(key) & h.mask;
    for (uint32_t n = 0; n <= h.mask; n++) {
        const uint32_t w = h.t[2 * s];
        if (w == key + 1) return s;
        if (w == 0u) return 0xFFFFFFFFu;
        s = (s + 1) & h.mask;
    }
    return 0xFFFFFFFFu;
}

// the group tail of a vertex in mode 1 / 2 moved the survivor now at slot hs (position x) of
// group k: its entry follows
__device__ __forceinline__ void gix_reslot(const MutateArgs &g, uint64_t o, uint32_t x, uint32_t k, uint32_t hs) {
    const GixT t = gix_table(g.gix, o);
    const uint32_t e = gix_find(t, gix_key(x, k));
    if (e != 0xFFFFFFFFu) t.t[2 * e + 1] = hs;
}

}  // namespace bingo
