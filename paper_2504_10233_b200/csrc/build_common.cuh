// build_common.cuh -- capacity policy, 32 B record load/store and the warp
// integer-Vose alias construction shared by build and update kernels.
#pragma once
#include <algorithm>
#include <cstdint>

#include "bingo_internal.cuh"

namespace bingo {

// Hornet-style growth headroom: slack is a fraction in [0, 4].
__host__ __device__ inline uint64_t arc_capacity(uint32_t d, double slack) {
    uint64_t extra = (uint64_t)((double)d * slack);
    if (extra < 4) extra = 4;
    return ((uint64_t)d + extra + 3) & ~3ull;
}
// member array capacity in 16 B units (2 entries per unit)
__host__ __device__ inline uint32_t member_units(uint32_t c, double slack) {
    uint64_t extra = (uint64_t)((double)c * slack);
    if (extra < 2) extra = 2;
    return (uint32_t)(((uint64_t)c + extra + 1) / 2);
}
__host__ __device__ inline uint32_t bucket_capacity(uint32_t n) { return n == 0 ? 0u : (n < 32 ? n + 1 : 32u); }
inline uint64_t pool_capacity(uint64_t used, double reserve, uint64_t min_extra) {
    uint64_t extra = (uint64_t)((double)used * reserve);
    return used + std::max<uint64_t>(extra, min_extra);
}

__device__ __forceinline__ void store_bucket(Bucket *p, const Bucket &b) {
    uint4 lo, hi;
    lo.x = (uint32_t)b.thr;
    lo.y = (uint32_t)(b.thr >> 32);
    lo.z = b.c;
    lo.w = b.ref;
    hi.x = b.a_c;
    hi.y = b.a_ref;
    hi.z = (uint32_t)b.kk | ((uint32_t)b.a_kk << 8) | ((uint32_t)b.alias << 16) | ((uint32_t)b.pad << 24);
    hi.w = b.aux;
    uint4 *q = reinterpret_cast<uint4 *>(p);
    q[0] = lo;
    q[1] = hi;
}

__device__ __forceinline__ Bucket unpack_bucket(uint4 lo, uint4 hi) {
    Bucket b;
    b.thr = ((uint64_t)lo.y << 32) | lo.x;
    b.c = lo.z;
    b.ref = lo.w;
    b.a_c = hi.x;
    b.a_ref = hi.y;
    b.kk = (uint8_t)(hi.z & 0xff);
    b.a_kk = (uint8_t)((hi.z >> 8) & 0xff);
    b.alias = (uint8_t)((hi.z >> 16) & 0xff);
    b.pad = (uint8_t)(hi.z >> 24);
    b.aux = hi.w;
    return b;
}

__device__ __forceinline__ Bucket load_bucket(const Bucket *p) {
    const uint4 *q = reinterpret_cast<const uint4 *>(p);
    return unpack_bucket(q[0], q[1]);
}

// Integer Vose over the group weights (R-4), one lane per bucket.
//   s_b = n W_b; while a small (s < T) and a large (s >= T) unassigned
//   bucket exist: l = lowest small, h = lowest large; thr[l] = s_l,
//   alias[l] = h, s_h -= T - s_l.  Remaining buckets: thr = T, alias = self.
// Exact integer arithmetic (no rounding).  Lanes with active = false take
// part in the ballots but own no bucket.
__device__ __forceinline__ void vose_warp(bool active, uint32_t n, uint64_t W, uint64_t T, uint64_t &thr,
                                          uint32_t &alias) {
    const uint32_t lane = threadIdx.x & 31u;
    uint64_t s = (uint64_t)n * W;
    bool un = active;
    thr = T;
    alias = lane;
    for (;;) {
        const uint32_t small = __ballot_sync(0xffffffffu, un && s < T);
        const uint32_t large = __ballot_sync(0xffffffffu, un && s >= T);
        if (!small || !large) break;
        const uint32_t l = __ffs(small) - 1, h = __ffs(large) - 1;
        const uint64_t sl = __shfl_sync(0xffffffffu, s, l);
        if (lane == l) { thr = sl; alias = h; un = false; }
        if (lane == h) s -= T - sl;
    }
}

}  // namespace bingo
