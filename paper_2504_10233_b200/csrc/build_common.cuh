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
// member array capacity in 16 B units of the dst array (4 entries per unit)
__host__ __device__ inline uint32_t member_units(uint32_t c, double slack) {
    uint64_t extra = (uint64_t)((double)c * slack);
    if (extra < 2) extra = 2;
    return (uint32_t)(((uint64_t)c + extra + 3) / 4);
}
// degree bins for the L2 hot-set plan: 4 bins per octave
static constexpr int HOT_BINS = 4 * 33;
__host__ __device__ inline int hot_bin(uint32_t d) {
    if (d < 4) return (int)d;
#ifdef __CUDA_ARCH__
    const int e = 31 - __clz(d);                       // floor(log2 d) >= 2
#else
    const int e = 31 - __builtin_clz(d);
#endif
    return 4 * (e - 1) + (int)((d >> (e - 2)) & 3u);   // next two bits
}
// smallest degree in bin b (inverse of hot_bin); b == HOT_BINS -> never hot
__host__ __device__ inline uint32_t hot_bin_floor(int b) {
    if (b >= HOT_BINS) return 0xFFFFFFFFu;
    if (b < 4) return (uint32_t)b;
    const int e = b / 4 + 1, m = b % 4;
    return (uint32_t)((4u + (uint32_t)m) << (e - 2));
}

__host__ __device__ inline uint32_t bucket_capacity(uint32_t n) { return n == 0 ? 0u : (n < 32 ? n + 1 : 32u); }
inline uint64_t pool_capacity(uint64_t used, double reserve, uint64_t min_extra) {
    uint64_t extra = (uint64_t)((double)used * reserve);
    return used + std::max<uint64_t>(extra, min_extra);
}

__device__ __forceinline__ void store_bucket(Bucket *p, const Bucket &b) {
    uint4 lo, hi;
    lo.x = (uint32_t)b.lim;
    lo.y = (uint32_t)(b.lim >> 32);
    lo.z = b.px;
    lo.w = b.py;
    hi.x = b.ax;
    hi.y = b.ay;
    hi.z = (uint32_t)b.kk | ((uint32_t)b.a_kk << 8) | ((uint32_t)b.alias << 16) | ((uint32_t)b.pad << 24);
    hi.w = b.spare;
    uint4 *q = reinterpret_cast<uint4 *>(p);
    q[0] = lo;
    q[1] = hi;
}

__device__ __forceinline__ Bucket unpack_bucket(uint4 lo, uint4 hi) {
    Bucket b;
    b.lim = ((uint64_t)lo.y << 32) | lo.x;
    b.px = lo.z;
    b.py = lo.w;
    b.ax = hi.x;
    b.ay = hi.y;
    b.kk = (uint8_t)(hi.z & 0xff);
    b.a_kk = (uint8_t)((hi.z >> 8) & 0xff);
    b.alias = (uint8_t)((hi.z >> 16) & 0xff);
    b.pad = (uint8_t)(hi.z >> 24);
    b.spare = hi.w;
    return b;
}

__device__ __forceinline__ Bucket load_bucket(const Bucket *p) {
    const uint4 *q = reinterpret_cast<const uint4 *>(p);
    return unpack_bucket(q[0], q[1]);
}

__device__ __forceinline__ void store_gcan(GCan *p, uint64_t thr, uint32_t c, uint32_t aux) {
    *reinterpret_cast<uint4 *>(p) = make_uint4((uint32_t)thr, (uint32_t)(thr >> 32), c, aux);
}
__device__ __forceinline__ GCan load_gcan(const GCan *p) {
    const uint4 v = *reinterpret_cast<const uint4 *>(p);
    GCan g;
    g.thr = ((uint64_t)v.y << 32) | v.x;
    g.c = v.z;
    g.aux = v.w;
    return g;
}

// lim = ceil(thr * 2^64 / T), saturated to 2^64 - 1 (R-4'): for a 64-bit draw R,
//   floor(R T / 2^64) < thr  <=>  R < ceil(thr 2^64 / T)
// (floor(x) < integer thr <=> x < thr; integer R < y <=> R < ceil(y)), so the
// walker's test R < lim takes exactly the decision of the canonical coin
// mulhi64(R, T) < thr.  Saturation only hits thr = T, i.e. an unassigned bucket
// whose alias is itself, where both branches pick the same group.
//
// The quotient floor(thr 2^64 / T) is computed without a 128-bit division: a
// double-precision estimate (off by at most ~2^13), one exact 128-bit remainder,
// a second double estimate of the correction (off by at most 1), and exact
// integer fix-ups until 0 <= remainder < T.  thr < T, so the quotient is below
// 2^64 - 1 and the ceiling cannot overflow.
__device__ __forceinline__ void rem128(uint64_t thr, uint64_t q, uint64_t T, int64_t &rh, uint64_t &rl) {
    // r = thr * 2^64 - q * T as a signed 128-bit (rh, rl); |r| < 2^126
    const uint64_t pl = q * T, ph = __umul64hi(q, T);
    rl = 0ull - pl;
    rh = (int64_t)(thr - ph - (pl != 0ull ? 1ull : 0ull));
}
__device__ __forceinline__ uint64_t alias_lim(uint64_t thr, uint64_t T) {
    if (thr >= T) return ~0ull;
    if (thr == 0) return 0ull;
    const double Td = (double)T;
    double qd = (double)thr / Td * 18446744073709551616.0;
    uint64_t q = qd >= 18446744073709549568.0 ? 18446744073709549568ull : (uint64_t)qd;
    int64_t rh;
    uint64_t rl;
    rem128(thr, q, T, rh, rl);
    const double cd = floor(((double)rh * 18446744073709551616.0 + (double)rl) / Td);
    q += (uint64_t)(int64_t)cd;
    rem128(thr, q, T, rh, rl);
    while (rh < 0) {                          // r < 0: q too large
        q--;
        const uint64_t o = rl;
        rl += T;
        rh += (rl < o) ? 1 : 0;
    }
    while (rh > 0 || rl >= T) {               // r >= T: q too small
        q++;
        const uint64_t o = rl;
        rl -= T;
        rh -= (rl > o) ? 1 : 0;
    }
    return q + ((rh != 0 || rl != 0) ? 1ull : 0ull);
}

// Walker view of group (k, kind): (x, y) as documented on Bucket.
__device__ __forceinline__ void group_view(uint32_t kind, uint32_t c, uint32_t moff, uint32_t one_dst, uint32_t d,
                                           uint64_t adj_off, uint32_t &x, uint32_t &y) {
    if (kind == K_ONE) { x = 1; y = one_dst; }
    else if (kind == K_DENSE) { x = d; y = (uint32_t)(adj_off >> 2); }
    else { x = c; y = moff; }
}

// Fill and store bucket b of a vertex from lane-held per-bucket values (warp-wide).
// Every lane calls it; lanes b < n own bucket b.
__device__ __forceinline__ void write_buckets(Bucket *bkt, GCan *gcan, uint64_t bo, uint32_t n, uint32_t lane,
                                              uint32_t kb, uint32_t kind_b, uint32_t c_b, uint32_t x_b, uint32_t y_b,
                                              uint32_t aux_b, uint64_t thr, uint32_t alias, uint64_t T) {
    Bucket B;
    B.lim = alias_lim(thr, T);
    B.px = x_b;
    B.py = y_b;
    B.kk = make_kk(kb, kind_b);
    B.alias = (uint8_t)alias;
    B.pad = 0;
    B.spare = 0;
    B.ax = __shfl_sync(0xffffffffu, x_b, alias);
    B.ay = __shfl_sync(0xffffffffu, y_b, alias);
    B.a_kk = (uint8_t)__shfl_sync(0xffffffffu, (uint32_t)B.kk, alias);
    if (lane < n) {
        store_bucket(&bkt[bo + lane], B);
        store_gcan(&gcan[bo + lane], thr, c_b, aux_b);
    }
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
