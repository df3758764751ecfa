// float_bias.cuh -- per-vertex decimal-group record of the floating-point bias mode (R-15)
#pragma once
#include <cstdint>

namespace bingo {

struct __align__(32) DecRec {
    uint64_t thrD;   // decimal group iff a 64-bit draw < thrD (0: none; ~0 with flag bit 1: always)
    uint64_t dmax;   // rejection bound: max D_i
    uint32_t doff;   // first decimal member (16 B entries {idx, dst, D lo, D hi})
    uint32_t dcnt;   // decimal members
    uint8_t lam;     // lambda = 10^lam
    uint8_t flags;   // bit 0: lambda constraint unmet, bit 1: integer part empty
    uint16_t pad;
    uint32_t pad2;
};
static_assert(sizeof(DecRec) == 32, "DecRec is one sector");

__host__ __device__ inline double pow10_exact(int j) {
    // 10^0 .. 10^9 are exact binary64 values
    double p = 1.0;
    for (int i = 0; i < j; i++) p *= 10.0;
    return p;
}

#ifdef __CUDACC__
// s = fl(w 10^j) (IEEE binary64, round to nearest, no contraction); I = floor(s) < 2^32,
// D = floor((s - I) 2^52) (exact).  false when s >= 2^32 (R-15).
__device__ __forceinline__ bool scale_one(double w, int j, uint32_t &I, uint64_t &D) {
    const double s = __dmul_rn(w, pow10_exact(j));
    if (!(s < 4294967296.0)) return false;
    const double fl = floor(s);
    I = (uint32_t)fl;
    D = (uint64_t)floor(__dmul_rn(__dsub_rn(s, fl), 4503599627370496.0));   // 2^52
    return true;
}

__device__ __forceinline__ unsigned __int128 warp_sum128(unsigned __int128 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t lo = __shfl_xor_sync(0xffffffffu, (uint64_t)v, o);
        const uint64_t hi = __shfl_xor_sync(0xffffffffu, (uint64_t)(v >> 64), o);
        v += ((unsigned __int128)hi << 64) | lo;
    }
    return v;
}

// floor(a 2^64 / b) for a < b, binary long division (exact)
__device__ __forceinline__ uint64_t frac64(unsigned __int128 a, unsigned __int128 b) {
    uint64_t q = 0;
    for (int i = 0; i < 64; i++) {
        a <<= 1;
        q <<= 1;
        if (a >= b) { a -= b; q |= 1; }
    }
    return q;
}

// decimal-member capacity of a vertex with c decimal members (growth slack, R-16)
__host__ __device__ inline uint32_t dec_capacity(uint32_t c) { return c ? c + c / 4 + 1 : 0; }
#endif

}  // namespace bingo
