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

}  // namespace bingo
