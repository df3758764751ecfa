// float_bias.cu -- floating-point biases (S4.3 P:344-363, S4.4 P:368-377; R-15), build side.
//
// Per vertex (warp): for lambda = 10^j, j = 0..9, s_i = fl(w_i lambda) (IEEE binary64,
// round-to-nearest, no contraction), I_i = floor(s_i) < 2^32, D_i = floor((s_i - I_i) 2^52)
// (exact), W_I = sum I_i, W_D = sum D_i (u128).  lambda = the smallest j with
// (d - 1) W_D < W_I 2^52 (W_D / (W_I + W_D) < 1/d in real units); none -> the largest
// valid j and flag "constraint unmet".  The integer parts I_i become the arcs' radix-
// decomposed biases (the integer build then runs unchanged); the decimal group is the
// arcs with D_i > 0, ascending; thrD = floor(W_D 2^64 / (W_I 2^52 + W_D)).
#include <cstdio>

#include "bingo.h"
#include "bingo_internal.cuh"
#include "build_common.cuh"
#include "float_bias.cuh"
#include "scan.cuh"

namespace bingo {

__global__ void k_float_lambda(uint32_t V, const uint64_t *__restrict__ ro, const double *__restrict__ wf,
                               uint32_t *__restrict__ ibias, DecRec *__restrict__ dec, uint64_t *__restrict__ dcnt_out,
                               int *__restrict__ flag, const uint32_t *__restrict__ perm) {
    const uint32_t warps = (blockDim.x >> 5) * gridDim.x;
    const uint32_t lane = lane_id();
    for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < V; j += warps) {
        const uint32_t u = perm ? perm[j] : j;   // external CSR row of internal vertex j
        const uint64_t b0 = ro[u];
        const uint32_t d = (uint32_t)(ro[u + 1] - b0);
        // input validation: w > 0, finite, <= 1e300
        bool bad = false;
        for (uint32_t i = lane; i < d; i += 32) {
            const double w = wf[b0 + i];
            if (!(w > 0.0) || !(w <= 1e300)) bad = true;
        }
        if (__any_sync(0xffffffffu, bad)) {
            if (lane == 0) atomicOr(flag, 1);
            continue;
        }
        int chosen = -1, last_valid = -1;
        for (int lj = 0; lj < 10 && chosen < 0; lj++) {
            unsigned __int128 wi = 0, wd = 0;
            bool valid = true;
            for (uint32_t i = lane; i < d; i += 32) {
                uint32_t I;
                uint64_t D;
                if (!scale_one(wf[b0 + i], lj, I, D)) { valid = false; break; }
                wi += I;
                wd += D;
            }
            if (!__all_sync(0xffffffffu, valid)) break;     // larger lambda only grows s_i
            wi = warp_sum128(wi);
            wd = warp_sum128(wd);
            last_valid = lj;
            if ((unsigned __int128)(d ? d - 1 : 0) * wd < (wi << 52)) chosen = lj;
        }
        if (last_valid < 0 && d > 0) {
            if (lane == 0) atomicOr(flag, 4);
            continue;
        }
        uint32_t fl = 0;
        if (chosen < 0) {
            chosen = last_valid < 0 ? 0 : last_valid;
            if (d) fl |= 1u;
        }
        if (d == 0) chosen = 0;   // R-15: the constraint is vacuous for d = 0 -> the smallest lambda
        unsigned __int128 wi = 0, wd = 0;
        uint64_t dmax = 0;
        uint32_t cnt = 0;
        for (uint32_t i = lane; i < d; i += 32) {
            uint32_t I;
            uint64_t D;
            scale_one(wf[b0 + i], chosen, I, D);
            ibias[b0 + i] = I;
            wi += I;
            wd += D;
            dmax = D > dmax ? D : dmax;
            cnt += D ? 1u : 0u;
        }
        wi = warp_sum128(wi);
        wd = warp_sum128(wd);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t m = __shfl_xor_sync(0xffffffffu, dmax, o);
            dmax = m > dmax ? m : dmax;
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
        if (lane == 0) {
            if (wi == 0 && d) fl |= 2u;
            DecRec r;
            r.thrD = wd == 0 ? 0ull : (wi == 0 ? ~0ull : frac64(wd, (wi << 52) + wd));
            r.dmax = dmax;
            r.doff = 0;
            r.dcnt = cnt;
            r.lam = (uint8_t)chosen;
            r.flags = (uint8_t)fl;
            r.pad = 0;
            r.pad2 = dec_capacity(cnt);   // decimal-member capacity (updates, R-16)
            dec[j] = r;
            dcnt_out[j] = dec_capacity(cnt);
        }
    }
}

// decimal members (ascending adjacency index), after the integer build placed the arcs
__global__ void k_float_fill(uint32_t V, const uint64_t *__restrict__ ro, const uint32_t *__restrict__ dst,
                             const double *__restrict__ wf, const uint64_t *__restrict__ doff,
                             DecRec *__restrict__ dec, uint4 *__restrict__ dmem, const VHdr *__restrict__ hdr,
                             uint64_t *__restrict__ arc_dval, const uint32_t *__restrict__ perm,
                             const uint32_t *__restrict__ inv) {
    const uint32_t warps = (blockDim.x >> 5) * gridDim.x;
    const uint32_t lane = lane_id();
    for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < V; j += warps) {
        const uint32_t u = perm ? perm[j] : j;
        const uint64_t b0 = ro[u];
        const uint32_t d = (uint32_t)(ro[u + 1] - b0);
        const int lam = dec[j].lam;
        const uint64_t base = doff[j];
        const uint64_t aoff = hdr[j].adj_off;   // the arc's D travels with it in updates (R-16)
        uint32_t run = 0;
        for (uint32_t c0 = 0; c0 < d; c0 += 32) {
            const uint32_t i = c0 + lane;
            uint32_t I = 0;
            uint64_t D = 0;
            if (i < d) {
                scale_one(wf[b0 + i], lam, I, D);
                arc_dval[aoff + i] = D;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, D != 0);
            if (D) dmem[base + run + __popc(bal & lanemask_lt())] = make_uint4(i, inv ? inv[dst[b0 + i]] : dst[b0 + i], (uint32_t)D, (uint32_t)(D >> 32));
            run += __popc(bal);
        }
        if (lane == 0) dec[j].doff = (uint32_t)base;
    }
}

}  // namespace bingo

using namespace bingo;

// Called by bingo_build in float mode: validates, picks lambda, writes the integer parts
// into `ibias` (device [A]) and the decimal records; the caller runs the integer build on
// ibias and then float_fill().
bingo_status float_prepare(bingo_graph *g, const bingo_build_desc *desc, uint32_t *ibias, uint64_t *dcnt,
                           uint64_t *dscan, uint64_t *tmp, cudaStream_t s, uint64_t *total_dec) {
    const uint32_t V = desc->num_vertices;
    const unsigned blocks = (unsigned)std::min<uint64_t>(((uint64_t)V + 7) / 8, 148ull * 64);
    int hflag = 0;
    if (cudaMemsetAsync(g->dev_flag, 0, sizeof(int), s) != cudaSuccess) return BINGO_E_CUDA;
    k_float_lambda<<<blocks, 256, 0, s>>>(V, desc->row_offsets, desc->bias_f64, ibias, g->dec, dcnt, g->dev_flag,
                                          g->perm);
    bingo_count_launch();
    if (cudaGetLastError() != cudaSuccess) return BINGO_E_CUDA;
    if (exclusive_scan_u64(dcnt, dscan, V, tmp, s) != cudaSuccess) return BINGO_E_CUDA;
    if (cudaMemcpyAsync(&hflag, g->dev_flag, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(total_dec, dscan + V, sizeof(uint64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return BINGO_E_CUDA;
    if (hflag & 1) return BINGO_E_INVAL;
    if (hflag & 4) return BINGO_E_OVERFLOW;
    return BINGO_OK;
}

bingo_status float_fill(bingo_graph *g, const bingo_build_desc *desc, const uint64_t *dscan, cudaStream_t s) {
    const uint32_t V = desc->num_vertices;
    const unsigned blocks = (unsigned)std::min<uint64_t>(((uint64_t)V + 7) / 8, 148ull * 64);
    k_float_fill<<<blocks, 256, 0, s>>>(V, desc->row_offsets, desc->dst, desc->bias_f64, dscan, g->dec, g->dmem,
                                        g->hdr, g->arc_dval, g->perm, g->inv);
    bingo_count_launch();
    return cudaGetLastError() == cudaSuccess ? BINGO_OK : BINGO_E_CUDA;
}
