// sort.cu -- stable LSD radix sort of (u32 key, u32 value) pairs, 8-bit digits.
// Used to segment an update batch by source vertex with batch order kept
// inside every segment ("put the graph updates of the same vertex
// together").
//
// Per pass: k_radix_hist (per-tile digit counts, digit-major), an exclusive
// scan over [digit][tile], k_radix_scatter (stable in-tile ranks by warp
// match + per-warp digit tables, then scatter).  Tiles of 2048 items are
// processed round-major (item = base + r * 256 + thread) so rank order is
// input order.
#include "scan.cuh"
#include "bingo_internal.cuh"
#include "sort.cuh"

namespace bingo {

static constexpr int RT = 256;        // threads per tile
static constexpr int RI = 8;          // items per thread
static constexpr uint32_t RTILE = RT * RI;

__global__ void __launch_bounds__(RT) k_radix_hist(const uint32_t *__restrict__ keys, uint64_t n, int shift,
                                                   uint64_t *__restrict__ hist, uint32_t tiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * RTILE;
#pragma unroll
    for (int r = 0; r < RI; r++) {
        const uint64_t i = base + (uint64_t)r * RT + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[(uint64_t)threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(RT) k_radix_scatter(const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin,
                                                      uint32_t *__restrict__ kout, uint32_t *__restrict__ vout,
                                                      uint64_t n, int shift, const uint64_t *__restrict__ off,
                                                      uint32_t tiles) {
    __shared__ uint32_t wcnt[RT / 32][256];
    __shared__ uint32_t run[256];
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    run[threadIdx.x] = 0;
    for (int w = 0; w < RT / 32; w++) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * RTILE;
    const uint64_t tile_off = off[(uint64_t)threadIdx.x * tiles + blockIdx.x];  // thread = digit
    __shared__ uint64_t s_off[256];
    s_off[threadIdx.x] = tile_off;
    __syncthreads();
    for (int r = 0; r < RI; r++) {
        const uint64_t i = base + (uint64_t)r * RT + threadIdx.x;
        const bool valid = i < n;
        uint32_t key = 0, val = 0, dig = 0xFFFFFFFFu;
        if (valid) {
            key = kin[i];
            val = vin[i];
            dig = (key >> shift) & 255u;
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, dig);
        const uint32_t lt = peers & ((1u << lane) - 1u);
        if (valid && lt == 0) wcnt[wid][dig] = __popc(peers);   // group leader records the count
        __syncthreads();
        {   // thread d: exclusive prefix over warps, carried across rounds
            const uint32_t d = threadIdx.x;
            uint32_t acc = run[d];
            for (int w = 0; w < RT / 32; w++) {
                const uint32_t t = wcnt[w][d];
                wcnt[w][d] = acc;
                acc += t;
            }
            run[d] = acc;
        }
        __syncthreads();
        if (valid) {
            const uint64_t dst = s_off[dig] + wcnt[wid][dig] + __popc(lt);
            kout[dst] = key;
            vout[dst] = val;
        }
        __syncthreads();
        for (int w = 0; w < RT / 32; w++) wcnt[w][threadIdx.x] = 0;
        __syncthreads();
    }
}

size_t radix_tmp_words(uint64_t n) {
    const uint64_t tiles = (n + RTILE - 1) / RTILE;
    return 2 * (256 * tiles + 1) + scan_tmp_words(256 * tiles);
}

cudaError_t radix_sort_pairs(uint32_t *k0, uint32_t *v0, uint32_t *k1, uint32_t *v1, uint64_t n, int key_bits,
                             uint64_t *tmp, cudaStream_t s, bool *result_in_1) {
    *result_in_1 = false;
    if (n <= 1) return cudaSuccess;
    const uint32_t tiles = (uint32_t)((n + RTILE - 1) / RTILE);
    uint64_t *hist = tmp;
    uint64_t *off = tmp + 256ull * tiles + 1;
    uint64_t *stmp = off + 256ull * tiles + 1;
    uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
    for (int shift = 0; shift < key_bits; shift += 8) {
        k_radix_hist<<<tiles, RT, 0, s>>>(ki, n, shift, hist, tiles);
        bingo_count_launch();
        cudaError_t e = exclusive_scan_u64(hist, off, 256ull * tiles, stmp, s);
        if (e != cudaSuccess) return e;
        k_radix_scatter<<<tiles, RT, 0, s>>>(ki, vi, ko, vo, n, shift, off, tiles);
        bingo_count_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        uint32_t *t = ki; ki = ko; ko = t;
        t = vi; vi = vo; vo = t;
        *result_in_1 = !*result_in_1;
    }
    return cudaSuccess;
}

}  // namespace bingo
