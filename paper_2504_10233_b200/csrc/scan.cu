// scan.cu -- single-pass exclusive scan over u64 (decoupled look-back).
// Tiles of 2048 elements (256 threads x 8).
#include <algorithm>

#include "scan.cuh"
#include "bingo_internal.cuh"

namespace bingo {

static constexpr int SCAN_THREADS = 256;
static constexpr int SCAN_ITEMS = 8;
static constexpr uint64_t SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

size_t scan_tmp_words(uint64_t n) {
    const uint64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    return (size_t)(tiles + 2);   // look-back status per tile + the tile counter
}

__device__ __forceinline__ uint64_t block_exclusive(uint64_t v, uint64_t *total) {
    __shared__ uint64_t warp_tot[SCAN_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint64_t t = lane < SCAN_THREADS / 32 ? warp_tot[lane] : 0;
        uint64_t s = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < SCAN_THREADS / 32) warp_tot[lane] = s - t;
        if (lane == SCAN_THREADS / 32 - 1) *total = s;
    }
    __syncthreads();
    uint64_t r = x - v + warp_tot[wid];
    __syncthreads();
    return r;
}

// tile scan with optional carry-in array (per tile) ; writes total at out[n]
__global__ void k_tile_scan(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, uint64_t n,
                            const uint64_t *__restrict__ carry) {
    uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
    uint64_t v[SCAN_ITEMS];
    uint64_t acc = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        uint64_t i = base + (uint64_t)threadIdx.x * SCAN_ITEMS + j;
        v[j] = i < n ? in[i] : 0;
        acc += v[j];
    }
    __shared__ uint64_t tot;
    uint64_t pre = block_exclusive(acc, &tot) + (carry ? carry[blockIdx.x] : 0);
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        uint64_t i = base + (uint64_t)threadIdx.x * SCAN_ITEMS + j;
        if (i < n) out[i] = pre;
        pre += v[j];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == SCAN_THREADS - 1) out[n] = pre;
}

// Single-pass exclusive scan (decoupled look-back): tiles take ids from an atomic
// counter in launch order, publish their aggregate, then their inclusive prefix once
// the look-back over predecessors is resolved.  One kernel instead of three.
// Status word: bits 63..62 = flag (1 aggregate, 2 inclusive prefix), 61..0 = value
// (every scanned quantity here is < 2^62).  tmp: [tiles] status words + counter.
static constexpr uint64_t ST_A = 1ull << 62, ST_P = 2ull << 62, ST_V = (1ull << 62) - 1;

struct ScanMulti {
    const uint64_t *in[SCAN_MULTI_MAX];
    uint64_t *out[SCAN_MULTI_MAX];
};

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_lookback(const ScanMulti m, uint64_t n,
                                                                unsigned long long *status_all, unsigned *counter_all,
                                                                uint64_t tiles, const unsigned long long *pn) {
    // pn: the length is read from device memory (clamped to n, the launch's capacity);
    // tiles past it leave at once (nothing looks back at them)
    if (pn) n = min((uint64_t)*pn, n);
    // blockIdx.y selects the array; each array has its own tile counter and status words
    const uint64_t *__restrict__ in = m.in[blockIdx.y];
    uint64_t *__restrict__ out = m.out[blockIdx.y];
    unsigned long long *status = status_all + blockIdx.y * tiles;
    unsigned *counter = counter_all + 2 * blockIdx.y;
    __shared__ unsigned s_tile;
    __shared__ uint64_t s_excl, tot;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * SCAN_TILE;
    if (tile && base >= n) return;
    uint64_t v[SCAN_ITEMS];
    uint64_t acc = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        const uint64_t i = base + (uint64_t)threadIdx.x * SCAN_ITEMS + j;
        v[j] = i < n ? in[i] : 0;
        acc += v[j];
    }
    uint64_t pre = block_exclusive(acc, &tot);
    if (threadIdx.x < 32) {
        // warp 0 publishes the tile aggregate, then looks back over a window of 32
        // predecessors at once (lane l reads tile - 1 - l): the nearest inclusive prefix
        // plus the aggregates in front of it; tiles before 0 count as a prefix of 0
        const uint32_t lane = threadIdx.x;
        volatile unsigned long long *st = status;
        uint64_t excl = 0;
        if (tile == 0) {
            if (lane == 0) st[0] = ST_P | (tot & ST_V);
        } else {
            if (lane == 0) st[tile] = ST_A | (tot & ST_V);
            __threadfence();
            int64_t j0 = (int64_t)tile - 1;
            unsigned spins = 0;
            for (;;) {
                const int64_t j = j0 - (int64_t)lane;
                const unsigned long long w = j >= 0 ? st[j] : ST_P;
                const unsigned long long f = w & ~ST_V;
                const unsigned notready = __ballot_sync(0xffffffffu, f == 0);
                const unsigned isp = __ballot_sync(0xffffffffu, f == ST_P);
                const unsigned upto = isp ? ((isp & (0u - isp)) << 1) - 1u : 0xffffffffu;   // lanes 0..first P
                if (notready & upto) {   // a predecessor has not published yet (it started earlier: it will)
                    if (++spins > (1u << 26)) __trap();   // never hang the device silently
                    continue;
                }
                uint64_t x = ((upto >> lane) & 1u) ? (w & ST_V) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                excl += x;
                if (isp) break;
                j0 -= 32;
            }
            __threadfence();
            if (lane == 0) st[tile] = ST_P | ((excl + tot) & ST_V);
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    pre += s_excl;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        const uint64_t i = base + (uint64_t)threadIdx.x * SCAN_ITEMS + j;
        if (i < n) out[i] = pre;
        pre += v[j];
    }
    if (base + SCAN_TILE >= n && threadIdx.x == SCAN_THREADS - 1) out[n] = pre;   // the last tile: the total
}

static cudaError_t scan_multi(const uint64_t *const *in, uint64_t *const *out, int count, uint64_t n,
                              uint64_t *tmp, cudaStream_t s, const unsigned long long *pn) {
    if (count <= 0) return cudaSuccess;
    if (n == 0) {
        for (int a = 0; a < count; a++) {
            cudaError_t e = cudaMemsetAsync(out[a], 0, sizeof(uint64_t), s);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    const uint64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles == 1 && !pn) {
        for (int a = 0; a < count; a++) {
            k_tile_scan<<<1, SCAN_THREADS, 0, s>>>(in[a], out[a], n, nullptr);
            bingo_count_launch();
        }
        return cudaGetLastError();
    }
    ScanMulti m;
    for (int a = 0; a < count; a++) {
        m.in[a] = in[a];
        m.out[a] = out[a];
    }
    // tmp: [count][tiles] status words, then [count][2] u32 counters (one u64 each)
    unsigned long long *status = reinterpret_cast<unsigned long long *>(tmp);
    unsigned *counter = reinterpret_cast<unsigned *>(tmp + (uint64_t)count * tiles);
    cudaError_t e = cudaMemsetAsync(tmp, 0, sizeof(uint64_t) * ((uint64_t)count * tiles + count), s);
    if (e != cudaSuccess) return e;
    k_scan_lookback<<<dim3((unsigned)tiles, (unsigned)count), SCAN_THREADS, 0, s>>>(m, n, status, counter, tiles, pn);
    bingo_count_launch();
    return cudaGetLastError();
}

cudaError_t exclusive_scan_u64_multi(const uint64_t *const *in, uint64_t *const *out, int count, uint64_t n,
                                     uint64_t *tmp, cudaStream_t s) {
    return scan_multi(in, out, count, n, tmp, s, nullptr);
}

cudaError_t exclusive_scan_u64_multi_dn(const uint64_t *const *in, uint64_t *const *out, int count,
                                        const unsigned long long *pn, uint64_t nmax, uint64_t *tmp, cudaStream_t s) {
    return scan_multi(in, out, count, std::max<uint64_t>(nmax, 1), tmp, s, pn);
}

cudaError_t exclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t *tmp, cudaStream_t s) {
    return exclusive_scan_u64_multi(&in, &out, 1, n, tmp, s);
}

}  // namespace bingo
