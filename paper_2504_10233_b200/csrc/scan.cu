// scan.cu -- three-phase exclusive scan over u64 (tile reduce, scan of tile
// sums, tile scan + carry).  Tiles of 2048 elements (256 threads x 8).
#include "scan.cuh"
#include "bingo_internal.cuh"

namespace bingo {

static constexpr int SCAN_THREADS = 256;
static constexpr int SCAN_ITEMS = 8;
static constexpr uint64_t SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

size_t scan_tmp_words(uint64_t n) {
    uint64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles <= 1) return 1;
    return (size_t)(tiles + (tiles + 1)) + scan_tmp_words(tiles);
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

__global__ void k_tile_reduce(const uint64_t *__restrict__ in, uint64_t n, uint64_t *__restrict__ sums) {
    uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
    uint64_t acc = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        uint64_t i = base + (uint64_t)threadIdx.x * SCAN_ITEMS + j;
        if (i < n) acc += in[i];
    }
    __shared__ uint64_t tot;
    block_exclusive(acc, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
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

cudaError_t exclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t *tmp, cudaStream_t s) {
    if (n == 0) {
        return cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
    }
    uint64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles == 1) {
        k_tile_scan<<<1, SCAN_THREADS, 0, s>>>(in, out, n, nullptr);
        bingo_count_launch();
        return cudaGetLastError();
    }
    uint64_t *sums = tmp;               // [tiles]
    uint64_t *sums_scan = tmp + tiles + 1; // [tiles + 1]
    uint64_t *rest = sums_scan + tiles + 1;
    k_tile_reduce<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, n, sums);
    bingo_count_launch();
    cudaError_t e = exclusive_scan_u64(sums, sums_scan, tiles, rest, s);
    if (e != cudaSuccess) return e;
    k_tile_scan<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, out, n, sums_scan);
    bingo_count_launch();
    return cudaGetLastError();
}

}  // namespace bingo
