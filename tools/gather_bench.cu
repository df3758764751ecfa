// gather_bench.cu -- the HBM random-access roofline for the walker.
// Measurement infrastructure only (not part of the Bingo method).
//
//  gb_fill       fills a buffer of 32 B slots; slot s holds a pseudo-random
//                successor index (a random functional graph) in its first word.
//  gb_independent  each thread issues `iters` independent random 32 B loads,
//                `ilp` in flight per thread (the random-sector throughput peak).
//  gb_chase      each thread follows `chains` dependent pointer chains of
//                `steps` hops (1 chain per thread = the walker's access pattern:
//                every load's address depends on the previous load).
// Every load is one full 32 B sector (two 16 B vector loads of the same
// sector), so bytes = 32 x loads.  nslots must be a power of two.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__global__ void gb_fill(uint4 *buf, uint64_t nslots, uint64_t seed) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nslots; s += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t nx = mix64(s ^ seed) & (nslots - 1);
        buf[2 * s] = make_uint4((uint32_t)nx, (uint32_t)(nx >> 32), (uint32_t)s, 0u);
        buf[2 * s + 1] = make_uint4(1u, 2u, 3u, 4u);
    }
}

template <int ILP>
__global__ void gb_independent(const uint4 *__restrict__ buf, uint64_t nslots, uint32_t iters, uint64_t seed, uint32_t *out) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; it += ILP) {
        uint4 v[ILP], w[ILP];
#pragma unroll
        for (int j = 0; j < ILP; j++) {
            const uint64_t s = mix64(tid * 0x9E3779B97F4A7C15ull + (it + j) + seed) & (nslots - 1);
            v[j] = __ldg(buf + 2 * s);
            w[j] = __ldg(buf + 2 * s + 1);
        }
#pragma unroll
        for (int j = 0; j < ILP; j++) acc ^= v[j].x ^ w[j].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int Q>
__device__ __forceinline__ uint4 ld16(const uint4 *p) {
    uint4 v;
    if (Q == 0) v = __ldg(p);
    else if (Q == 1) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (Q == 2) asm volatile("ld.global.ca.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (Q == 3) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (Q == 4) asm volatile("ld.global.nc.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else asm volatile("ld.global.nc.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// dependent chase reading only 16 B (first half of each 32 B slot) with load qualifier Q
template <int Q>
__global__ void gb_chase_q(const uint4 *__restrict__ buf, uint64_t nslots, uint32_t steps, uint64_t seed, uint32_t *out) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t cur = mix64(tid + seed) & (nslots - 1);
    uint32_t acc = 0;
    for (uint32_t it = 0; it < steps; it++) {
        const uint4 v = ld16<Q>(buf + 2 * cur);
        cur = ((uint64_t)v.y << 32) | v.x;
        acc ^= v.z;
    }
    if (acc == 0x12345678u) out[0] = (uint32_t)cur;
}

template <int CH>
__global__ void gb_chase(const uint4 *__restrict__ buf, uint64_t nslots, uint32_t steps, uint64_t seed, uint32_t *out) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t cur[CH];
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) cur[c] = mix64(tid * CH + c + seed) & (nslots - 1);
    for (uint32_t it = 0; it < steps; it++) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
            const uint4 v = __ldg(buf + 2 * cur[c]);
            const uint4 w = __ldg(buf + 2 * cur[c] + 1);
            cur[c] = ((uint64_t)v.y << 32) | v.x;
            acc ^= w.w;
        }
    }
    if (acc == 0x12345678u) out[0] = (uint32_t)cur[0];
}

extern "C" int gather_fill(void *buf, uint64_t nslots, uint64_t seed, void *stream) {
    gb_fill<<<148 * 8, 256, 0, (cudaStream_t)stream>>>((uint4 *)buf, nslots, seed);
    return (int)cudaGetLastError();
}

// mode 0: independent (ilp 8); mode 1: chase, 1 chain/thread; mode 2: chase, 2 chains/thread;
// mode 3: chase, 4 chains/thread.  Returns elapsed ms via *ms (CUDA events), loads via *loads.
extern "C" int gather_run(void *buf, uint64_t nslots, int mode, uint32_t blocks, uint32_t threads, uint32_t iters,
                          uint64_t seed, void *scratch, float *ms, double *loads, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    const uint4 *B = (const uint4 *)buf;
    uint32_t *o = (uint32_t *)scratch;
    double total = (double)blocks * threads;
    switch (mode) {
        case 0: gb_independent<8><<<blocks, threads, 0, s>>>(B, nslots, iters, seed, o); total *= iters; break;
        case 1: gb_chase<1><<<blocks, threads, 0, s>>>(B, nslots, iters, seed, o); total *= iters; break;
        case 2: gb_chase<2><<<blocks, threads, 0, s>>>(B, nslots, iters, seed, o); total *= 2.0 * iters; break;
        case 3: gb_chase<4><<<blocks, threads, 0, s>>>(B, nslots, iters, seed, o); total *= 4.0 * iters; break;
        case 10: gb_chase_q<0><<<blocks, threads, 0, s>>>(B, nslots, iters, seed, o); total *= iters; break;
        case 11: gb_chase_q<1><<<blocks, threads, 0, s>>>(B, nslots, iters, seed, o); total *= iters; break;
        case 12: gb_chase_q<2><<<blocks, threads, 0, s>>>(B, nslots, iters, seed, o); total *= iters; break;
        case 14: gb_chase_q<4><<<blocks, threads, 0, s>>>(B, nslots, iters, seed, o); total *= iters; break;
        case 15: gb_chase_q<5><<<blocks, threads, 0, s>>>(B, nslots, iters, seed, o); total *= iters; break;
        case 13: gb_chase_q<3><<<blocks, threads, 0, s>>>(B, nslots, iters, seed, o); total *= iters; break;
        default: return -1;
    }
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *loads = total;
    return (int)cudaGetLastError();
}


// TLB-reach experiment: nslots logical 32 B slots, slot s placed at 128 B line
// s * spread_lines + (hash(s) mod spread_lines) of a buffer of nslots * spread_lines
// lines.  The set of touched lines (and so the L2 footprint) is the same for every
// spread; only the number of 2 MB pages they are scattered over changes.
__device__ __forceinline__ uint64_t spread_line(uint64_t s, uint64_t spread) {
    return s * spread + (spread > 1 ? (mix64(s * 0x2545F4914F6CDD1Dull) % spread) : 0);
}
__global__ void gb_fill_spread(uint4 *buf, uint64_t nslots, uint64_t spread, uint64_t seed) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nslots; s += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t nx = mix64(s ^ seed) & (nslots - 1);
        const uint64_t ln = spread_line(nx, spread);
        const uint64_t me = spread_line(s, spread);
        buf[8 * me] = make_uint4((uint32_t)ln, (uint32_t)(ln >> 32), (uint32_t)s, 0u);
    }
}
__global__ void gb_chase_spread(const uint4 *__restrict__ buf, uint64_t nslots, uint64_t spread, uint32_t steps,
                                uint64_t seed, uint32_t *out) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t cur = spread_line(mix64(tid + seed) & (nslots - 1), spread);
    uint32_t acc = 0;
    for (uint32_t it = 0; it < steps; it++) {
        const uint4 v = __ldg(buf + 8 * cur);
        cur = ((uint64_t)v.y << 32) | v.x;
        acc ^= v.z;
    }
    if (acc == 0x12345678u) out[0] = (uint32_t)cur;
}
extern "C" int gather_spread(void *buf, uint64_t nslots, uint64_t spread, uint32_t blocks, uint32_t threads,
                             uint32_t iters, uint64_t seed, void *scratch, float *ms, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    gb_fill_spread<<<148 * 8, 256, 0, s>>>((uint4 *)buf, nslots, spread, 12345);
    gb_chase_spread<<<blocks, threads, 0, s>>>((const uint4 *)buf, nslots, spread, iters, seed + 1, (uint32_t *)scratch);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    gb_chase_spread<<<blocks, threads, 0, s>>>((const uint4 *)buf, nslots, spread, iters, seed, (uint32_t *)scratch);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return (int)cudaGetLastError();
}

// L2 fetch-granularity limit (cudaLimitMaxL2FetchGranularity): returns the value in effect.
extern "C" int gather_set_l2_fetch(int bytes) {
    if (bytes >= 0) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes);
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    return (int)v;
}
