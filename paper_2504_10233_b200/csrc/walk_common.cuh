// walk_common.cuh -- the two-stage sample of Bingo (Eq.5 then Eq.6).
#pragma once
#include <cstdint>

#include "bingo_internal.cuh"
#include "build_common.cuh"

namespace bingo {

// walk profile counters (bingo_walk_profile): loads issued per record type
enum { PR_STEPS = 0, PR_HDR, PR_BKT, PR_MEM, PR_ARC, PR_PROBE, PR_VISIT, PR_WALKERS, BINGO_PROF_N_ };
#define BINGO_PROF_N 8

struct WalkProf {
    unsigned long long steps = 0, hdr = 0, bkt = 0, mem = 0, arc = 0, probe = 0, visit = 0, walkers = 0;
    __device__ void flush(unsigned long long *out) {
        unsigned long long v[8] = {steps, hdr, bkt, mem, arc, probe, visit, walkers};
#pragma unroll
        for (int j = 0; j < 8; j++) {
            unsigned long long x = v[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31u) == 0 && x) atomicAdd(&out[j], x);
        }
    }
};

struct WalkArgs {
    const VHdr *hdr;
    const Bucket *bkt;
    const uint2 *arc;
    const uint2 *mem;
    unsigned long long *visit;
    const uint32_t *starts;
    uint32_t *paths;
    uint32_t *lengths;
    uint32_t W, V, L, first_walker;
    uint32_t k0, k1;
    unsigned long long n2v_thr[3];
    uint32_t n2v_always[3];
    unsigned long long stop_thr;
    uint32_t stop_always;
    unsigned long long *prof;
};

__device__ __forceinline__ VHdr load_hdr(const VHdr *p) {
    const uint4 *q = reinterpret_cast<const uint4 *>(p);
    const uint4 lo = __ldg(q), hi = __ldg(q + 1);
    VHdr h;
    h.T = ((uint64_t)lo.y << 32) | lo.x;
    h.adj_off = ((uint64_t)lo.w << 32) | lo.z;
    h.bkt_off = hi.x;
    h.d = hi.y;
    h.n = (uint8_t)(hi.z & 0xff);
    h.ncap = (uint8_t)((hi.z >> 8) & 0xff);
    h.pad = (uint16_t)(hi.z >> 16);
    h.adj_cap = hi.w;
    return h;
}

__device__ __forceinline__ Bucket ldg_bucket(const Bucket *p) {
    const uint4 *q = reinterpret_cast<const uint4 *>(p);
    return unpack_bucket(__ldg(q), __ldg(q + 1));
}

// One first-order sample at a vertex with d > 0 (P:215 two stages).
//  (i)  inter-group: bucket b = floor(r0 n / 2^32), coin = floor(r1r2 T / 2^64),
//       group = coin < thr[b] ? b : alias[b]                 (Eq.5, alias P:191)
//  (ii) intra-group: ONE -> its member; REGULAR/SPARSE -> member
//       floor(x c / 2^64) (Eq.6); DENSE -> rejection over the adjacency,
//       accept iff bias AND 2^k != 0, re-drawing only the index (A-23).
template <bool PROF>
__device__ __forceinline__ uint32_t sample_dst(const WalkArgs &a, const VHdr &h, uint32_t w, uint32_t t,
                                               uint32_t outer, WalkProf &prof) {
    const P4 r = philox10(w, t, outer << 16, 0u, a.k0, a.k1);
    const uint32_t b = __umulhi(r.x, (uint32_t)h.n);
    const Bucket B = ldg_bucket(a.bkt + h.bkt_off + b);
    if (PROF) prof.bkt++;
    const uint64_t coin = __umul64hi(join64(r.y, r.z), h.T);
    const bool alt = coin >= B.thr;
    const uint32_t c = alt ? B.a_c : B.c;
    const uint32_t ref = alt ? B.a_ref : B.ref;
    const uint32_t kk = alt ? B.a_kk : B.kk;
    const uint32_t kind = kk >> 5;
    if (kind == K_ONE) return ref;
    if (kind != K_DENSE) {
        const P4 q = philox10(w, t, outer << 16, 1u, a.k0, a.k1);
        const uint64_t j = __umul64hi(join64(q.x, q.y), (uint64_t)c);
        if (PROF) prof.mem++;
        return __ldg(a.mem + (uint64_t)ref * 2 + j).y;
    }
    const uint32_t k = kk & 31u;
    for (uint32_t att = 0;; att++) {
        const P4 q = philox10(w, t, (outer << 16) + att, 1u, a.k0, a.k1);
        const uint64_t j = __umul64hi(join64(q.x, q.y), (uint64_t)h.d);
        const uint2 e = __ldg(a.arc + h.adj_off + j);
        if (PROF) prof.arc++;
        if ((e.y >> k) & 1u) return e.x;
    }
}

// node2vec distance-1 test (Eq.1, A-17): does a live arc prev -> v exist?
template <bool PROF>
__device__ __forceinline__ bool probe_arc(const WalkArgs &a, uint32_t prev, uint32_t v, WalkProf &prof) {
    const VHdr h = load_hdr(a.hdr + prev);
    if (PROF) prof.probe++;
    for (uint32_t i = 0; i < h.d; i++) {
        if (PROF && (i & 3u) == 0) prof.probe++;   // one 32 B sector per 4 arcs scanned
        if (__ldg(a.arc + h.adj_off + i).x == v) return true;
    }
    return false;
}

}  // namespace bingo
