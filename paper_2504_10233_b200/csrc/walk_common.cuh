// walk_common.cuh -- the two-stage sample of Bingo (Eq.5 then Eq.6).
#pragma once
#include <cstdint>

#include "bingo_internal.cuh"
#include "build_common.cuh"
#include "nbr_index.cuh"

namespace bingo {

// walk profile counters (bingo_walk_profile): loads issued per record type
enum { PR_STEPS = 0, PR_HDR, PR_BKT, PR_MEM, PR_ARC, PR_PROBE, PR_VISIT, PR_WALKERS, BINGO_PROF_N_ };
#define BINGO_PROF_N 8

// access trace (bingo_walk_trace, measurement only): one 16 B record per accepted step,
// the loads the step made:
//   x: vertex (internal id) whose thin header was read
//   y: bucket pool index | L2 keep policy << 31
//   z: member or dense attempt 0, w: dense attempt 1 -- TR_EMPTY, or
//      kind << 31 (0 member dst, 1 arc) | keep << 30 | granule (30 bits): 16 B of the member
//      pool or the 32 B sector of the arc pool (4 arcs) -- inside the sector the walk read
#define TR_EMPTY 0xFFFFFFFFu
__device__ __forceinline__ uint32_t tr_intra(bool arc, bool keep, uint64_t elem) {
    return ((uint32_t)arc << 31) | ((uint32_t)keep << 30) | (uint32_t)((elem >> 2) & 0x3FFFFFFFu);
}

struct WalkProf {
    unsigned long long steps = 0, hdr = 0, bkt = 0, mem = 0, arc = 0, probe = 0, visit = 0, walkers = 0;
    uint4 rec = make_uint4(0u, 0u, TR_EMPTY, TR_EMPTY);   // trace mode: this step's loads
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
    const ThinHdr *thdr;
    const VHdr *hdr;
    const Bucket *bkt;
    const uint2 *arc;
    const uint32_t *mdst;
    const uint32_t *nbt;
    const uint64_t *nbo;
    const DecRec *dec;      // float mode (R-15) or null
    const uint4 *dmem;
    unsigned long long *visit;
    const uint32_t *starts;
    const uint32_t *perm, *inv;   // internal <-> external vertex ids (paths and starts are external)
    uint32_t *paths;
    uint32_t *lengths;
    uint32_t W, V, L, first_walker;
    uint32_t k0, k1;
    unsigned long long n2v_thr[3];
    uint32_t n2v_always[3];
    unsigned long long stop_thr;
    uint32_t stop_always;
    unsigned long long *prof;
    // trace mode: record of step t of walker i at trace[trace_off[i] + t]
    uint4 *trace;
    const unsigned long long *trace_off;
    // shared-memory staging (k_walk): the first sm_hdr thin headers (relabelled graphs: the
    // hottest vertices) and the first sm_bkt buckets (hot-first pool) are copied into every
    // block's shared memory at launch; 0 = off
    uint32_t sm_hdr, sm_bkt;
    unsigned int *visit32;  // BINGO_VISIT32 A/B: per-launch u32 counters (null: the u64 counters)
};

#ifndef BINGO_SMEM_HDR
#define BINGO_SMEM_HDR 0
#endif
#ifndef BINGO_SMEM_BKT
#define BINGO_SMEM_BKT 0
#endif
#if BINGO_SMEM_HDR
__shared__ unsigned long long s_thdr[BINGO_SMEM_HDR];
#endif
#if BINGO_SMEM_BKT
__shared__ uint4 s_bkt[2 * BINGO_SMEM_BKT];
#endif

#ifdef BINGO_NO_L2_64B            // A/B experiment switch: no 64 B L2 fetch hint
#define BINGO_L2F ""
#else
#define BINGO_L2F ".L2::64B"
#endif
#ifdef BINGO_L1_NOALLOC           // A/B experiment switch: one-shot random reads bypass L1 allocation
#define BINGO_L1Q ".L1::no_allocate"
#else
#define BINGO_L1Q ""
#endif

struct Policies {
    uint64_t keep, stream;   // L2 cache-hint policies (createpolicy)
};

__device__ __forceinline__ ThinHdr load_thdr(const ThinHdr *p, const Policies &pol) {
    unsigned long long v;
    asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol.keep));
    ThinHdr h;
    h.bkt_off = (uint32_t)v;
    h.n = (uint8_t)(v >> 32);
    h.flags = (uint8_t)(v >> 40);
    h.pad1 = 0;
    return h;
}

// one 256-bit read-only load of a 32 B bucket (LDG.E.256 on sm_100a), 64 B L2
// fetch, with the vertex's L2 policy (hot: evict_last, cold: evict_first)
__device__ __forceinline__ Bucket ldg_bucket(const Bucket *p, uint64_t pol) {
    uint4 lo, hi;
    asm volatile("ld.global.nc" BINGO_L1Q ".L2::cache_hint" BINGO_L2F ".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p), "l"(pol));
    return unpack_bucket(lo, hi);
}

// 4 B random read with an explicit L2 policy, 64 B fetch
__device__ __forceinline__ uint32_t ldg4(const uint32_t *p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc" BINGO_L1Q ".L2::cache_hint" BINGO_L2F ".u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

// 8 B random read with an explicit L2 policy, 64 B fetch
__device__ __forceinline__ uint2 ldg8(const uint2 *p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc" BINGO_L1Q ".L2::cache_hint" BINGO_L2F ".v2.u32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}

// Speculative dense rejection width: S attempts' draws and loads are issued at
// once and the FIRST accepted attempt in order is taken -- the same result as
// the sequential loop of P:465 (A-23), without serialising a warp on the
// slowest lane's retries (acceptance > alpha = 40%, so P(all S rejected) < 0.6^S).
// Session 3 A/B on the bench workloads (profiles/r02_dense_spec_ab.txt): 1 attempt per round
// c2 8.49 -> 8.24 ms, c4 PPR 125.4 -> 124.9 ms; 3: slower (r01, before the later walk changes,
// 2 had been the best).
#ifndef BINGO_DENSE_SPEC
#define BINGO_DENSE_SPEC 1
#endif

// One first-order sample at a vertex with n > 0 (P:215 two stages).
//  (i)  inter-group: bucket b = floor(r0 n / 2^32); the group is b if the 64-bit
//       coin R = r1r2 satisfies R < lim_b, else alias[b]  (Eq.5, alias P:191;
//       R < lim_b <=> floor(R T / 2^64) < thr_b, R-4')
//  (ii) intra-group: ONE -> its member; REGULAR/SPARSE -> member
//       floor(x c / 2^64) (Eq.6); DENSE -> rejection over the adjacency,
//       accept iff bias AND 2^k != 0, re-drawing only the index (A-23).
template <bool PROF, bool TRACE = false>
__device__ __forceinline__ uint32_t sample_dst(const WalkArgs &a, const ThinHdr &h, uint32_t w, uint32_t t,
                                               uint32_t outer, WalkProf &prof, const Policies &pol) {
    const P4 r = draw_oi(w, t, outer, 0u, 0u, a.k0, a.k1);
    const uint32_t b = __umulhi(r.x, (uint32_t)h.n);
#if BINGO_SMEM_BKT
    const uint32_t bi = h.bkt_off + b;
    const Bucket B = bi < a.sm_bkt ? unpack_bucket(s_bkt[2 * bi], s_bkt[2 * bi + 1])
                                   : ldg_bucket(a.bkt + bi, (h.flags & 1u) ? pol.keep : pol.stream);
#else
    const Bucket B = ldg_bucket(a.bkt + h.bkt_off + b, (h.flags & 1u) ? pol.keep : pol.stream);
#endif
    if (PROF) prof.bkt++;
    if (TRACE) prof.rec.y = (h.bkt_off + b) | ((uint32_t)(h.flags & 1u) << 31);
    const bool alt = join64(r.y, r.z) >= B.lim;
    const uint32_t x = alt ? B.ax : B.px;
    const uint32_t y = alt ? B.ay : B.py;
    const uint32_t kk = alt ? B.a_kk : B.kk;
    const uint32_t kind = kk >> 5;
#ifdef BINGO_EXP_NO_MEMBER   // measurement experiment only: skip the intra-group load
    if (kind != K_ONE) return y & 0xFFFFFu;
#endif
#ifdef BINGO_EXP_NO_DENSE    // measurement experiment only: skip dense rejection
    if (kind == K_DENSE) return y & 0xFFFFFu;
#endif
    if (kind == K_ONE) return y;
    // the first intra-group draw (tag 1, inner 0) is the same for list and dense
    // groups: computed once, before the branch, so a warp whose lanes hold both
    // kinds does not run it twice
#ifdef BINGO_NO_HOIST            // A/B experiment switch: the draw inside each branch
    if (kind != K_DENSE) {
        const P4 q0 = draw_oi(w, t, outer, 0u, 1u, a.k0, a.k1);
        const uint64_t j0 = __umul64hi(join64(q0.x, q0.y), (uint64_t)x);
        if (PROF) prof.mem++;
        return ldg4(a.mdst + (uint64_t)y * 4 + j0, (h.flags & 2u) ? pol.keep : pol.stream);
    }
    const P4 q0 = draw_oi(w, t, outer, 0u, 1u, a.k0, a.k1);
    const uint64_t j0 = __umul64hi(join64(q0.x, q0.y), (uint64_t)x);
#else
    const P4 q0 = draw_oi(w, t, outer, 0u, 1u, a.k0, a.k1);
    const uint64_t j0 = __umul64hi(join64(q0.x, q0.y), (uint64_t)x);
    if (kind != K_DENSE) {
        if (PROF) prof.mem++;
        if (TRACE) prof.rec.z = tr_intra(false, h.flags & 2u, (uint64_t)y * 4 + j0);
        return ldg4(a.mdst + (uint64_t)y * 4 + j0, (h.flags & 2u) ? pol.keep : pol.stream);
    }
#endif
    const uint32_t k = kk & 31u;
    const uint2 *adj = a.arc + ((uint64_t)y << 2);
    for (uint32_t base = 0;; base += BINGO_DENSE_SPEC) {
        uint2 e[BINGO_DENSE_SPEC];
#pragma unroll
        for (int s = 0; s < BINGO_DENSE_SPEC; s++) {
            uint64_t j = j0;
            if (base + s) {
                const P4 q = draw_oi(w, t, outer, base + s, 1u, a.k0, a.k1);
                j = __umul64hi(join64(q.x, q.y), (uint64_t)x);
            }
            #ifdef BINGO_ARC_STREAM          // A/B experiment switch: dense arc reads always evict_first
            e[s] = ldg8(adj + j, pol.stream);
#else
            e[s] = ldg8(adj + j, (h.flags & 2u) ? pol.keep : pol.stream);
#endif
        }
        bool done = false;
        uint32_t res = 0;
#pragma unroll
        for (int s = 0; s < BINGO_DENSE_SPEC; s++) {
            const bool acc = !done && ((e[s].y >> k) & 1u);
            if (PROF && !done) prof.arc++;
            if (TRACE && !done && base + s < 2) {   // the sequential attempts 0 and 1 (R-5)
                uint64_t j = j0;
                if (base + s) {
                    const P4 q = draw_oi(w, t, outer, base + s, 1u, a.k0, a.k1);
                    j = __umul64hi(join64(q.x, q.y), (uint64_t)x);
                }
                const uint32_t code = tr_intra(true, h.flags & 2u, ((uint64_t)y << 2) + j);
                if (base + s == 0) prof.rec.z = code;
                else prof.rec.w = code;
            }
            res = acc ? e[s].x : res;
            done = done || acc;
        }
        if (done) return res;
    }
}

__device__ __forceinline__ DecRec load_dec(const DecRec *p) {
    uint4 lo, hi;
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
    DecRec r;
    r.thrD = ((uint64_t)lo.y << 32) | lo.x;
    r.dmax = ((uint64_t)lo.w << 32) | lo.z;
    r.doff = hi.x;
    r.dcnt = hi.y;
    r.lam = (uint8_t)(hi.z & 0xff);
    r.flags = (uint8_t)((hi.z >> 8) & 0xff);
    r.pad = 0;
    r.pad2 = 0;
    return r;
}

// Float mode (R-15): the decimal group with probability thrD / 2^64 (tag 5), sampled by
// rejection (tag 4: index floor(x |D| / 2^64), accept iff floor(y Dmax / 2^64) < D_j);
// otherwise the integer two-stage sample over the radix groups of floor(w lambda).
template <bool PROF>
__device__ __forceinline__ uint32_t sample_dst_f(const WalkArgs &a, const ThinHdr &h, const DecRec &dr, uint32_t w,
                                                 uint32_t t, uint32_t outer, WalkProf &prof, const Policies &pol) {
    if (dr.thrD) {
        bool decimal = true;
        if (!(dr.flags & 2u)) {
            const P4 r = draw_oi(w, t, outer, 0u, 5u, a.k0, a.k1);
            decimal = join64(r.x, r.y) < dr.thrD;
        }
        if (decimal) {
            for (uint32_t att = 0;; att++) {
                const P4 q = draw_oi(w, t, outer, att, 4u, a.k0, a.k1);
                const uint64_t j = __umul64hi(join64(q.x, q.y), (uint64_t)dr.dcnt);
                const uint4 e = __ldg(a.dmem + dr.doff + j);
                if (PROF) prof.arc++;
                if (__umul64hi(join64(q.z, q.w), dr.dmax) < (((uint64_t)e.w << 32) | e.z)) return e.y;
            }
        }
    }
    return sample_dst<PROF>(a, h, w, t, outer, prof, pol);
}

// node2vec distance-1 test (Eq.1, A-17): does a live arc prev -> v exist?
// With the neighbour index: one hash-set probe (prev's table base/mask were
// loaded while the walker stood at prev).  Without: a scan of adj(prev).
template <bool PROF>
__device__ __forceinline__ bool probe_arc(const WalkArgs &a, uint32_t prev, uint64_t prev_nbo, uint32_t v,
                                          WalkProf &prof) {
    if (a.nbt) {
        if (PROF) prof.probe++;
        return nb_contains(a.nbt + nb_base(prev_nbo), nb_mask(prev_nbo), v);
    }
    const VHdr h = a.hdr[prev];
    if (PROF) prof.probe++;
    for (uint32_t i = 0; i < h.d; i++) {
        if (PROF && (i & 3u) == 0) prof.probe++;   // one 32 B sector per 4 arcs scanned
        if (__ldg(a.arc + h.adj_off + i).x == v) return true;
    }
    return false;
}

}  // namespace bingo
