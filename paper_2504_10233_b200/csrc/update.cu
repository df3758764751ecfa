// update.cu -- batched edge insert/delete (PAPER S5.2).
//
// Pipeline for one batch of n arc records (all on `stream`):
//   k_upd_validate   record checks (EINVAL) + radix keys (src) / values (index)
//   radix sort       stable by src -> per-vertex segments in batch order
//   k_upd_heads + scan + k_upd_segments   touched-vertex segments
//   k_upd_plan       (warp per touched vertex) overflow checks and the exact
//                    pool demand of the batch -- nothing is mutated
//   -- host: one sync; EINVAL / EOVERFLOW / pool growth (NOMEM) decided here --
//   k_upd_mutate     (block per touched vertex) insert -> delete -> rebuild:
//                    (1) inserts append to the adjacency and to groups that are
//                        REGULAR/SPARSE before the batch, in batch order
//                    (2) deletes: each (u,v) takes the live instance with the
//                        smallest (epoch, position) (R-8) -- selected by an
//                        atomicMin over packed (epoch << 32 | position) keys per
//                        distinct v; then the two-phase parallel delete-and-swap
//                        (pairing R-6) on every list group and on the
//                        adjacency, and the rename of moved arcs
//                    (3) rebuild: Eq.9 reclassification, member materialisation
//                        on kind change, integer Vose alias (R-4)
//   k_upd_stats      reduce per-vertex statistics
// Untouched vertices are never read or written.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>

#include "bingo.h"
#include "bingo_internal.cuh"
#include "build_common.cuh"
#include "nbr_index.cuh"
#include "scan.cuh"
#include "sort.cuh"

using namespace bingo;

namespace bingo {

static constexpr uint32_t EMPTY_KEY = 0xFFFFFFFFu;
static constexpr uint32_t DEL_MARK = 0xFFFFFFFFu;
static constexpr int MT = 256;   // threads per block (warp-per-vertex mutate, other kernels)
static constexpr int LT = 1024;  // threads per block for large (hub) vertices

// per-touched-vertex statistics: [0] deleted, [1] missing, [2..26] transitions
static constexpr int VST = 28;

struct UpdCounters {        // device, zeroed per batch
    unsigned long long need_arc, need_bkt, need_mem, reserve_mem;
    unsigned long long scratch_words;
    unsigned long long need_hix;   // hub delete index: upper bound of new table words (BSP plan)
    unsigned long long need_gix;   // group index: upper bound of new table words (BSP plan)
    int flag;
    unsigned n_small, n_large;
    int pad;
};

// touched vertices whose post-insert adjacency or delete count exceed these go
// to the block-per-vertex kernel; the rest are handled by one warp each
// (BINGO_UPD_SMALL_L overrides the first, e.g. 0 to route everything to blocks in tests)
static constexpr uint32_t SMALL_L = 2048, SMALL_Q = 128;

__device__ __forceinline__ uint32_t hash_slot(uint32_t x, uint32_t mask) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x & mask;
}

__device__ __forceinline__ uint32_t next_pow2(uint32_t x) {
    return x <= 1 ? 1u : 1u << (32 - __clz(x - 1));
}

// ------------------------------------------------------------------ validate
// validates every record and writes it to `out` with src/dst translated to internal ids
// (hot-first relabelling; in == out is allowed)
__global__ void k_upd_validate(const uint4 *in, uint4 *out, uint64_t n, uint32_t V, const uint32_t *__restrict__ inv,
                               uint32_t *__restrict__ keys, uint32_t *__restrict__ vals, UpdCounters *cnt,
                               bool allow_zero) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 r = in[i];
        // float mode (R-16): the integer part of an inserted bias is set later and may be 0
        const bool bad = r.x > 1u || r.y >= V || r.z >= V || (r.x == 0u && r.w == 0u && !allow_zero);
        if (bad) {
            atomicOr(&cnt->flag, 1);
        } else {
            if (inv) {
                r.y = __ldg(inv + r.y);
                r.z = __ldg(inv + r.z);
            }
        }
        out[i] = r;
        keys[i] = bad ? 0u : r.y;
        vals[i] = (uint32_t)i;
    }
}

// head flags over the sorted keys
__global__ void k_upd_heads(const uint32_t *__restrict__ skeys, uint64_t n, uint64_t *__restrict__ head) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || skeys[i] != skeys[i - 1]) ? 1ull : 0ull;
}

// segments: touched vertex t covers sorted positions [seg[t], seg[t + 1])
__global__ void k_upd_segments(const uint64_t *__restrict__ head_ex, const uint32_t *__restrict__ skeys, uint64_t n,
                               uint32_t *__restrict__ seg, uint32_t *__restrict__ tv) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const bool h = (i == 0 || skeys[i] != skeys[i - 1]);
        if (h) {
            const uint64_t t = head_ex[i];
            seg[t] = (uint32_t)i;
            tv[t] = skeys[i];
        }
        if (i == n - 1) seg[head_ex[n]] = (uint32_t)n;
    }
}

// ------------------------------------------------------------------ segmentation without a sort (default)
// Touched vertices get dense ids by claiming a per-vertex slot (vslot, all EMPTY between
// batches), records are counted and placed per id, and only the order INSIDE a segment is
// then restored (batch order): short segments by one thread, long ones by a block.
// Six small launches instead of a 3-pass radix sort + heads + scan + segments.  Touched ids
// come in claim order (any order is valid: vertices are independent).
static constexpr uint32_t SEG_SHORT = 32, SEG_LONG_MAX = 8192;

// Touched ids are ranked by source-id bin (2^SEG_BSH consecutive ids; claim order inside a
// bin), so consecutive touched vertices sit on the same pages of the per-vertex arrays --
// every later phase walks them in that order (a fully unsorted order cost ~10% at c2).
static constexpr uint32_t SEG_BSH = 11;

// validate (as k_upd_validate) + claim: the first record of each source owns its vertex and
// takes a rank inside the vertex's bin
__global__ void k_seg_claim(const uint4 *in, uint4 *out, uint64_t n, uint32_t V, const uint32_t *__restrict__ inv,
                            uint32_t *vslot, uint32_t *__restrict__ key, uint32_t *__restrict__ otix,
                            unsigned long long *bcnt, uint32_t *nlong, UpdCounters *cnt, bool allow_zero) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *nlong = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 r = in[i];
        const bool bad = r.x > 1u || r.y >= V || r.z >= V || (r.x == 0u && r.w == 0u && !allow_zero);
        if (bad) {
            atomicOr(&cnt->flag, 1);
        } else if (inv) {
            r.y = __ldg(inv + r.y);
            r.z = __ldg(inv + r.z);
        }
        out[i] = r;
        const uint32_t k = bad ? 0u : r.y;   // an invalid batch is rejected whole; its records go to vertex 0
        key[i] = k;
        const bool own = atomicCAS(&vslot[k], EMPTY_KEY, (uint32_t)i) == EMPTY_KEY;
        otix[i] = own ? (uint32_t)atomicAdd(&bcnt[k >> SEG_BSH], 1ull) : EMPTY_KEY;
    }
}

// touched id t = bin offset + rank in bin; per-id record counts
__global__ void k_seg_count(uint64_t n, const uint32_t *__restrict__ key, uint32_t *__restrict__ otix,
                            const uint32_t *__restrict__ vslot, const uint64_t *__restrict__ boff,
                            uint32_t *__restrict__ kt, uint32_t *__restrict__ tv, unsigned long long *cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = key[i];
        const uint32_t o = vslot[k];
        const uint32_t t = (uint32_t)boff[k >> SEG_BSH] + otix[o];
        kt[i] = t;
        if (o == (uint32_t)i) tv[t] = k;
        atomicAdd(&cnt[t], 1ull);
    }
}

// places every record in its segment (any order), releases the vertex slots
__global__ void k_seg_place(uint64_t n, const uint32_t *__restrict__ key, const uint32_t *__restrict__ otix,
                            const uint32_t *__restrict__ kt, unsigned long long *cnt, const uint64_t *__restrict__ off,
                            uint32_t *__restrict__ sv, uint32_t *__restrict__ seg, uint32_t *vslot,
                            const unsigned long long *pnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = kt[i];
        const unsigned long long r = atomicAdd(&cnt[t], ~0ull);   // old count: ranks n_t - 1 .. 0
        sv[off[t] + r - 1] = (uint32_t)i;
        if (otix[i] != EMPTY_KEY) {
            seg[t] = (uint32_t)off[t];
            vslot[key[i]] = EMPTY_KEY;
        }
        if (i == 0) seg[*pnt] = (uint32_t)n;
    }
}

// batch order inside each segment: one segment per lane; two records by the lane itself,
// up to 32 by the warp together (a shuffle sort per segment), longer ones are listed for
// k_seg_order_long
__global__ void k_seg_order(const uint32_t *__restrict__ seg, uint32_t *__restrict__ sv, const unsigned long long *pnt,
                            uint32_t *__restrict__ longs, uint32_t *nlong) {
    const uint32_t nt = (uint32_t)*pnt;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t ntr = (nt + 31u) & ~31u;   // whole warps (the shuffle sorts)
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ntr; t += gridDim.x * blockDim.x) {
        uint32_t b = 0, len = 0;
        if (t < nt) {
            b = seg[t];
            len = seg[t + 1] - b;
        }
        if (len == 2) {
            const uint32_t x = sv[b], y = sv[b + 1];
            if (x > y) {
                sv[b] = y;
                sv[b + 1] = x;
            }
        } else if (len > SEG_SHORT) {
            longs[atomicAdd(nlong, 1u)] = t;
        }
        uint32_t m = __ballot_sync(0xffffffffu, len > 2 && len <= SEG_SHORT);
        while (m) {
            const int l = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t bb = __shfl_sync(0xffffffffu, b, l), ll = __shfl_sync(0xffffffffu, len, l);
            uint32_t x = lane < ll ? sv[bb + lane] : 0xFFFFFFFFu;
#pragma unroll
            for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
                for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
                    const bool up = (lane & k) == 0, lower = (lane & j) == 0;
                    x = (lower == up) ? min(x, y) : max(x, y);
                }
            }
            if (lane < ll) sv[bb + lane] = x;
        }
    }
}

// one block per long segment: bitonic sort of its record indices in shared memory; a segment
// above SEG_LONG_MAX records sets flag 8 and the batch is re-segmented by the radix sort
__global__ void __launch_bounds__(1024) k_seg_order_long(const uint32_t *__restrict__ seg, uint32_t *__restrict__ sv,
                                                         const uint32_t *__restrict__ longs, const uint32_t *nlong,
                                                         UpdCounters *cnt) {
    __shared__ uint32_t x[SEG_LONG_MAX];
    const uint32_t nl = *nlong;
    for (uint32_t j = blockIdx.x; j < nl; j += gridDim.x) {
        const uint32_t t = longs[j];
        const uint32_t b = seg[t], len = seg[t + 1] - b;
        if (len > SEG_LONG_MAX) {
            if (threadIdx.x == 0) atomicOr(&cnt->flag, 8);
            continue;
        }
        const uint32_t P = next_pow2(len);
        for (uint32_t q = threadIdx.x; q < P; q += blockDim.x) x[q] = q < len ? sv[b + q] : 0xFFFFFFFFu;
        __syncthreads();
        for (uint32_t k = 2; k <= P; k <<= 1) {
            for (uint32_t h = k >> 1; h > 0; h >>= 1) {
                for (uint32_t q = threadIdx.x; q < P; q += blockDim.x) {
                    const uint32_t r = q ^ h;
                    if (r > q) {
                        const uint32_t u = x[q], v = x[r];
                        if ((u > v) == ((q & k) == 0)) {
                            x[q] = v;
                            x[r] = u;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (uint32_t q = threadIdx.x; q < len; q += blockDim.x) sv[b + q] = x[q];
        __syncthreads();
    }
}

// ------------------------------------------------------------------ per-vertex pre-batch view
struct OldGroups {
    uint32_t mask;      // nonempty groups (bit k)
    uint32_t list_mask; // REGULAR/SPARSE groups
};

// lane b < n loads bucket b; returns (kind, c, ref, aux) of lane k's group in lane k
// (ref: REGULAR/SPARSE member offset; aux: member capacity or the ONE arc index)
__device__ __forceinline__ void load_old_groups(const Bucket *bkt, const GCan *gcan, const VHdr &h, uint32_t &kind_k,
                                                uint32_t &c_k, uint32_t &ref_k, uint32_t &aux_k, OldGroups &og) {
    const uint32_t lane = lane_id();
    uint32_t k_b = 0, kind_b = K_EMPTY, c_b = 0, ref_b = 0, aux_b = 0;
    if (lane < h.n) {
        const Bucket B = load_bucket(bkt + h.bkt_off + lane);
        const GCan G = load_gcan(gcan + h.bkt_off + lane);
        k_b = kk_k(B.kk);
        kind_b = kk_kind(B.kk);
        c_b = G.c;
        ref_b = B.py;
        aux_b = G.aux;
    }
    const uint32_t m = __reduce_or_sync(0xffffffffu, lane < h.n ? (1u << k_b) : 0u);
    og.mask = m;
    og.list_mask = __reduce_or_sync(0xffffffffu, (lane < h.n && is_list(kind_b)) ? (1u << k_b) : 0u);
    // lane k pulls from lane b = rank of k in mask
    const uint32_t b = __popc(m & ((1u << lane) - 1u));
    const bool has = (m >> lane) & 1u;
    const uint32_t src = has ? b : 0u;
    const uint32_t kd = __shfl_sync(0xffffffffu, kind_b, src);
    const uint32_t cc = __shfl_sync(0xffffffffu, c_b, src);
    const uint32_t rf = __shfl_sync(0xffffffffu, ref_b, src);
    const uint32_t ax = __shfl_sync(0xffffffffu, aux_b, src);
    kind_k = has ? kd : K_EMPTY;
    c_k = has ? cc : 0u;
    ref_k = has ? rf : 0u;
    aux_k = has ? ax : 0u;
}

// ------------------------------------------------------------------ plan (no mutation)
// Per touched vertex (one warp): overflow check (R-10) and the exact pool demand
// of the batch -- relocations are exact, kind transitions a tight upper bound.
struct PlanOut {
    bool overflow;
    uint32_t L, q;
    unsigned long long arc, bkt, mem, res, words;
};
// per-lane (lane = radix bit k) pre-batch view of group k, for the bulk-synchronous path
struct PlanLane {
    uint32_t kind, c, ref, aux, insk, list0;
};

__device__ __forceinline__ PlanOut plan_vertex(const uint4 *__restrict__ recs, const uint32_t *__restrict__ sval,
                                               uint32_t beg, uint32_t end, const VHdr &h,
                                               const Bucket *__restrict__ bkt, const GCan *__restrict__ gcan,
                                               uint32_t alpha, bool bs, double arc_slack, double mem_slack,
                                               PlanLane *pl = nullptr) {
    const uint32_t lane = lane_id();
    uint32_t kind_k, c_k, ref_k, aux_k;
    OldGroups og;
    load_old_groups(bkt, gcan, h, kind_k, c_k, ref_k, aux_k, og);
    uint32_t m = 0, q = 0, ins_or = 0, insk = 0;
    uint64_t ins_sum = 0;
    for (uint32_t base = beg; base < end; base += 32) {
        const uint32_t p = base + lane;
        uint4 r = make_uint4(2u, 0u, 0u, 0u);
        if (p < end) r = recs[sval[p]];
        const bool ins = r.x == 0u, del = r.x == 1u;
        const uint32_t w = ins ? r.w : 0u;
        m += __popc(__ballot_sync(0xffffffffu, ins));
        q += __popc(__ballot_sync(0xffffffffu, del));
        ins_or |= w;
        ins_sum += w;
        uint32_t mk = __reduce_or_sync(0xffffffffu, w);
        while (mk) {
            const int k = __ffs(mk) - 1;
            mk &= mk - 1;
            const uint32_t bal = __ballot_sync(0xffffffffu, (w >> k) & 1u);
            if (lane == (uint32_t)k) insk += __popc(bal);
        }
    }
    ins_or = __reduce_or_sync(0xffffffffu, ins_or);
    ins_sum = warp_sum(ins_sum);
    PlanOut o;
    // overflow: (T + inserted) * popc(mask | inserted) < 2^64 and d + m < 2^32 - 1 (R-10)
    const uint32_t nb = __popc(og.mask | ins_or);
    const uint64_t Tn = h.T + ins_sum;
    o.overflow = Tn < h.T || __umul64hi(Tn, (uint64_t)nb) != 0 || (uint64_t)h.d + m >= 0xFFFFFFFFull;
    const uint32_t L = h.d + m;
    uint64_t need_mem = 0, reserve = 0;
    const uint32_t cin = c_k + insk;
    if (is_list(kind_k)) {
        if (cin > aux_k) need_mem = member_units(cin, mem_slack);
    } else if (bs) {
        if (cin >= 1 && kind_k == K_EMPTY) reserve = member_units(cin, mem_slack);
    } else if (kind_k == K_EMPTY) {
        if (insk >= 2) reserve = member_units(cin, mem_slack);
    } else if (kind_k == K_ONE) {
        if (insk >= 1) reserve = member_units(cin, mem_slack);
    } else if (kind_k == K_DENSE) {
        const uint32_t cmin = c_k > q ? c_k - q : 0u;
        if ((uint64_t)100 * cmin <= (uint64_t)alpha * L) reserve = member_units(cin, mem_slack);
    }
    o.mem = warp_sum(need_mem);
    o.res = warp_sum(reserve);
    o.arc = L > h.adj_cap ? arc_capacity(L, arc_slack) : 0;
    o.bkt = nb > h.ncap ? bucket_capacity(nb) : 0;
    uint64_t words = 0;
    if (q) {
        const uint64_t Hq = next_pow2(2 * q);
        words = (uint64_t)(L + 31) / 32 + 8 * Hq + 3ull * q + 8;
        words = (words + 7) & ~7ull;
    }
    o.words = words;
    o.L = L;
    o.q = q;
    if (pl) {
        pl->kind = kind_k;
        pl->c = c_k;
        pl->ref = ref_k;
        pl->aux = aux_k;
        pl->insk = insk;
        pl->list0 = og.list_mask;
    }
    return o;
}

__global__ void k_upd_plan(const uint4 *__restrict__ recs, const uint32_t *__restrict__ sval,
                           const uint32_t *__restrict__ seg, const uint32_t *__restrict__ tv, uint32_t ntouch,
                           const VHdr *__restrict__ hdr, const Bucket *__restrict__ bkt,
                           const GCan *__restrict__ gcan, uint32_t alpha, bool bs,
                           double arc_slack, double mem_slack, uint64_t *__restrict__ scr_need, UpdCounters *cnt,
                           uint8_t *__restrict__ route, uint32_t *__restrict__ large_list, uint32_t small_L) {
    // demand counters are aggregated per block in shared memory (one global atomic per
    // block and counter instead of one per touched vertex)
    __shared__ unsigned long long b_arc, b_bkt, b_mem, b_res;
    __shared__ int b_flag;
    if (threadIdx.x == 0) { b_arc = b_bkt = b_mem = b_res = 0; b_flag = 0; }
    __syncthreads();
    const uint32_t lane = lane_id();
    const uint32_t warps = (blockDim.x >> 5) * gridDim.x;
    for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntouch; t += warps) {
        const VHdr h = hdr[tv[t]];
        const PlanOut o = plan_vertex(recs, sval, seg[t], seg[t + 1], h, bkt, gcan, alpha, bs, arc_slack, mem_slack);
        if (lane == 0) {
            if (o.overflow) atomicOr(&b_flag, 4);
            if (o.arc) atomicAdd(&b_arc, o.arc);
            if (o.bkt) atomicAdd(&b_bkt, o.bkt);
            if (o.mem) atomicAdd(&b_mem, o.mem);
            if (o.res) atomicAdd(&b_res, o.res);
            scr_need[t] = o.words;
            const bool large = !(o.L <= small_L && o.q <= SMALL_Q);
            route[t] = large ? 1 : 0;
            if (large) large_list[atomicAdd(&cnt->n_large, 1u)] = t;   // hubs: few, so little contention
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (b_arc) atomicAdd(&cnt->need_arc, b_arc);
        if (b_bkt) atomicAdd(&cnt->need_bkt, b_bkt);
        if (b_mem) atomicAdd(&cnt->need_mem, b_mem);
        if (b_res) atomicAdd(&cnt->reserve_mem, b_res);
        if (b_flag) atomicOr(&cnt->flag, b_flag);
    }
}

// ------------------------------------------------------------------ block helpers
// block-wide exclusive scan of one u32 per thread; returns prefix, *total via smem
template <int NT>
__device__ __forceinline__ uint32_t block_scan_u32(uint32_t v, uint32_t *s_tmp /*[NT/32+1]*/, uint32_t &total) {
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) s_tmp[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int w = 0; w < NT / 32; w++) {
            const uint32_t t = s_tmp[w];
            s_tmp[w] = acc;
            acc += t;
        }
        s_tmp[NT / 32] = acc;
    }
    __syncthreads();
    const uint32_t r = x - v + s_tmp[wid];
    total = s_tmp[NT / 32];
    __syncthreads();
    return r;
}

__device__ __forceinline__ bool bit_test(const uint32_t *bm, uint32_t p) { return (bm[p >> 5] >> (p & 31u)) & 1u; }

// ------------------------------------------------------------------ mutate (block per touched vertex)
struct MutateArgs {
    const uint4 *recs;
    const uint32_t *sval;
    const uint32_t *seg;
    const uint32_t *tv;
    const uint64_t *scr_off;
    uint32_t *scr;
    VHdr *hdr;
    ThinHdr *thdr;
    uint2 *arc;
    uint32_t *arc_epoch;
    uint64_t *arc_dval;         // float mode: D per arc, moves with the arc (R-16); else null
    const uint64_t *dins;       // float mode: D of each record (batch order); else null
    Bucket *bkt;
    GCan *gcan;
    uint32_t *mdst, *midx;
    uint32_t *nbt;
    uint64_t *nbo;
    uint32_t *nbtomb;
    uint64_t *hixo;             // hub delete index offsets: routes that do not maintain it invalidate
    uint32_t *hixt, *hix;       // its tombstone counts and table pool (BSP route)
    uint32_t hix_min;           // vertices with more arcs get (and may lazily rebuild) a table
    unsigned long long hix_cap; // hub index pool words (bump pointer bump[5])
    uint64_t *gixo;             // group index (group_index.cuh): per-vertex table offsets, null = off
    uint32_t *gixt, *gix;       // its tombstone counts and table pool
    uint32_t gix_min;           // vertices with more arcs may get a table
    unsigned long long gix_cap; // pool words (bump pointer bump[6])
    unsigned long long *bump;   // [0] arc, [1] bkt, [2] mem units, [5] hub index, [6] group index
    uint32_t *vstats;           // [ntouch][VST]
    uint32_t epoch, alpha, beta, hot_b, hot_m;
    bool bs;
    double arc_slack, mem_slack;
};

struct MutSmem {
    uint32_t kind0[32], c[32], insk[32], delk[32], moff[32], cap[32], one[32], kind1[32];
    uint32_t tmp[LT / 32 + 1];
    uint32_t list0, m, q, N, missing, fill_mask, find_mask, adj_cap;
    uint64_t adj_off;
};

template <int GT>
struct Grp;
template <>
struct Grp<32> {
    static __device__ __forceinline__ uint32_t rank() { return threadIdx.x & 31u; }
    static __device__ __forceinline__ void sync() { __syncwarp(); }
    static __device__ __forceinline__ bool any(bool p) { return __any_sync(0xffffffffu, p); }
    static __device__ __forceinline__ uint32_t scan(uint32_t v, uint32_t *, uint32_t &total) {
        const uint32_t lane = threadIdx.x & 31u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        total = __shfl_sync(0xffffffffu, x, 31);
        return x - v;
    }
};
template <>
struct Grp<LT> {
    static __device__ __forceinline__ uint32_t rank() { return threadIdx.x; }
    static __device__ __forceinline__ void sync() { __syncthreads(); }
    static __device__ __forceinline__ bool any(bool p) { return __syncthreads_or(p) != 0; }
    static __device__ __forceinline__ uint32_t scan(uint32_t v, uint32_t *tmp, uint32_t &total) {
        return block_scan_u32<LT>(v, tmp, total);
    }
};

// Per-vertex insert -> delete -> rebuild, executed by a group of GT threads:
// one warp (GT = 32, small vertices, 8 per block) or a whole block (GT = MT,
// large vertices).  Lanes 0..31 of the group own radix bit k = lane.
template <int GT>
__device__ __forceinline__ void mutate_vertex(const MutateArgs &a, const uint32_t t, MutSmem &sm,
                                              uint32_t *local_scr = nullptr, uint32_t local_words = 0) {
    using G = Grp<GT>;
    const uint32_t tid = G::rank(), lane = tid & 31u, wid = tid >> 5;
    uint32_t *s_kind0 = sm.kind0, *s_c = sm.c, *s_insk = sm.insk, *s_delk = sm.delk, *s_moff = sm.moff,
             *s_cap = sm.cap, *s_one = sm.one, *s_kind1 = sm.kind1, *s_tmp = sm.tmp;
    uint32_t &s_list0 = sm.list0, &s_m = sm.m, &s_q = sm.q, &s_N = sm.N, &s_missing = sm.missing;
    uint32_t &s_fill_mask = sm.fill_mask, &s_find_mask = sm.find_mask, &s_adj_cap = sm.adj_cap;
    uint64_t &s_adj_off = sm.adj_off;
    G::sync();   // the group's shared slot may still be read by its previous vertex

    const uint32_t u = a.tv[t];
    const uint32_t beg = a.seg[t], end = a.seg[t + 1];
    const VHdr h = a.hdr[u];

    // ---------------- phase 0: pre-batch groups, relocations
    if (wid == 0) {
        uint32_t kind_k, c_k, ref_k, aux_k;
        OldGroups og;
        load_old_groups(a.bkt, a.gcan, h, kind_k, c_k, ref_k, aux_k, og);
        // insert counts per bit for capacity decisions
        uint32_t m = 0, q = 0, insk = 0;
        for (uint32_t base = beg; base < end; base += 32) {
            const uint32_t p = base + lane;
            uint4 r = make_uint4(2u, 0u, 0u, 0u);
            if (p < end) r = a.recs[a.sval[p]];
            const uint32_t w = r.x == 0u ? r.w : 0u;
            m += __popc(__ballot_sync(0xffffffffu, r.x == 0u));
            q += __popc(__ballot_sync(0xffffffffu, r.x == 1u));
            uint32_t mk = __reduce_or_sync(0xffffffffu, w);
            while (mk) {
                const int k = __ffs(mk) - 1;
                mk &= mk - 1;
                const uint32_t bal = __ballot_sync(0xffffffffu, (w >> k) & 1u);
                if (lane == (uint32_t)k) insk += __popc(bal);
            }
        }
        s_kind0[lane] = kind_k;
        s_c[lane] = c_k;
        s_insk[lane] = 0;      // filled by the insert phase
        s_delk[lane] = 0;
        s_one[lane] = (kind_k == K_ONE) ? aux_k : 0xFFFFFFFFu;
        uint32_t moff = ref_k, cap = aux_k;
        const uint32_t cin = c_k + insk;
        bool grow = is_list(kind_k) && cin > cap;
        if (grow) {
            const uint32_t units = member_units(cin, a.mem_slack);
            moff = (uint32_t)atomicAdd(&a.bump[2], (unsigned long long)units);
            cap = units * 4;
        }
        s_moff[lane] = is_list(kind_k) ? moff : 0u;
        s_cap[lane] = is_list(kind_k) ? cap : 0u;
        if (lane == 0) {
            s_list0 = og.list_mask;
            s_m = m;
            s_q = q;
            s_N = 0;
            s_missing = 0;
            const uint32_t L = h.d + m;
            if (L > h.adj_cap) {
                const uint64_t cap2 = arc_capacity(L, a.arc_slack);
                s_adj_off = atomicAdd(&a.bump[0], (unsigned long long)cap2);
                s_adj_cap = (uint32_t)cap2;
            } else {
                s_adj_off = h.adj_off;
                s_adj_cap = h.adj_cap;
            }
        }
        // copy growing member arrays (warp-cooperative, one group at a time)
        uint32_t gm = __ballot_sync(0xffffffffu, grow);
        while (gm) {
            const int k = __ffs(gm) - 1;
            gm &= gm - 1;
            const uint32_t from = __shfl_sync(0xffffffffu, ref_k, k);
            const uint32_t to = __shfl_sync(0xffffffffu, moff, k);
            const uint32_t cnt = __shfl_sync(0xffffffffu, c_k, k);
            for (uint32_t j = lane; j < cnt; j += 32) {
                a.mdst[(uint64_t)to * 4 + j] = a.mdst[(uint64_t)from * 4 + j];
                a.midx[(uint64_t)to * 4 + j] = a.midx[(uint64_t)from * 4 + j];
            }
        }
    }
    G::sync();
    const uint64_t aoff = s_adj_off;
    const uint32_t m = s_m, q = s_q;
    const uint32_t L = h.d + m;
    if (aoff != h.adj_off) {
        for (uint32_t i = tid; i < h.d; i += GT) {
            a.arc[aoff + i] = a.arc[h.adj_off + i];
            a.arc_epoch[aoff + i] = a.arc_epoch[h.adj_off + i];
            if (a.arc_dval) a.arc_dval[aoff + i] = a.arc_dval[h.adj_off + i];
        }
    }
    G::sync();

    // ---------------- phase 1: inserts, batch order
    if (wid == 0 && m) {
        uint32_t run = 0;          // inserts so far
        uint32_t insk = 0;         // lane k: inserts with bit k so far
        const uint32_t kind_l = s_kind0[lane];
        const uint32_t c_l = s_c[lane];
        const uint32_t moff_l = s_moff[lane];
        for (uint32_t base = beg; base < end; base += 32) {
            const uint32_t p = base + lane;
            uint4 r = make_uint4(2u, 0u, 0u, 0u);
            if (p < end) r = a.recs[a.sval[p]];
            const bool ins = r.x == 0u;
            const uint32_t bal_i = __ballot_sync(0xffffffffu, ins);
            const uint32_t idx = h.d + run + __popc(bal_i & lanemask_lt());
            const uint32_t w = ins ? r.w : 0u;
            if (ins) {
                a.arc[aoff + idx] = make_uint2(r.z, r.w);
                a.arc_epoch[aoff + idx] = a.epoch;
                if (a.arc_dval) a.arc_dval[aoff + idx] = a.dins[a.sval[p]];
            }
            uint32_t mk = __reduce_or_sync(0xffffffffu, w);
            while (mk) {
                const int k = __ffs(mk) - 1;
                mk &= mk - 1;
                const uint32_t bal = __ballot_sync(0xffffffffu, (w >> k) & 1u);
                const uint32_t kind_kk = __shfl_sync(0xffffffffu, kind_l, k);
                const uint32_t start = __shfl_sync(0xffffffffu, c_l + insk, k);
                const uint32_t mo = __shfl_sync(0xffffffffu, moff_l, k);
                if (is_list(kind_kk) && ((w >> k) & 1u)) {
                    const uint64_t e = (uint64_t)mo * 4 + start + __popc(bal & lanemask_lt());
                    a.mdst[e] = r.z;
                    a.midx[e] = idx;
                }
                if (lane == (uint32_t)k) insk += __popc(bal);
            }
            run += __popc(bal_i);
        }
        s_insk[lane] = insk;
    }
    G::sync();

    // ---------------- phase 2: deletes
    uint32_t N = 0;
    uint32_t Lp = L;
    uint32_t *bm = nullptr, *holes = nullptr, *R = nullptr, *gh = nullptr;
    if (q) {
        // delete scratch: the caller's shared-memory slice when it fits, else global
        const uint64_t so = a.scr_off[t], words = a.scr_off[t + 1] - so;
        uint32_t *scr = (local_scr && words <= local_words) ? local_scr : a.scr + so;
        const uint32_t Hq = next_pow2(2 * q), hmask = Hq - 1;
        const uint32_t bw = (L + 31) / 32;
        bm = scr;
        uint32_t *hkey = bm + bw;
        uint32_t *hk = hkey + Hq;
        uint32_t *hfound = hk + Hq;
        uint32_t *hsel = hfound + Hq;
        unsigned long long *hbest = reinterpret_cast<unsigned long long *>(
            (reinterpret_cast<uintptr_t>(hsel + Hq) + 7) & ~(uintptr_t)7);
        unsigned long long *hprev = hbest + Hq;
        holes = reinterpret_cast<uint32_t *>(hprev + Hq);
        R = holes + q;
        gh = R + q;
        for (uint32_t i = tid; i < bw; i += GT) bm[i] = 0;
        for (uint32_t i = tid; i < Hq; i += GT) {
            hkey[i] = EMPTY_KEY;
            hk[i] = 0;
            hfound[i] = 0;
            hsel[i] = 0;
            hbest[i] = ~0ull;
            hprev[i] = 0;
        }
        G::sync();
        // distinct deleted destinations with multiplicity
        for (uint32_t p = beg + tid; p < end; p += GT) {
            const uint4 r = a.recs[a.sval[p]];
            if (r.x != 1u) continue;
            uint32_t s = hash_slot(r.z, hmask);
            for (;;) {
                const uint32_t old = atomicCAS(&hkey[s], EMPTY_KEY, r.z);
                if (old == EMPTY_KEY || old == r.z) {
                    atomicAdd(&hk[s], 1u);
                    break;
                }
                s = (s + 1) & hmask;
            }
        }
        G::sync();
        // selection rounds: round r picks, per distinct v still owed a delete, the
        // live instance with the smallest (epoch, position) key above the last pick
        for (uint32_t round = 0;; round++) {
#pragma unroll 4
            for (uint32_t p = tid; p < L; p += GT) {
                const uint32_t x = __ldg(&a.arc[aoff + p].x);
                uint32_t s = hash_slot(x, hmask);
                uint32_t hit = EMPTY_KEY;
                for (;;) {
                    const uint32_t kx = hkey[s];
                    if (kx == x) { hit = s; break; }
                    if (kx == EMPTY_KEY) break;
                    s = (s + 1) & hmask;
                }
                if (hit == EMPTY_KEY) continue;
                const unsigned long long key = ((unsigned long long)a.arc_epoch[aoff + p] << 32) | p;
                if (round == 0) {
                    atomicAdd(&hfound[hit], 1u);
                    atomicMin(&hbest[hit], key);
                } else if (hsel[hit] < hk[hit] && key > hprev[hit]) {
                    atomicMin(&hbest[hit], key);
                }
            }
            G::sync();
            uint32_t more = 0;
            for (uint32_t s = tid; s < Hq; s += GT) {
                if (hkey[s] == EMPTY_KEY || hsel[s] >= hk[s]) continue;
                const unsigned long long b = hbest[s];
                if (b == ~0ull) continue;
                const uint32_t p = (uint32_t)b;
                atomicOr(&bm[p >> 5], 1u << (p & 31u));
                hsel[s]++;
                hprev[s] = b;
                hbest[s] = ~0ull;
                atomicAdd(&s_N, 1u);
                uint32_t w = a.arc[aoff + p].y;
                while (w) {
                    const int k = __ffs(w) - 1;
                    w &= w - 1;
                    atomicAdd(&s_delk[k], 1u);
                }
                if (hsel[s] < hk[s] && hsel[s] < hfound[s]) more = 1;
            }
            if (!G::any(more != 0)) break;
        }
        for (uint32_t s = tid; s < Hq; s += GT)
            if (hkey[s] != EMPTY_KEY) atomicAdd(&s_missing, hk[s] - hsel[s]);
        G::sync();
        N = s_N;
        Lp = L - N;
        if (N) {
            // holes = marked positions < L' ascending (rank by block scan over bitmap words)
            const uint32_t wl = (Lp + 31) / 32;
            uint32_t carry = 0;
            for (uint32_t w0 = 0; w0 < wl; w0 += GT) {
                const uint32_t w = w0 + tid;
                uint32_t word = 0;
                if (w < wl) {
                    word = bm[w];
                    const uint32_t lim = Lp - w * 32;
                    if (lim < 32) word &= (1u << lim) - 1u;
                }
                uint32_t tot;
                const uint32_t pre = G::scan(__popc(word), s_tmp, tot);
                uint32_t r = carry + pre;
                while (word) {
                    const int b = __ffs(word) - 1;
                    word &= word - 1;
                    holes[r++] = w * 32 + b;
                }
                carry += tot;
            }
            G::sync();
            // adjacency tail window [L', L): survivors fill holes in rank order
            uint32_t scarry = 0;
            for (uint32_t t0 = Lp; t0 < L; t0 += GT) {
                const uint32_t tt = t0 + tid;
                const bool in = tt < L;
                const bool surv = in && !bit_test(bm, tt);
                uint32_t tot;
                const uint32_t rank = scarry + G::scan(surv ? 1u : 0u, s_tmp, tot);
                if (in) {
                    if (surv) {
                        const uint32_t dstp = holes[rank];
                        a.arc[aoff + dstp] = a.arc[aoff + tt];
                        a.arc_epoch[aoff + dstp] = a.arc_epoch[aoff + tt];
                        if (a.arc_dval) a.arc_dval[aoff + dstp] = a.arc_dval[aoff + tt];
                        R[tt - Lp] = dstp;
                    } else {
                        R[tt - Lp] = DEL_MARK;
                    }
                }
                scarry += tot;
            }
            G::sync();
        }
    }
    // ---------------- groups: delete-and-swap, rename (lists that existed before the batch)
    if (N) {
        uint32_t lm = s_list0;
        while (lm) {
            const int k = __ffs(lm) - 1;
            lm &= lm - 1;
            const uint32_t cp = s_c[k] + s_insk[k];
            const uint32_t Nk = s_delk[k];
            uint32_t *Md = a.mdst + (uint64_t)s_moff[k] * 4;
            uint32_t *Mi = a.midx + (uint64_t)s_moff[k] * 4;
            const uint32_t Lk = cp - Nk;
            // pass 1 over the front [0, L_k'): deleted slots become holes (ranked in slot
            // order); surviving entries that point into the adjacency tail are renamed
            // in place.  pass 2 over the tail window [L_k', c'): survivors, renamed,
            // fill the holes in rank order (R-6).
            uint32_t carry = 0;
            for (uint32_t s0 = 0; s0 < Lk; s0 += GT) {
                const uint32_t s = s0 + tid;
                bool del = false;
                if (s < Lk) {
                    const uint32_t x = Mi[s];
                    del = bit_test(bm, x);
                    if (!del && x >= Lp) Mi[s] = R[x - Lp];
                }
                uint32_t tot = 0;
                const uint32_t rank = Nk ? carry + G::scan(del ? 1u : 0u, s_tmp, tot) : 0u;
                if (del) gh[rank] = s;
                carry += tot;
            }
            G::sync();
            uint32_t scarry = 0;
            for (uint32_t s0 = Lk; s0 < cp; s0 += GT) {
                const uint32_t s = s0 + tid;
                uint32_t x = 0;
                const bool surv = s < cp && !bit_test(bm, (x = Mi[s]));
                uint32_t tot;
                const uint32_t rank = scarry + G::scan(surv ? 1u : 0u, s_tmp, tot);
                if (surv) {
                    Md[gh[rank]] = Md[s];
                    Mi[gh[rank]] = x >= Lp ? R[x - Lp] : x;
                }
                scarry += tot;
            }
            G::sync();
        }
    }
    // ---------------- phase 3: rebuild
    const uint32_t dn = Lp;
    if (wid == 0) {
        const uint32_t k = lane;
        const uint32_t kind0 = s_kind0[k];
        const uint32_t cn = s_c[k] + s_insk[k] - s_delk[k];
        const uint32_t kind1 = classify(cn, dn, a.alpha, a.beta, a.bs);
        s_kind1[k] = kind1;
        s_c[k] = cn;
        bool fill = false, find = false;
        uint32_t one = 0xFFFFFFFFu;
        if (is_list(kind1) && !is_list(kind0)) {
            const uint32_t units = member_units(cn, a.mem_slack);
            s_moff[k] = (uint32_t)atomicAdd(&a.bump[2], (unsigned long long)units);
            s_cap[k] = units * 4;
            fill = true;
        } else if (kind1 == K_ONE) {
            if (is_list(kind0)) {
                one = a.midx[(uint64_t)s_moff[k] * 4];
            } else if (kind0 == K_ONE) {
                const uint32_t mo = s_one[k];
                if (q && N && bit_test(bm, mo)) find = true;
                else one = (N && mo >= Lp) ? R[mo - Lp] : mo;
                if (!find && one == DEL_MARK) find = true;
            } else {
                find = true;
            }
        }
        s_one[k] = one;
        const uint32_t fm = __ballot_sync(0xffffffffu, fill);
        const uint32_t fd = __ballot_sync(0xffffffffu, find);
        if (lane == 0) {
            s_fill_mask = fm;
            s_find_mask = fd;
        }
        // stats: transitions
        uint32_t *vs = a.vstats + (uint64_t)t * VST;
        if (lane < 25) vs[2 + lane] = 0;
        __syncwarp();
        if (kind0 != K_EMPTY || kind1 != K_EMPTY) atomicAdd(&vs[2 + 5 * kind0 + kind1], 1u);
        if (lane == 0) {
            vs[0] = N;
            vs[1] = s_missing;
        }
    }
    G::sync();
    if (wid == 0 && (s_fill_mask | s_find_mask)) {
        // one ascending pass over the post-batch adjacency materialises new lists
        // (scan order = ascending index, R-2) and finds the unique member of ONE groups
        const uint32_t fm = s_fill_mask, fd = s_find_mask;
        uint32_t fillc = 0;     // lane k: entries written
        uint32_t onev = s_one[lane];
        for (uint32_t base = 0; base < dn; base += 32) {
            const uint32_t i = base + lane;
            uint2 e = make_uint2(0u, 0u);
            if (i < dn) e = a.arc[aoff + i];
            uint32_t mk = (fm | fd) & __reduce_or_sync(0xffffffffu, e.y);
            while (mk) {
                const int k = __ffs(mk) - 1;
                mk &= mk - 1;
                const uint32_t bal = __ballot_sync(0xffffffffu, (e.y >> k) & 1u);
                if ((fd >> k) & 1u) {
                    if (lane == (uint32_t)k) onev = base + __ffs(bal) - 1;
                    continue;
                }
                const uint32_t start = __shfl_sync(0xffffffffu, fillc, k);
                const uint32_t mo = s_moff[k];
                if ((e.y >> k) & 1u) {
                    const uint64_t q = (uint64_t)mo * 4 + start + __popc(bal & lanemask_lt());
                    a.mdst[q] = e.x;
                    a.midx[q] = i;
                }
                if (lane == (uint32_t)k) fillc += __popc(bal);
            }
        }
        s_one[lane] = onev;
    }
    G::sync();
    if (wid == 0) {
        const uint32_t k = lane;
        const uint32_t kind1 = s_kind1[k];
        const uint32_t cn = s_c[k];
        uint32_t onedst = 0;
        if (kind1 == K_ONE) onedst = a.arc[aoff + s_one[k]].x;
        const uint32_t mask = __ballot_sync(0xffffffffu, cn != 0);
        const uint32_t n = __popc(mask);
        uint64_t Tp = cn ? ((uint64_t)cn << k) : 0ull;
        const uint64_t T = warp_sum(Tp);
        // bucket b <- group k_b
        const uint32_t kb = (lane < n) ? (uint32_t)__fns(mask, 0, lane + 1) : 0u;
        const uint32_t c_b = __shfl_sync(0xffffffffu, cn, kb);
        const uint32_t kind_b = __shfl_sync(0xffffffffu, kind1, kb);
        const uint32_t moff_b = __shfl_sync(0xffffffffu, s_moff[k], kb);
        const uint32_t cap_b = __shfl_sync(0xffffffffu, s_cap[k], kb);
        const uint32_t one_b = __shfl_sync(0xffffffffu, s_one[k], kb);
        const uint32_t od_b = __shfl_sync(0xffffffffu, onedst, kb);
        uint64_t thr;
        uint32_t alias;
        vose_warp(lane < n, n, (uint64_t)c_b << kb, T, thr, alias);
        uint32_t bo = h.bkt_off, ncap = h.ncap;
        if (n > h.ncap) {
            // plan reserved bucket_capacity(popc(mask | inserted)) >= n
            if (lane == 0) bo = (uint32_t)atomicAdd(&a.bump[1], (unsigned long long)bucket_capacity(n));
            bo = __shfl_sync(0xffffffffu, bo, 0);
            ncap = bucket_capacity(n);
        }
        uint32_t x_b, y_b;
        group_view(kind_b, c_b, moff_b, od_b, dn, aoff, x_b, y_b);
        const uint32_t aux_b = is_list(kind_b) ? cap_b : (kind_b == K_ONE ? one_b : 0u);
        write_buckets(a.bkt, a.gcan, bo, n, lane, kb, kind_b, c_b, x_b, y_b, aux_b, thr, alias, T);
        if (lane == 0) {
            VHdr nh;
            nh.T = T;
            nh.adj_off = aoff;
            nh.bkt_off = bo;
            nh.d = dn;
            nh.n = (uint8_t)n;
            nh.ncap = (uint8_t)ncap;
            nh.pad = 0;
            nh.adj_cap = s_adj_cap;
            a.hdr[u] = nh;
            ThinHdr th;
            th.bkt_off = bo;
            th.n = (uint8_t)n;
            th.flags = (dn >= a.hot_b ? 1 : 0) | (dn >= a.hot_m ? 2 : 0);
            th.pad1 = 0;
            a.thdr[u] = th;
        }
    }
    if (a.nbt) {
        // neighbour hash set of the post-batch adjacency (node2vec distance test)
        const uint32_t lg = nb_log2size(dn);
        uint32_t *tbl = a.nbt + 4 * aoff;
        for (uint32_t j = tid; j < (1u << lg); j += GT) tbl[j] = NB_EMPTY;
        G::sync();
        for (uint32_t i = tid; i < dn; i += GT) nb_insert(tbl, (1u << lg) - 1, a.arc[aoff + i].x);
        if (tid == 0) {
            a.nbo[u] = nb_pack(4 * aoff, lg);
            a.nbtomb[u] = 0;
        }
    }
    if (tid == 0 && a.hixo && a.hixo[u]) a.hixo[u] = 0;   // this route does not maintain the hub index
    if (tid == 0 && a.gixo && a.gixo[u]) a.gixo[u] = 0;   // ... nor the group index
}

// small touched vertices: one warp each, 8 per block (grid-stride over all touched
// vertices, skipping those routed to the block kernel); each warp keeps its delete
// scratch (bitmap, hash of deleted destinations, holes, rename table) in a 4 KB
// shared-memory slice when it fits
static constexpr uint32_t WARP_SCR_WORDS = 1024;
__global__ void __launch_bounds__(MT) k_upd_mutate_warp(const MutateArgs a, const uint8_t *__restrict__ route,
                                                        uint32_t count) {
    __shared__ MutSmem sm[MT / 32];
    __shared__ __align__(16) uint32_t wscr[MT / 32][WARP_SCR_WORDS];
    const uint32_t w = threadIdx.x >> 5;
    for (uint32_t i = blockIdx.x * (MT / 32) + w; i < count; i += gridDim.x * (MT / 32))
        if (!route[i]) mutate_vertex<32>(a, i, sm[w], wscr[w], WARP_SCR_WORDS);
}

// large touched vertices (hubs): one 1024-thread block each
__global__ void __launch_bounds__(LT) k_upd_mutate_block(const MutateArgs a, const uint32_t *__restrict__ list,
                                                         uint32_t count) {
    __shared__ MutSmem sm;
    for (uint32_t i = blockIdx.x; i < count; i += gridDim.x) {
        mutate_vertex<LT>(a, list[i], sm);
        __syncthreads();
    }
}

__global__ void k_upd_stats(const uint32_t *__restrict__ vstats, uint32_t ntouch, unsigned long long *__restrict__ out,
                            const unsigned long long *pnt = nullptr) {
    if (pnt) ntouch = (uint32_t)*pnt;   // one-sync route: the count is on the device
    __shared__ unsigned long long acc[VST];
    if (threadIdx.x < VST) acc[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long loc[VST];
    for (int j = 0; j < VST; j++) loc[j] = 0;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ntouch; t += gridDim.x * blockDim.x)
        for (int j = 0; j < 27; j++) loc[j] += vstats[(uint64_t)t * VST + j];
    for (int j = 0; j < 27; j++) {
        unsigned long long v = loc[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31u) == 0 && v) atomicAdd(&acc[j], v);
    }
    __syncthreads();
    if (threadIdx.x < 27 && acc[threadIdx.x]) atomicAdd(&out[threadIdx.x], acc[threadIdx.x]);
}

// ------------------------------------------------------------------ small-batch fast path (a11)
// Streaming updates (S4.2; BJ.c5): for n <= FAST_N records a single
// 1024-thread block validates, groups by source (stable rank sort in shared
// memory), runs the same per-vertex plan and, when everything fits, the same
// per-vertex mutate (one warp per touched vertex) -- one launch, no host round
// trips before the mutation.  Status and statistics land in mapped pinned host
// memory.  If a vertex is too large for the preallocated scratch or a pool would
// have to grow, nothing is mutated and the host runs the general pipeline.
static constexpr uint32_t FAST_N = 256;       // records per single-block batch
static constexpr uint32_t FAST_INLINE = 64;   // host records passed inline as kernel parameters
static constexpr uint32_t FAST_MAXL = 1u << 16;
// a touched vertex above this many (post-insert) arcs hands the batch to the bulk-synchronous
// pipeline, whose chunk items spread the vertex's scans over the GPU (one block here walks
// them alone: c5 batches of 16 records took 0.9 ms on the fast path, profiles/r01_streaming_c5)
static constexpr uint32_t FAST_HANDOFF_L = 8192;
// the streaming kernel (one record, 1024 threads) mutates a vertex above this many arcs with
// the whole block instead of one warp
static constexpr uint32_t FAST_BLOCK_L = 512;
enum : uint32_t { FAST_OK = 0, FAST_INVAL = 1, FAST_OVERFLOW = 4, FAST_SLOW = 8 };

struct FastOut {
    uint32_t status, ntouch;
    unsigned long long stats[27];
    unsigned long long inserted;
};

struct FastArgs {
    MutateArgs m;                     // graph, allocator and policy fields (pointers set in-kernel)
    uint4 recs[FAST_INLINE];          // small host batches, inline (no copy)
    const uint4 *drecs;               // or a device batch
    const uint32_t *inv;              // external -> internal vertex ids
    uint32_t n, V;
    unsigned long long arc_cap, bkt_cap, mem_units_cap;
    uint32_t *scr;                    // FAST_N * fast_words() words
    unsigned long long scr_cap;
    uint32_t *vstats;                 // FAST_N * VST
    FastOut *out;                     // mapped pinned host memory
};

__host__ __device__ inline unsigned long long fast_words_per_vertex() {
    return (FAST_MAXL + 31) / 32 + 8ull * (2 * FAST_N) + 3ull * FAST_N + 16;
}

// the whole small-batch update in one block (k_upd_fast; the streaming queue's persistent
// kernel k_stream_upd runs it with one warp per record).  Records come from `src` (device or
// shared memory, fa.n of them); status / statistics go to fa.out.
__device__ __forceinline__ uint32_t fast_status(uint32_t f) {
    return (f & FAST_INVAL) ? FAST_INVAL : (f & FAST_OVERFLOW) ? FAST_OVERFLOW : (f & FAST_SLOW) ? FAST_SLOW : FAST_OK;
}

#ifdef BINGO_SQ_TRACE
// measurement build only (tools/sq_trace.py): globaltimer marks of the streaming kernel's phases
static constexpr uint32_t SQT_N = 8192;
__device__ unsigned long long g_sqt[SQT_N][8];
__shared__ unsigned long long s_sqt[8];
#define SQ_MARK(j)                                                                               \
    do {                                                                                         \
        if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s_sqt[j]));      \
    } while (0)
#else
#define SQ_MARK(j) \
    do {       \
    } while (0)
#endif

__device__ __forceinline__ uint32_t upd_fast_body(const FastArgs &fa, const uint4 *src) {
    __shared__ uint4 recs[FAST_N];
    __shared__ uint32_t sval[FAST_N], seg[FAST_N + 1], tv[FAST_N];
    __shared__ unsigned long long scr_off[FAST_N + 1];
    __shared__ MutSmem sm[32];
    __shared__ unsigned long long need_arc, need_bkt, need_mem;
    __shared__ uint32_t flag, ntouch, go, blockwide, lite;
    __shared__ uint32_t s_vst[VST];   // one touched vertex: its statistics stay in shared memory
    const uint32_t tid = threadIdx.x, lane = tid & 31u, w = tid >> 5;
    // the pool bump pointers, read now so their latency hides behind the validation and plan
    unsigned long long bump0 = 0, bump1 = 0, bump2 = 0;
    if (tid == 0) {
        bump0 = fa.m.bump[0];
        bump1 = fa.m.bump[1];
        bump2 = fa.m.bump[2];
    }
    // a whole 1024-thread block on one touched vertex (the streaming kernel): its O(d) scans
    // are spread over 32 warps, so vertices up to FAST_MAXL arcs stay on this path
    const bool block_mode = blockDim.x == LT;
    const uint32_t n = fa.n;
    if (tid == 0) { need_arc = need_bkt = need_mem = 0; flag = 0; blockwide = 0; }
    if (tid < n) recs[tid] = src[tid];
    __syncthreads();
    // validation (whole batch, before anything else)
    if (tid < n) {
        uint4 r = recs[tid];
        if (r.x > 1u || r.y >= fa.V || r.z >= fa.V || (r.x == 0u && r.w == 0u)) {
            atomicOr(&flag, FAST_INVAL);
        } else if (fa.inv) {   // internal vertex ids from here on
            r.y = fa.inv[r.y];
            r.z = fa.inv[r.z];
            recs[tid] = r;
        }
    }
    __syncthreads();
    SQ_MARK(1);
    // an invalid batch is rejected whole before anything is read through its ids (a src >= V
    // must never index hdr[]): uniform exit, nothing mutated (bingo.h: EINVAL)
    if (flag & FAST_INVAL) {
        if (tid == 0) {
            fa.out->status = FAST_INVAL;
            fa.out->ntouch = 0;
            fa.out->inserted = 0;
        }
        return FAST_INVAL;
    }
    // stable grouping by src: rank = #{j : src_j < src_i, or src_j == src_i and j < i}
    if (tid < n) {
        const uint32_t si = recs[tid].y;
        uint32_t rank = 0;
        for (uint32_t j = 0; j < n; j++) {
            const uint32_t sj = recs[j].y;
            rank += (sj < si || (sj == si && j < tid)) ? 1u : 0u;
        }
        sval[rank] = tid;
    }
    __syncthreads();
    if (w == 0) {
        uint32_t cntv = 0;
        for (uint32_t base = 0; base < FAST_N; base += 32) {
            const uint32_t p = base + lane;
            const bool head = p < n && (p == 0 || recs[sval[p]].y != recs[sval[p - 1]].y);
            const uint32_t bal = __ballot_sync(0xffffffffu, head);
            if (head) {
                const uint32_t t = cntv + __popc(bal & lanemask_lt());
                seg[t] = p;
                tv[t] = recs[sval[p]].y;
            }
            cntv += __popc(bal);
        }
        if (lane == 0) {
            ntouch = cntv;
            seg[cntv] = n;
        }
    }
    __syncthreads();
    const uint32_t nt = ntouch;
    const uint32_t nw = blockDim.x >> 5;   // launched with 32 * clamp(n, 2, 32) threads
#ifndef BINGO_SQ_NO_LITE
    // A single record (the persistent queue's 1024-thread block, or a one-record launch): a
    // conservative plan from the header alone.  Every demand is bounded from above -- groups after the record
    // <= n + popc(w), each list <= L members -- so if the bounded demand fits the pools the
    // exact one does, and if the bounded overflow test passes the exact one (R-10) does; the
    // vertex's buckets are prefetched into L1 for the mutation.  Anything the bounds cannot
    // decide takes the exact plan below.  Saves the plan's group loads and reductions and a
    // block barrier on the dependent path (BINGO_SQ_NO_LITE: A/B).
    bool use_lite = false;   // block-uniform: decided from n, nt and (after a barrier) `lite`
    if (n == 1 && nt == 1) {
        if (w == 0) {
            const VHdr h = fa.m.hdr[tv[0]];
            if (lane < h.n) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(fa.m.bkt + h.bkt_off + lane));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(fa.m.gcan + h.bkt_off + lane));
            }
            if (lane == 0) {
                const uint4 r = recs[0];
                const uint32_t m = r.x == 0u ? 1u : 0u, q = r.x == 1u ? 1u : 0u, wb = m ? r.w : 0u;
                const uint32_t L = h.d + m, nbmax = h.n + __popc(wb);
                const uint64_t Tn = h.T + wb;
                bool ok = Tn >= h.T && __umul64hi(Tn, (uint64_t)nbmax) == 0 && (uint64_t)h.d + m < 0xFFFFFFFFull;
                uint32_t f = flag;
                if (L > (block_mode ? FAST_MAXL : FAST_HANDOFF_L)) f |= FAST_SLOW;
                const uint64_t need_a = L > h.adj_cap ? arc_capacity(L, fa.m.arc_slack) : 0ull;
                const uint64_t need_b = nbmax > h.ncap ? bucket_capacity(nbmax) : 0ull;
                const uint64_t need_m = (uint64_t)nbmax * member_units(L, fa.m.mem_slack);
                uint64_t words = 0;
                if (q) words = ((uint64_t)(L + 31) / 32 + 8ull * next_pow2(2) + 3ull + 8ull + 7ull) & ~7ull;
                ok = ok && bump0 + need_a <= fa.arc_cap && bump1 + need_b <= fa.bkt_cap &&
                     bump2 + need_m <= fa.mem_units_cap && words <= fa.scr_cap;
                if (ok || (f & FAST_SLOW)) {
                    scr_off[0] = 0;
                    scr_off[1] = words;
                    blockwide = block_mode && L > FAST_BLOCK_L ? 1u : 0u;
                    flag = f;
                    go = f == 0 ? 1u : 0u;
                    lite = 1;
                } else {
                    lite = 0;
                }
            }
        }
        __syncthreads();
        use_lite = lite != 0;
    }
    if (!use_lite) {
#endif
    // plan, one warp per touched vertex
    for (uint32_t t = w; t < nt; t += nw) {
        const VHdr h = fa.m.hdr[tv[t]];
        const PlanOut o = plan_vertex(recs, sval, seg[t], seg[t + 1], h, fa.m.bkt, fa.m.gcan, fa.m.alpha, fa.m.bs,
                                      fa.m.arc_slack, fa.m.mem_slack);
        if (lane == 0) {
            if (o.overflow) atomicOr(&flag, FAST_OVERFLOW);
            const bool single = block_mode && nt == 1;
            if (o.L > (single ? FAST_MAXL : FAST_HANDOFF_L) || o.q > FAST_N) atomicOr(&flag, FAST_SLOW);
            if (single && o.L > FAST_BLOCK_L) blockwide = 1;
            atomicAdd(&need_arc, o.arc);
            atomicAdd(&need_bkt, o.bkt);
            atomicAdd(&need_mem, o.mem + o.res);
            scr_off[t] = o.words;
        }
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long acc = 0;
        for (uint32_t t = 0; t < nt; t++) {
            const unsigned long long x = scr_off[t];
            scr_off[t] = acc;
            acc += x;
        }
        scr_off[nt] = acc;
        uint32_t f = flag;
        if (!(f & (FAST_INVAL | FAST_OVERFLOW))) {
            if (bump0 + need_arc > fa.arc_cap || bump1 + need_bkt > fa.bkt_cap || bump2 + need_mem > fa.mem_units_cap ||
                acc > fa.scr_cap)
                f |= FAST_SLOW;
        }
        flag = f;
        go = f == 0 ? 1u : 0u;
    }
    __syncthreads();
#ifndef BINGO_SQ_NO_LITE
    }
#endif
    SQ_MARK(2);
    if (go) {
        MutateArgs a = fa.m;
        a.recs = recs;
        a.sval = sval;
        a.seg = seg;
        a.tv = tv;
        a.scr_off = reinterpret_cast<const uint64_t *>(scr_off);
        a.scr = fa.scr;
        a.vstats = nt == 1 ? s_vst : fa.vstats;
        // each warp's delete scratch in dynamic shared memory when it fits (else global)
        extern __shared__ __align__(16) uint32_t fast_wscr[];
        if (blockwide) mutate_vertex<LT>(a, 0, sm[0]);   // uniform: the single vertex, every thread
        else
            for (uint32_t t = w; t < nt; t += nw)
                mutate_vertex<32>(a, t, sm[w], fast_wscr + w * WARP_SCR_WORDS, WARP_SCR_WORDS);
    }
    __syncthreads();
    SQ_MARK(3);
    const uint32_t fin = flag;   // final since the barrier before the mutation
    if (tid == 0) {
        FastOut *o = fa.out;
        o->status = fast_status(fin);
        o->ntouch = nt;
        unsigned long long ins = 0;
        for (uint32_t i = 0; i < n; i++) ins += recs[i].x == 0u ? 1ull : 0ull;
        o->inserted = ins;
    }
    if (go && tid < 27) {
        const uint32_t *vst = nt == 1 ? s_vst : fa.vstats;
        unsigned long long acc = 0;
        for (uint32_t t = 0; t < nt; t++) acc += vst[(uint64_t)t * VST + tid];
        fa.out->stats[tid] = acc;
    }
    return fast_status(fin);
}

__global__ void __launch_bounds__(1024) k_upd_fast(const FastArgs fa) {
    upd_fast_body(fa, fa.drecs ? fa.drecs : fa.recs);
}

// ------------------------------------------------------------------ streaming queue
// A persistent single-warp kernel that applies single-record updates as the host posts them,
// without a launch per record.  Host -> device: slots of a ring in mapped pinned host memory
// (seq + record); device -> host: the FastOut of the record, then done_seq, in mapped memory.
// The kernel runs on the caller's stream, so every later operation on that stream is ordered
// after it (the epoch fence: the library stops the kernel before any other operation on the
// graph).  It exits on stop, after SQ_IDLE_NS without a record (a caller that synchronises
// its stream does not wait forever), or after a record the single-warp path cannot take
// (FAST_SLOW: pool growth, a vertex above FAST_HANDOFF_L arcs) -- the host applies that one
// through the batched pipeline and relaunches on the next record.
static constexpr uint32_t SQ_N = 64;
static constexpr unsigned long long SQ_IDLE_NS = 2000000ull;
struct alignas(32) StreamSlot {
    unsigned int seq;         // record k is valid when seq == k + 1 ...
    unsigned int gen;         // ... for the kernel generation gen only
    unsigned int chk;         // = seq, written first (the host writes chk, rec, gen, seq in order)
    unsigned int pad;
    uint4 rec;
};
// The completion of a streamed record: ONE 32 B system-scope store (st.v8, a single PCIe
// write), so no __threadfence_system is needed between the result and the sequence number that
// publishes it (the fence cost 1.7 us per record, tools/sq_trace.py).  w0 = records completed;
// w1 = status | ntouch << 4 | inserted << 8 | missing << 16 (bit 31: the statistics did not fit
// and are in StreamQ::out, written and fenced before this store); w2 = deleted; w3..w7 = the 25
// kind-transition counts, 6 bits each (a single touched vertex has <= 32 groups), and w7's top
// 10 bits repeat w0's low 10 bits so the host can tell a torn read.
struct alignas(32) SqDone {
    unsigned int w[8];
};
struct StreamQ {
    unsigned int run_gen;     // host -> device: the generation that may run
    unsigned int done_seq;    // (unused since the packed completion)
    unsigned int exit_gen;    // device -> host: the generation that exited ...
    unsigned int exit_seq;    // ... without taking record exit_seq (or after a FAST_SLOW record)
    unsigned int pad[12];
    SqDone done;              // device -> host: the last record's completion (packed)
    unsigned int pad2[8];
    FastOut out;              // device -> host: statistics that do not fit the packed completion
    StreamSlot slot[SQ_N];
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned int ld_volatile_u32(const unsigned int *p) {
    return *reinterpret_cast<const volatile unsigned int *>(p);
}

// one 32 B system-scope load of a whole slot (LDG.E.256.STRONG.SYS): a single PCIe read of
// one host cache line, so seq and the record it guards come from one snapshot (x86 stores
// become visible in program order: a snapshot holding seq = k + 1 holds chk, rec and gen too)
struct SlotView {
    unsigned int seq, gen, chk, pad;
    uint4 rec;
};
__device__ __forceinline__ SlotView ld_slot(const StreamSlot *p) {
    SlotView v;
    asm volatile("ld.relaxed.sys.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.seq), "=r"(v.gen), "=r"(v.chk), "=r"(v.pad), "=r"(v.rec.x), "=r"(v.rec.y), "=r"(v.rec.z),
                   "=r"(v.rec.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ uint4 ld_volatile_u4(const uint4 *p) {
    uint4 v;
    asm volatile("ld.volatile.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ void st_done(SqDone *p, const unsigned int (&d)[8]) {
    asm volatile("st.relaxed.sys.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(d[0]), "r"(d[1]),
                 "r"(d[2]), "r"(d[3]), "r"(d[4]), "r"(d[5]), "r"(d[6]), "r"(d[7])
                 : "memory");
}

// pack a record's result (SqDone); false if a field does not fit
__device__ __forceinline__ bool sq_pack(const FastOut &o, unsigned int st, unsigned int seq, unsigned int (&d)[8]) {
    const bool ok = st == FAST_OK;   // other statuses carry no statistics (the body leaves them unset)
    bool fits = !ok || (o.ntouch < 16 && o.inserted < 256 && o.stats[1] < 256 && o.stats[0] <= 0xFFFFFFFFull);
    unsigned long long f[3] = {0, 0, 0};   // 150-bit transition field, then w7's check bits
    for (int i = 0; i < 25; i++) {
        const unsigned long long c = ok ? o.stats[2 + i] : 0ull;
        fits = fits && c < 64;
        const int b = 6 * i;
        f[b >> 6] |= (c & 63ull) << (b & 63);
        if ((b & 63) > 58) f[(b >> 6) + 1] |= (c & 63ull) >> (64 - (b & 63));
    }
    d[0] = seq;
    d[1] = ok ? ((st & 15u) | (o.ntouch & 15u) << 4 | ((unsigned int)o.inserted & 255u) << 8 |
                 ((unsigned int)o.stats[1] & 255u) << 16 | (fits ? 0u : 1u << 31))
              : (st & 15u);
    d[2] = ok ? (unsigned int)o.stats[0] : 0u;
    d[3] = (unsigned int)f[0];
    d[4] = (unsigned int)(f[0] >> 32);
    d[5] = (unsigned int)f[1];
    d[6] = (unsigned int)(f[1] >> 32);
    d[7] = ((unsigned int)f[2] & 0x3FFFFFu) | (seq & 0x3FFu) << 22;
    return fits;
}

#ifndef BINGO_SQ_CHECK_EVERY   // polls per stop / idle check (a check is one more PCIe read)
#define BINGO_SQ_CHECK_EVERY 16u
#endif
__global__ void __launch_bounds__(LT) k_stream_upd(const FastArgs fa0, StreamQ *q, unsigned int seq0, unsigned int gen) {
    __shared__ uint4 rec;
    __shared__ unsigned int cmd;   // 0 process, 1 exit
    __shared__ FastOut s_out;      // the body's result, packed into ONE store below
    FastArgs fa = fa0;
    fa.n = 1;
    fa.out = &s_out;
    unsigned int k = seq0;
    for (;;) {
        if (threadIdx.x == 0) {
            unsigned int c = 1;
            const unsigned long long t0 = globaltimer_ns();
            const StreamSlot *sl = &q->slot[k % SQ_N];
            for (unsigned int poll = 0;; poll++) {
                const SlotView v = ld_slot(sl);   // back-to-back polls: one PCIe read each
                if (v.seq == k + 1 && v.chk == k + 1 && v.gen == gen) {
                    rec = v.rec;
                    c = 0;
                    SQ_MARK(0);
                    break;
                }
                // stopped, or idle: exit without taking record k (the host relaunches)
                if ((poll % BINGO_SQ_CHECK_EVERY) == BINGO_SQ_CHECK_EVERY - 1 &&
                    (ld_volatile_u32(&q->run_gen) != gen || globaltimer_ns() - t0 > SQ_IDLE_NS))
                    break;
            }
            cmd = c;
        }
        __syncthreads();
        if (cmd) break;
        const unsigned int st = upd_fast_body(fa, &rec);
        __syncthreads();
        SQ_MARK(4);
        k++;
        if (threadIdx.x == 0) {
            if (st == FAST_SLOW) {   // the host applies this record through the batched pipeline
                *reinterpret_cast<volatile unsigned int *>(&q->exit_seq) = k;
                *reinterpret_cast<volatile unsigned int *>(&q->exit_gen) = gen;
            }
            unsigned int d[8];
            if (!sq_pack(s_out, st, k, d)) {   // statistics too wide: the full FastOut, fenced first
                q->out = s_out;
                __threadfence_system();
            }
            SQ_MARK(5);
            st_done(&q->done, d);
#ifdef BINGO_SQ_TRACE
            for (int j = 0; j < 6; j++) g_sqt[(k - 1) % SQT_N][j] = s_sqt[j];
            g_sqt[(k - 1) % SQT_N][6] = st;
#endif
        }
        if (st == FAST_SLOW) return;
        if (st == FAST_OK) fa.m.epoch++;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *reinterpret_cast<volatile unsigned int *>(&q->exit_seq) = k;
        __threadfence_system();
        *reinterpret_cast<volatile unsigned int *>(&q->exit_gen) = gen;
        __threadfence_system();
    }
}

}  // namespace bingo

#include "gix_table.cuh"
#include "update_bsp.cuh"
#include "float_update.cuh"
#include "hub_index.cuh"
#include "group_index.cuh"
#include "exchange.cuh"

// ------------------------------------------------------------------ host side
namespace {

struct Carve {
    char *base;
    size_t pos;
    template <typename T>
    T *take(size_t count) {
        pos = (pos + 255) & ~(size_t)255;
        T *p = reinterpret_cast<T *>(base + pos);
        pos += sizeof(T) * count;
        return p;
    }
};

size_t batch_scratch_bytes(uint64_t n) {
    size_t b = 0;
    auto add = [&](size_t x) { b = ((b + 255) & ~(size_t)255) + x; };
    add(16 * n);                                   // recs copy
    add(4 * n); add(4 * n); add(4 * n); add(4 * n); // keys/vals ping-pong
    add(8 * radix_tmp_words(n));
    add(8 * (n + 1)); add(8 * (n + 2));            // head, head_ex
    add(8 * scan_tmp_words(n + 1));
    add(4 * (n + 1)); add(4 * n);                  // seg, tv
    add(8 * (n + 1)); add(8 * (n + 2));            // scr_need, scr_off
    add(4 * VST * n);                              // vstats
    add(4 * n); add(4 * n);                        // small / large touched lists
    add(sizeof(UpdCounters) + 8 * 32);             // counters, stats
    add(8 * n); add(8 * n);                        // float mode: dins, device copy of the real biases
    add(4 * n); add(4 * n);                        // float mode: decimal-member offsets / capacities
    return b + 4096;
}

bingo_status grow_pool(bingo_graph *g, int which, uint64_t need_total, cudaStream_t s) {
    // which: 0 arcs, 1 buckets, 2 members (units)
    if (which == 0) {
        uint64_t cap = std::max<uint64_t>(need_total + need_total / 4, g->arc_cap + g->arc_cap / 4);
        uint2 *na = (uint2 *)bingo_dev_alloc(g, sizeof(uint2) * cap);
        uint32_t *ne = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * cap);
        if (!na || !ne) { bingo_dev_free(g, na); bingo_dev_free(g, ne); return BINGO_E_NOMEM; }
        if (g->arc_dval) {
            uint64_t *nv = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * cap);
            if (!nv) { bingo_dev_free(g, na); bingo_dev_free(g, ne); return BINGO_E_NOMEM; }
            if (cudaMemcpyAsync(nv, g->arc_dval, 8 * g->arc_cap, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
                cudaStreamSynchronize(s) != cudaSuccess)
                return BINGO_E_CUDA;
            bingo_dev_free(g, g->arc_dval);
            g->arc_dval = nv;
        }
        if (cudaMemcpyAsync(na, g->arc, sizeof(uint2) * g->arc_cap, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(ne, g->arc_epoch, 4 * g->arc_cap, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return BINGO_E_CUDA;
        if (g->nbt) {
            uint32_t *nt = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * 4 * cap);
            if (!nt) { bingo_dev_free(g, na); bingo_dev_free(g, ne); return BINGO_E_NOMEM; }
            if (cudaMemcpyAsync(nt, g->nbt, sizeof(uint32_t) * 4 * g->arc_cap, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
                cudaStreamSynchronize(s) != cudaSuccess)
                return BINGO_E_CUDA;
            bingo_dev_free(g, g->nbt);
            g->nbt = nt;
        }
        bingo_dev_free(g, g->arc);
        bingo_dev_free(g, g->arc_epoch);
        g->arc = na; g->arc_epoch = ne; g->arc_cap = cap;
    } else if (which == 1) {
        uint64_t cap = std::min<uint64_t>(std::max<uint64_t>(need_total + need_total / 4, g->bkt_cap + g->bkt_cap / 4),
                                          0xFFFFFFF0ull);
        if (cap < need_total) return BINGO_E_NOMEM;
        Bucket *nb = (Bucket *)bingo_dev_alloc(g, sizeof(Bucket) * cap);
        GCan *ng = (GCan *)bingo_dev_alloc(g, sizeof(GCan) * cap);
        if (!nb || !ng) { bingo_dev_free(g, nb); bingo_dev_free(g, ng); return BINGO_E_NOMEM; }
        if (cudaMemcpyAsync(nb, g->bkt, sizeof(Bucket) * g->bkt_cap, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(ng, g->gcan, sizeof(GCan) * g->bkt_cap, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return BINGO_E_CUDA;
        bingo_dev_free(g, g->bkt);
        bingo_dev_free(g, g->gcan);
        g->bkt = nb; g->gcan = ng; g->bkt_cap = cap;
    } else {
        uint64_t units = std::min<uint64_t>(std::max<uint64_t>(need_total + need_total / 4, g->mem_cap / 4 + g->mem_cap / 16),
                                            0xFFFFFFF0ull);
        if (units < need_total) return BINGO_E_NOMEM;
        uint32_t *nd = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * 4 * units);
        uint32_t *ni = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * 4 * units);
        if (!nd || !ni) { bingo_dev_free(g, nd); bingo_dev_free(g, ni); return BINGO_E_NOMEM; }
        if (cudaMemcpyAsync(nd, g->mdst, sizeof(uint32_t) * g->mem_cap, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(ni, g->midx, sizeof(uint32_t) * g->mem_cap, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return BINGO_E_CUDA;
        bingo_dev_free(g, g->mdst);
        bingo_dev_free(g, g->midx);
        g->mdst = nd; g->midx = ni; g->mem_cap = 4 * units;
    }
    return BINGO_OK;
}

int key_bits_for(uint32_t V) {
    int b = 0;
    while (b < 32 && (V - 1) >> b) b++;
    return b ? b : 1;
}

}  // namespace

static bingo_status upd_cuda_fail(bingo_graph *g, cudaError_t e, const char *w) {
    fprintf(stderr, "libbingo: CUDA error in %s: %s\n", w, cudaGetErrorString(e));
    g->poisoned = 1;
    return BINGO_E_CUDA;
}
#define UCK(call)                                                   \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return upd_cuda_fail(g, e_, #call);  \
    } while (0)

// BINGO_UPD_TRACE=1: device (CUDA events) and host timestamps at the phase boundaries of
// one bingo_apply_updates call, printed to stderr (measurement only)
struct UpdTrace {
    bool on = false;
    int n = 0;
    const char *tag[24];
    cudaEvent_t ev[24];
    std::chrono::steady_clock::time_point ht[24];
    void mark(const char *t, cudaStream_t s) {
        if (!on || n >= 24) return;
        tag[n] = t;
        cudaEventCreate(&ev[n]);
        cudaEventRecord(ev[n], s);
        ht[n] = std::chrono::steady_clock::now();
        n++;
    }
    void dump() {
        if (!on || !n) return;
        cudaEventSynchronize(ev[n - 1]);
        for (int i = 1; i < n; i++) {
            float ms = 0, at = 0;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            cudaEventElapsedTime(&at, ev[0], ev[i]);
            const double hus = std::chrono::duration<double, std::micro>(ht[i] - ht[i - 1]).count();
            fprintf(stderr, "upd-trace %-26s at %8.1f us  (+%7.1f device, +%7.1f host)\n", tag[i], 1e3 * at, 1e3 * ms,
                    hus);
        }
        for (int i = 0; i < n; i++) cudaEventDestroy(ev[i]);
        n = 0;
    }
};
static UpdTrace g_trace;

static void fill_mutate_common(bingo_graph *g, MutateArgs &ma, uint32_t e) {
    const bool bs = (g->flags & BINGO_BUILD_BS_MODE) != 0;
    ma.hdr = g->hdr;
    ma.thdr = g->thdr;
    ma.arc = g->arc;
    ma.arc_epoch = g->arc_epoch;
    ma.arc_dval = g->arc_dval;
    ma.dins = g->cur_dins;
    ma.bkt = g->bkt;
    ma.gcan = g->gcan;
    ma.mdst = g->mdst;
    ma.midx = g->midx;
    ma.nbt = g->nbt;
    ma.nbo = g->nbo;
    ma.nbtomb = g->nbtomb;
    ma.hixo = g->hixo;
    ma.hixt = g->hixt;
    ma.hix = g->hix;
    ma.hix_min = g->hix_min;
    ma.hix_cap = g->hix_cap;
    ma.gixo = g->gixo;
    ma.gixt = g->gixt;
    ma.gix = g->gix;
    ma.gix_min = g->gix_min;
    ma.gix_cap = g->gix_cap;
    ma.bump = g->counters;
    ma.epoch = e;
    ma.alpha = g->alpha;
    ma.beta = g->beta;
    ma.hot_b = g->hot_bkt_degree;
    ma.hot_m = g->hot_mem_degree;
    ma.bs = bs;
    ma.arc_slack = g->arc_slack;
    ma.mem_slack = g->member_slack;
}

// returns true when the fast path decided the call (OK / EINVAL / EOVERFLOW / CUDA)
static bool ensure_fast_scratch(bingo_graph *g) {
    if (!g->fast_scr) {
        const size_t words = (size_t)(FAST_N * fast_words_per_vertex());
        g->fast_scr = (uint32_t *)bingo_dev_alloc(g, 4 * words + 4 * FAST_N * VST + 16 * FAST_N + 64);
        if (!g->fast_scr) return false;
        void *h = nullptr;
        if (cudaHostAlloc(&h, sizeof(FastOut), cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        g->fast_out_host = h;
        if (cudaHostGetDevicePointer(&g->fast_out_dev, h, 0) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
    }
    return true;
}

static void fill_fast_common(bingo_graph *g, FastArgs &fa) {
    memset(&fa, 0, sizeof(fa));
    fill_mutate_common(g, fa.m, g->epoch + 1);
    fa.V = g->V;
    fa.inv = g->inv;
    fa.arc_cap = g->arc_cap;
    fa.bkt_cap = g->bkt_cap;
    fa.mem_units_cap = g->mem_cap / 4;
    fa.scr = g->fast_scr;
    fa.scr_cap = FAST_N * fast_words_per_vertex();
    fa.vstats = g->fast_scr + fa.scr_cap;
    fa.out = (FastOut *)g->fast_out_dev;
}

// returns true when the fast path decided the call (OK / EINVAL / EOVERFLOW / CUDA)
static bool try_fast_path(bingo_graph *g, const bingo_update *batch, uint64_t n, uint32_t flags,
                          bingo_update_stats *stats, cudaStream_t s, bingo_status *out) {
    if (!ensure_fast_scratch(g)) return false;
    FastArgs fa;
    fill_fast_common(g, fa);
    if ((flags & BINGO_UPD_HOST_BATCH) && n > FAST_INLINE) {   // larger host batches: one H2D copy
        uint4 *stage = reinterpret_cast<uint4 *>(g->fast_scr + FAST_N * fast_words_per_vertex() + FAST_N * VST);
        if (cudaMemcpyAsync(stage, batch, 16 * n, cudaMemcpyHostToDevice, s) != cudaSuccess) {
            *out = upd_cuda_fail(g, cudaGetLastError(), "fast-path batch copy");
            return true;
        }
        fa.drecs = stage;
    } else if (flags & BINGO_UPD_HOST_BATCH) {
        memcpy(fa.recs, batch, 16 * n);
        fa.drecs = nullptr;
    } else {
        fa.drecs = reinterpret_cast<const uint4 *>(batch);
    }
    fa.n = (uint32_t)n;
    FastOut *ho = (FastOut *)g->fast_out_host;
    ho->status = 0xFFFFFFFFu;
    // one warp per touched vertex at most (a vertex's records go to one warp): small
    // blocks keep the block-wide barriers of the single-record case cheap
    // up to 32 warps x WARP_SCR_WORDS of dynamic shared memory: the attribute is per device,
    // so it is raised once for every device this process launches the fast path on
    static std::atomic<uint64_t> smem_set{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(smem_set.load(std::memory_order_acquire) & bit)) {
        if (cudaFuncSetAttribute(k_upd_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 4 * WARP_SCR_WORDS) !=
            cudaSuccess) {
            *out = upd_cuda_fail(g, cudaGetLastError(), "k_upd_fast smem attribute");
            return true;
        }
        smem_set.fetch_or(bit, std::memory_order_acq_rel);
    }
    const unsigned fw = (unsigned)std::min<uint64_t>(32, std::max<uint64_t>(2, n));
    k_upd_fast<<<1, 32 * fw, 4 * WARP_SCR_WORDS * fw, s>>>(fa);
    bingo_count_launch();
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        *out = upd_cuda_fail(g, e, "k_upd_fast");
        return true;
    }
    const uint32_t st = ho->status;
    if (st == FAST_SLOW) return false;
    if (st == FAST_INVAL) { *out = BINGO_E_INVAL; return true; }
    if (st == FAST_OVERFLOW) { *out = BINGO_E_OVERFLOW; return true; }
    if (st != FAST_OK) { *out = upd_cuda_fail(g, cudaErrorUnknown, "k_upd_fast status"); return true; }
    g->epoch++;
    const uint64_t deleted = ho->stats[0];
    g->num_arcs = g->num_arcs + ho->inserted - deleted;
    if (stats) {
        stats->inserted = ho->inserted;
        stats->deleted = deleted;
        stats->missing_deletes = ho->stats[1];
        stats->touched_vertices = ho->ntouch;
        for (int i = 0; i < 25; i++) stats->kind_transitions[i / 5][i % 5] = ho->stats[2 + i];
        stats->epoch = g->epoch;
    }
    *out = BINGO_OK;
    return true;
}

// grow-on-demand device buffer owned by the graph
static bool ensure_buf(bingo_graph *g, void *&buf, size_t &have, size_t need) {
    if (have >= need) return true;
    bingo_dev_free(g, buf);
    buf = bingo_dev_alloc(g, need);
    have = buf ? need : 0;
    return buf != nullptr;
}

// pool growth for the batch's demand; nothing is mutated when this fails
static bingo_status check_capacity(bingo_graph *g, const UpdCounters &hc, const unsigned long long *bump,
                                   cudaStream_t s) {
    if (hc.flag & 1) return BINGO_E_INVAL;
    if (hc.flag & 4) return BINGO_E_OVERFLOW;
    bingo_status st;
    if (bump[0] + hc.need_arc > g->arc_cap && (st = grow_pool(g, 0, bump[0] + hc.need_arc, s)) != BINGO_OK)
        return st == BINGO_E_CUDA ? (g->poisoned = 1, st) : st;
    if (bump[1] + hc.need_bkt > g->bkt_cap && (st = grow_pool(g, 1, bump[1] + hc.need_bkt, s)) != BINGO_OK)
        return st == BINGO_E_CUDA ? (g->poisoned = 1, st) : st;
    const uint64_t mem_units_need = bump[2] + hc.need_mem + hc.reserve_mem;
    if (mem_units_need > g->mem_cap / 4 && (st = grow_pool(g, 2, mem_units_need, s)) != BINGO_OK)
        return st == BINGO_E_CUDA ? (g->poisoned = 1, st) : st;
    return BINGO_OK;
}

// The hub delete index (opt-in, BINGO_HUB_INDEX=1): tables are built with the graph for its
// largest vertices (hix_build_all) and maintained by the bulk-synchronous route; lazy
// (re)builds only above the build threshold (a build costs ~9x a scan).  Measured (DESIGN.md
// 10): the c4 selection phase drops 542 -> ~160 us serialised, but whole batches do not get
// faster (c4 1.67 ms either way, the group fronts and hole passes dominate; c2 0.87 vs 0.82 ms),
// so the scans stay the default.
static bool hix_disabled() {
    const char *ev = getenv("BINGO_HUB_INDEX");
    return ev && ev[0] == '0';
}

// Both update indices (hub delete index, group index) are kept only for vertices of more than
// BINGO_INDEX_MIN arcs (default 2048; the build raises it 4x at a time until the tables fit
// their memory budget).  Below that the O(d) scans of the bulk-synchronous route are cheaper
// than keeping a table exact across batches (measured; c4 after session 3's
// grid changes: 4096 1.19 ms, 2048 1.14 ms, 1024 1.14 ms per 100K-record batch).
static uint32_t index_min() {
    uint32_t m = 2 * CH;
    if (const char *ev = getenv("BINGO_INDEX_MIN")) m = std::max<uint32_t>(CH, (uint32_t)strtoul(ev, nullptr, 10));
    return m;
}
// Without BINGO_INDEX_MIN the indices are built only for graphs of >= 2^28 arcs: on smaller
// graphs the hubs are small enough that their scans beat keeping tables (c2: 0.82 ms per
// 100K-record batch without, 1.05-1.5 ms with; c4: 1.51 ms without, ~1.2 ms with).
static bool index_wanted(const bingo_graph *g) {
    return getenv("BINGO_INDEX_MIN") != nullptr || g->num_arcs >= (1ull << 28);
}

// hub delete index storage (hub_index.cuh): per-vertex offsets / tombstone counts on first
// use, and a table pool with room for every table this batch may build (tables are taken
// zeroed from the pool and never reused, so new words are zeroed)
static bingo_status ensure_hix(bingo_graph *g, unsigned long long used, unsigned long long need, cudaStream_t s) {
    if (!need) return BINGO_OK;
    if (!g->hixo) {
        g->hixo = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * std::max<uint64_t>(g->V, 1));
        g->hixt = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * std::max<uint64_t>(g->V, 1));
        if (!g->hixo || !g->hixt) return BINGO_E_NOMEM;
        if (cudaMemsetAsync(g->hixo, 0, sizeof(uint64_t) * std::max<uint64_t>(g->V, 1), s) != cudaSuccess ||
            cudaMemsetAsync(g->hixt, 0, sizeof(uint32_t) * std::max<uint64_t>(g->V, 1), s) != cudaSuccess)
            return BINGO_E_CUDA;
    }
    if (used + need <= g->hix_cap) return BINGO_OK;
    const uint64_t cap = std::max<uint64_t>((used + need) + (used + need) / 4, g->hix_cap + g->hix_cap / 2);
    uint32_t *nh = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * cap);
    if (!nh) return BINGO_E_NOMEM;
    if ((g->hix_cap && cudaMemcpyAsync(nh, g->hix, sizeof(uint32_t) * g->hix_cap, cudaMemcpyDeviceToDevice, s) != cudaSuccess) ||
        cudaMemsetAsync(nh + g->hix_cap, 0, sizeof(uint32_t) * (cap - g->hix_cap), s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return BINGO_E_CUDA;
    bingo_dev_free(g, g->hix);
    g->hix = nh;
    g->hix_cap = cap;
    return BINGO_OK;
}

// The group index (group_index.cuh) is on unless BINGO_GROUP_INDEX=0; tables are taken from
// a pool at batch time.  Growing the pool is best effort: without room the hubs keep the
// member-list scans (g->gix_full), never an error.
static bool gix_enabled() {
    const char *ev = getenv("BINGO_GROUP_INDEX");
    return !(ev && ev[0] == '0');
}
static bingo_status ensure_gix_arrays(bingo_graph *g, cudaStream_t s) {
    if (g->gixo || g->gix_full || !gix_enabled() || g->float_mode || !g->V) return BINGO_OK;
    uint64_t *o = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * g->V);
    uint32_t *t = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * g->V);
    if (!o || !t) {
        bingo_dev_free(g, o);
        bingo_dev_free(g, t);
        g->gix_full = true;
        return BINGO_OK;
    }
    if (cudaMemsetAsync(o, 0, sizeof(uint64_t) * g->V, s) != cudaSuccess ||
        cudaMemsetAsync(t, 0, sizeof(uint32_t) * g->V, s) != cudaSuccess)
        return BINGO_E_CUDA;
    g->gix_min = index_min();
    g->gixo = o;
    g->gixt = t;
    return BINGO_OK;
}
static bingo_status ensure_gix(bingo_graph *g, unsigned long long used, unsigned long long need, cudaStream_t s) {
    if (!need || !g->gixo || g->gix_full || used + need <= g->gix_cap) return BINGO_OK;
    const uint64_t cap = std::max<uint64_t>((used + need) + (used + need) / 2, g->gix_cap + g->gix_cap / 2);
    uint32_t *nh = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * cap);
    if (!nh) {
        g->gix_full = true;
        return BINGO_OK;
    }
    if ((g->gix_cap && cudaMemcpyAsync(nh, g->gix, sizeof(uint32_t) * std::min<uint64_t>(used, g->gix_cap),
                                       cudaMemcpyDeviceToDevice, s) != cudaSuccess) ||
        cudaMemsetAsync(nh + std::min<uint64_t>(used, g->gix_cap), 0,
                        sizeof(uint32_t) * (cap - std::min<uint64_t>(used, g->gix_cap)), s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return BINGO_E_CUDA;
    bingo_dev_free(g, g->gix);
    g->gix = nh;
    g->gix_cap = cap;
    return BINGO_OK;
}

static inline unsigned warp_grid(uint64_t units, unsigned cap) {
    const uint64_t b = (units + MT / 32 - 1) / (MT / 32);
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(b, cap));
}

// blocks per SM (148 SMs) from an environment override (A/B), else the default
static unsigned bsp_env_grid(const char *name, unsigned per_sm) {
    if (const char *ev = getenv(name)) per_sm = std::max(1u, (unsigned)strtoul(ev, nullptr, 10));
    return 148 * per_sm;
}

// grid cap of the warp-per-vertex kernels, in blocks (BINGO_BSP_WG blocks per SM, A/B): 64
// (about one touched vertex per warp at 100K-record batches; the block scheduler balances the
// waves) over 16: c2 0.778 -> 0.748 ms, c4 1.276 -> 1.226 ms (profiles/r02_update_wg_ab.txt)
static unsigned bsp_wg() {
    unsigned per_sm = 64;
    if (const char *ev = getenv("BINGO_BSP_WG")) per_sm = std::max(1u, (unsigned)strtoul(ev, nullptr, 10));
    return 148 * per_sm;
}

// BINGO_BSP_FUSED=1: small vertices by the fused k_bsp_small instead of k_bsp_finalize +
// k_bsp_rebuild (A/B: the fused kernel spills more and was 2-3% slower at c2 and c4)
static bool bsp_unfused() {
    const char *ev = getenv("BINGO_BSP_FUSED");
    return !(ev && ev[0] == '1');
}

// touched vertices per sub-batch (BINGO_BSP_MAXT: smaller sub-batches, tests)
static uint64_t bsp_maxt() {
    uint64_t maxt = BSP_MAXT;
    if (const char *ev = getenv("BINGO_BSP_MAXT")) maxt = std::max<uint64_t>(1, strtoull(ev, nullptr, 10));
    return maxt;
}

// per-vertex state of a (sub-)batch of up to ntmax touched vertices, carved from bscratch
struct BspBufs {
    uint64_t *p_copy, *p_sel, *p_grp, *p_all, *scr_need, *scr_off, *stmp;
    uint32_t *vstats;
    BspTotals *dt;
    int *abort;
};
static bingo_status bsp_scratch(bingo_graph *g, uint64_t ntmax, BspArgs &a, BspBufs &b) {
    size_t vb = 0;
    {
        auto add = [&](size_t x) { vb = ((vb + 255) & ~(size_t)255) + x; };
        for (int j = 0; j < 8; j++) add(4 * ntmax);
        add(8 * ntmax);
        add(4ull * GK_N * 32 * ntmax);
        for (int j = 0; j < 4; j++) add(8 * (ntmax + 1));
        for (int j = 0; j < 4; j++) add(8 * (ntmax + 2));
        add(8 * (ntmax + 1));
        add(8 * (ntmax + 2));
        add(4ull * VST * ntmax);
        add(8 * 5 * scan_tmp_words(ntmax + 1));   // up to five scans in one launch
        add(sizeof(BspTotals));
        add(4 * ntmax);
        add(4 * ntmax);
        add(8 * ntmax);
        add(4 * ntmax);
        add(4 * ntmax);
        add(4 * ntmax);
        add(8 * 33 * ntmax);
        add(4 * ntmax);
        add(4 * ntmax);
        add(64);
        add(64);
        vb += 4096;
    }
    if (!ensure_buf(g, g->bscratch, g->bscratch_bytes, vb)) return BINGO_E_NOMEM;
    Carve cv{(char *)g->bscratch, 0};
    memset(&a, 0, sizeof(a));
    a.vL = cv.take<uint32_t>(ntmax);
    a.vq = cv.take<uint32_t>(ntmax);
    a.vm = cv.take<uint32_t>(ntmax);
    a.vN = cv.take<uint32_t>(ntmax);
    a.vmiss = cv.take<uint32_t>(ntmax);
    a.vlist0 = cv.take<uint32_t>(ntmax);
    a.vacap = cv.take<uint32_t>(ntmax);
    a.vmoved = cv.take<uint32_t>(ntmax);
    a.vaoff = cv.take<uint64_t>(ntmax);
    a.gk = cv.take<uint32_t>((size_t)GK_N * 32 * ntmax);
    a.cc_copy = cv.take<uint64_t>(ntmax + 1);
    a.cc_sel = cv.take<uint64_t>(ntmax + 1);
    a.cc_grp = cv.take<uint64_t>(ntmax + 1);
    a.cc_all = cv.take<uint64_t>(ntmax + 1);
    b.p_copy = cv.take<uint64_t>(ntmax + 2);
    b.p_sel = cv.take<uint64_t>(ntmax + 2);
    b.p_grp = cv.take<uint64_t>(ntmax + 2);
    b.p_all = cv.take<uint64_t>(ntmax + 2);
    a.p_copy = b.p_copy;
    a.p_sel = b.p_sel;
    a.p_grp = b.p_grp;
    a.p_all = b.p_all;
    b.scr_need = cv.take<uint64_t>(ntmax + 1);
    b.scr_off = cv.take<uint64_t>(ntmax + 2);
    b.vstats = cv.take<uint32_t>((size_t)VST * ntmax);
    b.stmp = cv.take<uint64_t>(5 * scan_tmp_words(ntmax + 1));
    b.dt = cv.take<BspTotals>(1);
    a.hubs = cv.take<uint32_t>(ntmax);
    a.bigs = cv.take<uint32_t>(ntmax);
    a.vnbo = cv.take<uint64_t>(ntmax);
    a.vnbfull = cv.take<uint32_t>(ntmax);
    a.vhix = cv.take<uint32_t>(ntmax);
    a.vrank = cv.take<uint32_t>(ntmax);
    a.sorts = cv.take<uint2>(ntmax * 33);
    a.vgix = cv.take<uint32_t>(ntmax);
    a.vgixe = cv.take<uint32_t>(ntmax);
    a.nhubs = cv.take<uint32_t>(16);
    a.nbigs = a.nhubs + 1;
    b.abort = cv.take<int>(16);
    return BINGO_OK;
}

// per-chunk-item counts and their prefixes (hole ranks, group-hole ranks), sized with
// slack so later batches of the one-sync route fit without a host round trip
static bingo_status bsp_items(bingo_graph *g, uint64_t sel, uint64_t grp, BspArgs &a, uint64_t *&itmp) {
    if (sel > g->isc_sel || grp > g->isc_grp || !g->iscratch) {
        const uint64_t ns = std::max<uint64_t>(g->isc_sel, sel + sel / 2 + 64);
        const uint64_t ng = std::max<uint64_t>(g->isc_grp, grp + grp / 2 + 64);
        size_t ib = 0;
        auto add = [&](size_t x) { ib = ((ib + 255) & ~(size_t)255) + x; };
        add(8 * (ns + 1)); add(8 * (ns + 2)); add(8 * (ng + 1)); add(8 * (ng + 2));
        add(8 * scan_tmp_words(std::max(ns, ng) + 1));
        ib += 1024;
        if (!ensure_buf(g, g->iscratch, g->iscratch_bytes, ib)) return BINGO_E_NOMEM;
        g->isc_sel = ns;
        g->isc_grp = ng;
    }
    Carve ic{(char *)g->iscratch, 0};
    a.icnt = ic.take<uint64_t>(g->isc_sel + 1);
    a.ipref = ic.take<uint64_t>(g->isc_sel + 2);
    a.gcnt = ic.take<uint64_t>(g->isc_grp + 1);
    a.gpref = ic.take<uint64_t>(g->isc_grp + 2);
    itmp = ic.take<uint64_t>(scan_tmp_words(std::max(g->isc_sel, g->isc_grp) + 1));
    return BINGO_OK;
}

// delete scratch words (per-vertex bitmaps and hashes), grown with slack
static bingo_status bsp_vscratch(bingo_graph *g, uint64_t words) {
    const size_t need = 4 * (words + 64);
    if (g->vscratch_bytes >= need) return BINGO_OK;
    return ensure_buf(g, g->vscratch, g->vscratch_bytes, need + need / 2) ? BINGO_OK : BINGO_E_NOMEM;
}

// The hub chain (a long sequence of dependent, mostly small kernels) is the critical path of a
// batch; the small-vertex chain beside it is bulk work over all SMs.  The side stream gets the
// highest priority, so the block scheduler starts the hub kernels' blocks first whenever SMs
// free up (BINGO_AUX_PRIO=0: default priority, A/B).
static bingo_status ensure_aux_stream(bingo_graph *g) {
    if (g->aux_stream) return BINGO_OK;
    int least = 0, greatest = 0;
    const char *ev = getenv("BINGO_AUX_PRIO");
    if ((ev && ev[0] == '0') || cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) greatest = 0;
    if (cudaStreamCreateWithPriority(&g->aux_stream, cudaStreamNonBlocking, greatest) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_join, cudaEventDisableTiming) != cudaSuccess)
        return BINGO_E_CUDA;
    return BINGO_OK;
}

// Bulk-synchronous batch (update_bsp.cuh) over the touched vertices of a sorted,
// segmented batch.  Touched vertices are processed in sub-batches of at most
// BSP_MAXT (vertices are independent, all sub-batches use epoch e); the pool
// demand of the whole batch is reserved before anything is mutated.
static bingo_status apply_bsp(bingo_graph *g, const uint4 *recs, const uint32_t *sv, const uint32_t *seg,
                              const uint32_t *tv, uint64_t ntouch, uint32_t e, UpdCounters *dc,
                              unsigned long long *dstats, cudaStream_t s) {
    const uint64_t maxt = bsp_maxt();
    const uint64_t ntmax = std::min<uint64_t>(ntouch, maxt);
    BspArgs a;
    BspBufs b;
    {
        const bingo_status st = bsp_scratch(g, ntmax, a, b);
        if (st != BINGO_OK) return st;
    }
    if (g->hscratch_bytes < sizeof(BspTotals)) {
        if (g->hscratch) cudaFreeHost(g->hscratch);
        g->hscratch = nullptr;
        g->hscratch_bytes = 0;
        UCK(cudaMallocHost(&g->hscratch, sizeof(BspTotals)));
        g->hscratch_bytes = sizeof(BspTotals);
    }
    BspTotals *ht = (BspTotals *)g->hscratch;
    uint64_t *scr_need = b.scr_need, *scr_off = b.scr_off, *stmp = b.stmp;
    uint64_t *p_copy = b.p_copy, *p_sel = b.p_sel, *p_grp = b.p_grp, *p_all = b.p_all;
    uint32_t *vstats = b.vstats;
    BspTotals *dt = b.dt;
    auto refresh = [&]() {
        fill_mutate_common(g, a.g, e);
        a.g.recs = recs;
        a.g.sval = sv;
        a.g.seg = seg;
        a.g.tv = tv;
        a.g.scr_off = scr_off;
        a.g.vstats = vstats;
        a.err = dstats + 31;
    };
    refresh();
    const bool multi = ntouch > maxt;
    const unsigned WG = bsp_wg(), IG = 148 * 8;
    BspCaps nocaps;
    memset(&nocaps, 0, sizeof(nocaps));
    if (multi) {
        // demand of the whole batch first (read-only pass)
        a.t0 = 0;
        a.nt = (uint32_t)ntouch;
        a.gks = a.nt;
        k_bsp_plan<<<warp_grid(ntouch, WG), MT, 0, s>>>(a, scr_need, dc, true, false);
        bingo_count_launch();
        UCK(cudaGetLastError());
        UCK(cudaMemcpyAsync(&ht->c, dc, sizeof(UpdCounters), cudaMemcpyDeviceToHost, s));
        UCK(cudaMemcpyAsync(ht->bump, g->counters, sizeof(ht->bump), cudaMemcpyDeviceToHost, s));
        UCK(cudaMemcpyAsync(&ht->hix_used, g->counters + 5, 8, cudaMemcpyDeviceToHost, s));
        UCK(cudaMemcpyAsync(&ht->gix_used, g->counters + 6, 8, cudaMemcpyDeviceToHost, s));
        UCK(cudaStreamSynchronize(s));
        bingo_status st = check_capacity(g, ht->c, ht->bump, s);
        if (st == BINGO_OK && !hix_disabled()) st = ensure_hix(g, ht->hix_used, ht->c.need_hix, s);
        if (st == BINGO_OK) st = ensure_gix(g, ht->gix_used, ht->c.need_gix, s);
        if (st != BINGO_OK) return st == BINGO_E_CUDA ? (g->poisoned = 1, st) : st;
        refresh();
    }
    for (uint64_t t0 = 0; t0 < ntouch; t0 += maxt) {
        a.t0 = (uint32_t)t0;
        a.nt = (uint32_t)std::min<uint64_t>(maxt, ntouch - t0);
        a.gks = a.nt;
        const uint32_t nt = a.nt;
        UCK(cudaMemsetAsync(a.nhubs, 0, 32, s));   // hubs, bigs, rebuild fills, -, rank hubs, big sorts
        UCK(cudaMemsetAsync(a.vhix, 0, 4 * (size_t)nt, s));
        k_bsp_plan<<<warp_grid(nt, WG), MT, 0, s>>>(a, scr_need, dc, !multi, true);
        bingo_count_launch();
        UCK(cudaGetLastError());
        {   // the five per-vertex prefix sums of the plan in one launch
            const uint64_t *ins[5] = {scr_need, a.cc_copy, a.cc_sel, a.cc_grp, a.cc_all};
            uint64_t *outs[5] = {scr_off, p_copy, p_sel, p_grp, p_all};
            UCK(exclusive_scan_u64_multi(ins, outs, g->nbt ? 5 : 4, nt, stmp, s));
            if (!g->nbt) UCK(cudaMemsetAsync(p_all + nt, 0, 8, s));
        }
        k_bsp_totals<<<1, 32, 0, s>>>(a, dc, scr_off, dt, nocaps, nullptr);
        bingo_count_launch();
        UCK(cudaGetLastError());
        g_trace.mark("plan+scans", s);
        UCK(cudaMemcpyAsync(ht, dt, sizeof(BspTotals), cudaMemcpyDeviceToHost, s));
        UCK(cudaStreamSynchronize(s));
        g_trace.mark("sync plan totals", s);
        if (!multi) {
            bingo_status st = check_capacity(g, ht->c, ht->bump, s);
            if (st == BINGO_OK && !hix_disabled()) st = ensure_hix(g, ht->hix_used, ht->c.need_hix, s);
            if (st == BINGO_OK) st = ensure_gix(g, ht->gix_used, ht->c.need_gix, s);
            if (st != BINGO_OK) return st == BINGO_E_CUDA ? (g->poisoned = 1, st) : st;
            refresh();
        }
        // ---- from here on the (sub-)batch is applied
        const uint64_t sel = ht->sel, grp = ht->grp, copy = ht->copy, all = ht->all;
        if (ht->scr) {
            const bingo_status st = bsp_vscratch(g, ht->scr);
            if (st != BINGO_OK) return st;
            a.g.scr = (uint32_t *)g->vscratch;
        }
        uint64_t *itmp = nullptr;
        if (sel || grp) {
            const bingo_status st = bsp_items(g, sel, grp, a, itmp);
            if (st != BINGO_OK) return st;
        }
#define BSP_LAUNCH(kern, grid, strm, ...)                            \
        do {                                                         \
            kern<<<(grid), MT, 0, (strm)>>>(__VA_ARGS__);            \
            bingo_count_launch();                                    \
            UCK(cudaGetLastError());                                 \
        } while (0)
        BSP_LAUNCH(k_bsp_alloc_insert, warp_grid(nt, WG), s, a);
        g_trace.mark("alloc_insert", s);
        // two independent chains over disjoint vertex sets (shared state: bump
        // counters, atomics only): small vertices on `s`, large ones on the side stream
        const bool side = ht->bigs != 0;
        if (side) {
            const bingo_status st = ensure_aux_stream(g);
            if (st != BINGO_OK) return upd_cuda_fail(g, cudaGetLastError(), "aux stream");
        }
        cudaStream_t sh = side ? g->aux_stream : s;
        if (side) {
            UCK(cudaEventRecord(g->ev_fork, s));
            UCK(cudaStreamWaitEvent(sh, g->ev_fork, 0));
        }
        // -- large vertices
        if (copy) BSP_LAUNCH(k_bsp_copy, warp_grid(copy, IG), sh, a, copy);
        const bool hix = g->hixo != nullptr && ht->bigs && !hix_disabled();
        if (hix) {
            BSP_LAUNCH(k_hix_prep, warp_grid(ht->bigs, WG), sh, a);
            if (sel) BSP_LAUNCH(k_hix_build, warp_grid(sel, IG), sh, a, sel);
        }
        if (sel) {
            BSP_LAUNCH(k_bsp_select, warp_grid(sel, IG), sh, a, sel);
            if (hix) BSP_LAUNCH(k_hix_select, warp_grid(ht->hubs, WG), sh, a);
            BSP_LAUNCH(k_bsp_finalize, warp_grid(ht->hubs, WG), sh, a, true);
            if (hix) BSP_LAUNCH(k_hix_del, warp_grid(ht->hubs, WG), sh, a);
            BSP_LAUNCH(k_bsp_hub_sort, warp_grid(ht->hubs, WG), sh, a);
            k_bsp_sort_big<<<148, 256, 0, sh>>>(a);
            bingo_count_launch();
            UCK(cudaGetLastError());
            UCK(cudaMemsetAsync(a.nhubs + 5, 0, 4, sh));
            if (g->gixo) {
                BSP_LAUNCH(k_gix_prep, warp_grid(ht->bigs, WG), sh, a);
                if (grp) BSP_LAUNCH(k_gix_build, warp_grid(grp, IG), sh, a, grp);
            }
            g_trace.mark("hub: select+finalize", sh);
            BSP_LAUNCH(k_bsp_hole_count, warp_grid(sel, IG), sh, a, sel);
            UCK(exclusive_scan_u64(a.icnt, const_cast<uint64_t *>(a.ipref), sel, itmp, sh));
            BSP_LAUNCH(k_bsp_hole_write, warp_grid(sel, IG), sh, a, sel);
            BSP_LAUNCH(k_bsp_tail, warp_grid(ht->hubs, WG), sh, a);
            g_trace.mark("hub: holes+tail", sh);
            if (hix) BSP_LAUNCH(k_hix_ins, warp_grid(ht->bigs, WG), sh, a);
            if (g->gixo) BSP_LAUNCH(k_gix_front, warp_grid(ht->hubs, WG), sh, a);
            if (grp) {
                BSP_LAUNCH(k_bsp_grp_count, warp_grid(grp, IG), sh, a, grp);
                UCK(exclusive_scan_u64(a.gcnt, const_cast<uint64_t *>(a.gpref), grp, itmp, sh));
                BSP_LAUNCH(k_bsp_grp_write, warp_grid(grp, IG), sh, a, grp);
                BSP_LAUNCH(k_bsp_grp_sort, warp_grid(ht->hubs, WG), sh, a);
                k_bsp_sort_big<<<148, 256, 0, sh>>>(a);
                bingo_count_launch();
                UCK(cudaGetLastError());
                BSP_LAUNCH(k_bsp_grp_tail, warp_grid(ht->hubs, WG), sh, a);
                g_trace.mark("hub: group fronts+tails", sh);
            }
        }
        if (hix && !sel) BSP_LAUNCH(k_hix_ins, warp_grid(ht->bigs, WG), sh, a);   // inserts only
        if (g->gixo && !sel && ht->bigs) BSP_LAUNCH(k_gix_prep, warp_grid(ht->bigs, WG), sh, a);
        if (ht->bigs) {
            BSP_LAUNCH(k_bsp_rebuild_big, warp_grid(ht->bigs, WG), sh, a);
            k_bsp_rebuild_fill<<<(unsigned)std::min<uint64_t>(ht->bigs, 148 * 2), LT, 0, sh>>>(a);
            bingo_count_launch();
            UCK(cudaGetLastError());
            g_trace.mark("hub: rebuild_big", sh);
        }
        // -- small vertices
        if (bsp_unfused()) {
            if (ht->scr) BSP_LAUNCH(k_bsp_finalize, warp_grid(nt, WG), s, a, false);
            BSP_LAUNCH(k_bsp_rebuild, warp_grid(nt, WG), s, a);
        } else {
            BSP_LAUNCH(k_bsp_small, warp_grid(nt, WG), s, a);
        }
        g_trace.mark("small-vertex chain", s);
        if (side) {
            UCK(cudaEventRecord(g->ev_join, sh));
            UCK(cudaStreamWaitEvent(s, g->ev_join, 0));
        }
        g_trace.mark("join hub chain", s);
        if (g->nbt) BSP_LAUNCH(k_bsp_nb_incr, warp_grid(nt, WG), s, a);
        if (g->nbt && all) {
            BSP_LAUNCH(k_bsp_nb_clear, warp_grid(all, IG), s, a, all);
            BSP_LAUNCH(k_bsp_nb_fill, warp_grid(all, IG), s, a, all);
        }
#undef BSP_LAUNCH
        k_upd_stats<<<(unsigned)std::min<uint64_t>((nt + 255) / 256, 148), 256, 0, s>>>(vstats, nt, dstats);
        bingo_count_launch();
        UCK(cudaGetLastError());
    }
    return BINGO_OK;
}

// One-sync bulk-synchronous batch: the whole pipeline of apply_bsp is enqueued at once,
// before the host knows the touched-vertex count (*pnt, on the device) or any total of the
// plan.  Kernels read those on the device (BspArgs::pnt; item loops take their totals from
// the plan's prefix sums; grids are sized for the capacity, n touched vertices at most), and
// k_bsp_totals checks the batch against the pools and scratch allocated when it was
// enqueued.  If anything is short (or the batch is invalid) every mutating kernel returns at
// once, and the caller, after its single sync, grows what is short and re-runs the batch on
// the synchronous route (apply_bsp): the graph is untouched until the gate passes.
static bingo_status apply_bsp_async(bingo_graph *g, const uint4 *recs, const uint32_t *sv, const uint32_t *seg,
                                    const uint32_t *tv, const unsigned long long *pnt, uint64_t nmax, uint32_t e,
                                    UpdCounters *dc, unsigned long long *dstats, cudaStream_t s,
                                    BspTotals **dtot) {
    const uint64_t ntmax = std::max<uint64_t>(nmax, 1);
    BspArgs a;
    BspBufs b;
    {
        const bingo_status st = bsp_scratch(g, ntmax, a, b);
        if (st != BINGO_OK) return st;
    }
    uint64_t *itmp = nullptr;
    {
        const bingo_status st = bsp_items(g, 0, 0, a, itmp);
        if (st != BINGO_OK) return st;
    }
    {
        const bingo_status st = ensure_aux_stream(g);
        if (st != BINGO_OK) return upd_cuda_fail(g, cudaGetLastError(), "aux stream");
    }
    fill_mutate_common(g, a.g, e);
    a.g.recs = recs;
    a.g.sval = sv;
    a.g.seg = seg;
    a.g.tv = tv;
    a.g.scr_off = b.scr_off;
    a.g.vstats = b.vstats;
    a.err = dstats + 31;
    a.g.scr = (uint32_t *)g->vscratch;
    a.t0 = 0;
    a.nt = 0;
    a.pnt = pnt;
    a.gks = (uint32_t)ntmax;
    a.abort = b.abort;
    BspCaps caps;
    memset(&caps, 0, sizeof(caps));
    caps.arc = g->arc_cap;
    caps.bkt = g->bkt_cap;
    caps.mem_units = g->mem_cap / 4;
    caps.hix = g->hix_cap;
    caps.hix_on = !hix_disabled();
    if (caps.hix_on && !g->hixo) caps.hix = 0;   // tables need the offsets first: the sync route allocates them
    caps.scr_words = g->vscratch_bytes >= 4 * 64 ? g->vscratch_bytes / 4 - 64 : 0;
    caps.gix = g->gix_cap;
    caps.gix_on = g->gixo && !g->gix_full;
    caps.sel = g->isc_sel;
    caps.grp = g->isc_grp;
    // IG: item kernels, one wave of contiguous per-warp ranges; HG: the hub chain's per-hub kernels
    // (IG 16 and HG 16 per SM on graphs >= 2^28 arcs, whose hub scans fill more items and whose
    // hub chain is the critical path: c4 1.222 -> 1.177 ms (IG), 1.122 -> 1.09 ms (HG); c2 is 1-2%
    // faster at 8 / 4; profiles/r02_update_wg_ab.txt)
    const bool big_graph = g->num_arcs >= (1ull << 28);
    const unsigned WG = bsp_wg(), HG = bsp_env_grid("BINGO_BSP_HG", big_graph ? 16u : 4u),
                   IG = bsp_env_grid("BINGO_BSP_IG", big_graph ? 16u : 8u);
    const unsigned wg = warp_grid(ntmax, WG), hg = warp_grid(ntmax, HG);
    UCK(cudaMemsetAsync(a.nhubs, 0, 32, s));
    UCK(cudaMemsetAsync(a.vhix, 0, 4 * (size_t)ntmax, s));
    k_bsp_plan<<<wg, MT, 0, s>>>(a, b.scr_need, dc, true, true);
    bingo_count_launch();
    UCK(cudaGetLastError());
    {
        const uint64_t *ins[5] = {b.scr_need, a.cc_copy, a.cc_sel, a.cc_grp, a.cc_all};
        uint64_t *outs[5] = {b.scr_off, b.p_copy, b.p_sel, b.p_grp, b.p_all};
        UCK(exclusive_scan_u64_multi_dn(ins, outs, 5, pnt, ntmax, b.stmp, s));
    }
    k_bsp_totals<<<1, 32, 0, s>>>(a, dc, b.scr_off, b.dt, caps, b.abort);
    bingo_count_launch();
    UCK(cudaGetLastError());
    *dtot = b.dt;
    g_trace.mark("plan+scans+gate", s);
#define BSP_LAUNCH(kern, grid, strm, ...)                            \
    do {                                                             \
        kern<<<(grid), MT, 0, (strm)>>>(__VA_ARGS__);                \
        bingo_count_launch();                                        \
        UCK(cudaGetLastError());                                     \
    } while (0)
    BSP_LAUNCH(k_bsp_alloc_insert, wg, s, a);
    g_trace.mark("alloc_insert", s);
    cudaStream_t sh = g->aux_stream;
    UCK(cudaEventRecord(g->ev_fork, s));
    UCK(cudaStreamWaitEvent(sh, g->ev_fork, 0));
    // -- large vertices (side stream); item totals and hub counts are read on the device
    BSP_LAUNCH(k_bsp_copy, IG, sh, a, 0ull);
    const bool hix = g->hixo != nullptr && !hix_disabled();
    if (hix) {
        BSP_LAUNCH(k_hix_prep, hg, sh, a);
        BSP_LAUNCH(k_hix_build, IG, sh, a, 0ull);
    }
    BSP_LAUNCH(k_bsp_select, IG, sh, a, 0ull);
    if (hix) BSP_LAUNCH(k_hix_select, hg, sh, a);
    BSP_LAUNCH(k_bsp_finalize, hg, sh, a, true);
    if (hix) BSP_LAUNCH(k_hix_del, hg, sh, a);
    BSP_LAUNCH(k_bsp_hub_sort, hg, sh, a);
    k_bsp_sort_big<<<148, 256, 0, sh>>>(a);
    bingo_count_launch();
    UCK(cudaGetLastError());
    UCK(cudaMemsetAsync(a.nhubs + 5, 0, 4, sh));
    if (g->gixo) {
        BSP_LAUNCH(k_gix_prep, hg, sh, a);
        BSP_LAUNCH(k_gix_build, IG, sh, a, 0ull);
    }
    g_trace.mark("hub: select+finalize", sh);
    BSP_LAUNCH(k_bsp_hole_count, IG, sh, a, 0ull);
    UCK(exclusive_scan_u64_multi_dn(&a.icnt, const_cast<uint64_t **>(&a.ipref), 1, &b.dt->sel, g->isc_sel, itmp, sh));
    BSP_LAUNCH(k_bsp_hole_write, IG, sh, a, 0ull);
    BSP_LAUNCH(k_bsp_tail, hg, sh, a);
    g_trace.mark("hub: holes+tail", sh);
    if (hix) BSP_LAUNCH(k_hix_ins, hg, sh, a);
    if (g->gixo) BSP_LAUNCH(k_gix_front, hg, sh, a);
    BSP_LAUNCH(k_bsp_grp_count, IG, sh, a, 0ull);
    UCK(exclusive_scan_u64_multi_dn(&a.gcnt, const_cast<uint64_t **>(&a.gpref), 1, &b.dt->grp, g->isc_grp, itmp, sh));
    BSP_LAUNCH(k_bsp_grp_write, IG, sh, a, 0ull);
    BSP_LAUNCH(k_bsp_grp_sort, hg, sh, a);
    k_bsp_sort_big<<<148, 256, 0, sh>>>(a);
    bingo_count_launch();
    UCK(cudaGetLastError());
    BSP_LAUNCH(k_bsp_grp_tail, hg, sh, a);
    g_trace.mark("hub: group fronts+tails", sh);
    BSP_LAUNCH(k_bsp_rebuild_big, hg, sh, a);
    k_bsp_rebuild_fill<<<148 * 2, LT, 0, sh>>>(a);
    bingo_count_launch();
    UCK(cudaGetLastError());
    g_trace.mark("hub: rebuild_big", sh);
    // -- small vertices
    if (bsp_unfused()) {
        BSP_LAUNCH(k_bsp_finalize, wg, s, a, false);
        BSP_LAUNCH(k_bsp_rebuild, wg, s, a);
    } else {
        BSP_LAUNCH(k_bsp_small, wg, s, a);
    }
    g_trace.mark("small-vertex chain", s);
    UCK(cudaEventRecord(g->ev_join, sh));
    UCK(cudaStreamWaitEvent(s, g->ev_join, 0));
    g_trace.mark("join hub chain", s);
    if (g->nbt) {
        BSP_LAUNCH(k_bsp_nb_incr, wg, s, a);
        BSP_LAUNCH(k_bsp_nb_clear, IG, s, a, 0ull);
        BSP_LAUNCH(k_bsp_nb_fill, IG, s, a, 0ull);
    }
#undef BSP_LAUNCH
    k_upd_stats<<<(unsigned)std::min<uint64_t>((ntmax + 255) / 256, 148), 256, 0, s>>>(b.vstats, 0, dstats, pnt);
    bingo_count_launch();
    UCK(cudaGetLastError());
    return BINGO_OK;
}

static bingo_status finish_batch(bingo_graph *g, uint64_t n, uint64_t ntouch, uint32_t e,
                                 const unsigned long long *dstats, bingo_update_stats *stats, cudaStream_t s);

static cudaError_t float_fixup(bingo_graph *g, const uint32_t *tv, uint64_t ntouch, const uint32_t *fdoff,
                               const uint32_t *fdcap, cudaStream_t s) {
    if (!ntouch) return cudaSuccess;
    k_float_fixup<<<(unsigned)std::min<uint64_t>((ntouch + 7) / 8, 148 * 16), 256, 0, s>>>(
        tv, ntouch, g->hdr, g->arc, g->arc_dval, fdoff, fdcap, g->dec, g->dmem);
    bingo_count_launch();
    return cudaGetLastError();
}

static bool use_legacy_mutate() {
    const char *ev = getenv("BINGO_UPD_LEGACY");
    return ev && ev[0] == '1';
}

// BINGO_UPD_RADIX_FRONT=1: segment every batch with the radix sort (A/B, tests)
static bool use_radix_front() {
    const char *ev = getenv("BINGO_UPD_RADIX_FRONT");
    return ev && ev[0] == '1';
}

// BINGO_UPD_SYNC=1: the bulk-synchronous route with a host round trip after the front end
// and after the plan (apply_bsp) instead of the one-sync route (tests, A/B)
static bool use_sync_route() {
    const char *ev = getenv("BINGO_UPD_SYNC");
    return ev && ev[0] == '1';
}

// pinned host staging of the one-sync route: the plan totals / gate and the statistics
struct UpdHost {
    BspTotals t;
    unsigned long long stats[32];
};
static UpdHost *upd_host(bingo_graph *g) {
    if (!g->uhost) {
        void *h = nullptr;
        if (cudaMallocHost(&h, sizeof(UpdHost)) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        g->uhost = h;
    }
    return (UpdHost *)g->uhost;
}

static bingo_status finish_batch_host(bingo_graph *g, uint64_t n, uint64_t ntouch, uint32_t e,
                                      const unsigned long long *hs, bingo_update_stats *stats);

bingo_status apply_radix(bingo_graph *g, const bingo_update *batch, uint64_t n, uint32_t flags,
                         bingo_update_stats *stats, cudaStream_t s);

static bingo_status apply_impl(bingo_graph *g, const bingo_update *batch, const double *wf, uint64_t n,
                               uint32_t flags, bingo_update_stats *stats, void *stream);

extern "C" bingo_status bingo_apply_updates(bingo_graph *g, const bingo_update *batch, uint64_t n, uint32_t flags,
                                            bingo_update_stats *stats, void *stream) {
    return apply_impl(g, batch, nullptr, n, flags, stats, stream);
}

extern "C" bingo_status bingo_apply_updates_f64(bingo_graph *g, const bingo_update *batch, const double *bias_f64,
                                                uint64_t n, uint32_t flags, bingo_update_stats *stats, void *stream) {
    if (n && !bias_f64) return BINGO_E_INVAL;
    return apply_impl(g, batch, bias_f64, n, flags, stats, stream);
}

// restores g->cur_dins on every exit path of a float-mode batch
struct DinsGuard {
    bingo_graph *g;
    ~DinsGuard() { g->cur_dins = nullptr; }
};

// the batch again, segmented by the radix sort (a segment exceeded SEG_LONG_MAX records;
// nothing was mutated)
static bingo_status apply_radix_front(bingo_graph *g, const bingo_update *batch, const double *wf, uint64_t n,
                                      uint32_t flags, bingo_update_stats *stats, void *stream) {
    g->radix_front = true;
    const bingo_status st = apply_impl(g, batch, wf, n, flags, stats, stream);
    g->radix_front = false;
    return st;
}

static bingo_status apply_impl(bingo_graph *g, const bingo_update *batch, const double *wf, uint64_t n,
                               uint32_t flags, bingo_update_stats *stats, void *stream) {
    if (!g) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    if (n && !batch) return BINGO_E_INVAL;
    // float-bias graphs take real biases (bingo_apply_updates_f64, R-16); integer graphs do not
    if (n && g->float_mode != (wf != nullptr)) return BINGO_E_INVAL;
    if (n >= 0xFFFFFFFFull) return BINGO_E_INVAL;
    bingo_sq_quiesce(g, (cudaStream_t)stream);
    const bool fm = g->float_mode;
    g_trace.on = getenv("BINGO_UPD_TRACE") != nullptr;
    g_trace.mark("start", (cudaStream_t)stream);
    cudaStream_t s = (cudaStream_t)stream;
    if (stats) memset(stats, 0, sizeof(*stats));
    if (n == 0) {
        g->epoch++;
        if (stats) stats->epoch = g->epoch;
        return BINGO_OK;
    }
    if (g->radix_log2) return apply_radix(g, batch, n, flags, stats, s);   // radix-base graphs (radix.cu, R-19)
    // ---- small batches: single-launch fast path (falls through when it reports SLOW)
    if (n <= FAST_N && !fm) {
        bingo_status fst;
        if (try_fast_path(g, batch, n, flags, stats, s, &fst)) return fst;
    }
    // ---- scratch
    const size_t need = batch_scratch_bytes(n);
    if (g->scratch_bytes < need) {
        bingo_dev_free(g, g->scratch);
        g->scratch = bingo_dev_alloc(g, need);
        g->scratch_bytes = g->scratch ? need : 0;
        if (!g->scratch) return BINGO_E_NOMEM;
    }
    const size_t hneed = sizeof(UpdCounters) + 8 * 32;
    if (g->hscratch_bytes < hneed) {
        if (g->hscratch) cudaFreeHost(g->hscratch);
        g->hscratch = nullptr;
        g->hscratch_bytes = 0;
        UCK(cudaMallocHost(&g->hscratch, hneed));
        g->hscratch_bytes = hneed;
    }
    if (!use_legacy_mutate() && !fm) {
        const bingo_status st = ensure_gix_arrays(g, s);
        if (st != BINGO_OK) return upd_cuda_fail(g, cudaGetLastError(), "group index arrays");
    }
    Carve cv{(char *)g->scratch, 0};
    uint4 *drec = cv.take<uint4>(n);
    uint32_t *k0 = cv.take<uint32_t>(n), *v0 = cv.take<uint32_t>(n), *k1 = cv.take<uint32_t>(n),
             *v1 = cv.take<uint32_t>(n);
    uint64_t *rtmp = cv.take<uint64_t>(radix_tmp_words(n));
    uint64_t *head = cv.take<uint64_t>(n + 1), *head_ex = cv.take<uint64_t>(n + 2);
    uint64_t *stmp = cv.take<uint64_t>(scan_tmp_words(n + 1));
    uint32_t *seg = cv.take<uint32_t>(n + 1), *tv = cv.take<uint32_t>(n);
    uint64_t *scr_need = cv.take<uint64_t>(n + 1), *scr_off = cv.take<uint64_t>(n + 2);
    uint32_t *vstats = cv.take<uint32_t>((size_t)VST * n);
    uint8_t *route = cv.take<uint8_t>(n);
    uint32_t *large_list = cv.take<uint32_t>(n);
    UpdCounters *dc = cv.take<UpdCounters>(1);
    unsigned long long *dstats = cv.take<unsigned long long>(32);
    uint64_t *dins = cv.take<uint64_t>(n);
    double *dwf = cv.take<double>(n);
    uint32_t *fdoff = cv.take<uint32_t>(n), *fdcap = cv.take<uint32_t>(n);

    // records are validated into drec with internal vertex ids (the caller's batch is never written)
    const uint4 *src_recs = reinterpret_cast<const uint4 *>(batch);
    if (flags & BINGO_UPD_HOST_BATCH) {
        UCK(cudaMemcpyAsync(drec, batch, 16 * n, cudaMemcpyHostToDevice, s));
        src_recs = drec;
    }
    const uint4 *recs = drec;
    UCK(cudaMemsetAsync(dc, 0, sizeof(UpdCounters), s));
    UCK(cudaMemsetAsync(dstats, 0, 8 * 32, s));
    const unsigned gb = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
    // segmentation by source (a7): claim + count + place + in-segment order by default; the
    // 3-pass radix sort when BINGO_UPD_RADIX_FRONT=1 or a segment exceeds SEG_LONG_MAX records
    const bool radix_front = g->radix_front || use_radix_front();
    uint32_t *nlong = reinterpret_cast<uint32_t *>(head_ex + n + 1);
    const uint64_t nbins = ((uint64_t)std::max<uint32_t>(g->V, 1) + (1u << SEG_BSH) - 1) >> SEG_BSH;
    uint64_t *bcnt = nullptr, *boff = nullptr, *btmp = nullptr;
    if (!radix_front) {
        if (!g->vslot) {
            const size_t vs = 4 * (size_t)std::max<uint32_t>(g->V, 1);
            const size_t words = (nbins + 1) + (nbins + 2) + scan_tmp_words(nbins + 1);
            g->vslot = (uint32_t *)bingo_dev_alloc(g, vs + 8 * words + 256);
            if (!g->vslot) return BINGO_E_NOMEM;
            UCK(cudaMemsetAsync(g->vslot, 0xFF, vs, s));
        }
        bcnt = reinterpret_cast<uint64_t *>(((uintptr_t)(g->vslot + std::max<uint32_t>(g->V, 1)) + 255) & ~(uintptr_t)255);
        boff = bcnt + nbins + 1;
        btmp = boff + nbins + 2;
        UCK(cudaMemsetAsync(bcnt, 0, 8 * nbins, s));
        UCK(cudaMemsetAsync(head, 0, 8 * n, s));   // per-id record counts
        k_seg_claim<<<gb, 256, 0, s>>>(src_recs, drec, n, g->V, g->inv, g->vslot, k0, v0,
                                       reinterpret_cast<unsigned long long *>(bcnt), nlong, dc, fm);
    } else {
        k_upd_validate<<<gb, 256, 0, s>>>(src_recs, drec, n, g->V, g->inv, k0, v0, dc, fm);
    }
    bingo_count_launch();
    UCK(cudaGetLastError());
    DinsGuard dguard{g};
    if (fm) {
        const double *w = wf;
        if (flags & BINGO_UPD_HOST_BATCH) {
            UCK(cudaMemcpyAsync(dwf, wf, 8 * n, cudaMemcpyHostToDevice, s));
            w = dwf;
        }
        k_float_scale<<<gb, 256, 0, s>>>(drec, w, n, g->V, g->dec, dins, dc);
        bingo_count_launch();
        UCK(cudaGetLastError());
        g->cur_dins = dins;
    }
    const uint32_t *sv;
    const unsigned long long *d_ntouch;
    if (!radix_front) {
        UCK(exclusive_scan_u64(bcnt, boff, nbins, btmp, s));   // boff[nbins] = #touched
        const unsigned long long *ntc = reinterpret_cast<const unsigned long long *>(boff + nbins);
        unsigned long long *cnt = reinterpret_cast<unsigned long long *>(head);
        k_seg_count<<<gb, 256, 0, s>>>(n, k0, v0, g->vslot, boff, k1, tv, cnt);
        bingo_count_launch();
        UCK(cudaGetLastError());
        {
            const uint64_t *in = head;
            uint64_t *out = head_ex;
            UCK(exclusive_scan_u64_multi_dn(&in, &out, 1, ntc, n, stmp, s));
        }
        k_seg_place<<<gb, 256, 0, s>>>(n, k0, v0, k1, cnt, head_ex, v1, seg, g->vslot, ntc);
        bingo_count_launch();
        UCK(cudaGetLastError());
        k_seg_order<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(seg, v1, ntc, large_list,
                                                                                          nlong);
        bingo_count_launch();
        UCK(cudaGetLastError());
        k_seg_order_long<<<148, 1024, 0, s>>>(seg, v1, large_list, nlong, dc);
        bingo_count_launch();
        UCK(cudaGetLastError());
        sv = v1;
        d_ntouch = ntc;
    } else {
        bool in1 = false;
        UCK(radix_sort_pairs(k0, v0, k1, v1, n, key_bits_for(g->V), rtmp, s, &in1));
        const uint32_t *sk = in1 ? k1 : k0;
        sv = in1 ? v1 : v0;
        k_upd_heads<<<gb, 256, 0, s>>>(sk, n, head);
        bingo_count_launch();
        UCK(cudaGetLastError());
        UCK(exclusive_scan_u64(head, head_ex, n, stmp, s));   // head_ex[n] = #touched
        k_upd_segments<<<gb, 256, 0, s>>>(head_ex, sk, n, seg, tv);
        bingo_count_launch();
        UCK(cudaGetLastError());
        d_ntouch = reinterpret_cast<const unsigned long long *>(head_ex + n);
    }
    uint64_t ntouch = 0;
    g_trace.mark("front (validate+sort+seg)", s);
    const uint32_t e = g->epoch + 1;
    if (!fm && !use_legacy_mutate() && n <= bsp_maxt() && !use_sync_route()) {
        // one host sync per batch: the plan, the gate and every phase are enqueued at once
        BspTotals *dtot = nullptr;
        bingo_status st = apply_bsp_async(g, recs, sv, seg, tv, d_ntouch, n, e, dc, dstats, s, &dtot);
        if (st != BINGO_OK) return st;
        UpdHost *hh = upd_host(g);
        if (!hh) return BINGO_E_NOMEM;
        UCK(cudaMemcpyAsync(&hh->t, dtot, sizeof(BspTotals), cudaMemcpyDeviceToHost, s));
        UCK(cudaMemcpyAsync(hh->stats, dstats, sizeof(hh->stats), cudaMemcpyDeviceToHost, s));
        g_trace.mark("tail (stats)", s);
        UCK(cudaStreamSynchronize(s));
        g_trace.mark("sync", s);
        g_trace.dump();
        const int ab = hh->t.abort;
        ntouch = hh->t.nt;
        if (ab & 1) return BINGO_E_INVAL;
        if (ab & 4) return BINGO_E_OVERFLOW;
        if (ab & 8) return apply_radix_front(g, batch, wf, n, flags, stats, stream);
        if (!ab) return finish_batch_host(g, n, ntouch, e, hh->stats, stats);
        // something was short: nothing was mutated; the synchronous route grows and applies
        g->n_sync_reruns++;
        UCK(cudaMemsetAsync(dc, 0, sizeof(UpdCounters), s));   // the batch is valid (checked above)
        UCK(cudaMemsetAsync(dstats, 0, 8 * 32, s));
        st = apply_bsp(g, recs, sv, seg, tv, ntouch, e, dc, dstats, s);
        if (st != BINGO_OK) return st;
        return finish_batch(g, n, ntouch, e, dstats, stats, s);
    }
    UCK(cudaMemcpyAsync(&ntouch, d_ntouch, 8, cudaMemcpyDeviceToHost, s));
    {
        int *hfl = reinterpret_cast<int *>(g->hscratch);
        UCK(cudaMemcpyAsync(hfl, &dc->flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        UCK(cudaStreamSynchronize(s));
        if (*hfl & 8) return apply_radix_front(g, batch, wf, n, flags, stats, stream);
    }
    g_trace.mark("sync #touched", s);
    if (fm && ntouch) {
        // decimal-member regions for the batch; validation errors and pool growth before any mutation
        k_float_plan<<<(unsigned)std::min<uint64_t>((ntouch + 255) / 256, 148 * 16), 256, 0, s>>>(
            recs, sv, seg, tv, ntouch, dins, g->dec, g->counters, fdoff, fdcap);
        bingo_count_launch();
        UCK(cudaGetLastError());
        unsigned long long used = 0;
        int fl = 0;
        UCK(cudaMemcpyAsync(&used, g->counters + 3, 8, cudaMemcpyDeviceToHost, s));
        UCK(cudaMemcpyAsync(&fl, &dc->flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        UCK(cudaStreamSynchronize(s));
        if (fl & 1) return BINGO_E_INVAL;
        if (fl & 4) return BINGO_E_OVERFLOW;
        if (used > g->dmem_cap) {
            const uint64_t cap = std::max<uint64_t>(used + used / 4, g->dmem_cap + g->dmem_cap / 4);
            uint4 *nd = (uint4 *)bingo_dev_alloc(g, sizeof(uint4) * cap);
            if (!nd) return BINGO_E_NOMEM;
            UCK(cudaMemcpyAsync(nd, g->dmem, sizeof(uint4) * g->dmem_cap, cudaMemcpyDeviceToDevice, s));
            UCK(cudaStreamSynchronize(s));
            bingo_dev_free(g, g->dmem);
            g->dmem = nd;
            g->dmem_cap = cap;
        }
    }
    if (!use_legacy_mutate()) {
        const bingo_status st = apply_bsp(g, recs, sv, seg, tv, ntouch, e, dc, dstats, s);
        if (st != BINGO_OK) return st;
        if (fm) UCK(float_fixup(g, tv, ntouch, fdoff, fdcap, s));
        return finish_batch(g, n, ntouch, e, dstats, stats, s);
    }
    const bool bs = (g->flags & BINGO_BUILD_BS_MODE) != 0;
    uint32_t small_L = SMALL_L;
    if (const char *ev = getenv("BINGO_UPD_SMALL_L")) small_L = (uint32_t)strtoul(ev, nullptr, 10);
    const unsigned gp = (unsigned)std::min<uint64_t>((ntouch + 7) / 8, 148 * 32);
    k_upd_plan<<<gp ? gp : 1, 256, 0, s>>>(recs, sv, seg, tv, (uint32_t)ntouch, g->hdr, g->bkt, g->gcan, g->alpha, bs,
                                          g->arc_slack, g->member_slack, scr_need, dc, route, large_list,
                                          small_L);
    bingo_count_launch();
    UCK(cudaGetLastError());
    UCK(exclusive_scan_u64(scr_need, scr_off, ntouch, stmp, s));
    UpdCounters hc;
    unsigned long long bump[3];
    uint64_t scr_total = 0;
    UCK(cudaMemcpyAsync(&hc, dc, sizeof(hc), cudaMemcpyDeviceToHost, s));
    UCK(cudaMemcpyAsync(bump, g->counters, sizeof(bump), cudaMemcpyDeviceToHost, s));
    UCK(cudaMemcpyAsync(&scr_total, scr_off + ntouch, 8, cudaMemcpyDeviceToHost, s));
    UCK(cudaStreamSynchronize(s));
    // ---- capacity (grow pools before any mutation; NOMEM leaves the graph untouched)
    {
        const bingo_status st = check_capacity(g, hc, bump, s);
        if (st != BINGO_OK) return st;
    }
    // per-vertex delete scratch
    uint32_t *vscr = nullptr;
    const size_t vbytes = 4 * (scr_total + 64);
    if (scr_total) {
        if (g->vscratch_bytes < vbytes) {
            bingo_dev_free(g, g->vscratch);
            g->vscratch = bingo_dev_alloc(g, vbytes);
            g->vscratch_bytes = g->vscratch ? vbytes : 0;
            if (!g->vscratch) return BINGO_E_NOMEM;
        }
        vscr = (uint32_t *)g->vscratch;
    }
    // ---- mutate (from here on the batch is applied)
    MutateArgs ma;
    ma.recs = recs;
    ma.sval = sv;
    ma.seg = seg;
    ma.tv = tv;
    ma.scr_off = scr_off;
    ma.scr = vscr;
    ma.hdr = g->hdr;
    ma.thdr = g->thdr;
    ma.arc = g->arc;
    ma.arc_epoch = g->arc_epoch;
    ma.arc_dval = g->arc_dval;
    ma.dins = g->cur_dins;
    ma.bkt = g->bkt;
    ma.gcan = g->gcan;
    ma.mdst = g->mdst;
    ma.midx = g->midx;
    ma.nbt = g->nbt;
    ma.nbo = g->nbo;
    ma.nbtomb = g->nbtomb;
    ma.hixo = g->hixo;
    ma.hixt = g->hixt;
    ma.hix = g->hix;
    ma.hix_min = g->hix_min;
    ma.hix_cap = g->hix_cap;
    ma.gixo = g->gixo;
    ma.gixt = g->gixt;
    ma.gix = g->gix;
    ma.gix_min = g->gix_min;
    ma.gix_cap = g->gix_cap;
    ma.bump = g->counters;
    ma.vstats = vstats;
    ma.epoch = e;
    ma.alpha = g->alpha;
    ma.beta = g->beta;
    ma.hot_b = g->hot_bkt_degree;
    ma.hot_m = g->hot_mem_degree;
    ma.bs = bs;
    ma.arc_slack = g->arc_slack;
    ma.mem_slack = g->member_slack;
    if (ntouch) {
        // hubs (block kernel, side stream) overlap the small vertices (warp kernel): the two
        // sets are disjoint and only share the bump counters (atomics)
        const bool both = hc.n_large && hc.n_large < ntouch;
        if (both && !g->aux_stream) {
            UCK(cudaStreamCreateWithFlags(&g->aux_stream, cudaStreamNonBlocking));
            UCK(cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming));
            UCK(cudaEventCreateWithFlags(&g->ev_join, cudaEventDisableTiming));
        }
        cudaStream_t sl = both ? g->aux_stream : s;
        if (both) {
            UCK(cudaEventRecord(g->ev_fork, s));
            UCK(cudaStreamWaitEvent(sl, g->ev_fork, 0));
        }
        if (hc.n_large) {
            k_upd_mutate_block<<<(unsigned)std::min<uint64_t>(hc.n_large, 148ull * 2), LT, 0, sl>>>(ma, large_list,
                                                                                                hc.n_large);
            bingo_count_launch();
            UCK(cudaGetLastError());
        }
        if (hc.n_large < ntouch) {
            const unsigned gs = (unsigned)std::min<uint64_t>((ntouch + MT / 32 - 1) / (MT / 32), 148ull * 8);
            k_upd_mutate_warp<<<gs, MT, 0, s>>>(ma, route, (uint32_t)ntouch);
            bingo_count_launch();
            UCK(cudaGetLastError());
        }
        if (both) {
            UCK(cudaEventRecord(g->ev_join, sl));
            UCK(cudaStreamWaitEvent(s, g->ev_join, 0));
        }
        k_upd_stats<<<(unsigned)std::min<uint64_t>((ntouch + 255) / 256, 148), 256, 0, s>>>(vstats, (uint32_t)ntouch,
                                                                                            dstats);
        bingo_count_launch();
        UCK(cudaGetLastError());
    }
    if (fm) UCK(float_fixup(g, tv, ntouch, fdoff, fdcap, s));
    return finish_batch(g, n, ntouch, e, dstats, stats, s);
}

static bingo_status finish_batch(bingo_graph *g, uint64_t n, uint64_t ntouch, uint32_t e,
                                 const unsigned long long *dstats, bingo_update_stats *stats, cudaStream_t s) {
    unsigned long long hs[32];
    g_trace.mark("tail (nb, stats)", s);
    UCK(cudaMemcpyAsync(hs, dstats, sizeof(hs), cudaMemcpyDeviceToHost, s));
    UCK(cudaStreamSynchronize(s));
    g_trace.mark("sync stats", s);
    g_trace.dump();
    return finish_batch_host(g, n, ntouch, e, hs, stats);
}

static bingo_status finish_batch_host(bingo_graph *g, uint64_t n, uint64_t ntouch, uint32_t e,
                                      const unsigned long long *hs, bingo_update_stats *stats) {
    if (hs[31]) {   // an internal index inconsistency (never expected): fail loudly, graph unusable
        fprintf(stderr, "libbingo: group index inconsistency in %llu vertices\n", hs[31]);
        g->poisoned = 1;
        return BINGO_E_CUDA;
    }
    g->epoch = e;
    // inserted = number of insert records (validated batch)
    uint64_t inserted = 0;
    {
        // count inserts on the host side cheaply from the stats: deleted + missing = #delete records
        const uint64_t dels = hs[0] + hs[1];
        inserted = n - dels;
    }
    g->num_arcs = g->num_arcs + inserted - hs[0];
    if (stats) {
        stats->inserted = inserted;
        stats->deleted = hs[0];
        stats->missing_deletes = hs[1];
        stats->touched_vertices = ntouch;
        for (int i = 0; i < 25; i++) stats->kind_transitions[i / 5][i % 5] = hs[2 + i];
        stats->epoch = e;
    }
    return BINGO_OK;
}


// ---------------------------------------------------------------- hub delete index at build time
// Tables for every vertex with d > min_d, min_d the smallest of 1024 / 4096 / 16384 / 65536
// whose tables fit 15% of the free device memory (c2: 2,411 vertices, 13.5% of the arcs,
// 212 MB).  Called by bingo_build; a graph without room keeps no tables (scans only).
bingo_status hix_build_all(bingo_graph *g, cudaStream_t s) {
    if (hix_disabled() || g->V == 0 || g->float_mode || !index_wanted(g)) return BINGO_OK;
    const uint64_t V = g->V;
    uint64_t *items = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * (V + 1));
    uint64_t *words = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * (V + 1));
    uint64_t *pref = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * (V + 2));
    uint64_t *woff = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * (V + 2));
    uint64_t *tmp = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * scan_tmp_words(V + 1));
    bingo_status st = BINGO_OK;
    auto fin = [&](bingo_status r) {
        bingo_dev_free(g, items); bingo_dev_free(g, words); bingo_dev_free(g, pref); bingo_dev_free(g, woff);
        bingo_dev_free(g, tmp);
        return r;
    };
    if (!items || !words || !pref || !woff || !tmp) return fin(BINGO_OK);   // no room: no tables
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const unsigned eg = (unsigned)std::min<uint64_t>((V + 255) / 256, 148ull * 16);
    const uint32_t m0 = index_min();
    const uint32_t mins[4] = {m0, 4 * m0, 16 * m0, 64 * m0};
    for (uint32_t min_d : mins) {
        k_hix_sizes<<<eg, 256, 0, s>>>(g->V, g->hdr, min_d, items, words);
        bingo_count_launch();
        const uint64_t *ins[2] = {items, words};
        uint64_t *outs[2] = {pref, woff};
        if (cudaGetLastError() != cudaSuccess || exclusive_scan_u64_multi(ins, outs, 2, V, tmp, s) != cudaSuccess)
            return fin(BINGO_E_CUDA);
        uint64_t tot[2] = {0, 0};
        if (cudaMemcpyAsync(&tot[0], pref + V, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaMemcpyAsync(&tot[1], woff + V, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return fin(BINGO_E_CUDA);
        if (!tot[0]) break;                                   // no vertex that large
        if (4.0 * (double)tot[1] > 0.15 * (double)free_b) continue;   // does not fit: a higher threshold
        const uint64_t cap = tot[1] + tot[1] / 4 + 1024;
        g->hixo = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * V);
        g->hixt = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * V);
        g->hix = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * cap);
        if (!g->hixo || !g->hixt || !g->hix) {
            bingo_dev_free(g, g->hixo); bingo_dev_free(g, g->hixt); bingo_dev_free(g, g->hix);
            g->hixo = nullptr; g->hixt = nullptr; g->hix = nullptr;
            return fin(BINGO_OK);
        }
        g->hix_cap = cap;
        g->hix_min = min_d;
        const unsigned long long used = tot[1];
        if (cudaMemsetAsync(g->hix, 0, sizeof(uint32_t) * cap, s) != cudaSuccess ||
            cudaMemsetAsync(g->hixt, 0, sizeof(uint32_t) * V, s) != cudaSuccess ||
            cudaMemcpyAsync(g->counters + 5, &used, 8, cudaMemcpyHostToDevice, s) != cudaSuccess)
            return fin(BINGO_E_CUDA);
        k_hix_offsets<<<eg, 256, 0, s>>>(g->V, g->hdr, min_d, woff, g->hixo);
        bingo_count_launch();
        k_hix_fill<<<(unsigned)std::min<uint64_t>((tot[0] + 7) / 8, 148ull * 32), MT, 0, s>>>(
            g->V, pref, tot[0], g->hdr, g->arc, g->hixo, g->hix);
        bingo_count_launch();
        if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) return fin(BINGO_E_CUDA);
        break;
    }
    return fin(st);
}


// ---------------------------------------------------------------- group index at build time
// Tables for every vertex with d > min_d, min_d the smallest of 1024 / 4096 / 16384 / 65536
// whose tables fit 15% of the free device memory; the pool gets 25% more for the tables that
// later batches rebuild (a dropped index, a vertex growing past min_d).  Called by bingo_build
// after the hub delete index; a graph without room keeps no tables (member-list scans only).
bingo_status gix_build_all(bingo_graph *g, cudaStream_t s) {
    if (!gix_enabled() || g->V == 0 || g->float_mode) return BINGO_OK;
    if (!index_wanted(g)) {
        g->gix_full = true;   // no group index for this graph (no lazy arrays either)
        return BINGO_OK;
    }
    const uint64_t V = g->V;
    uint64_t *words = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * (V + 1));
    uint64_t *woff = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * (V + 2));
    uint64_t *tmp = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * scan_tmp_words(V + 1));
    uint32_t *list = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * (V + 1));
    auto fin = [&](bingo_status r) {
        bingo_dev_free(g, words); bingo_dev_free(g, woff); bingo_dev_free(g, tmp); bingo_dev_free(g, list);
        return r;
    };
    if (!words || !woff || !tmp || !list) return fin(BINGO_OK);   // no room: no tables
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const unsigned eg = (unsigned)std::min<uint64_t>((V + 255) / 256, 148ull * 16);
    const unsigned wg = (unsigned)std::min<uint64_t>((V + 7) / 8, 148ull * 32);
    const uint32_t m0 = index_min();
    const uint32_t mins[4] = {m0, 4 * m0, 16 * m0, 64 * m0};
    uint32_t *nlist = list + V;
    for (uint32_t min_d : mins) {
        k_gix_sizes<<<wg, MT, 0, s>>>(g->V, g->hdr, g->bkt, g->gcan, min_d, words, nullptr, nullptr);
        bingo_count_launch();
        if (cudaGetLastError() != cudaSuccess || exclusive_scan_u64(words, woff, V, tmp, s) != cudaSuccess)
            return fin(BINGO_E_CUDA);
        uint64_t tot = 0;
        if (cudaMemcpyAsync(&tot, woff + V, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return fin(BINGO_E_CUDA);
        if (!tot) break;                                                   // no vertex that large
        if (4.0 * 1.25 * (double)tot > 0.15 * (double)free_b) continue;   // does not fit: a higher threshold
        const uint64_t cap = std::max<uint64_t>(tot + tot / 4, 1u << 20);
        g->gixo = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * V);
        g->gixt = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * V);
        g->gix = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * cap);
        if (!g->gixo || !g->gixt || !g->gix) {
            bingo_dev_free(g, g->gixo); bingo_dev_free(g, g->gixt); bingo_dev_free(g, g->gix);
            g->gixo = nullptr; g->gixt = nullptr; g->gix = nullptr;
            return fin(BINGO_OK);
        }
        g->gix_cap = cap;
        g->gix_min = min_d;
        const unsigned long long used = tot;
        if (cudaMemsetAsync(g->gix, 0, sizeof(uint32_t) * cap, s) != cudaSuccess ||
            cudaMemsetAsync(g->gixt, 0, sizeof(uint32_t) * V, s) != cudaSuccess ||
            cudaMemsetAsync(nlist, 0, 4, s) != cudaSuccess ||
            cudaMemcpyAsync(g->counters + 6, &used, 8, cudaMemcpyHostToDevice, s) != cudaSuccess)
            return fin(BINGO_E_CUDA);
        k_gix_sizes<<<wg, MT, 0, s>>>(g->V, g->hdr, g->bkt, g->gcan, min_d, words, list, nlist);
        bingo_count_launch();
        k_gix_offsets<<<eg, 256, 0, s>>>(g->V, words, woff, g->gixo);
        bingo_count_launch();
        uint32_t nl = 0;
        if (cudaGetLastError() != cudaSuccess || cudaMemcpyAsync(&nl, nlist, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return fin(BINGO_E_CUDA);
        if (nl) {
            k_gix_fill<<<(unsigned)std::min<uint32_t>(nl, 148u * 8), 256, 0, s>>>(list, nl, g->hdr, g->bkt, g->gcan,
                                                                                   g->midx, g->gixo, g->gix);
            bingo_count_launch();
        }
        if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) return fin(BINGO_E_CUDA);
        return fin(BINGO_OK);
    }
    g->gix_full = true;   // no threshold fits the budget: no group index for this graph
    return fin(BINGO_OK);
}


// ---------------------------------------------------------------- streaming queue (host side)
void bingo_sq_quiesce(bingo_graph *g, cudaStream_t s) {
    if (!g || !g->sq_running) return;
    StreamQ *q = (StreamQ *)g->sq_host;
    __atomic_store_n(&q->run_gen, 0u, __ATOMIC_SEQ_CST);   // generations start at 1: the kernel exits
    if (s != g->sq_stream) cudaStreamWaitEvent(s, g->sq_ev, 0);
    g->sq_running = false;
}

void bingo_sq_release(bingo_graph *g) {
    if (!g || !g->sq_host) return;
    bingo_sq_quiesce(g, g->sq_stream);
    if (g->sq_ev) {
        cudaEventSynchronize(g->sq_ev);
        cudaEventDestroy(g->sq_ev);
    }
    cudaFreeHost(g->sq_host);
    g->sq_host = g->sq_dev = nullptr;
    g->sq_ev = nullptr;
}

static bingo_status sq_launch(bingo_graph *g, cudaStream_t s) {
    if (!g->sq_host) {
        void *h = nullptr;
        if (cudaHostAlloc(&h, sizeof(StreamQ), cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            return BINGO_E_NOMEM;
        }
        memset(h, 0, sizeof(StreamQ));
        if (cudaHostGetDevicePointer(&g->sq_dev, h, 0) != cudaSuccess ||
            cudaEventCreateWithFlags(&g->sq_ev, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            cudaFreeHost(h);
            return BINGO_E_CUDA;
        }
        g->sq_host = h;
    }
    if (!ensure_fast_scratch(g)) return BINGO_E_NOMEM;
    {   // the static shared memory of upd_fast_body plus one warp's delete scratch exceed 48 KB:
        // raise the dynamic limit once per device (the attribute is per device)
        static std::atomic<uint64_t> sq_smem_set{0};
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t bit = 1ull << (dev & 63);
        if (!(sq_smem_set.load(std::memory_order_acquire) & bit)) {
            if (cudaFuncSetAttribute(k_stream_upd, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * WARP_SCR_WORDS) !=
                cudaSuccess)
                return upd_cuda_fail(g, cudaGetLastError(), "k_stream_upd smem attribute");
            sq_smem_set.fetch_or(bit, std::memory_order_acq_rel);
        }
    }
    StreamQ *q = (StreamQ *)g->sq_host;
    FastArgs fa;
    fill_fast_common(g, fa);
    fa.n = 1;
    const unsigned gen = ++g->sq_gen ? g->sq_gen : ++g->sq_gen;   // never 0 (0 = stopped)
    __atomic_store_n(&q->run_gen, gen, __ATOMIC_SEQ_CST);
    k_stream_upd<<<1, LT, 4 * WARP_SCR_WORDS, s>>>(fa, (StreamQ *)g->sq_dev, g->sq_seq, gen);
    bingo_count_launch();
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaEventRecord(g->sq_ev, s);
    if (e != cudaSuccess) return upd_cuda_fail(g, e, "k_stream_upd");
    g->sq_stream = s;
    g->sq_running = true;
    return BINGO_OK;
}

extern "C" bingo_status bingo_stream_update(bingo_graph *g, const bingo_update *rec, bingo_update_stats *stats,
                                            void *stream) {
    if (!g || !rec) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    if (g->float_mode || g->radix_log2) return BINGO_E_INVAL;   // float graphs take real biases; radix graphs update through bingo_apply_updates (R-19)
    cudaStream_t s = (cudaStream_t)stream;
    if (stats) memset(stats, 0, sizeof(*stats));
    if (g->sq_running && g->sq_stream != s) bingo_sq_quiesce(g, s);
    StreamQ *q = (StreamQ *)g->sq_host;
    const unsigned k = g->sq_seq;
    unsigned int dw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int attempt = 0;; attempt++) {
        if (!g->sq_running) {
            const bingo_status st = sq_launch(g, s);
            if (st != BINGO_OK) return st;
            q = (StreamQ *)g->sq_host;
        }
        const unsigned gen = g->sq_gen;
        StreamSlot *sl = &q->slot[k % SQ_N];
        __atomic_store_n(&sl->chk, k + 1, __ATOMIC_RELEASE);
        memcpy((void *)&sl->rec, rec, 16);
        __atomic_store_n(&sl->gen, gen, __ATOMIC_RELEASE);
        __atomic_store_n(&sl->seq, k + 1, __ATOMIC_SEQ_CST);
        bool taken = false;
        for (uint64_t spin = 0;; spin++) {
            if (__atomic_load_n(&q->done.w[0], __ATOMIC_ACQUIRE) == k + 1) {
                // one 32 B device store: re-read until w0 and w7's check bits agree (a torn read)
                for (;;) {
                    for (int j = 7; j >= 0; j--) dw[j] = __atomic_load_n(&q->done.w[j], __ATOMIC_ACQUIRE);
                    if (dw[0] == k + 1 && (dw[7] >> 22) == ((k + 1) & 0x3FFu)) break;
                }
                taken = true;
                break;
            }
            if (__atomic_load_n(&q->exit_gen, __ATOMIC_ACQUIRE) == gen &&
                __atomic_load_n(&q->exit_seq, __ATOMIC_ACQUIRE) == k &&
                __atomic_load_n(&q->done.w[0], __ATOMIC_ACQUIRE) != k + 1) {
                g->sq_running = false;   // idle exit raced with the post: relaunch and repost
                break;
            }
            if ((spin & 0xFFFFF) == 0xFFFFF) {   // a dead context must not spin forever
                const cudaError_t e = cudaStreamQuery(s);
                if (e != cudaSuccess && e != cudaErrorNotReady) return upd_cuda_fail(g, e, "k_stream_upd");
            }
        }
        if (taken) break;
        if (attempt >= 2) {
            // the kernel keeps exiting before it sees the record: launches are being serialised
            // (a profiler replaying kernels one at a time).  Apply this record with one launch.
            __atomic_store_n(&sl->seq, 0u, __ATOMIC_SEQ_CST);
            return apply_impl(g, rec, nullptr, 1, BINGO_UPD_HOST_BATCH, stats, stream);
        }
    }
    g->sq_seq = k + 1;
    const uint32_t st = dw[1] & 15u;
    if (st == FAST_INVAL) return BINGO_E_INVAL;
    if (st == FAST_OVERFLOW) return BINGO_E_OVERFLOW;
    if (st == FAST_SLOW) {   // the kernel has exited; this record goes through the batched pipeline
        g->sq_running = false;
        return apply_impl(g, rec, nullptr, 1, BINGO_UPD_HOST_BATCH, stats, stream);
    }
    if (st != FAST_OK) return upd_cuda_fail(g, cudaErrorUnknown, "k_stream_upd status");
    g->epoch++;
    uint64_t inserted, deleted, missing, ntouch, tr[25];
    if (dw[1] >> 31) {   // the statistics did not fit the packed completion
        const FastOut &o = q->out;
        inserted = o.inserted;
        deleted = o.stats[0];
        missing = o.stats[1];
        ntouch = o.ntouch;
        for (int i = 0; i < 25; i++) tr[i] = o.stats[2 + i];
    } else {
        inserted = (dw[1] >> 8) & 255u;
        missing = (dw[1] >> 16) & 255u;
        ntouch = (dw[1] >> 4) & 15u;
        deleted = dw[2];
        const uint64_t f0 = (uint64_t)dw[3] | (uint64_t)dw[4] << 32, f1 = (uint64_t)dw[5] | (uint64_t)dw[6] << 32,
                       f2 = dw[7] & 0x3FFFFFu;
        const uint64_t f[3] = {f0, f1, f2};
        for (int i = 0; i < 25; i++) {
            const int b = 6 * i;
            uint64_t c = f[b >> 6] >> (b & 63);
            if ((b & 63) > 58) c |= f[(b >> 6) + 1] << (64 - (b & 63));
            tr[i] = c & 63u;
        }
    }
    g->num_arcs = g->num_arcs + inserted - deleted;
    if (stats) {
        stats->inserted = inserted;
        stats->deleted = deleted;
        stats->missing_deletes = missing;
        stats->touched_vertices = ntouch;
        for (int i = 0; i < 25; i++) stats->kind_transitions[i / 5][i % 5] = tr[i];
        stats->epoch = g->epoch;
    }
    return BINGO_OK;
}

#ifdef BINGO_SQ_TRACE
extern "C" int bingo_sq_trace_read(unsigned long long *host, int n) {
    if (n > (int)SQT_N) n = SQT_N;
    return (int)cudaMemcpyFromSymbol(host, g_sqt, sizeof(unsigned long long) * 8 * n);
}
#endif

// ---------------------------------------------------------------- replica state exchange (f1)
// bingo_export_vertices / bingo_import_vertices: include/bingo.h, exchange.cuh.
static bool exchange_supported(const bingo_graph *g) {
    return !g->float_mode && !g->radix_log2 && !g->nbt;
}

extern "C" bingo_status bingo_export_vertices(bingo_graph *g, const uint32_t *ids, uint32_t n, uint32_t *buf,
                                              uint64_t cap_words, uint64_t *offsets, uint64_t *words_out,
                                              void *stream) {
    if (!g || !offsets || !words_out || (n && !ids)) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    if (!exchange_supported(g)) return BINGO_E_INVAL;
    cudaStream_t s = (cudaStream_t)stream;
    bingo_sq_quiesce(g, s);
    *words_out = 0;
    if (n == 0) {
        if (cudaMemsetAsync(offsets, 0, sizeof(uint64_t), s) != cudaSuccess) return upd_cuda_fail(g, cudaGetLastError(), "export");
        return BINGO_OK;
    }
    uint64_t *sizes = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * (n + 1));
    uint64_t *tmp = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * scan_tmp_words(n + 1));
    int *bad = (int *)bingo_dev_alloc(g, sizeof(int));
    auto fin = [&](bingo_status r) {
        bingo_dev_free(g, sizes);
        bingo_dev_free(g, tmp);
        bingo_dev_free(g, bad);
        return r;
    };
    if (!sizes || !tmp || !bad) return fin(BINGO_E_NOMEM);
    ExArgs a;
    a.hdr = g->hdr;
    a.arc = g->arc;
    a.ep = g->arc_epoch;
    a.bkt = g->bkt;
    a.gcan = g->gcan;
    a.midx = g->midx;
    a.inv = g->inv;
    a.ids = ids;
    a.n = n;
    a.V = g->V;
    a.words = sizes;
    a.buf = buf;
    int hbad = 0;
    uint64_t total = 0;
    cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), s);
    if (e == cudaSuccess) {
        k_check_ids<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 1184), 256, 0, s>>>(ids, n, g->V, bad);
        bingo_count_launch();
        k_ex_sizes<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 1184), 256, 0, s>>>(a);
        bingo_count_launch();
        e = exclusive_scan_u64(sizes, offsets, n, tmp, s);
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&total, offsets + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fin(upd_cuda_fail(g, e, "export sizes"));
    if (hbad) return fin(BINGO_E_INVAL);
    *words_out = total;
    if (!buf) return fin(BINGO_OK);
    if (total > cap_words) return fin(BINGO_E_OVERFLOW);
    a.words = offsets;
    k_ex_fill<<<(unsigned)std::min<uint64_t>(((uint64_t)n + 7) / 8, 148ull * 16), 256, 0, s>>>(a);
    bingo_count_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fin(upd_cuda_fail(g, e, "export fill"));
    return fin(BINGO_OK);
}

extern "C" bingo_status bingo_import_vertices(bingo_graph *g, const uint32_t *buf, const uint64_t *offsets, uint32_t n,
                                              void *stream) {
    if (!g || (n && (!buf || !offsets))) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    if (!exchange_supported(g)) return BINGO_E_INVAL;
    if (n == 0) return BINGO_OK;
    cudaStream_t s = (cudaStream_t)stream;
    bingo_sq_quiesce(g, s);
    uint64_t *need = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * 3 * (n + 1));
    uint64_t *pref = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * 3 * (n + 1));
    uint64_t *tmp = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * 3 * scan_tmp_words(n + 1));
    long long *darcs = (long long *)bingo_dev_alloc(g, sizeof(long long) * 2);   // [0] arcs delta, [1] bad flag
    auto fin = [&](bingo_status r) {
        bingo_dev_free(g, need);
        bingo_dev_free(g, pref);
        bingo_dev_free(g, tmp);
        bingo_dev_free(g, darcs);
        return r;
    };
    if (!need || !pref || !tmp || !darcs) return fin(BINGO_E_NOMEM);
    ImArgs a;
    memset(&a, 0, sizeof(a));
    a.buf = buf;
    a.off = offsets;
    a.n = n;
    a.hdr = g->hdr;
    a.bkt = g->bkt;
    a.gcan = g->gcan;
    a.arc_slack = g->arc_slack;
    a.mem_slack = g->member_slack;
    a.hot_b = g->hot_bkt_degree;
    a.hot_m = g->hot_mem_degree;
    a.need = need;
    a.pref = pref;
    a.darcs = darcs;
    a.bad = reinterpret_cast<int *>(darcs + 1);
    a.V = g->V;
    const unsigned grid = (unsigned)std::min<uint64_t>(((uint64_t)n + 7) / 8, 148ull * 16);
    unsigned long long bump[3] = {0, 0, 0};
    uint64_t tot[3] = {0, 0, 0};
    cudaError_t e = cudaMemsetAsync(darcs, 0, sizeof(long long) * 2, s);
    if (e == cudaSuccess) {
        k_im_plan<<<grid, 256, 0, s>>>(a);
        bingo_count_launch();
        const uint64_t *in[3] = {need, need + (n + 1), need + 2 * (n + 1)};
        uint64_t *out[3] = {pref, pref + (n + 1), pref + 2 * (n + 1)};
        e = exclusive_scan_u64_multi(in, out, 3, n, tmp, s);
    }
    for (int k = 0; k < 3 && e == cudaSuccess; k++)
        e = cudaMemcpyAsync(&tot[k], pref + k * (n + 1) + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(bump, g->counters, sizeof(bump), cudaMemcpyDeviceToHost, s);
    int hbad = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, a.bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fin(upd_cuda_fail(g, e, "import plan"));
    if (hbad) return fin(BINGO_E_INVAL);
    // pool growth first: nothing is written before every pool is large enough
    bingo_status st;
    if (bump[0] + tot[0] > g->arc_cap && (st = grow_pool(g, 0, bump[0] + tot[0], s)) != BINGO_OK)
        return fin(st == BINGO_E_CUDA ? (g->poisoned = 1, st) : st);
    if (bump[1] + tot[1] > g->bkt_cap && (st = grow_pool(g, 1, bump[1] + tot[1], s)) != BINGO_OK)
        return fin(st == BINGO_E_CUDA ? (g->poisoned = 1, st) : st);
    if (bump[2] + tot[2] > g->mem_cap / 4 && (st = grow_pool(g, 2, bump[2] + tot[2], s)) != BINGO_OK)
        return fin(st == BINGO_E_CUDA ? (g->poisoned = 1, st) : st);
    a.thdr = g->thdr;
    a.arc = g->arc;
    a.ep = g->arc_epoch;
    a.bkt = g->bkt;
    a.gcan = g->gcan;
    a.midx = g->midx;
    a.mdst = g->mdst;
    a.hixo = g->hixo;
    a.gixo = g->gixo;
    for (int k = 0; k < 3; k++) a.bump[k] = bump[k];
    k_im_install<<<grid, 256, 0, s>>>(a);
    bingo_count_launch();
    unsigned long long nb[3] = {bump[0] + tot[0], bump[1] + tot[1], bump[2] + tot[2]};
    long long hd = 0;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->counters, nb, sizeof(nb), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hd, darcs, sizeof(long long), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fin(upd_cuda_fail(g, e, "import install"));
    g->num_arcs = (uint64_t)((long long)g->num_arcs + hd);
    return fin(BINGO_OK);
}
