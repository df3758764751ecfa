// update_bsp.cuh -- the bulk-synchronous batched update (included by update.cu).
//
// Same semantics as mutate_vertex (insert -> delete -> rebuild per touched
// vertex, readings R-6/R-8), restructured for the GPU: every phase is
// ONE wide kernel over all touched vertices of the batch, with the per-vertex
// state held in global structure-of-arrays between phases, and every O(degree)
// scan split into chunk ITEMS of CH adjacency positions (or member slots) that
// are spread over the whole GPU, one warp per item.  A hub's delete scan
// therefore runs on hundreds of SMs instead of one block, and a small vertex's
// ~25 dependent round trips are paid once per phase for the whole batch instead
// of once per vertex-wave.
//
//   plan          (warp / vertex)  pre-batch groups, demand, chunk-item counts
//   alloc_insert  (warp / vertex)  relocations, member growth, inserts (batch
//                                  order), delete-scratch init
//   copy          (warp / item)    adjacency relocation copies
//   select        (warp / item)    round 0 of the (epoch, position) selection
//   finalize      (warp / vertex)  picks, further rounds for repeated deletes,
//                                  per-group delete counts
//   hole_count / scan / hole_write (warp / item)   holes = marked positions
//                                  < L' in ascending order
//   tail          (warp / vertex)  adjacency tail window fills the holes (R-6)
//   grp_count / scan / grp_write (warp / item)     group fronts: holes in slot
//                                  order + renames of moved arcs
//   grp_tail      (warp / vertex)  group tail windows fill the holes (R-6)
//   rebuild       (warp / vertex)  Eq.9 reclassification, member
//                                  materialisation, integer Vose (R-4)
//   nb_clear / nb_fill (warp / item)   node2vec neighbour sets (optional)
#pragma once

namespace bingo {

// minimum resident blocks for the latency-bound warp-per-vertex / chunk-item kernels
// (more warps in flight hide the dependent round trips of each vertex)
#ifndef BINGO_BSP_MINB
#define BINGO_BSP_MINB 8
#endif

static constexpr uint32_t CH = 1024;   // adjacency positions / member slots per chunk item (32 per lane)
static constexpr uint32_t BSP_MAXT = 1u << 21;   // touched vertices per sub-batch (state ~1.1 KB each)
enum : uint32_t { GK_KIND0 = 0, GK_C, GK_INSK, GK_DELK, GK_MOFF, GK_CAP, GK_ONE, GK_GHO, GK_GHN, GK_N };
// hubs whose batch deletes at most SORT_MAX arcs take their holes by sorting their picks and
// their group holes by one pass over each group front (appends, then a sort); larger ones
// use the counted-rank passes (k_bsp_hole_count / k_bsp_grp_count + scans)
static constexpr uint32_t SORT_MAX = 4096;

struct BspArgs {
    MutateArgs g;                  // graph, batch (global touched index), delete scratch, vstats (local)
    uint32_t t0, nt;               // this sub-batch: touched vertices [t0, t0 + nt); local i = t - t0
    uint32_t *vL, *vq, *vm, *vN, *vmiss, *vlist0, *vacap, *vmoved;
    uint64_t *vaoff;
    uint32_t *gk;                  // [GK_N][nt][32]: lane k = radix group k
    uint64_t *cc_copy, *cc_sel, *cc_grp, *cc_all;          // chunk items per vertex (plan)
    const uint64_t *p_copy, *p_sel, *p_grp, *p_all;        // their exclusive prefixes [nt + 1]
    uint64_t *icnt;                // per select item: holes in its chunk
    const uint64_t *ipref;
    uint64_t *gcnt;                // per group item: deleted slots in its chunk
    const uint64_t *gpref;
    uint32_t *hubs, *nhubs;        // large vertices (L > CH) with deletes, any order
    uint32_t *bigs, *nbigs;        // all large vertices, any order
    uint32_t *vhix;                // hub delete index: 0 not maintained (invalidated), 1 used, 2 built + used
    uint64_t *vnbo;                // pre-batch nbo[u] (node2vec neighbour sets)
    uint32_t *vnbfull;             // 1: the vertex's neighbour set is rebuilt from its adjacency
    uint32_t *vrank;               // hubs: 1 = counted-rank passes (N > SORT_MAX), 0 = sorted picks
    uint2 *sorts;                  // (vertex, 32 = picks | group k) lists longer than a warp, for k_bsp_sort_big
    uint32_t *vgix;                // group index this batch: 0 none, 1 used, 2 built + used, 3 build failed (scan)
    uint32_t *vgixe;               // plan: list-group members after the inserts (group index entries)
    unsigned long long *err;       // internal inconsistencies found (group index); the host fails the call
    // one-sync route (apply_bsp_async): the launches are enqueued before the host knows the
    // touched-vertex count or the item totals, so kernels read them on the device
    const unsigned long long *pnt; // non-null: nt = *pnt (t0 = 0); else the host value nt
    uint32_t gks;                  // stride of the gk slots (>= nt)
    const int *abort;              // non-null: k_bsp_check's verdict; nonzero = mutate nothing
};

__device__ __forceinline__ uint32_t *gkp(const BspArgs &a, uint32_t f, uint32_t i) {
    return a.gk + ((uint64_t)f * a.gks + i) * 32;
}
__device__ __forceinline__ uint32_t bsp_nt(const BspArgs &a) {
    return a.pnt ? (uint32_t)*a.pnt : a.nt;
}
// item totals: the host value, or (one-sync route) the prefix total of the plan
__device__ __forceinline__ uint64_t bsp_total(const BspArgs &a, const uint64_t *pref, uint64_t total) {
    return a.pnt ? pref[bsp_nt(a)] : total;
}
#define BSP_ABORTED(a) ((a).abort && *(volatile const int *)(a).abort)

// per-vertex delete scratch (words from plan: bsp_scr_words)
struct DelScr {
    uint32_t *bm, *hkey, *hk, *hfound, *hsel, *holes, *R, *gh;
    uint2 *pk;                      // hubs: the picks (position, bias) in pick order (group index)
    unsigned long long *hbest, *hprev;
    uint32_t Hq;
};
__host__ __device__ inline uint64_t bsp_scr_words(uint32_t L, uint32_t q, uint32_t nlist) {
    if (!q) return 0;
    uint64_t Hq = 1;
    while (Hq < 2ull * q) Hq <<= 1;
    uint64_t w = (uint64_t)(L + 31) / 32 + 8 * Hq + (4ull + nlist) * q + 8;
    return (w + 7) & ~7ull;
}
__device__ __forceinline__ DelScr del_scr(uint32_t *base, uint32_t L, uint32_t q) {
    DelScr s;
    s.Hq = next_pow2(2 * q);
    s.bm = base;
    s.hkey = base + (L + 31) / 32;
    s.hk = s.hkey + s.Hq;
    s.hfound = s.hk + s.Hq;
    s.hsel = s.hfound + s.Hq;
    s.hbest = reinterpret_cast<unsigned long long *>((reinterpret_cast<uintptr_t>(s.hsel + s.Hq) + 7) & ~(uintptr_t)7);
    s.hprev = s.hbest + s.Hq;
    s.holes = reinterpret_cast<uint32_t *>(s.hprev + s.Hq);
    s.R = s.holes + q;
    s.pk = reinterpret_cast<uint2 *>(s.R + q);
    s.gh = s.R + 3 * q;
    return s;
}

// largest i in [0, n) with pref[i] <= x  (pref nondecreasing, pref[0] = 0, x < pref[n])
__device__ __forceinline__ uint32_t owner_of(const uint64_t *pref, uint32_t n, uint64_t x) {
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(pref + mid) <= x) lo = mid;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t hash_find(const uint32_t *hkey, uint32_t hmask, uint32_t x) {
    uint32_t s = hash_slot(x, hmask);
    for (;;) {
        const uint32_t kx = hkey[s];
        if (kx == x) return s;
        if (kx == EMPTY_KEY) return EMPTY_KEY;
        s = (s + 1) & hmask;
    }
}

#define BSP_WARP_LOOP(i, n)                                                                     \
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < (n);                    \
         i += (gridDim.x * blockDim.x) >> 5)
#define BSP_ITEM_LOOP(it, total)                                                                \
    for (uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < (total);    \
         it += ((uint64_t)gridDim.x * blockDim.x) >> 5)

// the owner of item it, given the owner of an earlier item of the same warp
__device__ __forceinline__ uint32_t owner_next(const uint64_t *pref, uint32_t i, uint64_t it) {
    while (__ldg(pref + i + 1) <= it) i++;
    return i;
}
// Chunk items [0, total) in one contiguous range per warp; i = the item's owner (largest i
// with pref[i] <= it).  One binary search per warp, then the owner advances with the items
// (a hub's items are consecutive), instead of a dependent binary search of ~17 steps per item.
#define BSP_ITEM_RANGE(it, i, total, pref, n)                                                   \
    const uint64_t nw_##it = ((uint64_t)gridDim.x * blockDim.x) >> 5;                          \
    const uint64_t per_##it = ((uint64_t)(total) + nw_##it - 1) / nw_##it;                     \
    const uint64_t b_##it = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * per_##it; \
    const uint64_t e_##it = min((uint64_t)(total), b_##it + per_##it);                          \
    uint32_t i = b_##it < e_##it ? owner_of(pref, n, b_##it) : 0u;                             \
    for (uint64_t it = b_##it; it < e_##it && ((i = owner_next(pref, i, it)), true); it++)

// ------------------------------------------------------------------ plan
// count: add the batch's pool demand to cnt; state: write the per-vertex state
__global__ void __launch_bounds__(MT, BINGO_BSP_MINB) k_bsp_plan(const BspArgs a, uint64_t *__restrict__ scr_need, UpdCounters *cnt,
                                                 bool count, bool state) {
    __shared__ unsigned long long b_arc, b_bkt, b_mem, b_res, b_hix, b_gix;
    __shared__ int b_flag;
    __shared__ uint32_t b_done;
    if (threadIdx.x == 0) { b_arc = b_bkt = b_mem = b_res = b_hix = b_gix = 0; b_flag = 0; b_done = 0; }
    __syncthreads();
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    const uint32_t NT = bsp_nt(a);
    BSP_WARP_LOOP(i, NT) {
        const uint32_t t = a.t0 + i;
        const VHdr h = g.hdr[g.tv[t]];
        PlanLane pl;
        const PlanOut o = plan_vertex(g.recs, g.sval, g.seg[t], g.seg[t + 1], h, g.bkt, g.gcan, g.alpha, g.bs,
                                      g.arc_slack, g.mem_slack, &pl);
        if (count && lane == 0) {
            if (o.overflow) atomicOr(&b_flag, 4);
            if (o.arc) atomicAdd(&b_arc, o.arc);
            if (o.bkt) atomicAdd(&b_bkt, o.bkt);
            if (o.mem) atomicAdd(&b_mem, o.mem);
            if (o.res) atomicAdd(&b_res, o.res);
            // hub delete index: words of a (re)built table, an upper bound
            // (only vertices without a table: a table dropped at k_hix_prep is re-taken from the
            // pool's slack, or the vertex scans this batch)
            if (g.hixo && o.L > CH && o.L > g.hix_min && o.q && !g.hixo[g.tv[t]])
                atomicAdd(&b_hix, 2ull << nb_log2size(o.L));
        }
        const bool lst = is_list(pl.kind);
        // group index: entries of a table built this batch (list members after the inserts)
        const uint32_t gixe = g.gixo ? warp_sum(lst ? pl.c + pl.insk : 0u) : 0u;
        if (count && lane == 0 && g.gixo && o.L > CH && o.L > g.gix_min && o.L <= GIX_MAXL && o.q &&
            !g.gixo[g.tv[t]])
            atomicAdd(&b_gix, 2ull << nb_log2size(max(gixe, 1u)));
        if (!state) continue;
        gkp(a, GK_KIND0, i)[lane] = pl.kind;
        gkp(a, GK_C, i)[lane] = pl.c;
        gkp(a, GK_INSK, i)[lane] = pl.insk;
        gkp(a, GK_MOFF, i)[lane] = lst ? pl.ref : 0u;
        gkp(a, GK_CAP, i)[lane] = lst ? pl.aux : 0u;
        gkp(a, GK_ONE, i)[lane] = pl.kind == K_ONE ? pl.aux : 0xFFFFFFFFu;
        const uint32_t gch = warp_sum(lst ? (pl.c + pl.insk + CH - 1) / CH : 0u);
        if (lane == 0) {
            a.vL[i] = o.L;
            a.vq[i] = o.q;
            a.vm[i] = o.L - h.d;
            a.vlist0[i] = pl.list0;
            a.vgixe[i] = gixe;
            scr_need[i] = bsp_scr_words(o.L, o.q, __popc(pl.list0));
            // chunk items only for LARGE vertices (L > CH); a small vertex's scans are
            // done by its own warp inside alloc_insert / finalize
            const bool large = o.L > CH;
            a.cc_copy[i] = (o.L > h.adj_cap && h.d > CH) ? (h.d + CH - 1) / CH : 0;
            a.cc_sel[i] = (o.q && large) ? (o.L + CH - 1) / CH : 0;
            a.cc_grp[i] = (o.q && large) ? gch : 0;
            if (o.q && large) a.hubs[atomicAdd(a.nhubs, 1u)] = i;
            if (large) a.bigs[atomicAdd(a.nbigs, 1u)] = i;
            a.cc_all[i] = o.L ? (o.L + CH - 1) / CH : 1;
        }
    }
    if (!count) return;
    // the block's last warp to finish publishes its totals (no block barrier: a warp that is
    // done does not wait for the block's slowest vertex)
    if (lane != 0) return;
    __threadfence_block();
    if (atomicAdd(&b_done, 1u) != (blockDim.x >> 5) - 1) return;
    __threadfence_block();
    {
        const unsigned long long x_arc = *(volatile unsigned long long *)&b_arc, x_bkt = *(volatile unsigned long long *)&b_bkt,
                                 x_mem = *(volatile unsigned long long *)&b_mem, x_res = *(volatile unsigned long long *)&b_res,
                                 x_hix = *(volatile unsigned long long *)&b_hix, x_gix = *(volatile unsigned long long *)&b_gix;
        const int x_flag = *(volatile int *)&b_flag;
        if (x_arc) atomicAdd(&cnt->need_arc, x_arc);
        if (x_bkt) atomicAdd(&cnt->need_bkt, x_bkt);
        if (x_mem) atomicAdd(&cnt->need_mem, x_mem);
        if (x_res) atomicAdd(&cnt->reserve_mem, x_res);
        if (x_hix) atomicAdd(&cnt->need_hix, x_hix);
        if (x_gix) atomicAdd(&cnt->need_gix, x_gix);
        if (x_flag) atomicOr(&cnt->flag, x_flag);
    }
}

// host-visible totals after the plan (one D2H copy, one sync)
struct BspTotals {
    UpdCounters c;
    unsigned long long bump[3];
    unsigned long long scr, copy, sel, grp, all, hubs, bigs, hix_used, gix_used;
    unsigned long long nt;     // touched vertices
    int abort;                 // one-sync route: 1 EINVAL, 4 EOVERFLOW, 2 capacity (the host grows, re-runs)
    int pad;
};
// capacities the one-sync route was enqueued with
struct BspCaps {
    unsigned long long arc, bkt, mem_units, hix, scr_words, sel, grp, gix;
    int hix_on, gix_on;
};
// Totals of the plan.  One-sync route (abort != null): also its gate -- the totals against
// what was allocated when the batch was enqueued.  Anything that does not fit (or an invalid
// / overflowing batch) sets *abort and every later kernel of the batch returns at once:
// nothing is mutated, and the host grows what is short and re-runs the batch on the
// synchronous route.
__global__ void k_bsp_totals(const BspArgs a, const UpdCounters *cnt, const uint64_t *scr_off, BspTotals *out,
                             const BspCaps caps, int *abort) {
    if (threadIdx.x != 0) return;
    const uint32_t nt = bsp_nt(a);
    BspTotals t;
    t.c = *cnt;
    for (int j = 0; j < 3; j++) t.bump[j] = a.g.bump[j];
    t.scr = scr_off[nt];
    t.copy = a.p_copy[nt];
    t.sel = a.p_sel[nt];
    t.grp = a.p_grp[nt];
    t.all = a.p_all[nt];
    t.hubs = *a.nhubs;
    t.bigs = *a.nbigs;
    t.hix_used = a.g.bump[5];
    t.gix_used = a.g.bump[6];
    t.nt = nt;
    t.pad = 0;
    int ab = 0;
    if (abort) {
        if (t.c.flag & 1) ab |= 1;
        if (t.c.flag & 4) ab |= 4;
        if (t.c.flag & 8) ab |= 8;   // a segment was too long to order: re-segment (radix sort), re-run
        if (t.bump[0] + t.c.need_arc > caps.arc || t.bump[1] + t.c.need_bkt > caps.bkt ||
            t.bump[2] + t.c.need_mem + t.c.reserve_mem > caps.mem_units)
            ab |= 2;
        if (caps.hix_on && t.c.need_hix && t.hix_used + t.c.need_hix > caps.hix) ab |= 2;
        if (caps.gix_on && t.c.need_gix && t.gix_used + t.c.need_gix > caps.gix) ab |= 2;
        if (t.scr > caps.scr_words || t.sel > caps.sel || t.grp > caps.grp) ab |= 2;
        *abort = ab;
    }
    t.abort = ab;
    *out = t;
}

// ------------------------------------------------------------------ relocations, inserts, scratch init
__global__ void __launch_bounds__(MT, BINGO_BSP_MINB) k_bsp_alloc_insert(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    const uint32_t NT = bsp_nt(a);
    BSP_WARP_LOOP(i, NT) {
        const uint32_t t = a.t0 + i;
        const uint32_t beg = g.seg[t], end = g.seg[t + 1];
        const VHdr h = g.hdr[g.tv[t]];
        const uint32_t L = a.vL[i], q = a.vq[i], m = a.vm[i];
        // adjacency relocation (the copy of the d live arcs is the chunked k_bsp_copy)
        uint64_t aoff = h.adj_off;
        uint32_t acap = h.adj_cap;
        if (L > h.adj_cap) {
            const uint64_t cap2 = arc_capacity(L, g.arc_slack);
            unsigned long long o = 0;
            if (lane == 0) o = atomicAdd(&g.bump[0], (unsigned long long)cap2);
            aoff = __shfl_sync(0xffffffffu, o, 0);
            acap = (uint32_t)cap2;
        }
        if (lane == 0) {
            a.vaoff[i] = aoff;
            a.vacap[i] = acap;
            a.vN[i] = 0;
            a.vmiss[i] = 0;
            if (g.nbt) a.vnbo[i] = g.nbo[g.tv[t]];
        }
        if (aoff != h.adj_off && h.d <= CH) {
            // small relocation: copied here (larger ones by k_bsp_copy items)
            for (uint32_t p = lane; p < h.d; p += 32) {
                g.arc[aoff + p] = g.arc[h.adj_off + p];
                g.arc_epoch[aoff + p] = g.arc_epoch[h.adj_off + p];
                if (g.arc_dval) g.arc_dval[aoff + p] = g.arc_dval[h.adj_off + p];
            }
        }
        // member arrays that overflow their capacity (lists before the batch)
        const uint32_t kind = gkp(a, GK_KIND0, i)[lane];
        const uint32_t c = gkp(a, GK_C, i)[lane];
        const uint32_t insk_tot = gkp(a, GK_INSK, i)[lane];
        const uint32_t ref = gkp(a, GK_MOFF, i)[lane];
        uint32_t moff = ref, cap = gkp(a, GK_CAP, i)[lane];
        const bool grow = is_list(kind) && c + insk_tot > cap;
        if (grow) {
            const uint32_t units = member_units(c + insk_tot, g.mem_slack);
            moff = (uint32_t)atomicAdd(&g.bump[2], (unsigned long long)units);
            cap = units * 4;
            gkp(a, GK_MOFF, i)[lane] = moff;
            gkp(a, GK_CAP, i)[lane] = cap;
        }
        gkp(a, GK_DELK, i)[lane] = 0;
        gkp(a, GK_GHN, i)[lane] = 0;
        uint32_t gm = __ballot_sync(0xffffffffu, grow);
        while (gm) {
            const int k = __ffs(gm) - 1;
            gm &= gm - 1;
            const uint32_t from = __shfl_sync(0xffffffffu, ref, k);
            const uint32_t to = __shfl_sync(0xffffffffu, moff, k);
            const uint32_t cnt = __shfl_sync(0xffffffffu, c, k);
#pragma unroll 4
            for (uint32_t j = lane; j < cnt; j += 32) {
                g.mdst[(uint64_t)to * 4 + j] = g.mdst[(uint64_t)from * 4 + j];
                g.midx[(uint64_t)to * 4 + j] = g.midx[(uint64_t)from * 4 + j];
            }
        }
        // inserts in batch order: adjacency appends at d + rank,
        // member appends to groups that are REGULAR/SPARSE before the batch (and their
        // group-index entries, when the vertex has a table)
        const uint64_t go = (g.gixo && m && L > CH) ? g.gixo[g.tv[t]] : 0ull;
        bool gok = true;
        if (m) {
            uint32_t run = 0, insk = 0;
            for (uint32_t base = beg; base < end; base += 32) {
                const uint32_t p = base + lane;
                uint4 r = make_uint4(2u, 0u, 0u, 0u);
                if (p < end) r = g.recs[g.sval[p]];
                const bool ins = r.x == 0u;
                const uint32_t bal_i = __ballot_sync(0xffffffffu, ins);
                const uint32_t idx = h.d + run + __popc(bal_i & lanemask_lt());
                const uint32_t w = ins ? r.w : 0u;
                if (ins) {
                    g.arc[aoff + idx] = make_uint2(r.z, r.w);
                    g.arc_epoch[aoff + idx] = g.epoch;
                    if (g.arc_dval) g.arc_dval[aoff + idx] = g.dins[g.sval[p]];
                }
                uint32_t mk = __reduce_or_sync(0xffffffffu, w);
                while (mk) {
                    const int k = __ffs(mk) - 1;
                    mk &= mk - 1;
                    const uint32_t bal = __ballot_sync(0xffffffffu, (w >> k) & 1u);
                    const uint32_t kind_kk = __shfl_sync(0xffffffffu, kind, k);
                    const uint32_t start = __shfl_sync(0xffffffffu, c + insk, k);
                    const uint32_t mo = __shfl_sync(0xffffffffu, moff, k);
                    if (is_list(kind_kk) && ((w >> k) & 1u)) {
                        const uint32_t sl = start + __popc(bal & lanemask_lt());
                        const uint64_t e = (uint64_t)mo * 4 + sl;
                        g.mdst[e] = r.z;
                        g.midx[e] = idx;
                        if (go) gok &= gix_insert(gix_table(g.gix, go), gix_key(idx, (uint32_t)k), sl);
                    }
                    if (lane == (uint32_t)k) insk += __popc(bal);
                }
                run += __popc(bal_i);
            }
        }
        if (go && !__all_sync(0xffffffffu, gok) && lane == 0) g.gixo[g.tv[t]] = 0;   // full: rebuilt when needed
        // delete scratch: bitmap, hash of the distinct deleted destinations
        if (q) {
            const DelScr s = del_scr(g.scr + g.scr_off[i], L, q);
            const uint32_t bw = (L + 31) / 32;
            for (uint32_t j = lane; j < bw; j += 32) s.bm[j] = 0;
            for (uint32_t j = lane; j < s.Hq; j += 32) {
                s.hkey[j] = EMPTY_KEY;
                s.hk[j] = 0;
                s.hfound[j] = 0;
                s.hsel[j] = 0;
                s.hbest[j] = ~0ull;
                s.hprev[j] = 0;
            }
            __syncwarp();
            const uint32_t hmask = s.Hq - 1;
            for (uint32_t p = beg + lane; p < end; p += 32) {
                const uint4 r = g.recs[g.sval[p]];
                if (r.x != 1u) continue;
                uint32_t sl = hash_slot(r.z, hmask);
                for (;;) {
                    const uint32_t old = atomicCAS(&s.hkey[sl], EMPTY_KEY, r.z);
                    if (old == EMPTY_KEY || old == r.z) {
                        atomicAdd(&s.hk[sl], 1u);
                        break;
                    }
                    sl = (sl + 1) & hmask;
                }
            }
        }
    }
}

// ------------------------------------------------------------------ adjacency relocation copies
__global__ void __launch_bounds__(MT) k_bsp_copy(const BspArgs a, uint64_t total) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    const uint32_t NT = bsp_nt(a);
    total = bsp_total(a, a.p_copy, total);
    BSP_ITEM_RANGE(it, i, total, a.p_copy, NT) {
        const uint32_t c = (uint32_t)(it - a.p_copy[i]);
        const VHdr h = g.hdr[g.tv[a.t0 + i]];
        const uint64_t to = a.vaoff[i];
        const uint32_t e = min(h.d, (c + 1) * CH);
#pragma unroll 4
        for (uint32_t p = c * CH + lane; p < e; p += 32) {
            g.arc[to + p] = g.arc[h.adj_off + p];
            g.arc_epoch[to + p] = g.arc_epoch[h.adj_off + p];
            if (g.arc_dval) g.arc_dval[to + p] = g.arc_dval[h.adj_off + p];
        }
    }
}

// ------------------------------------------------------------------ delete selection, round 0 (R-8)
// every live instance of a deleted destination: count it, and atomicMin its
// packed (epoch << 32 | position) key
__global__ void __launch_bounds__(MT, BINGO_BSP_MINB) k_bsp_select(const BspArgs a, uint64_t total) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    const uint32_t NT = bsp_nt(a);
    total = bsp_total(a, a.p_sel, total);
    BSP_ITEM_RANGE(it, i, total, a.p_sel, NT) {
        if (a.vhix[i]) continue;   // located through the hub delete index (k_hix_select)
        const uint32_t c = (uint32_t)(it - a.p_sel[i]);
        const uint32_t L = a.vL[i], q = a.vq[i];
        const uint64_t aoff = a.vaoff[i];
        const DelScr s = del_scr(g.scr + g.scr_off[i], L, q);
        const uint32_t hmask = s.Hq - 1;
        const uint32_t e = min(L, (c + 1) * CH);
        // 8 independent destination loads in flight per lane, then the (L1-resident) probes
        for (uint32_t p0 = c * CH + lane; p0 < e; p0 += 32 * 8) {
            uint32_t x[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const uint32_t p = p0 + 32 * j;
                x[j] = p < e ? __ldg(&g.arc[aoff + p].x) : EMPTY_KEY;
            }
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const uint32_t p = p0 + 32 * j;
                if (p >= e) continue;
                const uint32_t hit = hash_find(s.hkey, hmask, x[j]);
                if (hit == EMPTY_KEY) continue;
                const unsigned long long key = ((unsigned long long)g.arc_epoch[aoff + p] << 32) | p;
                atomicAdd(&s.hfound[hit], 1u);
                atomicMin(&s.hbest[hit], key);
            }
        }
    }
}

// ------------------------------------------------------------------ delete-and-swap pieces (warp-wide)
// adjacency tail window [L', L): survivors fill the holes in rank order (R-6),
// R maps tail position -> new position (or DEL_MARK)
__device__ __forceinline__ uint32_t tail_window(const MutateArgs &g, const DelScr &s, uint64_t aoff, uint32_t L,
                                                uint32_t Lp) {
    const uint32_t lane = lane_id();
    uint32_t carry = 0, moved = 0;   // moved: OR of the biases of the arcs that move (their groups need renames)
    for (uint32_t t0 = Lp; t0 < L; t0 += 32) {
        const uint32_t tt = t0 + lane;
        const bool in = tt < L;
        const bool surv = in && !bit_test(s.bm, tt);
        const uint32_t bal = __ballot_sync(0xffffffffu, surv);
        if (in) {
            if (surv) {
                const uint32_t dstp = s.holes[carry + __popc(bal & lanemask_lt())];
                const uint2 e = g.arc[aoff + tt];
                moved |= e.y;
                g.arc[aoff + dstp] = e;
                g.arc_epoch[aoff + dstp] = g.arc_epoch[aoff + tt];
                if (g.arc_dval) g.arc_dval[aoff + dstp] = g.arc_dval[aoff + tt];
                s.R[tt - Lp] = dstp;
            } else {
                s.R[tt - Lp] = DEL_MARK;
            }
        }
        carry += __popc(bal);
    }
    return __reduce_or_sync(0xffffffffu, moved);
}

// group front, slots [sb, se) of [0, L_k'): deleted slots are recorded as holes
// gh[r0 + rank] in slot order; surviving members pointing into the adjacency tail
// are renamed in place
__device__ __forceinline__ void group_front(const MutateArgs &g, const DelScr &s, uint32_t *Mi, uint32_t *gh,
                                            uint32_t sb, uint32_t se, uint32_t r0, uint32_t Lp) {
    const uint32_t lane = lane_id();
    uint32_t r = r0;
    for (uint32_t b0 = sb; b0 < se; b0 += 32 * 8) {
        uint32_t xs[8];   // 8 independent member loads in flight per lane
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t sl = b0 + 32 * j + lane;
            xs[j] = sl < se ? Mi[sl] : 0u;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t sl = b0 + 32 * j + lane;
            bool del = false;
            if (sl < se) {
                const uint32_t x = xs[j];
                del = bit_test(s.bm, x);
                if (!del && x >= Lp) Mi[sl] = s.R[x - Lp];
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, del);
            if (del) gh[r + __popc(bal & lanemask_lt())] = sl;
            r += __popc(bal);
        }
    }
}

// group front, slots [sb, se): as group_front, but the deleted slots are appended to gh
// through the group's counter in any order (sorted afterwards)
__device__ __forceinline__ void group_front_append(const MutateArgs &g, const DelScr &s, uint32_t *Mi, uint32_t *gh,
                                                   uint32_t *ghn, uint32_t sb, uint32_t se, uint32_t Lp) {
    const uint32_t lane = lane_id();
    for (uint32_t b0 = sb; b0 < se; b0 += 32 * 8) {
        uint32_t xs[8];   // 8 independent member loads in flight per lane
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t sl = b0 + 32 * j + lane;
            xs[j] = sl < se ? Mi[sl] : 0u;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t sl = b0 + 32 * j + lane;
            bool del = false;
            if (sl < se) {
                const uint32_t x = xs[j];
                del = bit_test(s.bm, x);
                if (!del && x >= Lp) Mi[sl] = s.R[x - Lp];
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, del);
            if (bal) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(ghn, (uint32_t)__popc(bal));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (del) gh[base + __popc(bal & lanemask_lt())] = sl;
            }
        }
    }
}

// ascending sort of x[0, n) in shared memory (bitonic; n <= cap, cap a power of two), the
// whole block
__device__ __forceinline__ void block_sort_u32(uint32_t *x, uint32_t n) {
    const uint32_t P = next_pow2(n);
    for (uint32_t q = n + threadIdx.x; q < P; q += blockDim.x) x[q] = 0xFFFFFFFFu;
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
}

// ascending sort of one value per lane (bitonic over the warp; pad with 0xFFFFFFFF)
__device__ __forceinline__ uint32_t warp_sort_u32(uint32_t x) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
            const bool up = (lane & k) == 0, lower = (lane & j) == 0;
            x = (lower == up) ? min(x, y) : max(x, y);
        }
    }
    return x;
}

// hubs with deletes: picks (appended by k_bsp_finalize) in ascending order; its prefix below
// L' is exactly the hole list of R-6 (the counted-rank route writes the same list).  One warp
// per hub: up to 32 picks in registers; up to SORT_MAX by k_bsp_sort_big; more take the
// counted-rank route (vrank = 1).
__global__ void __launch_bounds__(MT) k_bsp_hub_sort(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    BSP_WARP_LOOP(h, *a.nhubs) {
        const uint32_t i = a.hubs[h];
        const uint32_t N = a.vN[i];
        if (lane == 0) {
            a.vrank[i] = N > SORT_MAX ? 1u : 0u;
            if (N > SORT_MAX) atomicAdd(a.nhubs + 4, 1u);   // some hub takes the counted-rank passes
        }
        if (N < 2 || N > SORT_MAX) continue;
        const DelScr s = del_scr(g.scr + g.scr_off[i], a.vL[i], a.vq[i]);
        if (N > 32) {
            if (lane == 0) a.sorts[atomicAdd(a.nhubs + 5, 1u)] = make_uint2(i, 32u);
            continue;
        }
        const uint32_t x = warp_sort_u32(lane < N ? s.holes[lane] : 0xFFFFFFFFu);
        if (lane < N) s.holes[lane] = x;
    }
}

// sorted-picks hubs: each list group's appended deleted slots in ascending order (one warp
// per hub, a group at a time; longer lists by k_bsp_sort_big)
__global__ void __launch_bounds__(MT) k_bsp_grp_sort(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    BSP_WARP_LOOP(h, *a.nhubs) {
        const uint32_t i = a.hubs[h];
        if (!a.vN[i] || a.vrank[i]) continue;
        const DelScr s = del_scr(g.scr + g.scr_off[i], a.vL[i], a.vq[i]);
        const uint32_t n_l = ((a.vlist0[i] >> lane) & 1u) ? gkp(a, GK_GHN, i)[lane] : 0u;
        const uint32_t gho_l = gkp(a, GK_GHO, i)[lane];
        uint32_t m = __ballot_sync(0xffffffffu, n_l >= 2);
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t n = __shfl_sync(0xffffffffu, n_l, k);
            uint32_t *gh = s.gh + __shfl_sync(0xffffffffu, gho_l, k);
            if (n > 32) {
                if (lane == 0) a.sorts[atomicAdd(a.nhubs + 5, 1u)] = make_uint2(i, (uint32_t)k);
                continue;
            }
            const uint32_t x = warp_sort_u32(lane < n ? gh[lane] : 0xFFFFFFFFu);
            if (lane < n) gh[lane] = x;
        }
    }
}

// the listed longer sorts (a hub's picks: group 32; a group's deleted slots: group k), one
// block each, bitonic in shared memory; the list is consumed (its counter reset)
__global__ void __launch_bounds__(256) k_bsp_sort_big(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    __shared__ uint32_t x[SORT_MAX];
    const MutateArgs &g = a.g;
    const uint32_t ns = a.nhubs[5];
    for (uint32_t j = blockIdx.x; j < ns; j += gridDim.x) {
        const uint2 e = a.sorts[j];
        const uint32_t i = e.x;
        const DelScr s = del_scr(g.scr + g.scr_off[i], a.vL[i], a.vq[i]);
        uint32_t *v;
        uint32_t n;
        if (e.y == 32u) {
            v = s.holes;
            n = a.vN[i];
        } else {
            v = s.gh + gkp(a, GK_GHO, i)[e.y];
            n = gkp(a, GK_GHN, i)[e.y];
        }
        for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) x[q] = v[q];
        __syncthreads();
        block_sort_u32(x, n);
        for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) v[q] = x[q];
        __syncthreads();
    }
    __syncthreads();
}

// group tail window [L_k', c'): survivors, renamed, fill the holes in rank order (R-6)
__device__ __forceinline__ void group_tail(const MutateArgs &g, const DelScr &s, uint32_t *Md, uint32_t *Mi,
                                           const uint32_t *gh, uint32_t cp, uint32_t Nk, uint32_t Lp,
                                           uint64_t gixo = 0, uint32_t k = 0) {
    const uint32_t lane = lane_id();
    uint32_t carry = 0;
    for (uint32_t s0 = cp - Nk; s0 < cp; s0 += 32) {
        const uint32_t sl = s0 + lane;
        uint32_t x = 0;
        const bool surv = sl < cp && !bit_test(s.bm, (x = Mi[sl]));
        const uint32_t bal = __ballot_sync(0xffffffffu, surv);
        if (surv) {
            const uint32_t hslot = gh[carry + __popc(bal & lanemask_lt())];
            const uint32_t xn = x >= Lp ? s.R[x - Lp] : x;
            Md[hslot] = Md[sl];
            Mi[hslot] = xn;
            if (gixo) gix_reslot(g, gixo, xn, k, hslot);   // its group-index entry follows
        }
        carry += __popc(bal);
    }
}

// ------------------------------------------------------------------ picks, further rounds, per-group counts
// hubs = false: small vertices (all of their delete path here); hubs = true: the
// large vertices with deletes (picks only; the rest by the chunk-item kernels)
// one vertex of k_bsp_finalize (hubs: picks only; small vertices: the whole delete-and-swap);
// the warp's shared-memory slices are passed in
__device__ __forceinline__ void finalize_vertex(const BspArgs &a, const uint32_t i, const bool hubs, uint32_t *s_delk_w,
                                                uint32_t *s_np_w, uint32_t *s_bm_w, uint32_t *s_hol_w,
                                                uint32_t *s_R_w, uint32_t *s_gh_w) {
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    const uint32_t q = a.vq[i];
    const uint32_t L = a.vL[i];
    const bool small = L <= CH;
    if (!q || small == hubs) return;
    const uint64_t aoff = a.vaoff[i];
    const DelScr s = del_scr(g.scr + g.scr_off[i], L, q);
    const uint32_t hmask = s.Hq - 1;
    s_delk_w[lane] = 0;
    if (lane == 0) *s_np_w = 0;
    if (small) {
        // round 0 of a small vertex (large ones: k_bsp_select items)
        for (uint32_t p = lane; p < L; p += 32) {
            const uint32_t hit = hash_find(s.hkey, hmask, g.arc[aoff + p].x);
            if (hit == EMPTY_KEY) continue;
            const unsigned long long key = ((unsigned long long)g.arc_epoch[aoff + p] << 32) | p;
            atomicAdd(&s.hfound[hit], 1u);
            atomicMin(&s.hbest[hit], key);
        }
    }
    __syncwarp();
    uint32_t N = 0;
    for (uint32_t round = 0;; round++) {
        if (round) {
            // round r > 0: per destination still owed a delete, the smallest key
            // above the previous pick (repeated deletes of one (u, v), R-8)
            for (uint32_t p = lane; p < L; p += 32) {
                const uint32_t hit = hash_find(s.hkey, hmask, g.arc[aoff + p].x);
                if (hit == EMPTY_KEY) continue;
                const unsigned long long key = ((unsigned long long)g.arc_epoch[aoff + p] << 32) | p;
                if (s.hsel[hit] < s.hk[hit] && key > s.hprev[hit]) atomicMin(&s.hbest[hit], key);
            }
            __syncwarp();
        }
        bool more = false;
        for (uint32_t sl = lane; sl < s.Hq; sl += 32) {
            if (s.hkey[sl] == EMPTY_KEY || s.hsel[sl] >= s.hk[sl]) continue;
            const unsigned long long b = s.hbest[sl];
            if (b == ~0ull) continue;
            const uint32_t p = (uint32_t)b;
            atomicOr(&s.bm[p >> 5], 1u << (p & 31u));
            const uint32_t hs = ++s.hsel[sl];
            s.hprev[sl] = b;
            s.hbest[sl] = ~0ull;
            N++;
            uint32_t bits = g.arc[aoff + p].y;
            if (hubs) {   // unordered; k_bsp_hub_sort orders the positions, the group index reads the pairs
                const uint32_t j = atomicAdd(s_np_w, 1u);
                s.holes[j] = p;
                s.pk[j] = make_uint2(p, bits);
            }
            while (bits) {
                const int k = __ffs(bits) - 1;
                bits &= bits - 1;
                atomicAdd(&s_delk_w[k], 1u);
            }
            if (hs < s.hk[sl] && hs < s.hfound[sl]) more = true;
        }
        __syncwarp();
        if (!__any_sync(0xffffffffu, more)) break;
    }
    uint32_t miss = 0;
    for (uint32_t sl = lane; sl < s.Hq; sl += 32)
        if (s.hkey[sl] != EMPTY_KEY) miss += s.hk[sl] - s.hsel[sl];
    N = warp_sum(N);
    miss = warp_sum(miss);
    __syncwarp();
    const uint32_t delk = s_delk_w[lane];
    const uint32_t list0 = a.vlist0[i];
    // gh offsets: the deleted-slot lists of the list groups, packed in k order
    const uint32_t v = ((list0 >> lane) & 1u) ? delk : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    gkp(a, GK_DELK, i)[lane] = delk;
    gkp(a, GK_GHO, i)[lane] = x - v;
    if (lane == 0) {
        a.vN[i] = N;
        a.vmiss[i] = miss;
    }
    __syncwarp();
    if (!small || !N) return;
    // ---- small vertex: the whole delete-and-swap here (L <= CH: one bitmap word per lane)
    const uint32_t Lp = L - N;
    DelScr ls = s;
    ls.bm = s_bm_w;
    s_bm_w[lane] = lane < (L + 31) / 32 ? s.bm[lane] : 0u;
    if (N <= 32) {
        ls.holes = s_hol_w;
        ls.R = s_R_w;
    }
    if (__shfl_sync(0xffffffffu, x, 31) <= 64) ls.gh = s_gh_w;
    __syncwarp();
    {
        uint32_t word = 0;
        if (lane * 32 < Lp) {
            word = ls.bm[lane];
            const uint32_t lim = Lp - lane * 32;
            if (lim < 32) word &= (1u << lim) - 1u;
        }
        const uint32_t pc = __popc(word);
        uint32_t y = pc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= (uint32_t)o) y += z;
        }
        uint32_t r = y - pc;
        while (word) {
            const int b = __ffs(word) - 1;
            word &= word - 1;
            ls.holes[r++] = lane * 32 + b;
        }
    }
    __syncwarp();
    const uint32_t moved = tail_window(g, ls, aoff, L, Lp);
    __syncwarp();
    if (N <= 32 && lane < N) s.R[lane] = ls.R[lane];   // rebuild reads R (ONE groups)
    const uint32_t cp_l = gkp(a, GK_C, i)[lane] + gkp(a, GK_INSK, i)[lane];
    const uint32_t mo_l = gkp(a, GK_MOFF, i)[lane];
    // only groups that lost a member or hold an arc that moved change
    uint32_t lm = list0 & (__ballot_sync(0xffffffffu, delk != 0) | moved);
    while (lm) {
        const int k = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint32_t cp = __shfl_sync(0xffffffffu, cp_l, k);
        const uint32_t Nk = __shfl_sync(0xffffffffu, delk, k);
        const uint32_t mo = __shfl_sync(0xffffffffu, mo_l, k);
        const uint32_t gho = __shfl_sync(0xffffffffu, x - v, k);
        uint32_t *Md = g.mdst + (uint64_t)mo * 4;
        uint32_t *Mi = g.midx + (uint64_t)mo * 4;
        group_front(g, ls, Mi, ls.gh + gho, 0, cp - Nk, 0, Lp);
        __syncwarp();
        if (Nk) group_tail(g, ls, Md, Mi, ls.gh + gho, cp, Nk, Lp);
        __syncwarp();
    }
}

__global__ void __launch_bounds__(MT, BINGO_BSP_MINB) k_bsp_finalize(const BspArgs a, bool hubs) {
    __shared__ uint32_t s_delk[MT / 32][32];
    __shared__ uint32_t s_np[MT / 32];   // hubs: picks appended to the holes array so far
    // small vertices: bitmap, holes, rename table and group holes in shared memory
    __shared__ uint32_t s_bm[MT / 32][32], s_hol[MT / 32][32], s_R[MT / 32][32], s_gh[MT / 32][64];
    if (BSP_ABORTED(a)) return;
    const uint32_t w = threadIdx.x >> 5;
    const uint32_t NT = hubs ? *a.nhubs : bsp_nt(a);
    BSP_WARP_LOOP(j, NT) {
        const uint32_t i = hubs ? a.hubs[j] : j;
        finalize_vertex(a, i, hubs, s_delk[w], s_np + w, s_bm[w], s_hol[w], s_R[w], s_gh[w]);
    }
}

// ------------------------------------------------------------------ holes: marked positions < L', ascending
__device__ __forceinline__ uint32_t hole_word(const BspArgs &a, uint32_t i, uint32_t c, uint32_t &wi, DelScr &s) {
    const uint32_t L = a.vL[i], q = a.vq[i], N = a.vN[i];
    if (!N || !a.vrank[i]) return 0;   // sorted-picks hubs have their holes already
    const uint32_t Lp = L - N;
    s = del_scr(a.g.scr + a.g.scr_off[i], L, q);
    wi = c * 32 + lane_id();
    if (wi * 32 >= Lp) return 0;
    uint32_t word = s.bm[wi];
    const uint32_t lim = Lp - wi * 32;
    if (lim < 32) word &= (1u << lim) - 1u;
    return word;
}

__global__ void __launch_bounds__(MT) k_bsp_hole_count(const BspArgs a, uint64_t total) {
    if (BSP_ABORTED(a)) return;
    if (!a.nhubs[4]) return;   // no hub takes the counted-rank route this batch
    const uint32_t NT = bsp_nt(a);
    total = bsp_total(a, a.p_sel, total);
    BSP_ITEM_RANGE(it, i, total, a.p_sel, NT) {
        const uint32_t c = (uint32_t)(it - a.p_sel[i]);
        uint32_t wi;
        DelScr s;
        const uint32_t n = warp_sum((uint32_t)__popc(hole_word(a, i, c, wi, s)));
        if (lane_id() == 0) a.icnt[it] = n;
    }
}

__global__ void __launch_bounds__(MT) k_bsp_hole_write(const BspArgs a, uint64_t total) {
    if (BSP_ABORTED(a)) return;
    if (!a.nhubs[4]) return;   // no hub takes the counted-rank route this batch
    const uint32_t lane = lane_id();
    const uint32_t NT = bsp_nt(a);
    total = bsp_total(a, a.p_sel, total);
    BSP_ITEM_RANGE(it, i, total, a.p_sel, NT) {
        if (!a.vN[i] || !a.vrank[i]) continue;
        const uint32_t c = (uint32_t)(it - a.p_sel[i]);
        uint32_t wi = 0;
        DelScr s;
        uint32_t word = hole_word(a, i, c, wi, s);
        const uint32_t n = __popc(word);
        uint32_t x = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        uint32_t r = (uint32_t)(a.ipref[it] - a.ipref[a.p_sel[i]]) + x - n;
        while (word) {
            const int b = __ffs(word) - 1;
            word &= word - 1;
            s.holes[r++] = wi * 32 + b;
        }
    }
}

// ------------------------------------------------------------------ adjacency tail window [L', L) (R-6)
__global__ void __launch_bounds__(MT) k_bsp_tail(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    BSP_WARP_LOOP(h, *a.nhubs) {
        const uint32_t i = a.hubs[h];
        const uint32_t N = a.vN[i], L = a.vL[i];
        if (!N) continue;
        const uint32_t q = a.vq[i];
        const DelScr s = del_scr(g.scr + g.scr_off[i], L, q);
        const uint32_t moved = tail_window(g, s, a.vaoff[i], L, L - N);
        if (lane_id() == 0) a.vmoved[i] = moved;
    }
}

// ------------------------------------------------------------------ group fronts
// group item -> (vertex i, group k, chunk j of the slots [0, c + ins_k)); every
// lane computes the same answer
struct GrpItem {
    uint32_t i, k, j, first;   // first: item index of chunk 0 of (i, k)
    uint32_t cp, Nk, moff, gho;
};
__device__ __forceinline__ GrpItem grp_item(const BspArgs &a, uint64_t it, uint32_t owner) {
    const uint32_t lane = lane_id();
    GrpItem gi;
    gi.i = owner;
    const uint32_t c = (uint32_t)(it - a.p_grp[gi.i]);
    const uint32_t list0 = a.vlist0[gi.i];
    const bool lst = (list0 >> lane) & 1u;
    const uint32_t cp = lst ? gkp(a, GK_C, gi.i)[lane] + gkp(a, GK_INSK, gi.i)[lane] : 0u;
    const uint32_t nch = (cp + CH - 1) / CH;
    uint32_t x = nch;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    const uint32_t pre = x - nch;
    const uint32_t own = __ballot_sync(0xffffffffu, nch && pre <= c && c < pre + nch);
    gi.k = __ffs(own) - 1;
    gi.j = c - __shfl_sync(0xffffffffu, pre, gi.k);
    gi.first = (uint32_t)(it - gi.j);
    gi.cp = __shfl_sync(0xffffffffu, cp, gi.k);
    gi.Nk = gkp(a, GK_DELK, gi.i)[gi.k];
    gi.moff = gkp(a, GK_MOFF, gi.i)[gi.k];
    gi.gho = gkp(a, GK_GHO, gi.i)[gi.k];
    return gi;
}

__global__ void __launch_bounds__(MT, BINGO_BSP_MINB) k_bsp_grp_count(const BspArgs a, uint64_t total) {
    if (BSP_ABORTED(a)) return;
    if (!a.nhubs[4]) return;   // no hub takes the counted-rank route this batch
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    total = bsp_total(a, a.p_grp, total);
    const uint32_t NT = bsp_nt(a);
    BSP_ITEM_RANGE(it, own, total, a.p_grp, NT) {
        const GrpItem gi = grp_item(a, it, own);
        uint32_t n = 0;
        if (gi.Nk && a.vrank[gi.i]) {
            const uint32_t L = a.vL[gi.i], q = a.vq[gi.i];
            const DelScr s = del_scr(g.scr + g.scr_off[gi.i], L, q);
            const uint32_t *Mi = g.midx + (uint64_t)gi.moff * 4;
            const uint32_t e = min(gi.cp - gi.Nk, (gi.j + 1) * CH);
            for (uint32_t s0 = gi.j * CH + lane; s0 < e; s0 += 32 * 8) {
                uint32_t m[8];
#pragma unroll
                for (int j = 0; j < 8; j++) m[j] = s0 + 32 * j < e ? __ldg(Mi + s0 + 32 * j) : 0xFFFFFFFFu;
#pragma unroll
                for (int j = 0; j < 8; j++) n += (m[j] != 0xFFFFFFFFu && bit_test(s.bm, m[j])) ? 1u : 0u;
            }
            n = warp_sum(n);
        }
        if (lane == 0) a.gcnt[it] = n;
    }
}

// pass 1 over the front [0, L_k'): deleted slots become holes ranked in slot
// order; survivors pointing into the adjacency tail are renamed in place
__global__ void __launch_bounds__(MT, BINGO_BSP_MINB) k_bsp_grp_write(const BspArgs a, uint64_t total) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    total = bsp_total(a, a.p_grp, total);
    const uint32_t NT = bsp_nt(a);
    BSP_ITEM_RANGE(it, own, total, a.p_grp, NT) {
        const GrpItem gi = grp_item(a, it, own);
        const uint32_t N = a.vN[gi.i];
        if (!N || (!gi.Nk && !((a.vmoved[gi.i] >> gi.k) & 1u))) continue;   // group unchanged
        const uint32_t L = a.vL[gi.i], q = a.vq[gi.i], Lp = L - N;
        const DelScr s = del_scr(g.scr + g.scr_off[gi.i], L, q);
        uint32_t *Mi = g.midx + (uint64_t)gi.moff * 4;
        const uint32_t Lk = gi.cp - gi.Nk;
        if (g.gixo && (a.vgix[gi.i] == 1u || a.vgix[gi.i] == 2u || a.vgix[gi.i] == 4u)) continue;   // k_gix_front did it
        if (!a.vrank[gi.i]) {   // deleted slots appended (any order), sorted by k_bsp_grp_sort
            group_front_append(g, s, Mi, s.gh + gi.gho, gkp(a, GK_GHN, gi.i) + gi.k, gi.j * CH,
                               min(Lk, (gi.j + 1) * CH), Lp);
            continue;
        }
        const uint32_t r0 = gi.Nk ? (uint32_t)(a.gpref[it] - a.gpref[gi.first]) : 0u;
        group_front(g, s, Mi, s.gh + gi.gho, gi.j * CH, min(Lk, (gi.j + 1) * CH), r0, Lp);
    }
}

// pass 2 over each group's tail window [L_k', c'): survivors, renamed, fill the
// holes in rank order (R-6)
__global__ void __launch_bounds__(MT) k_bsp_grp_tail(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    BSP_WARP_LOOP(h, *a.nhubs) {
        const uint32_t i = a.hubs[h];
        const uint32_t N = a.vN[i], L = a.vL[i];
        if (!N) continue;
        const uint32_t q = a.vq[i], Lp = L - N;
        const DelScr s = del_scr(g.scr + g.scr_off[i], L, q);
        const uint32_t Nk_l = gkp(a, GK_DELK, i)[lane];
        uint32_t gm = __ballot_sync(0xffffffffu, ((a.vlist0[i] >> lane) & 1u) && Nk_l);
        const uint32_t cp_l = gkp(a, GK_C, i)[lane] + gkp(a, GK_INSK, i)[lane];
        const uint32_t mo_l = gkp(a, GK_MOFF, i)[lane];
        const uint32_t gho_l = gkp(a, GK_GHO, i)[lane];
        const uint64_t go = (g.gixo && (a.vgix[i] == 1u || a.vgix[i] == 2u)) ? g.gixo[g.tv[a.t0 + i]] : 0ull;
        while (gm) {
            const int k = __ffs(gm) - 1;
            gm &= gm - 1;
            const uint32_t cp = __shfl_sync(0xffffffffu, cp_l, k);
            const uint32_t Nk = __shfl_sync(0xffffffffu, Nk_l, k);
            const uint32_t mo = __shfl_sync(0xffffffffu, mo_l, k);
            const uint32_t gho = __shfl_sync(0xffffffffu, gho_l, k);
            group_tail(g, s, g.mdst + (uint64_t)mo * 4, g.midx + (uint64_t)mo * 4, s.gh + gho, cp, Nk, Lp, go,
                       (uint32_t)k);
        }
    }
}

// ------------------------------------------------------------------ rebuild
// lane k = radix group k of the vertex being rebuilt
struct RbLane {
    uint32_t kind1, cn, moff, cap, one;
};

// stage A (one warp): Eq.9 reclassification, member-array allocation for groups
// that become lists, the ONE member when it is known without a scan, statistics.
// Returns the (fill, find) masks of groups that need the adjacency scan.
__device__ __forceinline__ void rebuild_classify(const BspArgs &a, uint32_t i, RbLane &r, uint32_t &fm, uint32_t &fd) {
    const uint32_t lane = lane_id(), k = lane;
    const MutateArgs &g = a.g;
    const uint32_t L = a.vL[i], q = a.vq[i], N = a.vN[i], dn = L - N, Lp = dn;
    DelScr s;
    if (q) s = del_scr(g.scr + g.scr_off[i], L, q);
    const uint32_t kind0 = gkp(a, GK_KIND0, i)[k];
    r.cn = gkp(a, GK_C, i)[k] + gkp(a, GK_INSK, i)[k] - gkp(a, GK_DELK, i)[k];
    r.kind1 = classify(r.cn, dn, g.alpha, g.beta, g.bs);
    r.moff = gkp(a, GK_MOFF, i)[k];
    r.cap = gkp(a, GK_CAP, i)[k];
    r.one = 0xFFFFFFFFu;
    bool fill = false, find = false;
    if (is_list(r.kind1) && !is_list(kind0)) {
        const uint32_t units = member_units(r.cn, g.mem_slack);
        r.moff = (uint32_t)atomicAdd(&g.bump[2], (unsigned long long)units);
        r.cap = units * 4;
        fill = true;
    } else if (r.kind1 == K_ONE) {
        if (is_list(kind0)) {
            r.one = g.midx[(uint64_t)r.moff * 4];
        } else if (kind0 == K_ONE) {
            const uint32_t mo = gkp(a, GK_ONE, i)[k];
            if (q && N && bit_test(s.bm, mo)) find = true;
            else r.one = (N && mo >= Lp) ? s.R[mo - Lp] : mo;
            if (!find && r.one == DEL_MARK) find = true;
        } else {
            find = true;
        }
    }
    // statistics: deletes, missing deletes, kind transitions
    uint32_t *vs = g.vstats + (uint64_t)i * VST;
    if (lane < 25) vs[2 + lane] = 0;
    __syncwarp();
    if (kind0 != K_EMPTY || r.kind1 != K_EMPTY) atomicAdd(&vs[2 + 5 * kind0 + r.kind1], 1u);
    if (lane == 0) {
        vs[0] = N;
        vs[1] = a.vmiss[i];
    }
    fm = __ballot_sync(0xffffffffu, fill);
    fd = __ballot_sync(0xffffffffu, find);
}

// adjacency positions [pb, pe), one warp, ascending: lane k counts (count_only) or
// writes its fill-group members starting at slot base_k (R-2: ascending index), and
// records the first position of each find group in first_k
__device__ __forceinline__ void fill_scan(const MutateArgs &g, uint64_t aoff, uint32_t pb, uint32_t pe, uint32_t fm,
                                          uint32_t fd, uint32_t moff_l, bool count_only, uint32_t &cnt_l,
                                          uint32_t &first_l, uint64_t go = 0, uint32_t *vg = nullptr) {
    const uint32_t lane = lane_id();
    for (uint32_t base = pb; base < pe; base += 32) {
        const uint32_t p = base + lane;
        uint2 e = make_uint2(0u, 0u);
        if (p < pe) e = g.arc[aoff + p];
        uint32_t mk = (fm | fd) & __reduce_or_sync(0xffffffffu, e.y);
        while (mk) {
            const int kb = __ffs(mk) - 1;
            mk &= mk - 1;
            const uint32_t bal = __ballot_sync(0xffffffffu, (e.y >> kb) & 1u);
            if ((fd >> kb) & 1u) {
                if (lane == (uint32_t)kb && first_l == 0xFFFFFFFFu) first_l = base + __ffs(bal) - 1;
                continue;
            }
            if (!count_only) {
                const uint32_t start = __shfl_sync(0xffffffffu, cnt_l, kb);
                const uint32_t mo = __shfl_sync(0xffffffffu, moff_l, kb);
                if ((e.y >> kb) & 1u) {
                    const uint32_t sl = start + __popc(bal & lanemask_lt());
                    const uint64_t qq = (uint64_t)mo * 4 + sl;
                    g.mdst[qq] = e.x;
                    g.midx[qq] = p;
                    // a group that became a list: its members enter the vertex's group index
                    if (go && !gix_insert(gix_table(g.gix, go), gix_key(p, (uint32_t)kb), sl)) *vg = 4u;
                }
            }
            if (lane == (uint32_t)kb) cnt_l += __popc(bal);
        }
    }
}

// stage C (one warp): integer Vose (R-4), buckets, headers
__device__ __forceinline__ void rebuild_write(const BspArgs &a, uint32_t i, const RbLane &r) {
    const uint32_t lane = lane_id(), k = lane;
    const MutateArgs &g = a.g;
    const uint32_t u = g.tv[a.t0 + i];
    const VHdr h = g.hdr[u];
    const uint32_t dn = a.vL[i] - a.vN[i];
    const uint64_t aoff = a.vaoff[i];
    uint32_t onedst = 0;
    if (r.kind1 == K_ONE) onedst = g.arc[aoff + r.one].x;
    const uint32_t mask = __ballot_sync(0xffffffffu, r.cn != 0);
    const uint32_t n = __popc(mask);
    const uint64_t T = warp_sum(r.cn ? ((uint64_t)r.cn << k) : 0ull);
    const uint32_t kb = (lane < n) ? (uint32_t)__fns(mask, 0, lane + 1) : 0u;
    const uint32_t c_b = __shfl_sync(0xffffffffu, r.cn, kb);
    const uint32_t kind_b = __shfl_sync(0xffffffffu, r.kind1, kb);
    const uint32_t moff_b = __shfl_sync(0xffffffffu, r.moff, kb);
    const uint32_t cap_b = __shfl_sync(0xffffffffu, r.cap, kb);
    const uint32_t one_b = __shfl_sync(0xffffffffu, r.one, kb);
    const uint32_t od_b = __shfl_sync(0xffffffffu, onedst, kb);
    uint64_t thr;
    uint32_t alias;
    vose_warp(lane < n, n, (uint64_t)c_b << kb, T, thr, alias);
    uint32_t bo = h.bkt_off, ncap = h.ncap;
    if (n > h.ncap) {
        unsigned long long o = 0;
        if (lane == 0) o = atomicAdd(&g.bump[1], (unsigned long long)bucket_capacity(n));
        bo = (uint32_t)__shfl_sync(0xffffffffu, o, 0);
        ncap = bucket_capacity(n);
    }
    uint32_t x_b, y_b;
    group_view(kind_b, c_b, moff_b, od_b, dn, aoff, x_b, y_b);
    const uint32_t aux_b = is_list(kind_b) ? cap_b : (kind_b == K_ONE ? one_b : 0u);
    write_buckets(g.bkt, g.gcan, bo, n, lane, kb, kind_b, c_b, x_b, y_b, aux_b, thr, alias, T);
    if (lane == 0) {
        VHdr nh;
        nh.T = T;
        nh.adj_off = aoff;
        nh.bkt_off = bo;
        nh.d = dn;
        nh.n = (uint8_t)n;
        nh.ncap = (uint8_t)ncap;
        nh.pad = 0;
        nh.adj_cap = a.vacap[i];
        g.hdr[u] = nh;
        ThinHdr th;
        th.bkt_off = bo;
        th.n = (uint8_t)n;
        th.flags = (dn >= g.hot_b ? 1 : 0) | (dn >= g.hot_m ? 2 : 0);
        th.pad1 = 0;
        g.thdr[u] = th;
        if (g.nbt) g.nbo[u] = nb_pack(4 * aoff, nb_log2size(dn));
        if (!a.vhix[i] && g.hixo && g.hixo[u]) g.hixo[u] = 0;   // index not maintained by this batch
    }
    if (g.gixo) {   // group index: kept only if this batch maintained it and the list groups stay lists
        const uint32_t ent = warp_sum(is_list(r.kind1) ? r.cn : 0u);
        if (lane == 0) {
            const uint64_t o = g.gixo[u];
            if (o) {
                const uint32_t mode = a.vL[i] > CH ? a.vgix[i] : 0u;
                const bool keep = (mode == 1u || mode == 2u) && 4ull * ((uint64_t)ent + g.gixt[u]) <= (3ull << (o >> 48));
                if (!keep) g.gixo[u] = 0;
            }
        }
    }
}

// small vertices (L <= CH): one warp each
__global__ void __launch_bounds__(MT, BINGO_BSP_MINB) k_bsp_rebuild(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t NT = bsp_nt(a);
    BSP_WARP_LOOP(i, NT) {
        if (a.vL[i] > CH) continue;
        RbLane r;
        uint32_t fm, fd;
        rebuild_classify(a, i, r, fm, fd);
        if (fm | fd) {
            // one ascending pass over the post-batch adjacency materialises new lists
            // and finds the member of ONE groups
            uint32_t cnt = 0, first = 0xFFFFFFFFu;
            fill_scan(a.g, a.vaoff[i], 0, a.vL[i] - a.vN[i], fm, fd, r.moff, false, cnt, first);
            if ((fd >> lane_id()) & 1u) r.one = first;
        }
        rebuild_write(a, i, r);
    }
}

// small vertices (L <= CH): k_bsp_finalize(small) and k_bsp_rebuild fused -- the whole
// delete-and-swap, then the rebuild, by one warp per vertex in one launch (its state is read
// once, and no warp waits for the second kernel's launch and ramp)
__global__ void __launch_bounds__(MT, BINGO_BSP_MINB) k_bsp_small(const BspArgs a) {
    __shared__ uint32_t s_delk[MT / 32][32];
    __shared__ uint32_t s_np[MT / 32];
    __shared__ uint32_t s_bm[MT / 32][32], s_hol[MT / 32][32], s_R[MT / 32][32], s_gh[MT / 32][64];
    if (BSP_ABORTED(a)) return;
    const uint32_t w = threadIdx.x >> 5;
    const uint32_t NT = bsp_nt(a);
    BSP_WARP_LOOP(i, NT) {
        if (a.vL[i] > CH) continue;
        finalize_vertex(a, i, false, s_delk[w], s_np + w, s_bm[w], s_hol[w], s_R[w], s_gh[w]);
        __syncwarp();
        RbLane r;
        uint32_t fm, fd;
        rebuild_classify(a, i, r, fm, fd);
        if (fm | fd) {
            uint32_t cnt = 0, first = 0xFFFFFFFFu;
            fill_scan(a.g, a.vaoff[i], 0, a.vL[i] - a.vN[i], fm, fd, r.moff, false, cnt, first);
            if ((fd >> lane_id()) & 1u) r.one = first;
        }
        rebuild_write(a, i, r);
    }
}

// large vertices (L > CH): one warp each for the reclassification, the alias and the
// writes (a block per vertex left 31 warps idle behind barriers: 0.9 ms per c4 batch);
// the few that need an adjacency scan (a group turning into a list, or a ONE group
// whose member must be found) save their stage-A state in the gk slots and are
// finished by k_bsp_rebuild_fill, one block each
__global__ void __launch_bounds__(MT, BINGO_BSP_MINB) k_bsp_rebuild_big(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    BSP_WARP_LOOP(h, *a.nbigs) {
        const uint32_t i = a.bigs[h];
        const uint32_t kind0 = gkp(a, GK_KIND0, i)[lane];
        RbLane r;
        uint32_t fm, fd;
        rebuild_classify(a, i, r, fm, fd);
        const uint32_t gm = a.vgix[i];
        if (a.g.gixo && (gm == 1u || gm == 2u)) {
            // a group leaving the list layouts (-> one-element, dense or empty): its members
            // leave the group index (the list itself, compacted, is still in place)
            const uint32_t u = a.g.tv[a.t0 + i];
            const GixT t = gix_table(a.g.gix, a.g.gixo[u]);
            uint32_t lm = __ballot_sync(0xffffffffu, is_list(kind0) && !is_list(r.kind1) && r.cn);
            uint32_t rem = 0;
            while (lm) {
                const int k = __ffs(lm) - 1;
                lm &= lm - 1;
                const uint32_t cn = __shfl_sync(0xffffffffu, r.cn, k);
                const uint32_t *Mi = a.g.midx + (uint64_t)__shfl_sync(0xffffffffu, r.moff, k) * 4;
                for (uint32_t sl = lane; sl < cn; sl += 32) {
                    const uint32_t e = gix_find(t, gix_key(Mi[sl], (uint32_t)k));
                    if (e != 0xFFFFFFFFu) {
                        t.t[2 * e] = GIX_TOMB;
                        rem++;
                    }
                }
            }
            rem = warp_sum(rem);
            if (lane == 0 && rem) a.g.gixt[u] += rem;
        }
        if (!(fm | fd)) {
            rebuild_write(a, i, r);
            continue;
        }
        gkp(a, GK_KIND0, i)[lane] = r.kind1;
        gkp(a, GK_C, i)[lane] = r.cn;
        gkp(a, GK_MOFF, i)[lane] = r.moff;
        gkp(a, GK_CAP, i)[lane] = r.cap;
        gkp(a, GK_ONE, i)[lane] = r.one;
        gkp(a, GK_INSK, i)[lane] = lane == 0 ? fm : fd;
        if (lane == 0) a.hubs[atomicAdd(a.nhubs + 2, 1u)] = i;   // hubs[] is free again by now
    }
}

// large vertices with a fill/find scan: one 1024-thread block each; the scan is split
// over the 32 warps (count pass, per-group scan over warps, write pass)
__global__ void __launch_bounds__(LT) k_bsp_rebuild_fill(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    __shared__ RbLane s_r[32];
    __shared__ uint32_t s_fm, s_fd;
    __shared__ uint32_t s_cnt[32][33];     // [warp][group], then exclusive prefixes
    __shared__ uint32_t s_first[32][33];
    const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
    for (uint32_t h = blockIdx.x; h < a.nhubs[2]; h += gridDim.x) {
        const uint32_t i = a.hubs[h];
        if (w == 0) {
            RbLane r;
            r.kind1 = gkp(a, GK_KIND0, i)[lane];
            r.cn = gkp(a, GK_C, i)[lane];
            r.moff = gkp(a, GK_MOFF, i)[lane];
            r.cap = gkp(a, GK_CAP, i)[lane];
            r.one = gkp(a, GK_ONE, i)[lane];
            s_r[lane] = r;
            if (lane == 0) s_fm = gkp(a, GK_INSK, i)[0];
            if (lane == 1) s_fd = gkp(a, GK_INSK, i)[1];
        }
        __syncthreads();
        const uint32_t fm = s_fm, fd = s_fd;
        const uint32_t dn = a.vL[i] - a.vN[i];
        const uint64_t aoff = a.vaoff[i];
        const uint32_t seg = ((dn + 32 * 32 - 1) / (32 * 32)) * 32;   // positions per warp, multiple of 32
        const uint32_t pb = min(dn, w * seg), pe = min(dn, pb + seg);
        const uint32_t moff_l = s_r[lane].moff;
        uint32_t cnt = 0, first = 0xFFFFFFFFu;
        fill_scan(a.g, aoff, pb, pe, fm, 0u, moff_l, true, cnt, first);
        s_cnt[w][lane] = cnt;
        __syncthreads();
        if (w == 0) {
            uint32_t acc = 0;
            for (uint32_t j = 0; j < 32; j++) {
                const uint32_t c = s_cnt[j][lane];
                s_cnt[j][lane] = acc;
                acc += c;
            }
        }
        __syncthreads();
        cnt = s_cnt[w][lane];
        first = 0xFFFFFFFFu;
        const uint32_t gm = a.vgix[i];
        const uint64_t go = (a.g.gixo && (gm == 1u || gm == 2u)) ? a.g.gixo[a.g.tv[a.t0 + i]] : 0ull;
        fill_scan(a.g, aoff, pb, pe, fm, fd, moff_l, false, cnt, first, go, a.vgix + i);
        s_first[w][lane] = first;
        __syncthreads();
        if (w == 0 && ((fd >> lane) & 1u)) {
            uint32_t f = 0xFFFFFFFFu;
            for (uint32_t j = 0; j < 32; j++) f = min(f, s_first[j][lane]);
            s_r[lane].one = f;
        }
        __syncthreads();
        if (w == 0) rebuild_write(a, i, s_r[lane]);
        __syncthreads();
    }
}

// ------------------------------------------------------------------ node2vec neighbour sets of touched vertices
// Incremental when the set keeps its base and size (no relocation, same
// log2 size) and its tombstones stay <= size / 4: inserted destinations are
// added, a destination whose every live instance this batch deleted (all found
// instances selected, hsel = hfound > 0) is tombstoned.  Otherwise the vertex is
// flagged for the full rebuild by the chunk items below.
__global__ void __launch_bounds__(MT) k_bsp_nb_incr(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    const uint32_t NT = bsp_nt(a);
    BSP_WARP_LOOP(i, NT) {
        const uint32_t t = a.t0 + i;
        const uint32_t u = g.tv[t];
        const uint32_t L = a.vL[i], q = a.vq[i];
        const uint32_t dn = L - a.vN[i];
        const uint32_t lg = nb_log2size(dn);
        const uint64_t base = 4 * a.vaoff[i];
        const uint64_t old = a.vnbo[i];
        uint32_t tomb = g.nbtomb[u];
        bool full = nb_base(old) != base || (uint32_t)(old >> 48) != lg;
        DelScr s;
        uint32_t rem = 0;
        if (!full && q) {
            s = del_scr(g.scr + g.scr_off[i], L, q);
            for (uint32_t sl = lane; sl < s.Hq; sl += 32)
                if (s.hkey[sl] != EMPTY_KEY && s.hfound[sl] && s.hsel[sl] == s.hfound[sl]) rem++;
            rem = warp_sum(rem);
            if (tomb + rem > (1u << lg) / 4) full = true;
        }
        if (lane == 0) a.vnbfull[i] = full ? 1u : 0u;
        if (full) {
            if (lane == 0) g.nbtomb[u] = 0;
            continue;
        }
        uint32_t *tbl = g.nbt + base;
        const uint32_t mask = (1u << lg) - 1;
        for (uint32_t p = g.seg[t] + lane; p < g.seg[t + 1]; p += 32) {
            const uint4 r = g.recs[g.sval[p]];
            if (r.x == 0u) nb_insert(tbl, mask, r.z);
        }
        __syncwarp();
        __threadfence_block();
        uint32_t gone = 0;
        if (q)
            for (uint32_t sl = lane; sl < s.Hq; sl += 32)
                if (s.hkey[sl] != EMPTY_KEY && s.hfound[sl] && s.hsel[sl] == s.hfound[sl])
                    gone += nb_remove(tbl, mask, s.hkey[sl]) ? 1u : 0u;
        gone = warp_sum(gone);
        if (lane == 0) g.nbtomb[u] = tomb + gone;
    }
}

__global__ void __launch_bounds__(MT) k_bsp_nb_clear(const BspArgs a, uint64_t total) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    const uint32_t NT = bsp_nt(a);
    total = bsp_total(a, a.p_all, total);
    BSP_ITEM_RANGE(it, i, total, a.p_all, NT) {
        if (!a.vnbfull[i]) continue;
        const uint32_t c = (uint32_t)(it - a.p_all[i]);
        const uint32_t dn = a.vL[i] - a.vN[i];
        const uint32_t size = 1u << nb_log2size(dn);
        uint32_t *tbl = g.nbt + 4 * a.vaoff[i];
        const uint32_t e = min(size, (c + 1) * 4 * CH);
        for (uint32_t j = c * 4 * CH + lane; j < e; j += 32) tbl[j] = NB_EMPTY;
    }
}

__global__ void __launch_bounds__(MT) k_bsp_nb_fill(const BspArgs a, uint64_t total) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    const uint32_t NT = bsp_nt(a);
    total = bsp_total(a, a.p_all, total);
    BSP_ITEM_RANGE(it, i, total, a.p_all, NT) {
        if (!a.vnbfull[i]) continue;
        const uint32_t c = (uint32_t)(it - a.p_all[i]);
        const uint32_t dn = a.vL[i] - a.vN[i];
        const uint32_t mask = (1u << nb_log2size(dn)) - 1;
        const uint64_t aoff = a.vaoff[i];
        uint32_t *tbl = g.nbt + 4 * aoff;
        const uint32_t e = min(dn, (c + 1) * CH);
        for (uint32_t p = c * CH + lane; p < e; p += 32) nb_insert(tbl, mask, g.arc[aoff + p].x);
    }
}

}  // namespace bingo
