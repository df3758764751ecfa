// hub_index.cuh -- the hub delete index (included by update.cu after update_bsp.cuh).
//
// The paper locates a deleted edge by its index; the ABI deletes by (src, dst),
// so without an index every large vertex that receives a delete is scanned end to end
// (k_bsp_select: O(d) per touched hub, the dominant cost of c4/c5 batches).  Here every
// large vertex (L > CH) that receives deletes gets, on first use, a destination ->
// position multimap (open addressing, 2 words per entry {dst + 1, position}, 0 = empty,
// HIX_TOMB = removed; tables come zeroed from a bump pool), which the bulk-synchronous
// route keeps exact: deletes remove their entries, moved arcs (R-6 tail window) update
// theirs, inserted arcs add entries.  Selection through the index finds exactly the
// live instances the scan would find, so the picks (R-8) are the same.  The index is
// derived state: a vertex whose batch repeats a deleted destination, a vertex touched by
// another route (legacy, fast path, small-vertex BSP path) and a table past 3/4 load
// (entries + tombstones) drop their index; it is rebuilt from the adjacency when needed.
#pragma once

namespace bingo {

static constexpr uint32_t HIX_TOMB = 0xFFFFFFFFu;

struct HixT {
    uint32_t *t;
    uint32_t mask;
};
__device__ __forceinline__ HixT hix_table(const MutateArgs &g, uint64_t o) {
    HixT h;
    h.t = g.hix + (o & ((1ull << 48) - 1));
    h.mask = (uint32_t)((1ull << (o >> 48)) - 1);
    return h;
}
__device__ __forceinline__ void hix_insert(const HixT &h, uint32_t v, uint32_t p) {
    uint32_t s = nb_hash(v) & h.mask;
    for (;;) {
        if (atomicCAS(&h.t[2 * s], 0u, v + 1) == 0u) {
            h.t[2 * s + 1] = p;
            return;
        }
        s = (s + 1) & h.mask;
    }
}
// the entry (v, p) gets position np (np = HIX_TOMB: removed); false if absent
__device__ __forceinline__ bool hix_move(const HixT &h, uint32_t v, uint32_t p, uint32_t np) {
    uint32_t s = nb_hash(v) & h.mask;
    for (;;) {
        const uint32_t k = h.t[2 * s];
        if (k == 0u) return false;
        if (k == v + 1 && h.t[2 * s + 1] == p) {
            if (np == HIX_TOMB) h.t[2 * s] = HIX_TOMB;
            else h.t[2 * s + 1] = np;
            return true;
        }
        s = (s + 1) & h.mask;
    }
}

// per large touched vertex: decide whether this batch uses / builds / drops its index
__global__ void __launch_bounds__(MT) k_hix_prep(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    BSP_WARP_LOOP(h, *a.nbigs) {
        const uint32_t i = a.bigs[h];
        const uint32_t u = g.tv[a.t0 + i];
        const uint32_t L = a.vL[i], q = a.vq[i];
        const uint64_t o = g.hixo[u];
        const bool valid = o != 0 && 4ull * (L + g.hixt[u]) <= (3ull << (o >> 48));
        uint32_t mode = valid ? 1u : 0u;
        if (q) {
            const DelScr s = del_scr(g.scr + g.scr_off[i], L, q);
            bool dup = false;
            for (uint32_t sl = lane; sl < s.Hq; sl += 32) dup |= s.hkey[sl] != EMPTY_KEY && s.hk[sl] > 1u;
            if (__any_sync(0xffffffffu, dup)) {
                mode = 0;   // repeated deletes of one pair: the scan path (rounds) handles them
            } else if (!valid && L > g.hix_min) {
                // build a fresh table (zeroed pool words) for the pre-batch arcs, if the pool has room
                unsigned long long off = 0;
                const uint32_t lg = nb_log2size(L);
                if (lane == 0) off = atomicAdd(&g.bump[5], 2ull << lg);
                off = __shfl_sync(0xffffffffu, off, 0);
                if (off + (2ull << lg) <= g.hix_cap) {
                    mode = 2;
                    if (lane == 0) {
                        g.hixo[u] = (uint64_t)off | ((uint64_t)lg << 48);
                        g.hixt[u] = 0;
                    }
                } else {
                    mode = 0;   // no room: this batch scans
                }
            }
        }
        if (lane == 0) a.vhix[i] = mode;
    }
}

// table builds: the pre-batch positions [0, d) of every vertex in mode 2 (chunk items)
__global__ void __launch_bounds__(MT) k_hix_build(const BspArgs a, uint64_t total) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    const uint32_t NT = bsp_nt(a);
    total = bsp_total(a, a.p_sel, total);
    BSP_ITEM_RANGE(it, i, total, a.p_sel, NT) {
        if (a.vhix[i] != 2u) continue;
        const uint32_t c = (uint32_t)(it - a.p_sel[i]);
        const uint32_t d = a.vL[i] - a.vm[i];
        const uint64_t aoff = a.vaoff[i];
        const HixT t = hix_table(g, g.hixo[g.tv[a.t0 + i]]);
        const uint32_t e = min(d, (c + 1) * CH);
        for (uint32_t p = c * CH + lane; p < e; p += 32) hix_insert(t, __ldg(&g.arc[aoff + p].x), p);
    }
}

// round 0 of the selection (R-8) through the index: every live instance of each deleted
// destination, pre-batch ones from the table, this batch's inserts by a scan of [d, L)
__global__ void __launch_bounds__(MT) k_hix_select(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    BSP_WARP_LOOP(h, *a.nhubs) {
        const uint32_t i = a.hubs[h];
        if (!a.vhix[i]) continue;
        const uint32_t L = a.vL[i], q = a.vq[i], d = L - a.vm[i];
        const uint64_t aoff = a.vaoff[i];
        const DelScr s = del_scr(g.scr + g.scr_off[i], L, q);
        const HixT t = hix_table(g, g.hixo[g.tv[a.t0 + i]]);
        for (uint32_t sl = lane; sl < s.Hq; sl += 32) {
            const uint32_t v = s.hkey[sl];
            if (v == EMPTY_KEY) continue;
            unsigned long long best = ~0ull;
            uint32_t cnt = 0;
            for (uint32_t x = nb_hash(v) & t.mask;; x = (x + 1) & t.mask) {
                const uint32_t k = t.t[2 * x];
                if (k == 0u) break;
                if (k != v + 1) continue;
                const uint32_t p = t.t[2 * x + 1];
                const unsigned long long key = ((unsigned long long)g.arc_epoch[aoff + p] << 32) | p;
                best = key < best ? key : best;
                cnt++;
            }
            if (cnt) {
                atomicAdd(&s.hfound[sl], cnt);
                atomicMin(&s.hbest[sl], best);
            }
        }
        const uint32_t hmask = s.Hq - 1;
        for (uint32_t p = d + lane; p < L; p += 32) {
            const uint32_t hit = hash_find(s.hkey, hmask, g.arc[aoff + p].x);
            if (hit == EMPTY_KEY) continue;
            atomicAdd(&s.hfound[hit], 1u);
            atomicMin(&s.hbest[hit], ((unsigned long long)g.arc_epoch[aoff + p] << 32) | p);
        }
    }
}

// after the picks, before the arcs move: the picked pre-batch arcs leave the table
__global__ void __launch_bounds__(MT) k_hix_del(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    BSP_WARP_LOOP(h, *a.nhubs) {
        const uint32_t i = a.hubs[h];
        if (!a.vhix[i]) continue;
        const uint32_t L = a.vL[i], q = a.vq[i], d = L - a.vm[i];
        const uint32_t u = g.tv[a.t0 + i];
        const DelScr s = del_scr(g.scr + g.scr_off[i], L, q);
        const HixT t = hix_table(g, g.hixo[u]);
        uint32_t tomb = 0;
        for (uint32_t sl = lane; sl < s.Hq; sl += 32) {
            if (s.hkey[sl] == EMPTY_KEY || s.hsel[sl] == 0u) continue;   // hk = 1: at most one pick
            const uint32_t p = (uint32_t)s.hprev[sl];
            if (p < d && hix_move(t, s.hkey[sl], p, HIX_TOMB)) tomb++;
        }
        tomb = warp_sum(tomb);
        if (lane == 0) g.hixt[u] += tomb;
    }
}

// after the adjacency tail window moved (R-6): moved arcs update their entries, this batch's
// surviving inserts add theirs; a table past 3/4 load is dropped
__global__ void __launch_bounds__(MT) k_hix_ins(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    BSP_WARP_LOOP(h, *a.nbigs) {
        const uint32_t i = a.bigs[h];
        if (!a.vhix[i]) continue;
        const uint32_t L = a.vL[i], q = a.vq[i], N = a.vN[i], d = L - a.vm[i], Lp = L - N;
        const uint32_t u = g.tv[a.t0 + i];
        const uint64_t aoff = a.vaoff[i];
        const HixT t = hix_table(g, g.hixo[u]);
        if (q && N) {
            const DelScr s = del_scr(g.scr + g.scr_off[i], L, q);
            for (uint32_t x = Lp + lane; x < L; x += 32) {   // tail window: survivors moved to R
                if (bit_test(s.bm, x)) continue;
                const uint32_t np = s.R[x - Lp];
                const uint32_t v = g.arc[aoff + np].x;
                if (x < d) hix_move(t, v, x, np);
                else hix_insert(t, v, np);
            }
            for (uint32_t x = d + lane; x < Lp; x += 32)     // inserts that stayed in place
                if (!bit_test(s.bm, x)) hix_insert(t, g.arc[aoff + x].x, x);
        } else {
            for (uint32_t x = d + lane; x < L; x += 32) hix_insert(t, g.arc[aoff + x].x, x);
        }
        if (lane == 0) {
            const uint64_t o = g.hixo[u];
            if (4ull * (Lp + g.hixt[u]) > (3ull << (o >> 48))) g.hixo[u] = 0;
        }
    }
}

// ---- tables built with the graph (bingo_build): every vertex with d > min_d
__global__ void k_hix_sizes(uint32_t V, const VHdr *__restrict__ hdr, uint32_t min_d, uint64_t *__restrict__ items,
                            uint64_t *__restrict__ words) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < V; u += gridDim.x * blockDim.x) {
        const uint32_t d = hdr[u].d;
        const bool on = d > min_d;
        items[u] = on ? (d + CH - 1) / CH : 0;
        words[u] = on ? (2ull << nb_log2size(d)) : 0;
    }
}
__global__ void k_hix_offsets(uint32_t V, const VHdr *__restrict__ hdr, uint32_t min_d,
                              const uint64_t *__restrict__ woff, uint64_t *__restrict__ hixo) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < V; u += gridDim.x * blockDim.x) {
        const uint32_t d = hdr[u].d;
        hixo[u] = d > min_d ? (woff[u] | ((uint64_t)nb_log2size(d) << 48)) : 0ull;
    }
}
__global__ void __launch_bounds__(MT) k_hix_fill(uint32_t V, const uint64_t *__restrict__ pref, uint64_t total,
                                                 const VHdr *__restrict__ hdr, const uint2 *__restrict__ arc,
                                                 const uint64_t *__restrict__ hixo, uint32_t *__restrict__ hix) {
    const uint32_t lane = lane_id();
    for (uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < total;
         it += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t u = owner_of(pref, V, it);
        const uint32_t c = (uint32_t)(it - pref[u]);
        const VHdr h = hdr[u];
        HixT t;
        t.t = hix + (hixo[u] & ((1ull << 48) - 1));
        t.mask = (uint32_t)((1ull << (hixo[u] >> 48)) - 1);
        const uint32_t e = min(h.d, (c + 1) * CH);
        for (uint32_t p = c * CH + lane; p < e; p += 32) hix_insert(t, __ldg(&arc[h.adj_off + p].x), p);
    }
}

}  // namespace bingo
