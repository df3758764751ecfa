// group_index.cuh -- the per-hub group inverted index (included by update.cu after hub_index.cuh).
//
// deleting an arc must remove it from every group it belongs to, and moving an arc
// (the delete-and-swap of the adjacency) must rename it in every group that lists it;
// the paper keeps an inverted index from an edge to its position in each group for this.
// Without one, the bulk-synchronous route finds those member slots by scanning the front of
// every member list of every touched hub (k_bsp_grp_write: O(sum of list sizes) per hub --
// the dominant cost of a c4 batch).  Here every hub (L > CH arcs) that takes deletes keeps,
// from its first such batch on, a multimap (adjacency position p, radix group k) -> member
// slot of p in group k, over its REGULAR/SPARSE groups (open addressing, 2 words per entry
// {key + 1, slot}, key = p << 5 | k, 0 = empty, GIX_TOMB = removed; tables come zeroed from a
// bump pool, counters[6]).  The bulk-synchronous route keeps it exact:
//   inserts (k_bsp_alloc_insert)   every member appended for an inserted arc adds its entry;
//   picks (k_gix_front, phase 1)   every deleted arc's entries leave; the slots below the
//                                  group's new length L_k' are the group's holes (appended, then
//                                  sorted by k_bsp_grp_sort: the same list the front scan makes);
//   moves (k_gix_front, phase 2)   every survivor of the adjacency tail window that moved from t
//                                  to R[t - L'] is renamed in its front slots and its
//                                  entries re-keyed to the new position;
//   group tails (k_bsp_grp_tail)   a survivor moved from a group's tail window into a hole
//                                  gets its new slot.
// The index is derived state, dropped (and rebuilt from the member lists by k_gix_build at the
// next batch with deletes) when a route that does not maintain it touches the vertex, when a
// group changes between list and non-list layouts, when the batch deletes more than SORT_MAX
// of its arcs, or past 3/4 load (entries + tombstones).  Lookups find exactly the slots the
// scan would find, so the result is the same bit for bit.
#pragma once

namespace bingo {

// ---- per large touched vertex: use (1), build (2) or drop (0) the index this batch.  After
// k_bsp_hub_sort (vrank known) and k_bsp_alloc_insert (inserts entered into valid tables).
__global__ void __launch_bounds__(MT) k_gix_prep(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    const MutateArgs &g = a.g;
    for (uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x); h < *a.nbigs; h += gridDim.x * blockDim.x) {
        const uint32_t i = a.bigs[h];
        const uint32_t u = g.tv[a.t0 + i];
        const uint32_t L = a.vL[i], q = a.vq[i];
        const uint64_t o = g.gixo[u];
        const bool hub = q != 0;                       // in the hubs list: its group fronts change
        const bool sorted = !hub || (a.vN[i] <= SORT_MAX && !a.vrank[i]);
        uint32_t mode = 0;
        if (o != 0 && sorted && L <= GIX_MAXL) {
            mode = 1;
        } else if (o == 0 && hub && sorted && a.vN[i] && L <= GIX_MAXL && L > g.gix_min) {
            // a fresh table for the post-insert member lists: 2^lg >= 2 x entries
            const uint32_t lg = nb_log2size(max(a.vgixe[i], 1u));
            const unsigned long long words = 2ull << lg;
            const unsigned long long off = atomicAdd(&g.bump[6], words);
            if (off + words <= g.gix_cap) {
                g.gixo[u] = (uint64_t)off | ((uint64_t)lg << 48);
                g.gixt[u] = 0;
                mode = 2;
            }
        }
        if (mode == 0 && o != 0) g.gixo[u] = 0;       // not maintained by this batch
        a.vgix[i] = mode;
    }
}

// ---- builds: every member slot of every list group of the vertices in mode 2 (group items)
__global__ void __launch_bounds__(MT) k_gix_build(const BspArgs a, uint64_t total) {
    if (BSP_ABORTED(a)) return;
    const uint32_t lane = lane_id();
    const MutateArgs &g = a.g;
    const uint32_t NT = bsp_nt(a);
    total = bsp_total(a, a.p_grp, total);
    BSP_ITEM_RANGE(it, own, total, a.p_grp, NT) {
        if (a.vgix[own] != 2u) continue;
        const GrpItem gi = grp_item(a, it, own);
        const GixT t = gix_table(g.gix, g.gixo[g.tv[a.t0 + gi.i]]);
        const uint32_t *Mi = g.midx + (uint64_t)gi.moff * 4;
        const uint32_t e = min(gi.cp, (gi.j + 1) * CH);
        bool ok = true;
        for (uint32_t sl = gi.j * CH + lane; sl < e; sl += 32) ok &= gix_insert(t, gix_key(__ldg(Mi + sl), gi.k), sl);
        if (!__all_sync(0xffffffffu, ok) && lane == 0) a.vgix[gi.i] = 3u;   // full: scan this batch, drop
    }
}

// ---- after the adjacency tail window moved (k_bsp_tail): one warp per hub in mode 1 / 2.
// Phase 1: the picks' entries leave; their slots below L_k' are the group's front holes.
// Phase 2: moved survivors are renamed in their front slots and re-keyed.
__global__ void __launch_bounds__(MT) k_gix_front(const BspArgs a) {
    if (BSP_ABORTED(a)) return;
    __shared__ uint32_t s_lk[MT / 32][32];
    const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
    const MutateArgs &g = a.g;
    BSP_WARP_LOOP(h, *a.nhubs) {
        const uint32_t i = a.hubs[h];
        const uint32_t mode = a.vgix[i];
        if (mode == 0 || mode == 3) continue;
        const uint32_t u = g.tv[a.t0 + i];
        const uint32_t L = a.vL[i], q = a.vq[i], N = a.vN[i], Lp = L - N;
        const DelScr s = del_scr(g.scr + g.scr_off[i], L, q);
        const GixT t = gix_table(g.gix, g.gixo[u]);
        const uint32_t list0 = a.vlist0[i];
        const uint64_t aoff = a.vaoff[i];
        const uint32_t Nk = gkp(a, GK_DELK, i)[lane];
        s_lk[w][lane] = gkp(a, GK_C, i)[lane] + gkp(a, GK_INSK, i)[lane] - Nk;   // L_k'
        __syncwarp();
        uint32_t rem = 0;
        bool ok = true, ins_ok = true;   // ok: every looked-up entry exists (it always should)
        for (uint32_t j = lane; j < N; j += 32) {
            const uint2 pb = s.pk[j];
            uint32_t bits = pb.y & list0;
            while (bits) {
                const uint32_t k = __ffs(bits) - 1;
                bits &= bits - 1;
                const uint32_t e = gix_find(t, gix_key(pb.x, k));
                if (e == 0xFFFFFFFFu) {
                    ok = false;
                    continue;
                }
                const uint32_t sl = t.t[2 * e + 1];
                t.t[2 * e] = GIX_TOMB;
                rem++;
                if (sl < s_lk[w][k]) s.gh[gkp(a, GK_GHO, i)[k] + atomicAdd(gkp(a, GK_GHN, i) + k, 1u)] = sl;
            }
        }
        __syncwarp();
        __threadfence_block();
        for (uint32_t x = Lp + lane; x < L; x += 32) {
            if (bit_test(s.bm, x)) continue;
            const uint32_t np = s.R[x - Lp];
            uint32_t bits = g.arc[aoff + np].y & list0;
            while (bits) {
                const uint32_t k = __ffs(bits) - 1;
                bits &= bits - 1;
                const uint32_t e = gix_find(t, gix_key(x, k));
                if (e == 0xFFFFFFFFu) {
                    ok = false;
                    continue;
                }
                const uint32_t sl = t.t[2 * e + 1];
                t.t[2 * e] = GIX_TOMB;
                rem++;
                if (sl < s_lk[w][k]) g.midx[(uint64_t)gkp(a, GK_MOFF, i)[k] * 4 + sl] = np;   // front rename
                ins_ok &= gix_insert(t, gix_key(np, k), sl);   // tail slots: the group tail renames and re-slots
            }
        }
        rem = warp_sum(rem);
        const bool all_ok = __all_sync(0xffffffffu, ok), all_ins = __all_sync(0xffffffffu, ins_ok);
        if (lane == 0) {
            g.gixt[u] += rem;
            if (!all_ins) a.vgix[i] = 4u;             // table full: dropped after this batch (the result stands)
            if (!all_ok) atomicAdd(a.err, 1ull);      // a missing entry: the host fails the call loudly
        }
    }
}

// ---- tables built with the graph (gix_build_all): every vertex with min_d < d <= GIX_MAXL
// words[u] = table words of u (0 = none), ent[u] = its entries (list-group members)
__global__ void __launch_bounds__(MT) k_gix_sizes(uint32_t V, const VHdr *__restrict__ hdr, const Bucket *bkt,
                                                  const GCan *gcan, uint32_t min_d, uint64_t *__restrict__ words,
                                                  uint32_t *__restrict__ list, uint32_t *nlist) {
    const uint32_t lane = lane_id();
    for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < V; u += (gridDim.x * blockDim.x) >> 5) {
        const VHdr h = hdr[u];
        if (h.d <= min_d || h.d > GIX_MAXL) {
            if (lane == 0) words[u] = 0;
            continue;
        }
        uint32_t kind_k, c_k, ref_k, aux_k;
        OldGroups og;
        load_old_groups(bkt, gcan, h, kind_k, c_k, ref_k, aux_k, og);
        const uint32_t E = warp_sum(is_list(kind_k) ? c_k : 0u);
        if (lane == 0) {
            words[u] = E ? (2ull << nb_log2size(E)) : 0ull;
            if (E && list) list[atomicAdd(nlist, 1u)] = u;
        }
    }
}
__global__ void k_gix_offsets(uint32_t V, const uint64_t *__restrict__ words, const uint64_t *__restrict__ woff,
                              uint64_t *__restrict__ gixo) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < V; u += gridDim.x * blockDim.x) {
        const uint64_t w = words[u];
        gixo[u] = w ? (woff[u] | ((uint64_t)(62 - __clzll(w)) << 48)) : 0ull;   // w = 2 << lg
    }
}
// one block per listed vertex: every member slot of every list group enters the table
__global__ void __launch_bounds__(256) k_gix_fill(const uint32_t *__restrict__ list, uint32_t nl,
                                                  const VHdr *__restrict__ hdr, const Bucket *bkt, const GCan *gcan,
                                                  const uint32_t *__restrict__ midx, const uint64_t *__restrict__ gixo,
                                                  uint32_t *gix) {
    __shared__ uint32_t s_c[32], s_m[32], s_pre[33];
    for (uint32_t j = blockIdx.x; j < nl; j += gridDim.x) {
        const uint32_t u = list[j];
        if (threadIdx.x < 32) {
            const VHdr h = hdr[u];
            uint32_t kind_k, c_k, ref_k, aux_k;
            OldGroups og;
            load_old_groups(bkt, gcan, h, kind_k, c_k, ref_k, aux_k, og);
            const uint32_t c = is_list(kind_k) ? c_k : 0u;
            uint32_t x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (threadIdx.x >= (uint32_t)o) x += y;
            }
            s_c[threadIdx.x] = c;
            s_m[threadIdx.x] = ref_k;
            s_pre[threadIdx.x] = x - c;
            if (threadIdx.x == 31) s_pre[32] = x;
        }
        __syncthreads();
        const GixT t = gix_table(gix, gixo[u]);
        const uint32_t E = s_pre[32];
        for (uint32_t f = threadIdx.x; f < E; f += blockDim.x) {
            uint32_t k = 0;   // the group of flat index f: largest k with s_pre[k] <= f and c_k > 0
#pragma unroll
            for (int b = 16; b > 0; b >>= 1)
                if (k + b < 32 && s_pre[k + b] <= f) k += b;
            while (!s_c[k] || s_pre[k] + s_c[k] <= f) k++;
            const uint32_t sl = f - s_pre[k];
            gix_insert(t, gix_key(__ldg(midx + (uint64_t)s_m[k] * 4 + sl), k), sl);
        }
        __syncthreads();
    }
}

}  // namespace bingo
