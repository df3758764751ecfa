// build.cu -- sampling-space construction on the device.
//
//  k_build_sizes  (warp per vertex)  validates the CSR, counts the radix groups
//                 c_k (Eq.3/4) with one ballot per bit per 32 arcs,
//                 classifies them (Eq.9) and emits the capacity each
//                 pool needs for the vertex.
//  scans          exclusive prefix sums -> deterministic pool offsets.
//  k_build_fill   (warp per vertex)  copies the arcs, materialises REGULAR/SPARSE
//                 member lists in ascending adjacency order (R-2) by ballot
//                 compaction, finds one-element members, builds the integer Vose
//                 alias over the nonempty groups with one lane per bucket (R-4),
//                 and writes the 32 B buckets and the 32 B vertex header.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "bingo.h"
#include "bingo_internal.cuh"
#include "build_common.cuh"
#include "nbr_index.cuh"
#include "scan.cuh"
#include "sort.cuh"

using namespace bingo;

namespace bingo {

__global__ void k_build_sizes(uint32_t V, const uint64_t *__restrict__ ro, const uint32_t *__restrict__ dst,
                              const uint32_t *__restrict__ bias, uint32_t alpha, uint32_t beta, bool bs,
                              double arc_slack, double mem_slack, uint64_t *__restrict__ sz_arc,
                              uint64_t *__restrict__ sz_bkt, uint64_t *__restrict__ sz_mem, int *__restrict__ flag,
                              unsigned long long *__restrict__ hot_hist, bool allow_zero,
                              const uint32_t *__restrict__ perm) {
    __shared__ unsigned long long s_hist[2 * HOT_BINS];
    for (int i = threadIdx.x; i < 2 * HOT_BINS; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const uint32_t warps = (blockDim.x >> 5) * gridDim.x;
    const uint32_t lane = lane_id();
    for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < V; j += warps) {
        const uint32_t u = perm ? perm[j] : j;   // internal id j = hot rank of external vertex u
        const uint64_t b0 = ro[u], b1 = ro[u + 1];
        if (b1 < b0 || b1 - b0 >= 0xFFFFFFFFull) {
            if (lane == 0) atomicOr(flag, b1 < b0 ? 1 : 4);
            continue;
        }
        const uint32_t d = (uint32_t)(b1 - b0);
        uint32_t cnt = 0;       // lane k: c_k
        uint64_t tsum = 0;      // partial sum of biases
        uint32_t mask = 0;
        for (uint32_t base = 0; base < d; base += 32) {
            uint32_t i = base + lane;
            uint32_t w = 0;
            if (i < d) {
                w = bias[b0 + i];
                uint32_t v = dst[b0 + i];
                if ((w == 0 && !allow_zero) || v >= V) atomicOr(flag, 1);
                tsum += w;
            }
            mask |= w;
#pragma unroll
            for (int k = 0; k < 32; k++) {
                uint32_t bal = __ballot_sync(0xffffffffu, (w >> k) & 1u);
                if (lane == (uint32_t)k) cnt += __popc(bal);
            }
        }
        const uint64_t T = warp_sum(tsum);
        mask = __reduce_or_sync(0xffffffffu, mask);
        const uint32_t n = __popc(mask);
        if (lane == 0 && __umul64hi(T, (uint64_t)n) != 0) atomicOr(flag, 4);
        const uint32_t kind = classify(cnt, d, alpha, beta, bs);
        uint64_t units = is_list(kind) ? member_units(cnt, mem_slack) : 0;
        units = warp_sum(units);
        if (lane == 0) {
            sz_arc[j] = arc_capacity(d, arc_slack);
            sz_bkt[j] = bucket_capacity(n);
            sz_mem[j] = units;
            // walker-read bytes of this vertex by degree bin: buckets, member dsts
            atomicAdd(&s_hist[hot_bin(d)], (unsigned long long)(32ull * n));
            atomicAdd(&s_hist[HOT_BINS + hot_bin(d)], (unsigned long long)(16ull * units));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * HOT_BINS; i += blockDim.x)
        if (s_hist[i]) atomicAdd(&hot_hist[i], s_hist[i]);
}

__global__ void k_build_fill(uint32_t V, const uint64_t *__restrict__ ro, const uint32_t *__restrict__ dst,
                             const uint32_t *__restrict__ bias, uint32_t alpha, uint32_t beta, bool bs,
                             double mem_slack, const uint64_t *__restrict__ off_arc,
                             const uint64_t *__restrict__ off_bkt, const uint64_t *__restrict__ off_mem,
                             const uint64_t *__restrict__ sz_arc, VHdr *__restrict__ hdr, ThinHdr *__restrict__ thdr, uint2 *__restrict__ arc,
                             uint32_t *__restrict__ arc_epoch, Bucket *__restrict__ bkt, GCan *__restrict__ gcan,
                             uint32_t *__restrict__ mdst, uint32_t *__restrict__ midx, uint32_t hot_b,
                             uint32_t hot_m, const uint32_t *__restrict__ perm, const uint32_t *__restrict__ inv) {
    const uint32_t warps = (blockDim.x >> 5) * gridDim.x;
    const uint32_t lane = lane_id();
    for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < V; j += warps) {
        const uint32_t u = perm ? perm[j] : j;   // external row; everything stored uses internal ids
        const uint64_t b0 = ro[u];
        const uint32_t d = (uint32_t)(ro[u + 1] - b0);
        const uint64_t aoff = off_arc[j];
        // pass 1: copy arcs, count groups
        uint32_t cnt = 0;
        uint64_t tsum = 0;
        uint32_t mask = 0;
        for (uint32_t base = 0; base < d; base += 32) {
            uint32_t i = base + lane;
            uint32_t w = 0;
            if (i < d) {
                w = bias[b0 + i];
                arc[aoff + i] = make_uint2(inv ? inv[dst[b0 + i]] : dst[b0 + i], w);
                arc_epoch[aoff + i] = 0;
                tsum += w;
            }
            mask |= w;
#pragma unroll
            for (int k = 0; k < 32; k++) {
                uint32_t bal = __ballot_sync(0xffffffffu, (w >> k) & 1u);
                if (lane == (uint32_t)k) cnt += __popc(bal);
            }
        }
        const uint64_t T = warp_sum(tsum);
        mask = __reduce_or_sync(0xffffffffu, mask);
        const uint32_t n = __popc(mask);
        const uint32_t kind = classify(cnt, d, alpha, beta, bs);
        // member array of group k (lane k): offset in 16 B units, capacity in entries
        const uint32_t units = is_list(kind) ? member_units(cnt, mem_slack) : 0;
        uint32_t pre = units;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
            if ((int)lane >= o) pre += y;
        }
        pre -= units;
        const uint64_t my_off = off_mem[j] + pre;   // 16 B units
        // pass 2: members (ascending adjacency index) and one-element members
        uint32_t fill = 0;          // lane k: entries written so far
        uint32_t one_idx = 0, one_dst = 0;
        const bool any_member_kind = __any_sync(0xffffffffu, is_list(kind) || kind == K_ONE);
        if (any_member_kind) {
            for (uint32_t base = 0; base < d; base += 32) {
                uint32_t i = base + lane;
                uint32_t w = 0, v = 0;
                if (i < d) { w = bias[b0 + i]; v = inv ? inv[dst[b0 + i]] : dst[b0 + i]; }
                uint32_t mk = mask;
                while (mk) {
                    const int k = __ffs(mk) - 1;
                    mk &= mk - 1;
                    const uint32_t kind_k = __shfl_sync(0xffffffffu, kind, k);
                    if (!(is_list(kind_k) || kind_k == K_ONE)) continue;
                    const uint32_t bal = __ballot_sync(0xffffffffu, (w >> k) & 1u);
                    if (!bal) continue;
                    if (kind_k == K_ONE) {
                        const int src_lane = __ffs(bal) - 1;
                        const uint32_t vv = __shfl_sync(0xffffffffu, v, src_lane);
                        if (lane == (uint32_t)k) { one_idx = base + src_lane; one_dst = vv; }
                        continue;
                    }
                    const uint32_t start = __shfl_sync(0xffffffffu, fill, k);
                    const uint64_t goff = __shfl_sync(0xffffffffu, my_off, k);
                    if ((w >> k) & 1u) {
                        const uint64_t e = goff * 4 + start + __popc(bal & lanemask_lt());
                        mdst[e] = v;
                        midx[e] = i;
                    }
                    if (lane == (uint32_t)k) fill += __popc(bal);
                }
            }
        }
        // integer Vose over nonempty groups, lane b = bucket b (R-4)
        const uint32_t kb = (lane < n) ? (uint32_t)__fns(mask, 0, lane + 1) : 0;
        const uint32_t c_b = __shfl_sync(0xffffffffu, cnt, kb);
        const uint32_t kind_b = __shfl_sync(0xffffffffu, kind, kb);
        const uint64_t off_b = __shfl_sync(0xffffffffu, my_off, kb);
        const uint32_t oi_b = __shfl_sync(0xffffffffu, one_idx, kb);
        const uint32_t od_b = __shfl_sync(0xffffffffu, one_dst, kb);
        const uint32_t units_b = __shfl_sync(0xffffffffu, units, kb);
        uint64_t thr;
        uint32_t alias;
        vose_warp(lane < n, n, (uint64_t)c_b << kb, T, thr, alias);
        const uint64_t bo = off_bkt[j];
        uint32_t x_b, y_b;
        group_view(kind_b, c_b, (uint32_t)off_b, od_b, d, aoff, x_b, y_b);
        const uint32_t aux_b = is_list(kind_b) ? units_b * 4 : (kind_b == K_ONE ? oi_b : 0u);
        write_buckets(bkt, gcan, bo, n, lane, kb, kind_b, c_b, x_b, y_b, aux_b, thr, alias, T);
        if (lane == 0) {
            VHdr h;
            h.T = T;
            h.adj_off = aoff;
            h.bkt_off = (uint32_t)bo;
            h.d = d;
            h.n = (uint8_t)n;
            h.ncap = (uint8_t)bucket_capacity(n);
            h.pad = 0;
            h.adj_cap = (uint32_t)sz_arc[j];
            hdr[j] = h;
            ThinHdr th;
            th.bkt_off = (uint32_t)bo;
            th.n = (uint8_t)n;
            th.flags = (d >= hot_b ? 1 : 0) | (d >= hot_m ? 2 : 0);
            th.pad1 = 0;
            thdr[j] = th;
        }
    }
}

// Hot-first vertex relabelling: internal id j = rank of the vertex in descending
// out-degree (ties by id, a stable sort); perm[j] = external id, inv[u] = internal
// id.  Every per-vertex array (headers, visit counts, neighbour-set offsets, decimal
// records) is indexed by j and every stored destination is internal, so pool
// offsets (plain scans in j order) and the per-vertex arrays both put the vertices
// that serve most walk steps (walk visits are degree-skewed) into a few 2 MB pages:
// random access on B200 is bound by address translation once a footprint outgrows
// the TLB reach (~128-256 MB, profiles/r01_tlb_sweep.json).  The boundary
// translates: starts, update records and exports in, paths, counts and dumps out.
__global__ void k_hot_keys(uint32_t V, const uint64_t *__restrict__ ro, uint32_t *__restrict__ key,
                           uint32_t *__restrict__ val, bool hot) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < V; u += gridDim.x * blockDim.x) {
        key[u] = hot ? ~(uint32_t)(ro[u + 1] - ro[u]) : 0u;
        val[u] = u;
    }
}
__global__ void k_inverse(uint32_t V, const uint32_t *__restrict__ perm, uint32_t *__restrict__ inv) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < V; j += gridDim.x * blockDim.x) inv[perm[j]] = j;
}
// Hot-first pools without relabelling (graphs whose per-vertex arrays already fit
// the TLB reach): ids stay external, only the pool offsets follow the hot order.
__global__ void k_perm_gather(uint32_t V, const uint32_t *__restrict__ perm, const uint64_t *__restrict__ in,
                              uint64_t *__restrict__ out) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < V; j += gridDim.x * blockDim.x) out[j] = in[perm[j]];
}
__global__ void k_perm_scatter(uint32_t V, const uint32_t *__restrict__ perm, const uint64_t *__restrict__ in,
                               uint64_t *__restrict__ out) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= V; j += gridDim.x * blockDim.x)
        out[j < V ? perm[j] : V] = in[j];
}

// neighbour hash sets (node2vec distance test), warp per vertex
__global__ void k_build_nbt(uint32_t V, const VHdr *__restrict__ hdr, const uint2 *__restrict__ arc,
                            uint32_t *__restrict__ nbt, uint64_t *__restrict__ nbo) {
    const uint32_t warps = (blockDim.x >> 5) * gridDim.x;
    const uint32_t lane = lane_id();
    for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < V; u += warps) {
        const VHdr h = hdr[u];
        const uint32_t lg = nb_log2size(h.d);
        const uint64_t base = 4 * h.adj_off;
        uint32_t *tbl = nbt + base;
        for (uint32_t j = lane; j < (1u << lg); j += 32) tbl[j] = NB_EMPTY;
        __syncwarp();
        for (uint32_t i = lane; i < h.d; i += 32) nb_insert(tbl, (1u << lg) - 1, arc[h.adj_off + i].x);
        if (lane == 0) nbo[u] = nb_pack(base, lg);
    }
}

}  // namespace bingo

// ---------------------------------------------------------------- host side
// L2 residency plan: the walker loads every thin header with an
// evict_last policy, and the buckets / member arrays of "hot" vertices too; the
// hot set is the highest-degree vertices whose walker bytes fit in the
// persisting set-aside left after the thin headers.  Walk visits are
// degree-skewed, so this set serves most bucket and member reads.
static uint32_t degree_for_budget(const unsigned long long *hist, double budget) {
    if (budget <= 0) return 0xFFFFFFFFu;
    double acc = 0;
    int b = HOT_BINS - 1;
    for (; b >= 0; b--) {
        if (acc + (double)hist[b] > budget) break;
        acc += (double)hist[b];
    }
    return hot_bin_floor(b + 1);
}

static void choose_hot_degrees(bingo_graph *g, const unsigned long long *hist, uint64_t nV) {
    g->hot_bkt_degree = g->hot_mem_degree = 0xFFFFFFFFu;
    int dev = 0, max_persist = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess ||
        max_persist <= 0) {
        cudaGetLastError();
        g->persist_bytes = 0;
        return;
    }
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    if (cur < (size_t)max_persist) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist);
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    cudaGetLastError();
    g->persist_bytes = cur;
    const double thdr_bytes = (double)sizeof(ThinHdr) * (double)nV;
    const double budget = 0.9 * (double)cur - thdr_bytes;
    double share = 0.35;   // bucket share of the hot budget (buckets are read ~d/n times per byte more)
    if (const char *e = getenv("BINGO_L2_BUCKET_SHARE")) share = atof(e);
    g->hot_bkt_degree = degree_for_budget(hist, budget * share);
    g->hot_mem_degree = degree_for_budget(hist + HOT_BINS, budget * (1.0 - share));
}

static bingo_status fail_cuda(bingo_graph *g, cudaError_t e, const char *where) {
    fprintf(stderr, "libbingo: CUDA error in %s: %s\n", where, cudaGetErrorString(e));
    if (g) g->poisoned = 1;
    return BINGO_E_CUDA;
}
#define CK(call)                                                  \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) { st = fail_cuda(g, e_, #call); goto done; } \
    } while (0)

bingo_status float_prepare(bingo_graph *g, const bingo_build_desc *desc, uint32_t *ibias, uint64_t *dcnt,
                           uint64_t *dscan, uint64_t *tmp, cudaStream_t s, uint64_t *total_dec);
bingo_status float_fill(bingo_graph *g, const bingo_build_desc *desc, const uint64_t *dscan, cudaStream_t s);
bingo_status hix_build_all(bingo_graph *g, cudaStream_t s);
bingo_status gix_build_all(bingo_graph *g, cudaStream_t s);

extern "C" bingo_status bingo_build(const bingo_build_desc *desc, void *stream, bingo_graph **out) {
    if (!desc || !out) return BINGO_E_INVAL;
    *out = nullptr;
    const uint32_t V = desc->num_vertices;
    if (V == 0 && desc->num_arcs) return BINGO_E_INVAL;
    if (V >= 0x7FFFFFFFu) return BINGO_E_INVAL;
    if (!desc->row_offsets || (desc->num_arcs && (!desc->dst || !desc->bias))) return BINGO_E_INVAL;
    if (desc->alpha_pct > 100 || desc->beta_pct > 100) return BINGO_E_INVAL;
    cudaStream_t s = (cudaStream_t)stream;
    bingo_graph *g = new bingo_graph();
    bingo_status st = BINGO_OK;
    const bool bs = (desc->flags & BINGO_BUILD_BS_MODE) != 0;
    g->V = V;
    g->flags = desc->flags;
    g->alpha = bs ? 100 : desc->alpha_pct;
    g->beta = bs ? 0 : desc->beta_pct;
    g->alloc = desc->alloc;
    g->free_ = desc->free;
    g->alloc_ctx = desc->alloc_ctx;
    g->arc_slack = desc->arc_slack >= 0 ? desc->arc_slack : 0.25;
    g->member_slack = desc->member_slack >= 0 ? desc->member_slack : 0.25;
    g->pool_reserve = desc->pool_reserve >= 0 ? desc->pool_reserve : 0.1;
    g->num_arcs = desc->num_arcs;
    if (desc->flags & BINGO_BUILD_RADIX_MASK) {   // arbitrary radix base (radix.cu)
        const uint32_t b = (desc->flags & BINGO_BUILD_RADIX_MASK) >> 8;
        if (b > 5 || (desc->flags & (BINGO_BUILD_FLOAT_BIAS | BINGO_BUILD_NEIGHBOR_INDEX | BINGO_BUILD_BS_MODE))) {
            delete g;
            return BINGO_E_INVAL;
        }
        const bingo_status rs = build_radix(g, desc, b, s);
        if (rs != BINGO_OK) {
            bingo_destroy(g);
            return rs;
        }
        *out = g;
        return BINGO_OK;
    }

    const uint64_t nV = (uint64_t)V;
    const size_t tmpw = scan_tmp_words(nV);
    uint64_t *sz = nullptr, *off = nullptr, *tmp = nullptr;
    uint64_t tot[3] = {0, 0, 0};
    int hflag = 0;
    unsigned long long hc[4];
    unsigned long long *dhist = nullptr;
    unsigned long long hhist[2 * HOT_BINS];
    const bool fm = (desc->flags & BINGO_BUILD_FLOAT_BIAS) != 0;
    bingo_build_desc idesc = *desc;      // the integer build's view (float mode: integer parts)
    uint32_t *ibias = nullptr;
    uint64_t *dcnt = nullptr, *dscan = nullptr, total_dec = 0;
    const unsigned blocks = (unsigned)std::min<uint64_t>((nV + 7) / 8, 148ull * 64);
    // layout: 0 = vertex-id order; 1 = hot-first pools, external ids; 2 = hot-first
    // relabelling (internal ids = hot rank).  Default: 2 for V >= BINGO_RELABEL_MIN_V (the
    // per-vertex arrays outgrow the TLB reach), else 1.  BINGO_BUILD_ID_LAYOUT / BINGO_BUILD_RELABEL
    // force 0 / 2; env BINGO_LAYOUT=id|hot|relabel overrides (A/B).
    int layout = (desc->flags & BINGO_BUILD_ID_LAYOUT) ? 0
                 : (desc->flags & BINGO_BUILD_RELABEL) ? 2
                 : (V >= BINGO_RELABEL_MIN_V ? 2 : 1);
    if (const char *lay = getenv("BINGO_LAYOUT"))
        layout = strcmp(lay, "id") == 0 ? 0 : strcmp(lay, "hot") == 0 ? 1 : strcmp(lay, "relabel") == 0 ? 2 : layout;
    uint32_t *pk = nullptr, *hperm = nullptr;
    uint64_t *rtmp = nullptr, *pbuf = nullptr;

    g->counters = (unsigned long long *)bingo_dev_alloc(g, (16 + BINGO_WALK_SLOTS) * sizeof(unsigned long long));
    g->walk_ctr = g->counters ? g->counters + 16 : nullptr;
    g->dev_flag = (int *)bingo_dev_alloc(g, sizeof(int) * 4);
    g->hdr = (VHdr *)bingo_dev_alloc(g, sizeof(VHdr) * std::max<uint64_t>(nV, 1));
    g->thdr = (ThinHdr *)bingo_dev_alloc(g, sizeof(ThinHdr) * std::max<uint64_t>(nV, 1));
    g->visit = (unsigned long long *)bingo_dev_alloc(g, sizeof(unsigned long long) * std::max<uint64_t>(visit_words(V), 1));
    sz = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * 3 * (nV + 1));
    off = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * 3 * (nV + 1));
    tmp = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * tmpw);
    dhist = (unsigned long long *)bingo_dev_alloc(g, sizeof(unsigned long long) * 2 * HOT_BINS);
    if (nV && layout > 0) {
        pk = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * 4 * nV);
        rtmp = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * radix_tmp_words(nV));
        if (!pk || !rtmp) { st = BINGO_E_NOMEM; goto done; }
        const unsigned eg = (unsigned)std::min<uint64_t>((nV + 255) / 256, 148ull * 16);
        k_hot_keys<<<eg, 256, 0, s>>>(V, desc->row_offsets, pk, pk + nV, true);
        bingo_count_launch();
        CK(cudaGetLastError());
        bool in1 = false;
        CK(radix_sort_pairs(pk, pk + nV, pk + 2 * nV, pk + 3 * nV, nV, 32, rtmp, s, &in1));
        hperm = in1 ? pk + 3 * nV : pk + nV;
        if (layout == 2) {
            g->perm = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * nV);
            g->inv = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * nV);
            if (!g->perm || !g->inv) { st = BINGO_E_NOMEM; goto done; }
            CK(cudaMemcpyAsync(g->perm, hperm, sizeof(uint32_t) * nV, cudaMemcpyDeviceToDevice, s));
            k_inverse<<<eg, 256, 0, s>>>(V, g->perm, g->inv);
            bingo_count_launch();
            CK(cudaGetLastError());
        } else {
            pbuf = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * 2 * (nV + 1));
            if (!pbuf) { st = BINGO_E_NOMEM; goto done; }
        }
    }
    if (!g->counters || !g->dev_flag || !g->hdr || !g->thdr || !g->visit || !sz || !off || !tmp || !dhist) {
        st = BINGO_E_NOMEM;
        goto done;
    }
    CK(cudaMemsetAsync(dhist, 0, sizeof(unsigned long long) * 2 * HOT_BINS, s));
    if (fm) {
        g->float_mode = true;
        if (desc->num_arcs && !desc->bias_f64) { st = BINGO_E_INVAL; goto done; }
        g->dec = (DecRec *)bingo_dev_alloc(g, sizeof(DecRec) * std::max<uint64_t>(nV, 1));
        ibias = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * std::max<uint64_t>(desc->num_arcs, 1));
        dcnt = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * (nV + 1));
        dscan = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * (nV + 1));
        if (!g->dec || !ibias || !dcnt || !dscan) { st = BINGO_E_NOMEM; goto done; }
        CK(cudaMemsetAsync(g->dec, 0, sizeof(DecRec) * std::max<uint64_t>(nV, 1), s));
        if (V) {
            st = float_prepare(g, desc, ibias, dcnt, dscan, tmp, s, &total_dec);
            if (st != BINGO_OK) { if (st == BINGO_E_CUDA) g->poisoned = 1; goto done; }
        }
        idesc.bias = ibias;
    }
    CK(cudaMemsetAsync(g->counters, 0, 16 * sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(g->dev_flag, 0, sizeof(int) * 4, s));
    CK(cudaMemsetAsync(g->visit, 0, sizeof(unsigned long long) * std::max<uint64_t>(visit_words(V), 1), s));
    CK(cudaMemsetAsync(g->hdr, 0, sizeof(VHdr) * std::max<uint64_t>(nV, 1), s));
    CK(cudaMemsetAsync(g->thdr, 0, sizeof(ThinHdr) * std::max<uint64_t>(nV, 1), s));
    if (V) {
        k_build_sizes<<<blocks, 256, 0, s>>>(V, desc->row_offsets, desc->dst, idesc.bias, g->alpha, g->beta, bs,
                                             g->arc_slack, g->member_slack, sz, sz + (nV + 1), sz + 2 * (nV + 1),
                                             g->dev_flag, dhist, fm, g->perm);
        bingo_count_launch();
        CK(cudaGetLastError());
        if (layout == 1) {   // sizes are in external order; offsets follow the hot order
            const unsigned eg = (unsigned)std::min<uint64_t>((nV + 255) / 256, 148ull * 16);
            for (int p = 0; p < 3; p++) {
                k_perm_gather<<<eg, 256, 0, s>>>(V, hperm, sz + p * (nV + 1), pbuf);
                bingo_count_launch();
                CK(cudaGetLastError());
                CK(exclusive_scan_u64(pbuf, pbuf + (nV + 1), nV, tmp, s));
                k_perm_scatter<<<eg, 256, 0, s>>>(V, hperm, pbuf + (nV + 1), off + p * (nV + 1));
                bingo_count_launch();
                CK(cudaGetLastError());
            }
        } else {
            for (int p = 0; p < 3; p++) CK(exclusive_scan_u64(sz + p * (nV + 1), off + p * (nV + 1), nV, tmp, s));
        }
        CK(cudaMemcpyAsync(&hflag, g->dev_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        for (int p = 0; p < 3; p++)
            CK(cudaMemcpyAsync(&tot[p], off + p * (nV + 1) + nV, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hhist, dhist, sizeof(hhist), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        choose_hot_degrees(g, hhist, nV);
        uint64_t last_ro = 0;
        CK(cudaMemcpy(&last_ro, desc->row_offsets + V, sizeof(uint64_t), cudaMemcpyDeviceToHost));
        if (last_ro != desc->num_arcs) hflag |= 1;
        if (hflag & 1) { st = BINGO_E_INVAL; goto done; }
        if (hflag & 4) { st = BINGO_E_OVERFLOW; goto done; }
    }
    if (tot[1] >= 0xFFFFFFFFull || tot[2] >= 0xFFFFFFFFull) { st = BINGO_E_OVERFLOW; goto done; }
    g->arc_cap = pool_capacity(tot[0], g->pool_reserve, 1024);
    g->bkt_cap = std::min<uint64_t>(pool_capacity(tot[1], g->pool_reserve, 1024), 0xFFFFFFF0ull);
    g->mem_cap = 4 * std::min<uint64_t>(pool_capacity(tot[2], g->pool_reserve, 1024), 0xFFFFFFF0ull);
    g->arc = (uint2 *)bingo_dev_alloc(g, sizeof(uint2) * g->arc_cap);
    g->arc_epoch = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * g->arc_cap);
    g->bkt = (Bucket *)bingo_dev_alloc(g, sizeof(Bucket) * g->bkt_cap);
    g->gcan = (GCan *)bingo_dev_alloc(g, sizeof(GCan) * g->bkt_cap);
    g->mdst = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * g->mem_cap);
    g->midx = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * g->mem_cap);
    if (!g->arc || !g->arc_epoch || !g->bkt || !g->gcan || !g->mdst || !g->midx) { st = BINGO_E_NOMEM; goto done; }
    hc[0] = tot[0]; hc[1] = tot[1]; hc[2] = tot[2]; hc[3] = 0;
    CK(cudaMemcpyAsync(g->counters, hc, sizeof(hc), cudaMemcpyHostToDevice, s));
    if (V) {
        k_build_fill<<<blocks, 256, 0, s>>>(V, desc->row_offsets, desc->dst, idesc.bias, g->alpha, g->beta, bs,
                                            g->member_slack, off, off + (nV + 1), off + 2 * (nV + 1), sz, g->hdr, g->thdr,
                                            g->arc, g->arc_epoch, g->bkt, g->gcan, g->mdst, g->midx,
                                            g->hot_bkt_degree, g->hot_mem_degree, g->perm, g->inv);
        bingo_count_launch();
        CK(cudaGetLastError());
    }
    if (fm) {
        g->dmem_cap = std::max<uint64_t>(total_dec + total_dec / 8, 1024);
        g->dmem = (uint4 *)bingo_dev_alloc(g, sizeof(uint4) * g->dmem_cap);
        g->arc_dval = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * g->arc_cap);
        if (!g->dmem || !g->arc_dval) { st = BINGO_E_NOMEM; goto done; }
        CK(cudaMemsetAsync(g->arc_dval, 0, sizeof(uint64_t) * g->arc_cap, s));
        {
            const unsigned long long used = total_dec;   // decimal-member bump pointer (counters[3])
            CK(cudaMemcpyAsync(g->counters + 3, &used, sizeof(used), cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));
        }
        if (V) {
            st = float_fill(g, desc, dscan, s);
            if (st != BINGO_OK) { g->poisoned = 1; goto done; }
        }
    }
    if (desc->flags & BINGO_BUILD_NEIGHBOR_INDEX) {
        g->nbt = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * 4 * g->arc_cap);
        g->nbo = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * std::max<uint64_t>(nV, 1));
        g->nbtomb = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * std::max<uint64_t>(nV, 1));
        if (!g->nbt || !g->nbo || !g->nbtomb) { st = BINGO_E_NOMEM; goto done; }
        CK(cudaMemsetAsync(g->nbtomb, 0, sizeof(uint32_t) * std::max<uint64_t>(nV, 1), s));
        if (V) {
            k_build_nbt<<<blocks, 256, 0, s>>>(V, g->hdr, g->arc, g->nbt, g->nbo);
            bingo_count_launch();
            CK(cudaGetLastError());
        }
    }
    CK(cudaStreamSynchronize(s));
    st = hix_build_all(g, s);   // hub delete index (update-side, derived)
    if (st == BINGO_OK) st = gix_build_all(g, s);   // group index (update-side, derived)
    if (st == BINGO_E_CUDA) g->poisoned = 1;
done:
    bingo_dev_free(g, sz);
    bingo_dev_free(g, off);
    bingo_dev_free(g, tmp);
    bingo_dev_free(g, dhist);
    bingo_dev_free(g, pk);
    bingo_dev_free(g, rtmp);
    bingo_dev_free(g, pbuf);
    bingo_dev_free(g, ibias);
    bingo_dev_free(g, dcnt);
    bingo_dev_free(g, dscan);
    if (st != BINGO_OK) {
        bingo_destroy(g);
        return st;
    }
    *out = g;
    return BINGO_OK;
}
