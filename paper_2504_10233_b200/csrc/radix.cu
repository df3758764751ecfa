// radix.cu -- Bingo with an arbitrary radix base B = 2^b (reading R-17).
//
// A bias w = sum_i d_i B^i (digits d_i < B).  Group B^i holds the arcs with d_i != 0 and
// weighs W_i = B^i sum_j j c_ij; its neighbours no longer share one bias, so it is
// split into subgroups by digit value j (c_ij arcs each, ascending adjacency index) and an
// inter-subgroup alias over the weights j c_ij picks one before a member is
// drawn uniformly.  Fewer groups (K = 32 / b instead of 32: the complexity and memory term
// of Table timecmp) against one more dependent stage per step.
//
// HBM layout (vertex-id order).  The paper leaves nested dynamic structures to future work
// (P:927); here bingo_apply_updates rebuilds a touched vertex's structure from its updated
// adjacency (reading R-19, apply_radix below), which lives in the arc pool:
//   thdr[u]   {first bucket, n groups}
//   hdr[u]    T, d, adjacency offset / capacity (exports, updates)
//   arc, arc_epoch  the adjacency {dst, bias} and insert epochs (R-19), CSR order at build
//   bkt/gcan  per vertex: its n group buckets, then every group's subgroup buckets
//             (contiguous per group, ascending j).  A group bucket's view (px, py) is
//             (number of subgroups, pool index of its first subgroup bucket); a subgroup
//             bucket's view is (c, member offset in 16 B units) -- the same 32 B Bucket as
//             base 2, with lim = ceil(thr 2^64 / total) of its own alias (R-4').  gcan keeps
//             the canonical thr and (ns | c) for exports.
//   mdst      member dst of every subgroup, 4-entry (16 B) aligned.
// Walker step: thdr -> group bucket (tag 0) -> subgroup bucket (tag 6) -> member (tag 1).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "bingo.h"
#include "bingo_internal.cuh"
#include "build_common.cuh"
#include "scan.cuh"
#include "sort.cuh"
#include "walk_common.cuh"

using namespace bingo;

namespace bingo {

static constexpr int RB_WARPS = 8;                 // warps (vertices) per 256-thread block
static constexpr int RB_CELLS = 256;               // K x B <= 256 for b <= 5 (224 at b = 5)

__device__ __forceinline__ uint32_t rb_digit(uint32_t w, uint32_t i, uint32_t b) {
    const uint32_t sh = i * b;
    return sh >= 32 ? 0u : (w >> sh) & ((1u << b) - 1u);
}

// per-warp histogram c[i * B + j] of the vertex's digits (shared atomics), then the
// per-vertex sizes: buckets n + nsub, member units sum ceil(c / 4), T; overflow flag.
// A vertex's arcs as seen by the build: dst[a * st], bias[a * st] (st = 1: CSR arrays; st = 2:
// the {dst, bias} uint2 arc pool of an updatable radix graph).
struct RbArcs {
    const uint32_t *dst, *bias;
    uint32_t st;
    __device__ __forceinline__ uint32_t w(uint32_t a) const { return bias[(uint64_t)a * st]; }
    __device__ __forceinline__ uint32_t v(uint32_t a) const { return dst[(uint64_t)a * st]; }
};

__device__ __forceinline__ void rb_hist(const RbArcs &arcs, uint32_t d, uint32_t b, uint32_t *c) {
    const uint32_t lane = lane_id(), B = 1u << b, K = (32 + b - 1) / b;
    for (uint32_t x = lane; x < K * B; x += 32) c[x] = 0;
    __syncwarp();
    for (uint32_t a = lane; a < d; a += 32) {
        const uint32_t w = arcs.w(a);
        for (uint32_t i = 0; i < K; i++) {
            const uint32_t j = rb_digit(w, i, b);
            if (j) atomicAdd(&c[i * B + j], 1u);
        }
    }
    __syncwarp();
}

// one warp: the vertex's bucket count (groups + subgroups) and member units; T (overflow flags)
__device__ __forceinline__ void rb_sizes_vertex(const RbArcs &arcs, uint32_t d, uint32_t b, uint32_t *c,
                                                uint64_t &nb_out, uint64_t &units_out, uint64_t &T_out,
                                                int *__restrict__ flag) {
    const uint32_t lane = lane_id(), B = 1u << b, K = (32 + b - 1) / b;
    uint64_t T = 0;
    for (uint32_t a = lane; a < d; a += 32) {
        const uint32_t w = arcs.w(a);
        if (w == 0) atomicOr(flag, 1);
        T += w;
    }
    T = warp_sum(T);
    rb_hist(arcs, d, b, c);
    uint32_t ng = 0, nsub = 0;
    uint64_t units = 0;
    for (uint32_t i = lane; i < K; i += 32) {
        uint32_t ns = 0;
        for (uint32_t j = 1; j < B; j++) {
            const uint32_t cc = c[i * B + j];
            ns += cc ? 1u : 0u;
            units += (cc + 3) / 4;
        }
        nsub += ns;
        ng += ns ? 1u : 0u;
    }
    ng = warp_sum(ng);
    nsub = warp_sum(nsub);
    units = warp_sum(units);
    if (lane == 0 && (unsigned __int128)T * ng >= ((unsigned __int128)1 << 64)) atomicOr(flag, 4);
    nb_out = ng + nsub;
    units_out = units;
    T_out = T;
    __syncwarp();
}

__global__ void __launch_bounds__(256) k_rb_sizes(uint32_t V, const uint64_t *__restrict__ ro,
                                                  const uint32_t *__restrict__ bias, uint32_t b,
                                                  uint64_t *__restrict__ nbkt, uint64_t *__restrict__ nmem,
                                                  int *__restrict__ flag) {
    __shared__ uint32_t cs[RB_WARPS][RB_CELLS];
    const uint32_t wib = threadIdx.x >> 5, lane = lane_id();
    uint32_t *c = cs[wib];
    for (uint32_t u = blockIdx.x * RB_WARPS + wib; u < V; u += gridDim.x * RB_WARPS) {
        const uint64_t a0 = ro[u];
        const uint64_t dd = ro[u + 1] - a0;
        if (dd >= 0xFFFFFFFFull) {
            if (lane == 0) atomicOr(flag, 4);
            continue;
        }
        const RbArcs arcs{nullptr, bias + a0, 1u};
        uint64_t nb, units, T;
        rb_sizes_vertex(arcs, (uint32_t)dd, b, c, nb, units, T, flag);
        if (lane == 0) {
            nbkt[u] = nb;
            nmem[u] = units;
        }
    }
}

// One warp: from the digit histogram c (cells i * B + j) and T, the vertex's group and subgroup
// buckets at bo (both integer-Vose tables), and in cu the first member entry of every subgroup
// relative to munits * 4 (groups ascending i, subgroups ascending j).  Returns n (groups).
__device__ __forceinline__ uint32_t rb_tables(const uint32_t *c, uint32_t *cu, uint64_t T, uint32_t b, uint64_t bo,
                                              uint64_t munits, Bucket *__restrict__ bkt, GCan *__restrict__ gcan) {
    const uint32_t lane = lane_id(), B = 1u << b, K = (32 + b - 1) / b;
    // lane g < n owns nonempty group g (ascending i): its digit i, subgroup count ns and
    // S = sum_j j c_ij; lane-serial prefix of ns for the subgroup bucket bases
    uint32_t gi = 0, gns = 0;
    uint64_t gS = 0;
    uint32_t n = 0;
    for (uint32_t i = 0; i < K; i++) {
        uint32_t ns = 0;
        uint64_t S = 0;
        for (uint32_t j = 1; j < B; j++) {
            const uint32_t cc = c[i * B + j];
            ns += cc ? 1u : 0u;
            S += (uint64_t)j * cc;
        }
        if (!ns) continue;
        if (lane == n) { gi = i; gns = ns; gS = S; }
        n++;
    }
    uint32_t sub0 = 0;   // exclusive prefix of ns over the groups before lane's group
    {
        uint32_t v = lane < n ? gns : 0u;
        uint32_t incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        sub0 = incl - v;
    }
    // member offsets of every subgroup in (i ascending, j ascending) order, as entry
    // cursors relative to the vertex's first member unit (the pool index is u64)
    const uint64_t mbase = munits * 4;
    if (lane == 0) {
        uint32_t mo = 0;
        for (uint32_t i = 0; i < K; i++)
            for (uint32_t j = 1; j < B; j++) {
                const uint32_t cc = c[i * B + j];
                cu[i * B + j] = mo * 4;
                mo += (cc + 3) / 4;
            }
    }
    __syncwarp();
    // group alias (R-4) over W_g = B^i S_g, one lane per group
    const bool act = lane < n;
    const uint64_t W = act ? (gS << (gi * b)) : 0ull;
    uint64_t thr;
    uint32_t alias;
    vose_warp(act, n, W, T, thr, alias);
    const uint32_t sub_base = (uint32_t)(bo + n + sub0);
    {
        Bucket Bk;
        Bk.lim = alias_lim(thr, T);
        Bk.px = gns;
        Bk.py = sub_base;
        Bk.kk = make_kk(gi, K_REGULAR);
        Bk.alias = (uint8_t)alias;
        Bk.pad = 0;
        Bk.spare = 0;
        Bk.ax = __shfl_sync(0xffffffffu, gns, alias);
        Bk.ay = __shfl_sync(0xffffffffu, sub_base, alias);
        Bk.a_kk = (uint8_t)__shfl_sync(0xffffffffu, (uint32_t)Bk.kk, alias);
        if (act) {
            store_bucket(&bkt[bo + lane], Bk);
            store_gcan(&gcan[bo + lane], thr, gns, gi);
        }
    }
    // subgroup aliases (R-4), group by group, one lane per subgroup
    for (uint32_t g = 0; g < n; g++) {
        const uint32_t i = __shfl_sync(0xffffffffu, gi, g);
        const uint32_t ns = __shfl_sync(0xffffffffu, gns, g);
        const uint64_t S = __shfl_sync(0xffffffffu, gS, g);
        const uint32_t sb = __shfl_sync(0xffffffffu, sub_base, g);
        // lane s < ns owns the s-th nonempty subgroup (ascending j)
        uint32_t j_s = 0, c_s = 0, k = 0;
        for (uint32_t j = 1; j < B; j++) {
            const uint32_t cc = c[i * B + j];
            if (!cc) continue;
            if (lane == k) { j_s = j; c_s = cc; }
            k++;
        }
        const bool sact = lane < ns;
        uint64_t sthr;
        uint32_t salias;
        vose_warp(sact, ns, sact ? (uint64_t)j_s * c_s : 0ull, S, sthr, salias);
        const uint32_t mo_s = sact ? (uint32_t)(mbase / 4) + cu[i * B + j_s] / 4 : 0u;
        Bucket Bs;
        Bs.lim = alias_lim(sthr, S);
        Bs.px = c_s;
        Bs.py = mo_s;
        Bs.kk = make_kk(j_s, K_REGULAR);
        Bs.alias = (uint8_t)salias;
        Bs.pad = 0;
        Bs.spare = 0;
        Bs.ax = __shfl_sync(0xffffffffu, c_s, salias);
        Bs.ay = __shfl_sync(0xffffffffu, mo_s, salias);
        Bs.a_kk = (uint8_t)__shfl_sync(0xffffffffu, (uint32_t)Bs.kk, salias);
        if (sact) {
            store_bucket(&bkt[(uint64_t)sb + lane], Bs);
            store_gcan(&gcan[(uint64_t)sb + lane], sthr, c_s, j_s);
        }
    }
    __syncwarp();
    return n;
}

// One warp: the members of arcs [lo, hi) in ascending index appended to their subgroups at the
// cursors cu (entries relative to mbase; advanced).
__device__ __forceinline__ void rb_members(const RbArcs &arcs, uint32_t lo, uint32_t hi, uint32_t b, uint32_t *cu,
                                           uint64_t mbase, uint32_t *__restrict__ mdst) {
    const uint32_t lane = lane_id(), B = 1u << b, K = (32 + b - 1) / b;
    // members: arcs in ascending index, 32 at a time; for each digit position the lanes
    // with the same digit value are ranked by lane (= adjacency order) and appended
    for (uint32_t base = lo; base < hi; base += 32) {
        const uint32_t a = base + lane;
        const bool in = a < hi;
        const uint32_t w = in ? arcs.w(a) : 0u;
        const uint32_t v = in ? arcs.v(a) : 0u;
        for (uint32_t i = 0; i < K; i++) {
            const uint32_t j = rb_digit(w, i, b);
            const uint32_t key = in && j ? j : 0xFFFFFFFFu;
            const uint32_t same = __match_any_sync(0xffffffffu, key);
            uint32_t pos = 0;
            if (key != 0xFFFFFFFFu) pos = cu[i * B + j] + __popc(same & lanemask_lt());
            __syncwarp();
            if (key != 0xFFFFFFFFu) {
                mdst[mbase + pos] = v;
                if ((__ffs(same) - 1) == (int)lane) cu[i * B + j] += __popc(same);
            }
            __syncwarp();
        }
    }
    __syncwarp();
}

__device__ __forceinline__ void rb_headers(uint32_t u, uint64_t T, uint32_t d, uint64_t bo, uint32_t n,
                                           uint64_t adj_off, uint32_t adj_cap, VHdr *__restrict__ hdr,
                                           ThinHdr *__restrict__ thdr) {
    ThinHdr th;
    th.bkt_off = (uint32_t)bo;
    th.n = (uint8_t)n;
    th.flags = 0;
    th.pad1 = 0;
    thdr[u] = th;
    VHdr h;
    memset(&h, 0, sizeof(h));
    h.T = T;
    h.d = d;
    h.bkt_off = (uint32_t)bo;
    h.n = (uint8_t)n;
    h.adj_off = adj_off;
    h.adj_cap = adj_cap;
    hdr[u] = h;
}

// One warp builds vertex u's nested structure from its arcs into buckets [bo, bo + n + nsub)
// and member units from munits, and writes its headers (adj_off / adj_cap: where its arcs
// live, updatable graphs).  c, cu: the warp's shared digit histogram / cursors.
__device__ __forceinline__ void rb_fill_vertex(uint32_t u, const RbArcs &arcs, uint32_t d, uint32_t b, uint64_t bo,
                                               uint64_t munits, uint64_t adj_off, uint32_t adj_cap, uint32_t *c,
                                               uint32_t *cu, VHdr *__restrict__ hdr, ThinHdr *__restrict__ thdr,
                                               Bucket *__restrict__ bkt, GCan *__restrict__ gcan,
                                               uint32_t *__restrict__ mdst) {
    const uint32_t lane = lane_id();
    uint64_t T = 0;
    for (uint32_t a = lane; a < d; a += 32) T += arcs.w(a);
    T = warp_sum(T);
    rb_hist(arcs, d, b, c);
    const uint32_t n = rb_tables(c, cu, T, b, bo, munits, bkt, gcan);
    rb_members(arcs, 0, d, b, cu, munits * 4, mdst);
    if (lane == 0) rb_headers(u, T, d, bo, n, adj_off, adj_cap, hdr, thdr);
    __syncwarp();
}

__global__ void __launch_bounds__(256) k_rb_fill(uint32_t V, const uint64_t *__restrict__ ro,
                                                 const uint32_t *__restrict__ dst, const uint32_t *__restrict__ bias,
                                                 uint32_t b, const uint64_t *__restrict__ boff,
                                                 const uint64_t *__restrict__ moff, VHdr *__restrict__ hdr,
                                                 ThinHdr *__restrict__ thdr, Bucket *__restrict__ bkt,
                                                 GCan *__restrict__ gcan, uint32_t *__restrict__ mdst,
                                                 uint64_t *__restrict__ meta) {
    __shared__ uint32_t cs[RB_WARPS][RB_CELLS];
    __shared__ uint32_t cur[RB_WARPS][RB_CELLS];   // member write cursor of subgroup (i, j), 4-entry units x 4
    const uint32_t wib = threadIdx.x >> 5;
    for (uint32_t u = blockIdx.x * RB_WARPS + wib; u < V; u += gridDim.x * RB_WARPS) {
        const uint64_t a0 = ro[u];
        const uint32_t d = (uint32_t)(ro[u + 1] - a0);
        const RbArcs arcs{dst + a0, bias + a0, 1u};
        // the arcs live in the graph's arc pool at the same offsets (a copy of the CSR)
        rb_fill_vertex(u, arcs, d, b, boff[u], moff[u], a0, d, cs[wib], cur[wib], hdr, thdr, bkt, gcan, mdst);
        if (lane_id() == 0) {   // the vertex's structure space, for in-place rebuilds (R-19)
            meta[u] = moff[u];
            meta[V + u] = ((boff[u + 1] - boff[u]) << 32) | (moff[u + 1] - moff[u]);
        }
    }
}

// the CSR copied into the arc pool at the same offsets (updatable radix graphs keep their
// adjacency: reading R-19)
__global__ void k_rb_arcs(uint64_t A, const uint32_t *__restrict__ dst, const uint32_t *__restrict__ bias,
                          uint2 *__restrict__ arc) {
    for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < A; a += (uint64_t)gridDim.x * blockDim.x)
        arc[a] = make_uint2(dst[a], bias[a]);
}

// three-stage sample (R-17): group (tag 0), subgroup (tag 6), member (tag 1)
__device__ __forceinline__ uint32_t sample_dst_rb(const WalkArgs &a, const ThinHdr &h, uint32_t w, uint32_t t,
                                                  const Policies &pol) {
    const P4 r = draw_oi(w, t, 0u, 0u, 0u, a.k0, a.k1);
    const Bucket G = ldg_bucket(a.bkt + h.bkt_off + __umulhi(r.x, (uint32_t)h.n), pol.keep);
    const bool ga = join64(r.y, r.z) >= G.lim;
    const uint32_t ns = ga ? G.ax : G.px, sb = ga ? G.ay : G.py;
    const P4 r2 = draw_oi(w, t, 0u, 0u, 6u, a.k0, a.k1);
    const Bucket S = ldg_bucket(a.bkt + sb + __umulhi(r2.x, ns), pol.keep);
    const bool sa = join64(r2.y, r2.z) >= S.lim;
    const uint32_t c = sa ? S.ax : S.px, mo = sa ? S.ay : S.py;
    const P4 q = draw_oi(w, t, 0u, 0u, 1u, a.k0, a.k1);
    const uint64_t j = __umul64hi(join64(q.x, q.y), (uint64_t)c);
    return ldg4(a.mdst + (uint64_t)mo * 4 + j, pol.stream);
}

// persistent grid, one walker per lane, dynamic claiming (as k_walk); DeepWalk / PPR
template <int APP>
__global__ void __launch_bounds__(256, 2) k_walk_rb(const WalkArgs a, unsigned long long *__restrict__ claim) {
    uint64_t pol_keep, pol_stream;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    const Policies pol{pol_keep, pol_stream};
    const uint32_t lane = lane_id();
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool active = i < a.W;
    uint32_t w = 0, u = 0, t = 0;
    auto start = [&]() {
        w = a.first_walker + (uint32_t)i;
        u = a.starts ? a.starts[i] : (uint32_t)(((uint64_t)a.first_walker + i) % a.V);
        if (a.paths) __stcs(&a.paths[i], u);
        if (APP == BINGO_PPR && a.visit) atomicAdd(&a.visit[visit_slot(u)], 1ull);
        t = 0;
    };
    if (active) start();
    for (;;) {
        bool fin = false;
        if (active) {
            if (a.L != BINGO_NO_CAP && t >= a.L) {
                fin = true;
            } else {
                const ThinHdr h = load_thdr(a.thdr + u, pol);
                if (h.n == 0) {
                    fin = true;
                } else {
                    const uint32_t next = sample_dst_rb(a, h, w, t, pol);
                    if (a.paths) __stcs(&a.paths[(size_t)(t + 1) * a.W + i], next);
                    u = next;
                    if (APP == BINGO_PPR) {
                        if (a.visit) atomicAdd(&a.visit[visit_slot(u)], 1ull);
                        if (a.stop_always) {
                            fin = true;
                        } else {
                            const P4 r = philox10(w, t, 0u, 3u, a.k0, a.k1);
                            fin = join64(r.x, r.y) < a.stop_thr;
                        }
                    }
                    t++;
                    if (a.L != BINGO_NO_CAP && t >= a.L) fin = true;
                }
            }
            if (fin) {
                if (a.lengths) a.lengths[i] = t;
                if (a.paths && a.L != BINGO_NO_CAP)
                    for (uint32_t s = t + 1; s <= a.L; s++) __stcs(&a.paths[(size_t)s * a.W + i], 0xFFFFFFFFu);
            }
        }
        const unsigned fmask = __ballot_sync(0xffffffffu, fin);
        if (fmask) {
            const uint32_t leader = __ffs(fmask) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(claim, (unsigned long long)__popc(fmask));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (fin) {
                i = nthreads + base + __popc(fmask & lanemask_lt());
                active = i < a.W;
                if (active) start();
            }
        }
        if (!__any_sync(0xffffffffu, active)) break;
    }
}

}  // namespace bingo

static uint64_t rb_pool(uint64_t used, double reserve) {
    return std::max<uint64_t>(used + (uint64_t)((double)used * reserve) + 1024, 1024);
}

// bingo_build with BINGO_BUILD_RADIX_LOG2(b), b in [1, 5] (called by bingo_build)
bingo_status build_radix(bingo_graph *g, const bingo_build_desc *desc, uint32_t b, cudaStream_t s) {
    const uint32_t V = desc->num_vertices;
    const uint64_t nV = V;
    g->radix_log2 = b;
    g->counters = (unsigned long long *)bingo_dev_alloc(g, (16 + BINGO_WALK_SLOTS) * sizeof(unsigned long long));
    g->walk_ctr = g->counters ? g->counters + 16 : nullptr;
    g->dev_flag = (int *)bingo_dev_alloc(g, sizeof(int) * 4);
    g->hdr = (VHdr *)bingo_dev_alloc(g, sizeof(VHdr) * std::max<uint64_t>(nV, 1));
    g->thdr = (ThinHdr *)bingo_dev_alloc(g, sizeof(ThinHdr) * std::max<uint64_t>(nV, 1));
    g->visit = (unsigned long long *)bingo_dev_alloc(g, sizeof(unsigned long long) * std::max<uint64_t>(visit_words(V), 1));
    uint64_t *sz = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * 2 * (nV + 1));
    uint64_t *off = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * 2 * (nV + 1));
    uint64_t *tmp = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * scan_tmp_words(nV + 1));
    bingo_status st = BINGO_OK;
    auto done = [&](bingo_status r) {
        bingo_dev_free(g, sz);
        bingo_dev_free(g, off);
        bingo_dev_free(g, tmp);
        return r;
    };
    if (!g->counters || !g->dev_flag || !g->hdr || !g->thdr || !g->visit || !sz || !off || !tmp)
        return done(BINGO_E_NOMEM);
    const unsigned blocks = (unsigned)std::min<uint64_t>((nV + RB_WARPS - 1) / RB_WARPS, 148ull * 64);
    int hflag = 0;
    uint64_t tot[2] = {0, 0};
#define RCK(call)                                                            \
    do {                                                                     \
        if ((call) != cudaSuccess) { g->poisoned = 1; return done(BINGO_E_CUDA); } \
    } while (0)
    RCK(cudaMemsetAsync(g->counters, 0, (16 + BINGO_WALK_SLOTS) * sizeof(unsigned long long), s));
    RCK(cudaMemsetAsync(g->dev_flag, 0, sizeof(int) * 4, s));
    RCK(cudaMemsetAsync(g->visit, 0, sizeof(unsigned long long) * std::max<uint64_t>(visit_words(V), 1), s));
    RCK(cudaMemsetAsync(g->thdr, 0, sizeof(ThinHdr) * std::max<uint64_t>(nV, 1), s));
    RCK(cudaMemsetAsync(g->hdr, 0, sizeof(VHdr) * std::max<uint64_t>(nV, 1), s));
    if (V) {
        k_rb_sizes<<<blocks, 256, 0, s>>>(V, desc->row_offsets, desc->bias, b, sz, sz + (nV + 1), g->dev_flag);
        bingo_count_launch();
        RCK(cudaGetLastError());
        for (int p = 0; p < 2; p++) RCK(exclusive_scan_u64(sz + p * (nV + 1), off + p * (nV + 1), nV, tmp, s));
        RCK(cudaMemcpyAsync(&hflag, g->dev_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        for (int p = 0; p < 2; p++)
            RCK(cudaMemcpyAsync(&tot[p], off + p * (nV + 1) + nV, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        RCK(cudaStreamSynchronize(s));
        uint64_t last_ro = 0;
        RCK(cudaMemcpy(&last_ro, desc->row_offsets + V, sizeof(uint64_t), cudaMemcpyDeviceToHost));
        if (last_ro != desc->num_arcs) hflag |= 1;
        if (hflag & 1) return done(BINGO_E_INVAL);
        if (hflag & 4) return done(BINGO_E_OVERFLOW);
    }
    if (tot[0] >= 0x7FFFFFF0ull || tot[1] >= 0xFFFFFFF0ull) return done(BINGO_E_OVERFLOW);
    g->bkt_cap = rb_pool(tot[0], 0.0);
    g->mem_cap = 4 * rb_pool(tot[1], 0.0);
    g->bkt = (Bucket *)bingo_dev_alloc(g, sizeof(Bucket) * g->bkt_cap);
    g->gcan = (GCan *)bingo_dev_alloc(g, sizeof(GCan) * g->bkt_cap);
    g->mdst = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * g->mem_cap);
    // the adjacency (dst, bias) and arc epochs, for updates (R-19); slack for relocations
    const uint64_t A = desc->num_arcs;
    g->arc_cap = rb_pool(A, g->arc_slack);
    g->arc = (uint2 *)bingo_dev_alloc(g, sizeof(uint2) * g->arc_cap);
    g->arc_epoch = (uint32_t *)bingo_dev_alloc(g, sizeof(uint32_t) * g->arc_cap);
    g->rb_meta = (uint64_t *)bingo_dev_alloc(g, sizeof(uint64_t) * 2 * std::max<uint64_t>(nV, 1));
    if (!g->bkt || !g->gcan || !g->mdst || !g->arc || !g->arc_epoch || !g->rb_meta) return done(BINGO_E_NOMEM);
    RCK(cudaMemsetAsync(g->arc_epoch, 0, sizeof(uint32_t) * std::max<uint64_t>(A, 1), s));
    if (A) {
        k_rb_arcs<<<(unsigned)std::min<uint64_t>((A + 255) / 256, 148ull * 32), 256, 0, s>>>(A, desc->dst, desc->bias,
                                                                                             g->arc);
        bingo_count_launch();
        RCK(cudaGetLastError());
    }
    if (V) {
        k_rb_fill<<<blocks, 256, 0, s>>>(V, desc->row_offsets, desc->dst, desc->bias, b, off, off + (nV + 1), g->hdr,
                                         g->thdr, g->bkt, g->gcan, g->mdst, g->rb_meta);
        bingo_count_launch();
        RCK(cudaGetLastError());
        RCK(cudaStreamSynchronize(s));
    }
#undef RCK
    unsigned long long hc[3] = {A, tot[0], tot[1]};
    if (cudaMemcpy(g->counters, hc, sizeof(hc), cudaMemcpyHostToDevice) != cudaSuccess) {
        g->poisoned = 1;
        return done(BINGO_E_CUDA);
    }
    return done(st);
}

bingo_status launch_walk_radix(bingo_graph *g, const bingo_walk_desc *desc, const uint32_t *starts, uint32_t W,
                               uint32_t *paths, uint32_t *lengths, cudaStream_t s) {
    if (!(desc->app == BINGO_DEEPWALK || desc->app == BINGO_PPR) || (desc->flags & BINGO_WALK_WALKER_MAJOR))
        return BINGO_E_INVAL;
    WalkArgs a;
    memset(&a, 0, sizeof(a));
    a.thdr = g->thdr;
    a.bkt = g->bkt;
    a.mdst = g->mdst;
    a.visit = g->visit;
    a.starts = starts;
    a.paths = paths;
    a.lengths = lengths;
    a.W = W;
    a.V = g->V;
    a.L = desc->length;
    a.first_walker = desc->first_walker_id;
    a.k0 = (uint32_t)desc->seed;
    a.k1 = (uint32_t)(desc->seed >> 32);
    if (desc->stop_num >= desc->stop_den) {
        a.stop_always = 1;
        a.stop_thr = 0;
    } else {
        a.stop_always = 0;
        a.stop_thr = (unsigned long long)(((unsigned __int128)desc->stop_num << 64) / desc->stop_den);
    }
    unsigned long long *claim = g->walk_ctr + (__atomic_fetch_add(&g->walk_slot, 1u, __ATOMIC_RELAXED) % BINGO_WALK_SLOTS);
    if (cudaMemsetAsync(claim, 0, sizeof(unsigned long long), s) != cudaSuccess) {
        g->poisoned = 1;
        return BINGO_E_CUDA;
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (desc->app == BINGO_PPR) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_walk_rb<BINGO_PPR>, 256, 0);
        const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((W + 255) / 256, (uint64_t)sms * std::max(per_sm, 1)));
        k_walk_rb<BINGO_PPR><<<grid, 256, 0, s>>>(a, claim);
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_walk_rb<BINGO_DEEPWALK>, 256, 0);
        const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((W + 255) / 256, (uint64_t)sms * std::max(per_sm, 1)));
        k_walk_rb<BINGO_DEEPWALK><<<grid, 256, 0, s>>>(a, claim);
    }
    bingo_count_launch();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "libbingo: radix walk launch failed: %s\n", cudaGetErrorString(e));
        g->poisoned = 1;
        return BINGO_E_CUDA;
    }
    return BINGO_OK;
}

// canonical radix dump (R-18) from the device arrays; returns the byte count
bingo_status export_radix(bingo_graph *g, uint8_t *buf, size_t cap, size_t *size_out, cudaStream_t s) {
    const uint64_t V = g->V;
    std::vector<VHdr> hdr(V);
    std::vector<ThinHdr> th(V);
    uint64_t nb = 0, nm = 0;
    unsigned long long hc[3];
    if (cudaMemcpyAsync(hc, g->counters, sizeof(hc), cudaMemcpyDeviceToHost, s) != cudaSuccess) return BINGO_E_CUDA;
    if (V && (cudaMemcpyAsync(hdr.data(), g->hdr, sizeof(VHdr) * V, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
              cudaMemcpyAsync(th.data(), g->thdr, sizeof(ThinHdr) * V, cudaMemcpyDeviceToHost, s) != cudaSuccess))
        return BINGO_E_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return BINGO_E_CUDA;
    nb = hc[1];
    nm = hc[2];
    std::vector<Bucket> bk(nb);
    std::vector<GCan> gc(nb);
    std::vector<uint32_t> md(4 * nm);
    if (nb && (cudaMemcpyAsync(bk.data(), g->bkt, sizeof(Bucket) * nb, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
               cudaMemcpyAsync(gc.data(), g->gcan, sizeof(GCan) * nb, cudaMemcpyDeviceToHost, s) != cudaSuccess))
        return BINGO_E_CUDA;
    if (nm && cudaMemcpyAsync(md.data(), g->mdst, sizeof(uint32_t) * 4 * nm, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return BINGO_E_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return BINGO_E_CUDA;
    size_t pos = 0;
    auto put = [&](const void *p, size_t k) {
        if (buf && pos + k <= cap) memcpy(buf + pos, p, k);
        pos += k;
    };
    auto p32 = [&](uint32_t v) { put(&v, 4); };
    auto p64 = [&](uint64_t v) { put(&v, 8); };
    for (uint64_t u = 0; u < V; u++) {
        p32(hdr[u].d);
        const uint32_t n = th[u].n;
        p32(n);
        for (uint32_t q = 0; q < n; q++) {
            const uint64_t gb = th[u].bkt_off + q;
            const Bucket &G = bk[gb];
            p32(kk_k(G.kk));
            p64(gc[gb].thr);
            p32(G.alias);
            const uint32_t ns = G.px;
            p32(ns);
            for (uint32_t k = 0; k < ns; k++) {
                const uint64_t sb = (uint64_t)G.py + k;
                const Bucket &S = bk[sb];
                p32(kk_k(S.kk));
                p32(S.px);
                p64(gc[sb].thr);
                p32(S.alias);
                for (uint32_t e = 0; e < S.px; e++) p32(md[(uint64_t)S.py * 4 + e]);
            }
        }
        p64(hdr[u].T);
    }
    *size_out = pos;
    return BINGO_OK;
}

// ---------------------------------------------------------------- updates (reading R-19)
// The paper leaves the nested dynamic structure unbuilt.  A batch: whole-batch
// validation -> stable sort by source (batch order inside a vertex) -> per touched
// vertex (one warp): the adjacency copied to fresh space in the arc pool with the inserts
// appended (R-7), the deletes' picks (R-8) marked in a bitmap, the two-phase delete-and-swap
// (R-6) -> the nested structure rebuilt from the new adjacency into fresh bucket / member
// space (rb_fill_vertex, as the build) -> headers.  The headers change only in the last
// kernel, after every pool is known to be large enough, so EINVAL / EOVERFLOW / NOMEM leave
// the graph as it was.
namespace bingo {

struct RbuArgs {
    const uint4 *recs;                 // the batch, device copy
    const uint32_t *sval;              // record indices sorted by source (stable)
    const uint32_t *seg;               // [nt + 1] segment starts in sval order
    const uint32_t *tv;                // [nt] touched vertices
    uint32_t nt, b, epoch;             // epoch of this batch (R-9)
    VHdr *hdr;
    ThinHdr *thdr;
    uint2 *arc;
    uint32_t *arc_epoch;
    Bucket *bkt;
    GCan *gcan;
    uint32_t *mdst;
    uint64_t *meta;                    // g->rb_meta: [V] first member unit, [V] (bucket cap << 32 | unit cap)
    uint32_t V;
    uint2 *wa;                         // working adjacency (scratch): the new arcs of every touched vertex
    uint32_t *we;                      // ... and their epochs
    uint64_t *need_arc, *need_scr;     // plan: L = d + inserts, scratch words
    const uint64_t *arc_pref, *scr_pref;
    uint64_t arc_base, bkt_base, mem_base;   // pool bump pointers at this batch
    uint32_t *scr;
    uint32_t *newL;                    // post-batch degree
    // sizes: fresh pool space a vertex needs (0: its new adjacency / structure fits where it is;
    // else the size with 25% slack, which becomes its capacity)
    uint64_t *nfa, *nbk, *nun;
    const uint64_t *fa_pref, *bk_pref, *un_pref;
    unsigned long long *st;            // [3] inserted, deleted, missing
    int *flag;                         // 1 invalid, 4 overflow
    uint32_t *big;                     // touched indices t with newL > RBU_BIG (a block each)
    unsigned long long *nbig;
};

__global__ void k_rbu_validate(const uint4 *__restrict__ recs, uint64_t n, uint32_t V, int *flag,
                               uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 r = recs[i];
        if (r.x > 1u || r.y >= V || r.z >= V || (r.x == 0u && r.w == 0u)) atomicOr(flag, 1);
        keys[i] = r.y < V ? r.y : 0u;
        vals[i] = (uint32_t)i;
    }
}

__global__ void k_rbu_heads(const uint32_t *__restrict__ skeys, uint64_t n, uint64_t *__restrict__ head) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || skeys[i] != skeys[i - 1]) ? 1ull : 0ull;
}

__global__ void k_rbu_seg(const uint32_t *__restrict__ skeys, const uint64_t *__restrict__ head,
                          const uint64_t *__restrict__ hpref, uint64_t n, uint32_t *__restrict__ seg,
                          uint32_t *__restrict__ tv, unsigned long long *ntouch) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (head[i]) {
            seg[hpref[i]] = (uint32_t)i;
            tv[hpref[i]] = skeys[i];
        }
        if (i == n - 1) {
            const uint64_t nt = hpref[i] + head[i];
            seg[nt] = (uint32_t)n;
            *ntouch = nt;
        }
    }
}

// a vertex with more deletes than this finds its R-8 picks among candidates (one pass over
// the adjacency with a hash of the deleted dsts) instead of one adjacency scan per delete
static constexpr uint32_t RBU_SCAN_Q = 4;
// vertices with more arcs after the batch are sized and rebuilt by a whole block
static constexpr uint32_t RBU_BIG = 4096;
__host__ __device__ __forceinline__ uint64_t rbu_hash_size(uint32_t q) {
    uint64_t h = 16;
    while (h < 2ull * q) h <<= 1;
    return h;
}

#define RBU_WARP_LOOP(t, n) \
    for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < (n); t += (gridDim.x * blockDim.x) >> 5)

// per touched vertex: arc demand L = d + inserts, scratch (bitmap + holes + survivors), overflow
__global__ void __launch_bounds__(256) k_rbu_plan(const RbuArgs a) {
    const uint32_t lane = lane_id(), K = (32 + a.b - 1) / a.b;
    RBU_WARP_LOOP(t, a.nt) {
        const uint32_t beg = a.seg[t], end = a.seg[t + 1];
        uint32_t m = 0, q = 0;
        uint64_t ins = 0;
        for (uint32_t p = beg + lane; p < end; p += 32) {
            const uint4 r = a.recs[a.sval[p]];
            if (r.x == 0u) { m++; ins += r.w; }
            else q++;
        }
        m = warp_sum(m);
        q = warp_sum(q);
        ins = warp_sum(ins);
        if (lane == 0) {
            const VHdr h = a.hdr[a.tv[t]];
            const uint64_t L = (uint64_t)h.d + m;
            if (L >= 0xFFFFFFFFull || (unsigned __int128)(h.T + ins) * K >= ((unsigned __int128)1 << 64))
                atomicOr(a.flag, 4);
            a.need_arc[t] = L;
            // bitmap, holes + survivors, and (q > RBU_SCAN_Q) a hash of the deleted dsts plus
            // the candidate positions (arcs whose dst is deleted)
            a.need_scr[t] = (L + 31) / 32 + 2ull * q + (q > RBU_SCAN_Q ? rbu_hash_size(q) + L : 0ull);
        }
    }
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o);
        v = y < v ? y : v;
    }
    return v;
}

// enumerate, ascending, the positions p in [lo, hi) whose bitmap bit equals `want`, into out[]
__device__ __forceinline__ uint32_t rbu_enumerate(const uint32_t *bm, uint32_t lo, uint32_t hi, bool want,
                                                  uint32_t *out) {
    const uint32_t lane = lane_id();
    uint32_t total = 0;
    if (lo >= hi) return 0;
    for (uint32_t w0 = lo / 32; w0 * 32 < hi; w0 += 32) {
        const uint32_t w = w0 + lane;
        uint32_t bits = 0;
        if (w * 32 < hi) {
            bits = want ? bm[w] : ~bm[w];
            const uint32_t s = w * 32;
            if (s < lo) bits &= ~0u << (lo - s);
            if (hi - s < 32) bits &= (1u << (hi - s)) - 1u;
        }
        const uint32_t c = __popc(bits);
        uint32_t incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        uint32_t k = total + incl - c;
        while (bits) {
            const uint32_t bit = __ffs(bits) - 1;
            bits &= bits - 1;
            out[k++] = w * 32 + bit;
        }
        total += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    return total;
}

// per touched vertex: the new adjacency in fresh arc space (R-7, R-8, R-6)
__global__ void __launch_bounds__(256) k_rbu_mutate(const RbuArgs a) {
    const uint32_t lane = lane_id();
    RBU_WARP_LOOP(t, a.nt) {
        const uint32_t u = a.tv[t], beg = a.seg[t], end = a.seg[t + 1];
        const VHdr h = a.hdr[u];
        const uint32_t d = h.d;
        const uint64_t off = a.arc_pref[t], old = h.adj_off;   // working copy in scratch
        const uint32_t L = (uint32_t)a.need_arc[t];
        uint2 *const wa = a.wa;
        uint32_t *const we = a.we;
        for (uint32_t p = lane; p < d; p += 32) {
            wa[off + p] = a.arc[old + p];
            we[off + p] = a.arc_epoch[old + p];
        }
        // (1) inserts appended in batch order (R-7)
        uint32_t m = 0;
        for (uint32_t p0 = beg; p0 < end; p0 += 32) {
            const uint32_t p = p0 + lane;
            uint4 r = make_uint4(1u, 0u, 0u, 0u);
            if (p < end) r = a.recs[a.sval[p]];
            const bool ins = p < end && r.x == 0u;
            const uint32_t bal = __ballot_sync(0xffffffffu, ins);
            if (ins) {
                const uint32_t pos = d + m + __popc(bal & lanemask_lt());
                wa[off + pos] = make_uint2(r.z, r.w);
                we[off + pos] = a.epoch;
            }
            m += __popc(bal);
        }
        uint32_t *bm = a.scr + a.scr_pref[t];
        const uint32_t words = (L + 31) / 32;
        for (uint32_t w = lane; w < words; w += 32) bm[w] = 0;
        __syncwarp();
        // (2) deletes in batch order: the live instance with the smallest (epoch, position) (R-8).
        // Few deletes: scan the adjacency per delete.  Many: one pass collects the candidate
        // positions (arcs whose dst some delete names, via a hash of the deleted dsts) and each
        // delete scans only those -- the same picks, O(L + q x candidates) instead of O(q L).
        const uint32_t q = (uint32_t)(end - beg) - m;
        const uint32_t *cand = nullptr;
        uint32_t nc = L;
        if (q > RBU_SCAN_Q) {
            const uint32_t H = (uint32_t)rbu_hash_size(q);
            uint32_t *ht = bm + words + 2 * q, *cw = ht + H;
            for (uint32_t j = lane; j < H; j += 32) ht[j] = 0xFFFFFFFFu;
            __syncwarp();
            for (uint32_t p0 = beg; p0 < end; p0 += 32) {
                const uint32_t p = p0 + lane;
                if (p < end) {
                    const uint4 r = a.recs[a.sval[p]];
                    if (r.x == 1u) {
                        uint32_t sl = (r.z * 0x9E3779B1u) & (H - 1);
                        for (;;) {
                            const uint32_t o = atomicCAS(&ht[sl], 0xFFFFFFFFu, r.z);
                            if (o == 0xFFFFFFFFu || o == r.z) break;
                            sl = (sl + 1) & (H - 1);
                        }
                    }
                }
            }
            __syncwarp();
            nc = 0;
            for (uint32_t x0 = 0; x0 < L; x0 += 32) {
                const uint32_t x = x0 + lane;
                bool hit = false;
                if (x < L) {
                    const uint32_t v = wa[off + x].x;
                    for (uint32_t sl = (v * 0x9E3779B1u) & (H - 1);; sl = (sl + 1) & (H - 1)) {
                        const uint32_t k = ht[sl];
                        if (k == v) { hit = true; break; }
                        if (k == 0xFFFFFFFFu) break;
                    }
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, hit);
                if (hit) cw[nc + __popc(bal & lanemask_lt())] = x;
                nc += __popc(bal);
            }
            __syncwarp();
            cand = cw;
        }
        uint32_t N = 0, miss = 0;
        for (uint32_t p = beg; p < end; p++) {
            const uint4 r = a.recs[a.sval[p]];
            if (r.x != 1u) continue;
            unsigned long long best = ~0ull;
            for (uint32_t c = lane; c < nc; c += 32) {
                const uint32_t x = cand ? cand[c] : c;
                if (wa[off + x].x != r.z || ((bm[x >> 5] >> (x & 31)) & 1u)) continue;
                const unsigned long long key = ((unsigned long long)we[off + x] << 32) | x;
                best = key < best ? key : best;
            }
            best = warp_min_u64(best);
            if (best == ~0ull) {
                miss++;
            } else {
                const uint32_t x = (uint32_t)best;
                if (lane == 0) bm[x >> 5] |= 1u << (x & 31);
                N++;
            }
            __syncwarp();
        }
        // (3) two-phase delete-and-swap (R-6): survivor j of the tail window fills hole j
        const uint32_t Lp = L - N;
        if (N) {
            uint32_t *hl = bm + words, *sv = hl + N;
            const uint32_t nh = rbu_enumerate(bm, 0, Lp, true, hl);
            rbu_enumerate(bm, Lp, L, false, sv);
            for (uint32_t j = lane; j < nh; j += 32) {
                wa[off + hl[j]] = wa[off + sv[j]];
                we[off + hl[j]] = we[off + sv[j]];
            }
        }
        if (lane == 0) {
            a.newL[t] = Lp;
            if (Lp > RBU_BIG) a.big[atomicAdd(a.nbig, 1ull)] = t;
            if (m) atomicAdd(&a.st[0], (unsigned long long)m);
            if (N) atomicAdd(&a.st[1], (unsigned long long)N);
            if (miss) atomicAdd(&a.st[2], (unsigned long long)miss);
        }
    }
}

// fresh pool space for vertex t: none where the new adjacency / structure fits the vertex's
// current space (rebuilt in place), else the size plus 25% slack
__device__ __forceinline__ void rbu_demand(const RbuArgs &a, uint32_t t, uint64_t nb, uint64_t units) {
    const uint32_t u = a.tv[t], L = a.newL[t];
    const VHdr h = a.hdr[u];
    const uint64_t caps = a.meta[a.V + u];
    a.nfa[t] = L <= h.adj_cap ? 0ull : (uint64_t)L + L / 4;
    a.nbk[t] = nb <= (caps >> 32) ? 0ull : nb + nb / 4;
    a.nun[t] = units <= (caps & 0xFFFFFFFFull) ? 0ull : units + units / 4;
}

__global__ void __launch_bounds__(256) k_rbu_sizes(const RbuArgs a) {
    __shared__ uint32_t cs[RB_WARPS][RB_CELLS];
    const uint32_t wib = threadIdx.x >> 5, lane = lane_id();
    RBU_WARP_LOOP(t, a.nt) {
        if (a.newL[t] > RBU_BIG) continue;   // k_rbu_sizes_big
        const uint64_t off = a.arc_pref[t];
        const RbArcs arcs{&a.wa[off].x, &a.wa[off].y, 2u};
        uint64_t nb, units, T;
        rb_sizes_vertex(arcs, a.newL[t], a.b, cs[wib], nb, units, T, a.flag);
        if (lane == 0) rbu_demand(a, t, nb, units);
    }
}

// where vertex t's new adjacency and structure go (in place, or the fresh space of its demand);
// copies the working adjacency there (threads `id` of `nthr`) and records the structure space
struct RbuPlace {
    uint64_t aoff, bo, mu;
    uint32_t acap;
};
__device__ __forceinline__ RbuPlace rbu_place(const RbuArgs &a, uint32_t t, uint32_t id, uint32_t nthr) {
    const uint32_t u = a.tv[t], L = a.newL[t];
    const VHdr h = a.hdr[u];
    const uint64_t caps = a.meta[a.V + u];
    RbuPlace p;
    const bool fa = a.nfa[t] != 0, fb = a.nbk[t] != 0, fu = a.nun[t] != 0;
    p.aoff = fa ? a.arc_base + a.fa_pref[t] : h.adj_off;
    p.acap = fa ? (uint32_t)a.nfa[t] : h.adj_cap;
    p.bo = fb ? a.bkt_base + a.bk_pref[t] : h.bkt_off;
    p.mu = fu ? a.mem_base + a.un_pref[t] : a.meta[u];
    const uint64_t w = a.arc_pref[t];
    for (uint32_t x = id; x < L; x += nthr) {
        a.arc[p.aoff + x] = a.wa[w + x];
        a.arc_epoch[p.aoff + x] = a.we[w + x];
    }
    if (id == 0) {
        a.meta[u] = p.mu;
        a.meta[a.V + u] = ((fb ? a.nbk[t] : caps >> 32) << 32) | (fu ? a.nun[t] : caps & 0xFFFFFFFFull);
    }
    return p;
}

__global__ void __launch_bounds__(256) k_rbu_fill(const RbuArgs a) {
    __shared__ uint32_t cs[RB_WARPS][RB_CELLS];
    __shared__ uint32_t cur[RB_WARPS][RB_CELLS];
    const uint32_t wib = threadIdx.x >> 5;
    RBU_WARP_LOOP(t, a.nt) {
        if (a.newL[t] > RBU_BIG) continue;   // k_rbu_fill_big
        const RbuPlace pl = rbu_place(a, t, lane_id(), 32);
        const uint64_t off = a.arc_pref[t];
        const RbArcs arcs{&a.wa[off].x, &a.wa[off].y, 2u};
        rb_fill_vertex(a.tv[t], arcs, a.newL[t], a.b, pl.bo, pl.mu, pl.aoff, pl.acap, cs[wib], cur[wib], a.hdr,
                       a.thdr, a.bkt, a.gcan, a.mdst);
    }
}

// Large vertices, one 256-thread block each: per-warp digit counts over 8 contiguous chunks
// of the adjacency (their sum is the histogram), the tables by warp 0, then every warp appends
// its chunk's members at cursors offset by the earlier chunks' counts -- the same ascending
// member order as one warp over the whole adjacency.
__device__ __forceinline__ void rbu_block_counts(const RbArcs &arcs, uint32_t L, uint32_t b,
                                                 uint32_t (*cnt)[RB_CELLS], uint32_t *c, unsigned long long *sT) {
    const uint32_t B = 1u << b, K = (32 + b - 1) / b, wib = threadIdx.x >> 5, lane = lane_id();
    for (uint32_t x = threadIdx.x; x < RB_WARPS * RB_CELLS; x += blockDim.x) cnt[x / RB_CELLS][x % RB_CELLS] = 0;
    if (threadIdx.x == 0) *sT = 0;
    __syncthreads();
    const uint32_t chunk = (L + RB_WARPS - 1) / RB_WARPS, lo = min(L, wib * chunk), hi = min(L, lo + chunk);
    uint64_t T = 0;
    for (uint32_t a = lo + lane; a < hi; a += 32) {
        const uint32_t w = arcs.w(a);
        T += w;
        for (uint32_t i = 0; i < K; i++) {
            const uint32_t j = rb_digit(w, i, b);
            if (j) atomicAdd(&cnt[wib][i * B + j], 1u);
        }
    }
    T = warp_sum(T);
    if (lane == 0) atomicAdd(sT, (unsigned long long)T);
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < RB_CELLS; x += blockDim.x) {
        uint32_t sum = 0;
        for (uint32_t w = 0; w < RB_WARPS; w++) sum += cnt[w][x];
        c[x] = sum;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_rbu_sizes_big(const RbuArgs a) {
    __shared__ uint32_t cnt[RB_WARPS][RB_CELLS];
    __shared__ uint32_t c[RB_CELLS];
    __shared__ unsigned long long sT;
    const uint32_t B = 1u << a.b, K = (32 + a.b - 1) / a.b, lane = lane_id();
    for (uint32_t bi = blockIdx.x; bi < *a.nbig; bi += gridDim.x) {
        const uint32_t t = a.big[bi];
        const uint64_t off = a.arc_pref[t];
        const RbArcs arcs{&a.wa[off].x, &a.wa[off].y, 2u};
        rbu_block_counts(arcs, a.newL[t], a.b, cnt, c, &sT);
        if (threadIdx.x < 32) {
            uint32_t ng = 0, nsub = 0;
            uint64_t units = 0;
            for (uint32_t i = lane; i < K; i += 32) {
                uint32_t ns = 0;
                for (uint32_t j = 1; j < B; j++) {
                    const uint32_t cc = c[i * B + j];
                    ns += cc ? 1u : 0u;
                    units += (cc + 3) / 4;
                }
                nsub += ns;
                ng += ns ? 1u : 0u;
            }
            ng = warp_sum(ng);
            nsub = warp_sum(nsub);
            units = warp_sum(units);
            if (lane == 0) {
                if ((unsigned __int128)sT * ng >= ((unsigned __int128)1 << 64)) atomicOr(a.flag, 4);
                rbu_demand(a, t, ng + nsub, units);
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_rbu_fill_big(const RbuArgs a) {
    __shared__ uint32_t cnt[RB_WARPS][RB_CELLS];
    __shared__ uint32_t c[RB_CELLS], cu[RB_CELLS];
    __shared__ unsigned long long sT;
    __shared__ uint32_t sn;
    const uint32_t wib = threadIdx.x >> 5;
    for (uint32_t bi = blockIdx.x; bi < *a.nbig; bi += gridDim.x) {
        const uint32_t t = a.big[bi], L = a.newL[t];
        const RbuPlace pl = rbu_place(a, t, threadIdx.x, blockDim.x);
        const uint64_t off = a.arc_pref[t];
        const RbArcs arcs{&a.wa[off].x, &a.wa[off].y, 2u};
        rbu_block_counts(arcs, L, a.b, cnt, c, &sT);
        const uint64_t bo = pl.bo, munits = pl.mu;
        if (wib == 0) {
            const uint32_t n = rb_tables(c, cu, sT, a.b, bo, munits, a.bkt, a.gcan);
            if (lane_id() == 0) sn = n;
        }
        __syncthreads();
        for (uint32_t x = threadIdx.x; x < RB_CELLS; x += blockDim.x) {   // chunk w's cursor per cell
            uint32_t run = cu[x];
            for (uint32_t w = 0; w < RB_WARPS; w++) {
                const uint32_t k = cnt[w][x];
                cnt[w][x] = run;
                run += k;
            }
        }
        __syncthreads();
        const uint32_t chunk = (L + RB_WARPS - 1) / RB_WARPS, lo = min(L, wib * chunk), hi = min(L, lo + chunk);
        rb_members(arcs, lo, hi, a.b, cnt[wib], munits * 4, a.mdst);
        __syncthreads();
        if (threadIdx.x == 0)
            rb_headers(a.tv[t], sT, L, bo, sn, pl.aoff, pl.acap, a.hdr, a.thdr);
        __syncthreads();
    }
}

}  // namespace bingo

// grow a device array (realloc + copy): the pools are offset-addressed, so nothing else changes
template <typename T>
static bool rb_grow(bingo_graph *g, T *&p, uint64_t old_n, uint64_t new_n, cudaStream_t s) {
    T *q = (T *)bingo_dev_alloc(g, sizeof(T) * new_n);
    if (!q) return false;
    if (old_n && (cudaMemcpyAsync(q, p, sizeof(T) * old_n, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
                  cudaStreamSynchronize(s) != cudaSuccess)) {
        bingo_dev_free(g, q);
        return false;
    }
    bingo_dev_free(g, p);
    p = q;
    return true;
}

// bingo_apply_updates on a radix graph (called by apply_impl after the common checks)
bingo_status apply_radix(bingo_graph *g, const bingo_update *batch, uint64_t n, uint32_t flags,
                         bingo_update_stats *stats, cudaStream_t s) {
    const uint32_t V = g->V;
    std::vector<void *> tmp;
    auto take = [&](size_t bytes) {
        void *p = bingo_dev_alloc(g, std::max<size_t>(bytes, 16));
        if (p) tmp.push_back(p);
        return p;
    };
    auto fin = [&](bingo_status r) {
        for (void *p : tmp) bingo_dev_free(g, p);
        return r;
    };
    auto fail = [&](const char *w) {
        fprintf(stderr, "libbingo: CUDA error in %s: %s\n", w, cudaGetErrorString(cudaGetLastError()));
        g->poisoned = 1;
        return fin(BINGO_E_CUDA);
    };
#define RBU(call, w)                              \
    do {                                          \
        if ((call) != cudaSuccess) return fail(w); \
    } while (0)
    uint4 *recs = (uint4 *)take(16 * n);
    uint32_t *k0 = (uint32_t *)take(4 * n), *v0 = (uint32_t *)take(4 * n), *k1 = (uint32_t *)take(4 * n),
             *v1 = (uint32_t *)take(4 * n);
    uint64_t *rtmp = (uint64_t *)take(8 * radix_tmp_words(n));
    uint64_t *head = (uint64_t *)take(8 * (n + 1)), *hpref = (uint64_t *)take(8 * (n + 1));
    uint64_t *stmp = (uint64_t *)take(8 * scan_tmp_words(n + 1));
    uint32_t *seg = (uint32_t *)take(4 * (n + 1)), *tv = (uint32_t *)take(4 * n);
    // small device block: [0..2] stats, [3] ntouch, [4..6] bump pointers copy, [7] big vertices; flag after
    unsigned long long *dsm = (unsigned long long *)take(8 * 8 + 16);
    int *dflag = reinterpret_cast<int *>(dsm + 8);
    if (!recs || !k0 || !v0 || !k1 || !v1 || !rtmp || !head || !hpref || !stmp || !seg || !tv || !dsm)
        return fin(BINGO_E_NOMEM);
    RBU(cudaMemcpyAsync(recs, batch, 16 * n, (flags & BINGO_UPD_HOST_BATCH) ? cudaMemcpyHostToDevice
                                                                           : cudaMemcpyDeviceToDevice, s), "radix batch copy");
    RBU(cudaMemsetAsync(dsm, 0, 8 * 8 + 16, s), "radix memset");
    const unsigned G1 = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    k_rbu_validate<<<G1, 256, 0, s>>>(recs, n, V, dflag, k0, v0);
    bingo_count_launch();
    int kb = 1;
    while (kb < 32 && ((uint64_t)(V ? V - 1 : 0) >> kb)) kb++;
    bool in1 = false;
    RBU(radix_sort_pairs(k0, v0, k1, v1, n, kb, rtmp, s, &in1), "radix sort");
    const uint32_t *skeys = in1 ? k1 : k0, *sval = in1 ? v1 : v0;
    k_rbu_heads<<<G1, 256, 0, s>>>(skeys, n, head);
    bingo_count_launch();
    RBU(exclusive_scan_u64(head, hpref, n, stmp, s), "radix scan");
    k_rbu_seg<<<G1, 256, 0, s>>>(skeys, head, hpref, n, seg, tv, dsm + 3);
    bingo_count_launch();
    RBU(cudaMemcpyAsync(dsm + 4, g->counters, 3 * 8, cudaMemcpyDeviceToDevice, s), "radix bumps");
    unsigned long long h1[8];
    int hflag = 0;
    RBU(cudaMemcpyAsync(h1, dsm, sizeof(h1), cudaMemcpyDeviceToHost, s), "radix sync 1");
    RBU(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, s), "radix sync 1");
    RBU(cudaStreamSynchronize(s), "radix sync 1");
    if (hflag & 1) return fin(BINGO_E_INVAL);
    const uint32_t nt = (uint32_t)h1[3];
    RbuArgs a;
    memset(&a, 0, sizeof(a));
    a.recs = recs;
    a.sval = sval;
    a.seg = seg;
    a.tv = tv;
    a.nt = nt;
    a.b = g->radix_log2;
    a.epoch = g->epoch + 1;
    a.st = dsm;
    a.flag = dflag;
    uint64_t *need = (uint64_t *)take(8 * 2 * (nt + 1)), *pref = (uint64_t *)take(8 * 2 * (nt + 1));
    uint64_t *stmp2 = (uint64_t *)take(8 * 2 * scan_tmp_words(nt + 1));   // two scans at once
    a.newL = (uint32_t *)take(4 * (nt + 1));
    if (!need || !pref || !stmp2 || !a.newL) return fin(BINGO_E_NOMEM);
    a.need_arc = need;
    a.need_scr = need + (nt + 1);
    a.arc_pref = pref;
    a.scr_pref = pref + (nt + 1);
    a.hdr = g->hdr;
    const unsigned GW = (unsigned)std::min<uint64_t>((nt + 7) / 8, 148ull * 16);
    k_rbu_plan<<<GW, 256, 0, s>>>(a);
    bingo_count_launch();
    {
        const uint64_t *in[2] = {a.need_arc, a.need_scr};
        uint64_t *out[2] = {pref, pref + (nt + 1)};
        RBU(exclusive_scan_u64_multi(in, out, 2, nt, stmp2, s), "radix plan scan");
    }
    uint64_t tot[2] = {0, 0};
    RBU(cudaMemcpyAsync(&tot[0], pref + nt, 8, cudaMemcpyDeviceToHost, s), "radix sync 2");
    RBU(cudaMemcpyAsync(&tot[1], pref + (nt + 1) + nt, 8, cudaMemcpyDeviceToHost, s), "radix sync 2");
    RBU(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, s), "radix sync 2");
    RBU(cudaStreamSynchronize(s), "radix sync 2");
    if (hflag & 4) return fin(BINGO_E_OVERFLOW);
    const uint64_t bump0 = h1[4], bump1 = h1[5], bump2 = h1[6];
    // the working adjacency (scratch): every touched vertex's new arcs, then sizes and the
    // fresh pool space of the vertices that no longer fit where they are
    a.wa = (uint2 *)take(8 * (tot[0] + 1));
    a.we = (uint32_t *)take(4 * (tot[0] + 1));
    a.scr = (uint32_t *)take(4 * (tot[1] + 1));
    a.big = (uint32_t *)take(4 * (nt + 1));
    a.nbig = dsm + 7;
    a.nfa = (uint64_t *)take(8 * 3 * (nt + 1));
    uint64_t *bpref = (uint64_t *)take(8 * 3 * (nt + 1));
    uint64_t *stmp3 = (uint64_t *)take(8 * 3 * scan_tmp_words(nt + 1));
    if (!a.wa || !a.we || !a.scr || !a.big || !a.nfa || !bpref || !stmp3) return fin(BINGO_E_NOMEM);
    a.nbk = a.nfa + (nt + 1);
    a.nun = a.nfa + 2 * (nt + 1);
    a.fa_pref = bpref;
    a.bk_pref = bpref + (nt + 1);
    a.un_pref = bpref + 2 * (nt + 1);
    a.arc = g->arc;
    a.arc_epoch = g->arc_epoch;
    a.meta = g->rb_meta;
    a.V = V;
    k_rbu_mutate<<<GW, 256, 0, s>>>(a);
    bingo_count_launch();
    k_rbu_sizes<<<GW, 256, 0, s>>>(a);
    bingo_count_launch();
    k_rbu_sizes_big<<<148 * 2, 256, 0, s>>>(a);
    bingo_count_launch();
    {
        const uint64_t *in[3] = {a.nfa, a.nbk, a.nun};
        uint64_t *out[3] = {bpref, bpref + (nt + 1), bpref + 2 * (nt + 1)};
        RBU(exclusive_scan_u64_multi(in, out, 3, nt, stmp3, s), "radix sizes scan");
    }
    uint64_t tb[3] = {0, 0, 0};
    for (int k = 0; k < 3; k++)
        RBU(cudaMemcpyAsync(&tb[k], bpref + k * (nt + 1) + nt, 8, cudaMemcpyDeviceToHost, s), "radix sync 3");
    RBU(cudaStreamSynchronize(s), "radix sync 3");
    if (bump0 + tb[0] > g->arc_cap) {   // relocated adjacencies
        const uint64_t cap = std::max<uint64_t>(bump0 + tb[0] + (bump0 + tb[0]) / 4, g->arc_cap + g->arc_cap / 4);
        if (!rb_grow(g, g->arc, g->arc_cap, cap, s) || !rb_grow(g, g->arc_epoch, g->arc_cap, cap, s))
            return fin(BINGO_E_NOMEM);
        g->arc_cap = cap;
    }
    if (bump1 + tb[1] > g->bkt_cap) {
        const uint64_t cap = std::max<uint64_t>(bump1 + tb[1] + (bump1 + tb[1]) / 4, g->bkt_cap + g->bkt_cap / 4);
        if (cap >= 0x7FFFFFF0ull) return fin(BINGO_E_NOMEM);
        if (!rb_grow(g, g->bkt, g->bkt_cap, cap, s) || !rb_grow(g, g->gcan, g->bkt_cap, cap, s)) return fin(BINGO_E_NOMEM);
        g->bkt_cap = cap;
    }
    if (4 * (bump2 + tb[2]) > g->mem_cap) {
        const uint64_t units = std::max<uint64_t>(bump2 + tb[2] + (bump2 + tb[2]) / 4, g->mem_cap / 4 + g->mem_cap / 16);
        if (units >= 0xFFFFFFF0ull) return fin(BINGO_E_NOMEM);
        if (!rb_grow(g, g->mdst, g->mem_cap, 4 * units, s)) return fin(BINGO_E_NOMEM);
        g->mem_cap = 4 * units;
    }
    a.arc = g->arc;
    a.arc_epoch = g->arc_epoch;
    a.arc_base = bump0;
    a.bkt = g->bkt;
    a.gcan = g->gcan;
    a.mdst = g->mdst;
    a.thdr = g->thdr;
    a.bkt_base = bump1;
    a.mem_base = bump2;
    k_rbu_fill<<<GW, 256, 0, s>>>(a);
    bingo_count_launch();
    k_rbu_fill_big<<<148 * 2, 256, 0, s>>>(a);
    bingo_count_launch();
    RBU(cudaGetLastError(), "radix update kernels");
    unsigned long long nb[3] = {bump0 + tb[0], bump1 + tb[1], bump2 + tb[2]};
    RBU(cudaMemcpyAsync(g->counters, nb, sizeof(nb), cudaMemcpyHostToDevice, s), "radix bumps");
    RBU(cudaMemcpyAsync(h1, dsm, 3 * 8, cudaMemcpyDeviceToHost, s), "radix stats");
    RBU(cudaStreamSynchronize(s), "radix stats");
#undef RBU
    g->epoch++;
    g->num_arcs = g->num_arcs + h1[0] - h1[1];
    if (stats) {
        stats->inserted = h1[0];
        stats->deleted = h1[1];
        stats->missing_deletes = h1[2];
        stats->touched_vertices = nt;
        stats->epoch = g->epoch;
    }
    return fin(BINGO_OK);
}
