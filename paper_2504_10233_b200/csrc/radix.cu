// radix.cu -- Bingo with an arbitrary radix base B = 2^b (reading R-17).
//
// A bias w = sum_i d_i B^i (digits d_i < B).  Group B^i holds the arcs with d_i != 0 and
// weighs W_i = B^i sum_j j c_ij; its neighbours no longer share one bias, so it is
// split into subgroups by digit value j (c_ij arcs each, ascending adjacency index) and an
// inter-subgroup alias over the weights j c_ij picks one before a member is
// drawn uniformly.  Fewer groups (K = 32 / b instead of 32: the complexity and memory term
// of Table timecmp) against one more dependent stage per step.
//
// HBM layout (vertex-id order; static: the paper leaves nested dynamic structures to future
// work, so bingo_apply_updates returns EINVAL on these graphs):
//   thdr[u]   {first bucket, n groups}
//   hdr[u]    T, d (exports)
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
__device__ __forceinline__ void rb_hist(const uint32_t *bias, uint64_t a0, uint32_t d, uint32_t b, uint32_t *c) {
    const uint32_t lane = lane_id(), B = 1u << b, K = (32 + b - 1) / b;
    for (uint32_t x = lane; x < K * B; x += 32) c[x] = 0;
    __syncwarp();
    for (uint32_t a = lane; a < d; a += 32) {
        const uint32_t w = bias[a0 + a];
        for (uint32_t i = 0; i < K; i++) {
            const uint32_t j = rb_digit(w, i, b);
            if (j) atomicAdd(&c[i * B + j], 1u);
        }
    }
    __syncwarp();
}

__global__ void __launch_bounds__(256) k_rb_sizes(uint32_t V, const uint64_t *__restrict__ ro,
                                                  const uint32_t *__restrict__ bias, uint32_t b,
                                                  uint64_t *__restrict__ nbkt, uint64_t *__restrict__ nmem,
                                                  int *__restrict__ flag) {
    __shared__ uint32_t cs[RB_WARPS][RB_CELLS];
    const uint32_t wib = threadIdx.x >> 5, lane = lane_id(), B = 1u << b, K = (32 + b - 1) / b;
    uint32_t *c = cs[wib];
    for (uint32_t u = blockIdx.x * RB_WARPS + wib; u < V; u += gridDim.x * RB_WARPS) {
        const uint64_t a0 = ro[u];
        const uint64_t dd = ro[u + 1] - a0;
        if (dd >= 0xFFFFFFFFull) {
            if (lane == 0) atomicOr(flag, 4);
            continue;
        }
        const uint32_t d = (uint32_t)dd;
        uint64_t T = 0;
        for (uint32_t a = lane; a < d; a += 32) {
            const uint32_t w = bias[a0 + a];
            if (w == 0) atomicOr(flag, 1);
            T += w;
        }
        T = warp_sum(T);
        rb_hist(bias, a0, d, b, c);
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
            if ((unsigned __int128)T * ng >= ((unsigned __int128)1 << 64)) atomicOr(flag, 4);
            nbkt[u] = ng + nsub;
            nmem[u] = units;
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(256) k_rb_fill(uint32_t V, const uint64_t *__restrict__ ro,
                                                 const uint32_t *__restrict__ dst, const uint32_t *__restrict__ bias,
                                                 uint32_t b, const uint64_t *__restrict__ boff,
                                                 const uint64_t *__restrict__ moff, VHdr *__restrict__ hdr,
                                                 ThinHdr *__restrict__ thdr, Bucket *__restrict__ bkt,
                                                 GCan *__restrict__ gcan, uint32_t *__restrict__ mdst) {
    __shared__ uint32_t cs[RB_WARPS][RB_CELLS];
    __shared__ uint32_t cur[RB_WARPS][RB_CELLS];   // member write cursor of subgroup (i, j), 4-entry units x 4
    const uint32_t wib = threadIdx.x >> 5, lane = lane_id(), B = 1u << b, K = (32 + b - 1) / b;
    uint32_t *c = cs[wib];
    uint32_t *cu = cur[wib];
    for (uint32_t u = blockIdx.x * RB_WARPS + wib; u < V; u += gridDim.x * RB_WARPS) {
        const uint64_t a0 = ro[u];
        const uint32_t d = (uint32_t)(ro[u + 1] - a0);
        uint64_t T = 0;
        for (uint32_t a = lane; a < d; a += 32) T += bias[a0 + a];
        T = warp_sum(T);
        rb_hist(bias, a0, d, b, c);
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
        const uint64_t bo = boff[u];
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
        const uint64_t mbase = moff[u] * 4;
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
        // members: arcs in ascending index, 32 at a time; for each digit position the lanes
        // with the same digit value are ranked by lane (= adjacency order) and appended
        for (uint32_t base = 0; base < d; base += 32) {
            const uint32_t a = base + lane;
            const bool in = a < d;
            const uint32_t w = in ? bias[a0 + a] : 0u;
            const uint32_t v = in ? dst[a0 + a] : 0u;
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
        if (lane == 0) {
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
            hdr[u] = h;
        }
        __syncwarp();
    }
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
    if (!g->bkt || !g->gcan || !g->mdst) return done(BINGO_E_NOMEM);
    if (V) {
        k_rb_fill<<<blocks, 256, 0, s>>>(V, desc->row_offsets, desc->dst, desc->bias, b, off, off + (nV + 1), g->hdr,
                                         g->thdr, g->bkt, g->gcan, g->mdst);
        bingo_count_launch();
        RCK(cudaGetLastError());
        RCK(cudaStreamSynchronize(s));
    }
#undef RCK
    unsigned long long hc[3] = {0, tot[0], tot[1]};
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
