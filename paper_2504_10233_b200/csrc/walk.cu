// walk.cu -- the batched walker step.
//
// One walker per lane at a time, a persistent grid whose lanes claim walker ids
// dynamically (k_walk below), the whole walk kept in registers.  Each step is a chain of
// dependent 32 B sector loads through the read-only path:
//   VHdr[u] -> Bucket[bkt_off + b] -> (member | arc per dense attempt)
// and one coalesced, streaming (evict-first) store of the path column.
// Randomness: Philox4x32-10 keyed by the seed, counter (walker, step,
// (outer << 16) + inner, tag + ((outer >> 16) << 8)) (R-1, draw_oi) -- no RNG state in memory.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "bingo.h"
#include "bingo_internal.cuh"
#include "build_common.cuh"
#include "walk_common.cuh"

using namespace bingo;

namespace bingo {

// PPR visit-count increment: a reduction in L2 with the evict_last hint, so the counter lines
// stay resident between increments.  Without it each counter's line is evicted between its
// (random, repeated) increments and every increment pays a DRAM read-modify-write: c4 PPR
// 156.5 -> 134.7 ms (tools/ab_variants.sh, profiles/r02_visit_hint_ab.txt); evict_first for
// the non-padded counters instead: 172 ms.  BINGO_VISIT_NOHINT: plain atomicAdd (A/B).
__device__ __forceinline__ void visit_add(unsigned long long *p, unsigned long long v, const Policies &pol) {
#ifdef BINGO_VISIT_NOHINT
    atomicAdd(p, v);
#else
    asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol.keep)
                 : "memory");
#endif
}

#ifdef BINGO_VISIT32
__device__ __forceinline__ void visit_add32(unsigned int *p, unsigned int v, const Policies &pol) {
    asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol.keep)
                 : "memory");
}
#endif

template <int APP, bool PROF, bool WMAJOR>
__device__ __forceinline__ void walker_start(const WalkArgs &a, uint64_t i, uint32_t &w, uint32_t &u,
                                             const Policies &pol) {
    w = a.first_walker + (uint32_t)i;
    const uint32_t u0 = a.starts ? a.starts[i] : (uint32_t)(((uint64_t)a.first_walker + i) % a.V);   // external
    u = a.inv ? __ldg(a.inv + u0) : u0;
    if (a.paths) {
        if (WMAJOR) a.paths[i * ((size_t)a.L + 1)] = u0;
        else __stcs(&a.paths[i], u0);
    }
#ifdef BINGO_VISIT32
    if (APP == BINGO_PPR && a.visit32) visit_add32(&a.visit32[visit_slot(u)], 1u, pol);
    else
#endif
    if (APP == BINGO_PPR && a.visit) visit_add(a.visit + visit_slot(u), 1ull, pol);
}

#ifndef BINGO_WALK_MINB
#define BINGO_WALK_MINB 2
#endif
#ifndef BINGO_N2V_MINB
#define BINGO_N2V_MINB 2
#endif
// Each lane owns one walker at a time and every loop iteration advances every
// active lane by one step (node2vec: one proposal).  A lane whose walker ends
// (length reached, dead end, PPR stop) claims the next walker id at once from a
// per-launch counter (one warp-aggregated atomic per iteration in which some lane
// finished), so lanes never wait for the longest walk of their warp (PPR's
// geometric lengths, node2vec rejections, dead ends) and no SM idles while others
// still hold walkers (the static walker-to-thread split left ~20% of SM cycles
// idle at the tail).  DeepWalk lanes finish together, so a warp claims 32
// consecutive ids and the step-major path stores stay coalesced.  Results depend
// only on the walker id (R-1), never on which lane ran it.
// MODE: 0 plain, 1 load counters (bingo_walk_profile), 2 counters + access trace
// (bingo_walk_trace; DeepWalk / PPR, integer biases).
#ifndef WALK_CLAIM_CHUNK
#define WALK_CLAIM_CHUNK 32u
#endif
template <int APP, int MODE, bool WMAJOR, bool FLT>   // FLT: float-bias graph (decimal groups, R-15)
#ifndef BINGO_WALK_TPB
#define BINGO_WALK_TPB 256
#endif
__global__ void __launch_bounds__(BINGO_WALK_TPB, MODE ? 4 : (APP == BINGO_NODE2VEC ? BINGO_N2V_MINB : BINGO_WALK_MINB))
    k_walk(const WalkArgs a, unsigned long long *__restrict__ claim) {
    constexpr bool PROF = MODE >= 1;
    constexpr bool TRACE = MODE == 2;
    WalkProf prof;
    // L2 eviction priorities: the thin headers are re-read by every step of every
    // walker (keep), member/arc sectors are one-shot random reads (stream).
    uint64_t pol_keep, pol_stream;
#ifdef BINGO_NO_L2_POLICY         // A/B experiment switch: plain evict_normal everywhere
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_keep));
    pol_stream = pol_keep;
#else
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
#endif
    const Policies pol{pol_keep, pol_stream};
#if BINGO_SMEM_HDR
    for (uint32_t j = threadIdx.x; j < a.sm_hdr; j += blockDim.x)
        s_thdr[j] = __ldg(reinterpret_cast<const unsigned long long *>(a.thdr) + j);
#endif
#if BINGO_SMEM_BKT
    for (uint32_t j = threadIdx.x; j < 2 * a.sm_bkt; j += blockDim.x)
        s_bkt[j] = __ldg(reinterpret_cast<const uint4 *>(a.bkt) + j);
#endif
#if BINGO_SMEM_HDR || BINGO_SMEM_BKT
    __syncthreads();
#endif
    const size_t row = (size_t)a.L + 1;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;   // first walker: static
    bool active = i < a.W;
    uint32_t w = 0, u = 0, t = 0, o = 0, prev = 0xFFFFFFFFu;
    uint64_t prev_nbo = 0, cur_nbo = 0;
    ThinHdr h;
    DecRec dr;
    dr.dcnt = 0;
    if (active) walker_start<APP, PROF, WMAJOR>(a, i, w, u, pol);
    // PPR lanes finish one at a time (stop w.p. 1/80 per step): their walker ids beyond the
    // static first one come from a warp-private reserve refilled WALK_CLAIM_CHUNK ids at a
    // time, one chunk claimed ahead, so the launch counter's atomic (7.6% of the c4 PPR stall
    // samples when every refill waited for it, ncu s3) leaves the dependent path: c4 PPR
    // 134.0 -> 130.4 ms.  DeepWalk warps finish together (one refill per walk length) and
    // keep the direct claim (the reserve: c2 11% slower); node2vec too (8 more registers, one
    // block less per SM: c3 19.7 -> 25.8 ms).  A/B: profiles/r02_walk_claim_ab.txt.  Which
    // lane runs which walker never changes a result (R-1).
#ifdef BINGO_CLAIM_SINGLE
    constexpr bool CHUNKED = false;
#else
    constexpr bool CHUNKED = APP == BINGO_PPR;
#endif
    unsigned long long res_base = 0, res_next = 0;
    uint32_t res_left = 0;
    if (CHUNKED && lane == 0) res_next = atomicAdd(claim, (unsigned long long)WALK_CLAIM_CHUNK);
    for (;;) {
        bool fin = false;
        if (active) {
            if (a.L != BINGO_NO_CAP && t >= a.L) {
                fin = true;                                   // L = 0
            } else {
                if (APP != BINGO_NODE2VEC || o == 0) {        // node2vec keeps u's header across proposals
#if BINGO_SMEM_HDR
                    if (u < a.sm_hdr) {
                        const unsigned long long v = s_thdr[u];
                        h.bkt_off = (uint32_t)v;
                        h.n = (uint8_t)(v >> 32);
                        h.flags = (uint8_t)(v >> 40);
                        h.pad1 = 0;
                    } else
#endif
#ifdef BINGO_VISIT_REC
                    if (APP == BINGO_PPR && a.visit)
                        h = load_thdr(reinterpret_cast<const ThinHdr *>(a.visit + visit_rec(u)), pol);
                    else
#endif
                    h = load_thdr(a.thdr + u, pol);
                    if (APP == BINGO_NODE2VEC && a.nbo)
                        cur_nbo = __ldg(reinterpret_cast<const unsigned long long *>(a.nbo + u));
                    if (FLT) dr = load_dec(a.dec + u);
                    if (PROF) prof.hdr++;
                    if (TRACE) prof.rec.x = u;
                }
                if (h.n == 0 && dr.dcnt == 0) {
                    fin = true;                               // dead end (d = 0): truncate (R-13)
                } else {
                    const uint32_t next = FLT ? sample_dst_f<PROF>(a, h, dr, w, t, o, prof, pol)
                                                : sample_dst<PROF, TRACE>(a, h, w, t, o, prof, pol);
                    bool accept = true;
                    if (APP == BINGO_NODE2VEC && t >= 1) {
                        // KnightKing rejection: propose first-order, accept with f/f_max;
                        // a rejected proposal re-draws everything under outer attempt o + 1 (R-14)
                        // The accept draw (tag 2) does not depend on the class, so it is taken
                        // first and the distance-1 probe runs only when the two candidate
                        // classes (next != prev: distance 1 or 2) would decide differently --
                        // the same decisions as classifying first, with most probes skipped
                        // (p = 2, q = 0.5: half of them; p = 0.5, q = 2: three quarters).
                        if (next == prev) {
                            if (!a.n2v_always[0]) {
                                const P4 r = draw_oi(w, t, o, 0u, 2u, a.k0, a.k1);
                                accept = join64(r.x, r.y) < a.n2v_thr[0];
                            }
                        } else if (!(a.n2v_always[1] && a.n2v_always[2])) {
                            const P4 r = draw_oi(w, t, o, 0u, 2u, a.k0, a.k1);
                            const uint64_t x = join64(r.x, r.y);
                            const bool a1 = a.n2v_always[1] || x < a.n2v_thr[1];
                            const bool a2 = a.n2v_always[2] || x < a.n2v_thr[2];
                            accept = (a1 == a2) ? a1 : (probe_arc<PROF>(a, prev, prev_nbo, next, prof) ? a1 : a2);
                        }
                    }
                    if (!accept) {
                        o++;
                    } else {
                        if (PROF) prof.steps++;
                        if (a.paths) {   // paths hold external ids
                            const uint32_t xn = a.perm ? __ldg(a.perm + next) : next;
                            if (WMAJOR) a.paths[i * row + t + 1] = xn;
                            else __stcs(&a.paths[(size_t)(t + 1) * a.W + i], xn);
                        }
                        prev = u;
                        prev_nbo = cur_nbo;
                        u = next;
                        o = 0;
                        if (APP == BINGO_PPR) {
#ifndef BINGO_EXP_NO_VISIT       // measurement experiment only: skip the visit counts
#ifndef BINGO_VISIT_PLAIN          // one atomic per distinct vertex per warp iteration (A/B: plain)
                            if (a.visit) {
                                const unsigned act = __activemask();
                                const unsigned same = __match_any_sync(act, u);
                                if ((__ffs(same) - 1) == (int)(threadIdx.x & 31u)) {
#ifdef BINGO_VISIT32
                                    if (a.visit32) visit_add32(&a.visit32[visit_slot(u)], (unsigned)__popc(same), pol);
                                    else
#endif
                                    {
#ifdef BINGO_VISIT_REC
                                        visit_add(a.visit + visit_slot(u), (unsigned long long)__popc(same), pol);
#else
                                        const uint32_t r = ((threadIdx.x >> 5) + blockIdx.x) % BINGO_VISIT_COPIES;
#ifdef BINGO_VISIT_REDPOL        // A/B: counters of the non-padded (colder) vertices with an L2 evict_first hint
                                        if (u >= BINGO_VISIT_PAD)
                                            asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;"
                                                         :: "l"(a.visit + visit_slot_r(u, r)), "l"((unsigned long long)__popc(same)),
                                                            "l"(pol.stream) : "memory");
                                        else
#endif
                                        visit_add(a.visit + visit_slot_r(u, r), (unsigned long long)__popc(same), pol);
#endif
                                    }
                                }
                            }
#else
                            if (a.visit) visit_add(a.visit + visit_slot(u), 1ull, pol);
#endif
#endif
                            if (PROF) prof.visit++;
                            if (a.stop_always) {
                                fin = true;
                            } else {
                                const P4 r = philox10(w, t, 0u, 3u, a.k0, a.k1);
                                fin = join64(r.x, r.y) < a.stop_thr;
                            }
                        }
                        if (TRACE) {
                            const unsigned long long r = a.trace_off[i] + t;
                            if (r < a.trace_off[i + 1]) a.trace[r] = prof.rec;
                            prof.rec = make_uint4(0u, 0u, TR_EMPTY, TR_EMPTY);
                        }
                        t++;
                        if (a.L != BINGO_NO_CAP && t >= a.L) fin = true;
                    }
                }
            }
            if (fin) {
                if (PROF) prof.walkers++;
                if (a.lengths) a.lengths[i] = t;
                if (a.paths && a.L != BINGO_NO_CAP) {
                    for (uint32_t s = t + 1; s <= a.L; s++) {
                        if (WMAJOR) a.paths[i * row + s] = 0xFFFFFFFFu;
                        else __stcs(&a.paths[(size_t)s * a.W + i], 0xFFFFFFFFu);
                    }
                }
            }
        }
        // refill: the lanes that finished take consecutive walker ids in lane order
        const unsigned fmask = __ballot_sync(0xffffffffu, fin);
        if (fmask) {
            unsigned long long id;
            if (!CHUNKED) {   // one atomic on the launch counter per refill (the warp waits for it)
                const uint32_t leader = __ffs(fmask) - 1;
                unsigned long long base = 0;
                if (lane == leader) base = atomicAdd(claim, (unsigned long long)__popc(fmask));
                base = __shfl_sync(0xffffffffu, base, leader);
                id = base + __popc(fmask & ((1u << lane) - 1u));
            } else {
                // from the warp's reserve; when it runs out, switch to the chunk claimed ahead and
                // claim the next one (lane 0's atomic result is read only at the following switch)
                const uint32_t nf = __popc(fmask), rank = __popc(fmask & ((1u << lane) - 1u));
                if (nf <= res_left) {
                    id = res_base + rank;
                    res_base += nf;
                    res_left -= nf;
                } else {
                    const unsigned long long nb = __shfl_sync(0xffffffffu, res_next, 0);
                    id = rank < res_left ? res_base + rank : nb + (rank - res_left);
                    res_base = nb + (nf - res_left);
                    res_left = WALK_CLAIM_CHUNK - (nf - res_left);
                    if (lane == 0) res_next = atomicAdd(claim, (unsigned long long)WALK_CLAIM_CHUNK);
                }
            }
            if (fin) {
                i = nthreads + id;
                active = i < a.W;
                t = 0;
                o = 0;
                prev = 0xFFFFFFFFu;
                prev_nbo = cur_nbo = 0;
                if (active) walker_start<APP, PROF, WMAJOR>(a, i, w, u, pol);
            }
        }
        if (!__any_sync(0xffffffffu, active)) break;
    }
    if (PROF) prof.flush(a.prof);
}

}  // namespace bingo

// ---------------------------------------------------------------- host side
static void n2v_thresholds(double p, double q, unsigned long long thr[3], uint32_t always[3]) {
    const double f[3] = {1.0 / p, 1.0, 1.0 / q};
    double fmax = f[0];
    for (int i = 1; i < 3; i++) fmax = f[i] > fmax ? f[i] : fmax;
    for (int i = 0; i < 3; i++) {
        const double r = f[i] / fmax;
        if (r >= 1.0) {
            always[i] = 1;
            thr[i] = 0;
        } else {
            // floor(r * 2^64): r < 1 is a double, r * 2^64 is exact, conversion truncates
            always[i] = 0;
            thr[i] = (unsigned long long)ldexp(r, 64);
        }
    }
}

static void stop_threshold(uint32_t num, uint32_t den, unsigned long long *thr, uint32_t *always) {
    if (num >= den) {
        *always = 1;
        *thr = 0;
        return;
    }
    *always = 0;
    *thr = (unsigned long long)(((unsigned __int128)num << 64) / den);   // floor(num 2^64 / den)
}

// Persistent grid: exactly the resident capacity (SMs x occupancy), so every
// block runs from the start and strides over walkers -- no partial second wave.
template <typename K>
static unsigned walk_grid(K kernel, uint32_t W) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, BINGO_WALK_TPB, 0);
    if (const char *e = getenv("BINGO_WALK_BLOCKS_PER_SM")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
    cudaGetLastError();
    const size_t need = ((size_t)W + BINGO_WALK_TPB - 1) / BINGO_WALK_TPB;
    const size_t cap = (size_t)sms * (size_t)std::max(per_sm, 1);
    return (unsigned)std::max<size_t>(1, std::min(need, cap));
}

struct TraceOut {
    uint4 *trace;
    const unsigned long long *off;
};

#ifdef BINGO_VISIT32
// fold one launch's u32 counts into the u64 totals (and clear them)
__global__ void k_visit_fold(uint32_t V, unsigned int *v32, unsigned long long *visit) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < V; u += gridDim.x * blockDim.x) {
        const uint64_t sl = visit_slot(u);
        const unsigned int c = v32[sl];
        if (c) {
            visit[sl] += c;
            v32[sl] = 0;
        }
    }
}
#endif

#ifdef BINGO_VISIT_REC
__global__ void k_visit_hdr(uint32_t V, const ThinHdr *__restrict__ thdr, unsigned long long *visit) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < V; u += gridDim.x * blockDim.x)
        visit[visit_rec(u)] = *reinterpret_cast<const unsigned long long *>(thdr + u);
}
#endif

bingo_status launch_walk(bingo_graph *g, const bingo_walk_desc *desc, const uint32_t *starts, uint32_t W,
                         uint32_t *paths, uint32_t *lengths, cudaStream_t s, unsigned long long *prof = nullptr,
                         const TraceOut *tr = nullptr) {
    WalkArgs a;
    a.thdr = g->thdr;
    a.hdr = g->hdr;
    a.bkt = g->bkt;
    a.arc = g->arc;
    a.mdst = g->mdst;
    a.nbt = g->nbt;
    a.nbo = g->nbo;
    a.dec = g->float_mode ? g->dec : nullptr;
    a.dmem = g->dmem;
    a.visit = g->visit;
    a.starts = starts;
    a.perm = g->perm;
    a.inv = g->inv;
    a.paths = paths;
    a.lengths = lengths;
    a.W = W;
    a.V = g->V;
    a.L = desc->length;
    a.first_walker = desc->first_walker_id;
    a.k0 = (uint32_t)desc->seed;
    a.k1 = (uint32_t)(desc->seed >> 32);
    n2v_thresholds(desc->app == BINGO_NODE2VEC ? desc->p : 1.0, desc->app == BINGO_NODE2VEC ? desc->q : 1.0,
                   a.n2v_thr, a.n2v_always);
    // a class whose accept ratio f/f_max is below 2^-64 could never be accepted (its threshold
    // floors to 0): a walker whose proposals all fall in it would never finish -> EINVAL.
    // Otherwise the expected proposals per step are at most f_max / f_min (draw_oi never
    // repeats a counter, so the attempts are independent).
    for (int c = 0; c < 3; c++)
        if (desc->app == BINGO_NODE2VEC && !a.n2v_always[c] && a.n2v_thr[c] == 0) return BINGO_E_INVAL;
    stop_threshold(desc->stop_num, desc->stop_den, &a.stop_thr, &a.stop_always);
    a.prof = prof;
    // shared-memory staging: headers only where ids are hot-first (relabelled), not in the
    // trace / float kernels
    a.sm_hdr = (g->inv && !tr && !g->float_mode) ? (uint32_t)std::min<uint64_t>(BINGO_SMEM_HDR, g->V) : 0u;
    a.sm_bkt = (!tr && !g->float_mode) ? (uint32_t)std::min<uint64_t>(BINGO_SMEM_BKT, g->bkt_cap) : 0u;
    a.trace = tr ? tr->trace : nullptr;
    a.trace_off = tr ? tr->off : nullptr;
    a.visit32 = nullptr;
#ifdef BINGO_VISIT32
    if (desc->app == BINGO_PPR && !tr && g->V) {
        // a launch's visits (W x (1 + mean length)) must stay far below 2^32 per counter
        const double mean = desc->stop_num ? std::min<double>((double)desc->stop_den / desc->stop_num,
                                                              desc->length == BINGO_NO_CAP ? 1e30 : desc->length)
                                           : 1.0;
        if ((double)W * (1.0 + mean) < 2.0e9) {
            if (!g->visit32) {
                g->visit32 = (unsigned int *)bingo_dev_alloc(g, 4 * std::max<uint64_t>(visit_words(g->V), 1));
                if (g->visit32 && cudaMemsetAsync(g->visit32, 0, 4 * std::max<uint64_t>(visit_words(g->V), 1), s) != cudaSuccess)
                    return BINGO_E_CUDA;
            }
            a.visit32 = g->visit32;
        }
    }
#endif
    if (tr && (desc->app == BINGO_NODE2VEC || g->float_mode || (desc->flags & BINGO_WALK_WALKER_MAJOR) || !prof))
        return BINGO_E_INVAL;
    if (!g->walk_ctr) return BINGO_E_STATE;
#ifdef BINGO_VISIT_REC
    if (desc->app == BINGO_PPR && a.visit && g->V) {
        k_visit_hdr<<<(unsigned)std::min<uint64_t>((g->V + 255) / 256, 148ull * 16), 256, 0, s>>>(g->V, g->thdr, g->visit);
        bingo_count_launch();
    }
#endif
    unsigned long long *claim = g->walk_ctr + (__atomic_fetch_add(&g->walk_slot, 1u, __ATOMIC_RELAXED) % BINGO_WALK_SLOTS);
    if (cudaMemsetAsync(claim, 0, sizeof(unsigned long long), s) != cudaSuccess) {
        g->poisoned = 1;
        return BINGO_E_CUDA;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(BINGO_WALK_TPB);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cfg.attrs = nullptr;
    cfg.numAttrs = 0;
    cudaError_t le = cudaSuccess;
    const bool wmajor = (desc->flags & BINGO_WALK_WALKER_MAJOR) != 0;
#define BINGO_K3(APP_, PROF_, FLT_)                                                               \
    (wmajor ? (cfg.gridDim = dim3(walk_grid(k_walk<APP_, PROF_, true, FLT_>, W)),                 \
               cudaLaunchKernelEx(&cfg, k_walk<APP_, PROF_, true, FLT_>, a, claim))                      \
            : (cfg.gridDim = dim3(walk_grid(k_walk<APP_, PROF_, false, FLT_>, W)),                \
               cudaLaunchKernelEx(&cfg, k_walk<APP_, PROF_, false, FLT_>, a, claim)))
#define BINGO_K(APP_, PROF_) (a.dec ? BINGO_K3(APP_, PROF_, true) : BINGO_K3(APP_, PROF_, false))
    if (tr) {
        if (desc->app == BINGO_DEEPWALK) {
            cfg.gridDim = dim3(walk_grid(k_walk<BINGO_DEEPWALK, 2, false, false>, W));
            le = cudaLaunchKernelEx(&cfg, k_walk<BINGO_DEEPWALK, 2, false, false>, a, claim);
        } else {
            cfg.gridDim = dim3(walk_grid(k_walk<BINGO_PPR, 2, false, false>, W));
            le = cudaLaunchKernelEx(&cfg, k_walk<BINGO_PPR, 2, false, false>, a, claim);
        }
    } else if (prof) {
        switch (desc->app) {
            case BINGO_DEEPWALK: le = BINGO_K(BINGO_DEEPWALK, 1); break;
            case BINGO_NODE2VEC: le = BINGO_K(BINGO_NODE2VEC, 1); break;
            case BINGO_PPR: le = BINGO_K(BINGO_PPR, 1); break;
            default: return BINGO_E_INVAL;
        }
    } else {
        switch (desc->app) {
            case BINGO_DEEPWALK: le = BINGO_K(BINGO_DEEPWALK, 0); break;
            case BINGO_NODE2VEC: le = BINGO_K(BINGO_NODE2VEC, 0); break;
            case BINGO_PPR: le = BINGO_K(BINGO_PPR, 0); break;
            default: return BINGO_E_INVAL;
        }
    }
#undef BINGO_K
#undef BINGO_K3
    if (le != cudaSuccess) {
        fprintf(stderr, "libbingo: walk launch failed: %s\n", cudaGetErrorString(le));
        g->poisoned = 1;
        return BINGO_E_CUDA;
    }
    bingo_count_launch();
#ifdef BINGO_VISIT32
    if (a.visit32) {
        k_visit_fold<<<(unsigned)std::min<uint64_t>((g->V + 255) / 256, 148ull * 16), 256, 0, s>>>(g->V, a.visit32, g->visit);
        bingo_count_launch();
    }
#endif
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "libbingo: walk launch failed: %s\n", cudaGetErrorString(e));
        g->poisoned = 1;
        return BINGO_E_CUDA;
    }
    return BINGO_OK;
}

extern "C" bingo_status bingo_walk(bingo_graph *g, const bingo_walk_desc *desc, const uint32_t *starts_or_null,
                                   uint32_t num_walkers, uint32_t *paths_or_null, uint32_t *lengths_or_null,
                                   void *stream) {
    if (!g || !desc) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    bingo_sq_quiesce(g, (cudaStream_t)stream);
    if (desc->app > BINGO_PPR) return BINGO_E_INVAL;
    if (desc->app == BINGO_NODE2VEC && !(desc->p > 0 && desc->q > 0)) return BINGO_E_INVAL;
    if (desc->app == BINGO_PPR && desc->stop_den == 0) return BINGO_E_INVAL;
    if (desc->length == BINGO_NO_CAP && paths_or_null) return BINGO_E_INVAL;
    if (desc->length == BINGO_NO_CAP && desc->app != BINGO_PPR) return BINGO_E_INVAL;
    if (num_walkers == 0) return BINGO_OK;
    if (g->V == 0) return BINGO_E_INVAL;
    cudaStream_t s = (cudaStream_t)stream;
    if (g->radix_log2) {
        if (desc->flags & BINGO_WALK_HOST_OUTPUT) return BINGO_E_INVAL;
        return launch_walk_radix(g, desc, starts_or_null, num_walkers, paths_or_null, lengths_or_null, s);
    }
    if (!(desc->flags & BINGO_WALK_HOST_OUTPUT))
        return launch_walk(g, desc, starts_or_null, num_walkers, paths_or_null, lengths_or_null, s);
    // HOST buffers: the walkers run in chunks whose paths are staged in two device
    // buffers; each chunk's D2H copy (a strided 2-D copy for step-major paths) runs on
    // a side stream while the next chunk walks, so the PCIe transfer of the paths
    // overlaps the walk instead of following it.
    const uint64_t W = num_walkers;
    const uint64_t row = (uint64_t)desc->length + 1;
    const bool wmajor = (desc->flags & BINGO_WALK_WALKER_MAJOR) != 0;
    uint64_t Wc = W;
    if (paths_or_null) {
        Wc = std::max<uint64_t>(1 << 17, (W + 15) / 16);   // small chunks: the first copy starts early
        Wc = std::min<uint64_t>(Wc, W);
    }
    const uint64_t nchunks = (W + Wc - 1) / Wc;
    const size_t slot_words = paths_or_null ? (size_t)(row * Wc) : 0;
    const size_t need = sizeof(uint32_t) * (2 * slot_words + (lengths_or_null ? W : 0) + (starts_or_null ? W : 0)) + 256;
    if (g->wscratch_bytes < need) {
        bingo_dev_free(g, g->wscratch);
        g->wscratch = bingo_dev_alloc(g, need);
        g->wscratch_bytes = g->wscratch ? need : 0;
        if (!g->wscratch) return BINGO_E_NOMEM;
    }
    uint32_t *slots[2] = {(uint32_t *)g->wscratch, (uint32_t *)g->wscratch + slot_words};
    uint32_t *dl = (uint32_t *)g->wscratch + 2 * slot_words;
    uint32_t *ds = dl + (lengths_or_null ? W : 0);
    cudaError_t e = cudaSuccess;
    if (!g->copy_stream) {
        e = cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking);
        for (int i = 0; i < 2 && e == cudaSuccess; i++) {
            e = cudaEventCreateWithFlags(&g->ev_walk[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_copy[i], cudaEventDisableTiming);
        }
    }
    if (e == cudaSuccess && starts_or_null)
        e = cudaMemcpyAsync(ds, starts_or_null, sizeof(uint32_t) * W, cudaMemcpyHostToDevice, s);
    for (uint64_t c = 0; c < nchunks && e == cudaSuccess; c++) {
        const uint64_t c0 = c * Wc, wn = std::min<uint64_t>(Wc, W - c0);
        const int sl = (int)(c & 1);
        if (c >= 2 && paths_or_null) e = cudaStreamWaitEvent(s, g->ev_copy[sl], 0);
        if (e != cudaSuccess) break;
        bingo_walk_desc dc = *desc;
        dc.first_walker_id = desc->first_walker_id + (uint32_t)c0;
        bingo_status st = launch_walk(g, &dc, starts_or_null ? ds + c0 : nullptr, (uint32_t)wn,
                                      paths_or_null ? slots[sl] : nullptr, lengths_or_null ? dl + c0 : nullptr, s);
        if (st != BINGO_OK) return st;
        if (!paths_or_null) continue;
        e = cudaEventRecord(g->ev_walk[sl], s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(g->copy_stream, g->ev_walk[sl], 0);
        if (e == cudaSuccess) {
            if (wmajor)
                e = cudaMemcpyAsync(paths_or_null + c0 * row, slots[sl], sizeof(uint32_t) * wn * row,
                                    cudaMemcpyDeviceToHost, g->copy_stream);
            else
                e = cudaMemcpy2DAsync(paths_or_null + c0, sizeof(uint32_t) * W, slots[sl], sizeof(uint32_t) * wn,
                                      sizeof(uint32_t) * wn, row, cudaMemcpyDeviceToHost, g->copy_stream);
        }
        if (e == cudaSuccess) e = cudaEventRecord(g->ev_copy[sl], g->copy_stream);
    }
    if (e == cudaSuccess && lengths_or_null)
        e = cudaMemcpyAsync(lengths_or_null, dl, sizeof(uint32_t) * W, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && g->copy_stream) e = cudaStreamSynchronize(g->copy_stream);
    if (e != cudaSuccess) {
        fprintf(stderr, "libbingo: walk staging failed: %s\n", cudaGetErrorString(e));
        g->poisoned = 1;
        return BINGO_E_CUDA;
    }
    return BINGO_OK;
}

extern "C" bingo_status bingo_walk_profile(bingo_graph *g, const bingo_walk_desc *desc, const uint32_t *starts_or_null,
                                           uint32_t num_walkers, uint32_t *paths_or_null, uint32_t *lengths_or_null,
                                           uint64_t *counters_host, void *stream) {
    if (!g || !desc || !counters_host) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    bingo_sq_quiesce(g, (cudaStream_t)stream);
    if (g->radix_log2) return BINGO_E_INVAL;
    if (desc->app > BINGO_PPR || (desc->flags & BINGO_WALK_HOST_OUTPUT)) return BINGO_E_INVAL;
    if (desc->app == BINGO_NODE2VEC && !(desc->p > 0 && desc->q > 0)) return BINGO_E_INVAL;
    if (desc->app == BINGO_PPR && desc->stop_den == 0) return BINGO_E_INVAL;
    if (desc->length == BINGO_NO_CAP && (paths_or_null || desc->app != BINGO_PPR)) return BINGO_E_INVAL;
    if (g->V == 0) return BINGO_E_INVAL;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *dprof = (unsigned long long *)bingo_dev_alloc(g, sizeof(unsigned long long) * BINGO_PROF_N);
    if (!dprof) return BINGO_E_NOMEM;
    cudaError_t e = cudaMemsetAsync(dprof, 0, sizeof(unsigned long long) * BINGO_PROF_N, s);
    bingo_status st = BINGO_OK;
    if (e == cudaSuccess)
        st = launch_walk(g, desc, starts_or_null, num_walkers, paths_or_null, lengths_or_null, s, dprof);
    if (st == BINGO_OK && e == cudaSuccess)
        e = cudaMemcpyAsync(counters_host, dprof, sizeof(unsigned long long) * BINGO_PROF_N, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    bingo_dev_free(g, dprof);
    if (e != cudaSuccess) { g->poisoned = 1; return BINGO_E_CUDA; }
    return st;
}

// ---------------------------------------------------------------- access trace + replay
// (measurement only: the roofline's "achievable gather bandwidth" for the walk's OWN
// footprint and skew).  bingo_walk_trace re-runs a walk (same walks as bingo_walk) and
// records, per step, the loads the step made (16 B records, walk_common.cuh);
// k_replay then issues exactly those loads -- same addresses, widths, L2 policies and 64 B
// fetch hints -- walker by walker like the walk (a thread takes a walker and runs through
// its steps), but with no dependency between steps: REPLAY_AHEAD steps (up to 16 loads)
// in flight per thread.  That is the walk with perfect prefetching: what the memory system
// delivers for this access stream when latency is hidden -- the ceiling the dependent walk
// is measured against.
extern "C" bingo_status bingo_walk_trace(bingo_graph *g, const bingo_walk_desc *desc, const uint32_t *starts_or_null,
                                         uint32_t num_walkers, const uint64_t *rec_off, void *trace,
                                         uint64_t n_records, uint64_t *counters_host, void *stream) {
    if (!g || !desc || !counters_host || !rec_off || !trace) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    bingo_sq_quiesce(g, (cudaStream_t)stream);
    if (g->radix_log2) return BINGO_E_INVAL;
    if (!(desc->app == BINGO_DEEPWALK || desc->app == BINGO_PPR) || desc->flags || g->float_mode) return BINGO_E_INVAL;
    if (desc->app == BINGO_PPR && desc->stop_den == 0) return BINGO_E_INVAL;
    if (desc->length == BINGO_NO_CAP && desc->app != BINGO_PPR) return BINGO_E_INVAL;
    if (g->V == 0 || g->arc_cap >= (1ull << 32) || g->mem_cap >= (1ull << 32) || g->bkt_cap >= (1ull << 31))
        return BINGO_E_INVAL;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *dprof = (unsigned long long *)bingo_dev_alloc(g, sizeof(unsigned long long) * BINGO_PROF_N);
    if (!dprof) return BINGO_E_NOMEM;
    cudaError_t e = cudaMemsetAsync(dprof, 0, sizeof(unsigned long long) * BINGO_PROF_N, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(trace, 0xFF, sizeof(uint4) * n_records, s);
    const TraceOut tr{reinterpret_cast<uint4 *>(trace), reinterpret_cast<const unsigned long long *>(rec_off)};
    bingo_status st = BINGO_OK;
    if (e == cudaSuccess) st = launch_walk(g, desc, starts_or_null, num_walkers, nullptr, nullptr, s, dprof, &tr);
    if (st == BINGO_OK && e == cudaSuccess)
        e = cudaMemcpyAsync(counters_host, dprof, sizeof(unsigned long long) * BINGO_PROF_N, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    bingo_dev_free(g, dprof);
    if (e != cudaSuccess) { g->poisoned = 1; return BINGO_E_CUDA; }
    return st;
}

struct ReplayArgs {
    const uint4 *trace;
    const unsigned long long *off;
    uint32_t walkers;
    const ThinHdr *thdr;
    const Bucket *bkt;
    const uint32_t *mdst;
    const uint2 *arc;
    unsigned long long *counts;   // [4] loads issued: headers, buckets, members, arcs
    uint32_t *sink;
};

__device__ __forceinline__ uint32_t replay_intra(const ReplayArgs &a, uint32_t c, uint64_t keep, uint64_t strm,
                                                 uint32_t &nm, uint32_t &na) {
    if (c == TR_EMPTY) return 0;
    const uint64_t pol = (c >> 30) & 1u ? keep : strm;
    const uint64_t gr = c & 0x3FFFFFFFu;
    if (c >> 31) {
        na++;
        return ldg8(a.arc + (gr << 2), pol).x;
    }
    nm++;
    return ldg4(a.mdst + (gr << 2), pol);
}

template <int REPLAY_AHEAD>
__global__ void __launch_bounds__(256) k_replay(const ReplayArgs a) {
    uint64_t pol_keep, pol_stream;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    const Policies pol{pol_keep, pol_stream};
    uint32_t acc = 0, nh = 0, nm = 0, na = 0;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < a.walkers; j += gridDim.x * blockDim.x) {
        const unsigned long long r1 = a.off[j + 1];
        for (unsigned long long r = a.off[j]; r < r1; r += REPLAY_AHEAD) {
            uint4 c[REPLAY_AHEAD];
#pragma unroll
            for (int u = 0; u < REPLAY_AHEAD; u++)
                c[u] = r + u < r1 ? __ldcs(a.trace + r + u) : make_uint4(TR_EMPTY, TR_EMPTY, TR_EMPTY, TR_EMPTY);
            uint32_t v[REPLAY_AHEAD][4];
#pragma unroll
            for (int u = 0; u < REPLAY_AHEAD; u++) {
                v[u][0] = v[u][1] = 0;
                if (c[u].x != TR_EMPTY) {
                    v[u][0] = load_thdr(a.thdr + c[u].x, pol).bkt_off;
                    const Bucket B = ldg_bucket(a.bkt + (c[u].y & 0x7FFFFFFFu), c[u].y >> 31 ? pol_keep : pol_stream);
                    v[u][1] = B.px ^ B.ay;
                    nh++;
                }
                v[u][2] = replay_intra(a, c[u].z, pol_keep, pol_stream, nm, na);
                v[u][3] = replay_intra(a, c[u].w, pol_keep, pol_stream, nm, na);
            }
#pragma unroll
            for (int u = 0; u < REPLAY_AHEAD; u++) acc ^= v[u][0] ^ v[u][1] ^ v[u][2] ^ v[u][3];
        }
    }
    const unsigned long long x[3] = {warp_sum((unsigned long long)nh), warp_sum((unsigned long long)nm),
                                     warp_sum((unsigned long long)na)};
    if ((threadIdx.x & 31u) == 0) {
        if (x[0]) { atomicAdd(&a.counts[0], x[0]); atomicAdd(&a.counts[1], x[0]); }
        if (x[1]) atomicAdd(&a.counts[2], x[1]);
        if (x[2]) atomicAdd(&a.counts[3], x[2]);
    }
    if (acc == 0x9E3779B9u) a.sink[0] = acc;   // keeps the loads alive
}

extern "C" bingo_status bingo_walk_replay(bingo_graph *g, const void *trace, const uint64_t *rec_off,
                                          uint32_t num_walkers, uint32_t flags, uint64_t *counts_host, void *stream) {
    if (!g || !trace || !rec_off || !counts_host) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    bingo_sq_quiesce(g, (cudaStream_t)stream);
    if (g->radix_log2) return BINGO_E_INVAL;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *dc = (unsigned long long *)bingo_dev_alloc(g, sizeof(unsigned long long) * 8);
    if (!dc) return BINGO_E_NOMEM;
    ReplayArgs a;
    a.trace = reinterpret_cast<const uint4 *>(trace);
    a.off = reinterpret_cast<const unsigned long long *>(rec_off);
    a.walkers = num_walkers;
    a.thdr = g->thdr;
    a.bkt = g->bkt;
    a.mdst = g->mdst;
    a.arc = g->arc;
    a.counts = dc;
    a.sink = reinterpret_cast<uint32_t *>(dc + 7);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaMemsetAsync(dc, 0, sizeof(unsigned long long) * 8, s);
    // flags: bits 0-1 log2(steps in flight per thread: 1, 2, 4, 8), bits 8-15 blocks per SM (0: 8)
    const unsigned bps = ((flags >> 8) & 0xFFu) ? ((flags >> 8) & 0xFFu) : 8u;
    const dim3 grid((unsigned)sms * bps);
    if (e == cudaSuccess) {
        switch (flags & 3u) {
            case 0: k_replay<1><<<grid, 256, 0, s>>>(a); break;
            case 1: k_replay<2><<<grid, 256, 0, s>>>(a); break;
            case 2: k_replay<4><<<grid, 256, 0, s>>>(a); break;
            default: k_replay<8><<<grid, 256, 0, s>>>(a); break;
        }
        bingo_count_launch();
        e = cudaGetLastError();
    }
    uint64_t h[8] = {0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, dc, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    bingo_dev_free(g, dc);
    if (e != cudaSuccess) { g->poisoned = 1; return BINGO_E_CUDA; }
    for (int k = 0; k < 4; k++) counts_host[k] = h[k];
    return BINGO_OK;
}

// ---------------------------------------------------------------- 1-D partitioned walk
// The paper's multi-GPU design (after KnightKing): the graph is partitioned by
// vertex (each rank builds its graph over the full id space with only its own vertices'
// arcs) and WALKERS move to the rank that owns their current vertex.  One launch advances
// every walker of the inbox while it stays on owned vertices; a walker that steps onto a
// vertex another rank owns is written to that rank's outbox region and leaves.  Because
// every draw is keyed by (walker, step) (R-1), the partitioned walk takes exactly the
// single-GPU walk's steps, and the exchange order does not matter.
struct PartArgs {
    WalkArgs a;                       // graph, RNG, thresholds; paths / lengths indexed by i = w - first
    const uint4 *inbox;               // {walker id, current vertex (external), steps taken, fresh}
    uint32_t n_in;
    uint4 *outbox;                    // [parts][cap]
    unsigned long long cap;
    uint32_t *out_count;              // [parts] (pre-zeroed)
    const uint32_t *bounds;           // [parts + 1] owned external-id ranges
    uint32_t parts, me;
    unsigned long long *done;         // walkers that finished here
};

__device__ __forceinline__ uint32_t part_owner(const PartArgs &p, uint32_t x) {
    uint32_t r = 0;
    while (r + 1 < p.parts && x >= __ldg(p.bounds + r + 1)) r++;
    return r;
}

template <int APP>
__global__ void __launch_bounds__(BINGO_WALK_TPB) k_walk_part(const PartArgs p, unsigned long long *__restrict__ claim) {
    const WalkArgs &a = p.a;
    uint64_t pol_keep, pol_stream;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    const Policies pol{pol_keep, pol_stream};
    WalkProf prof;
    const uint32_t lane = threadIdx.x & 31u;
    unsigned long long fin_here = 0;
    for (;;) {
        unsigned long long j0 = 0;
        if (lane == 0) j0 = atomicAdd(claim, 32ull);
        j0 = __shfl_sync(0xffffffffu, j0, 0);
        if (j0 >= p.n_in) break;
        const unsigned long long j = j0 + lane;
        if (j < p.n_in) {   // the warp reconverges before its next claim
        const uint4 rec = p.inbox[j];
        const uint32_t w = rec.x;
        const uint64_t i = (uint64_t)(w - a.first_walker);
        uint32_t t = rec.z;
        uint32_t ux = rec.y;                                  // external id of the current vertex
        uint32_t u = a.inv ? __ldg(a.inv + ux) : ux;
        if (rec.w & 1u) {                                     // fresh walker: its start vertex is ours
            if (a.paths) __stcs(&a.paths[i], ux);
            if (APP == BINGO_PPR && a.visit) visit_add(a.visit + visit_slot(u), 1ull, pol);
        }
        bool finished = false;
        for (;;) {
            if (a.L != BINGO_NO_CAP && t >= a.L) { finished = true; break; }
            const ThinHdr h = load_thdr(a.thdr + u, pol);
            if (h.n == 0) { finished = true; break; }      // an owned dead end (d = 0): truncate (R-13)
            const uint32_t next = sample_dst<false>(a, h, w, t, 0u, prof, pol);
            const uint32_t nx = a.perm ? __ldg(a.perm + next) : next;
            if (a.paths) __stcs(&a.paths[(size_t)(t + 1) * a.W + i], nx);
            bool stop = false;
            if (APP == BINGO_PPR) {
                if (a.visit) visit_add(a.visit + visit_slot(next), 1ull, pol);
                if (a.stop_always) {
                    stop = true;
                } else {
                    const P4 r = philox10(w, t, 0u, 3u, a.k0, a.k1);
                    stop = join64(r.x, r.y) < a.stop_thr;
                }
            }
            t++;
            if (stop) { finished = true; break; }
            const uint32_t o = part_owner(p, nx);
            if (o != p.me) {                                  // leaves for the owner of its new vertex
                const unsigned long long pos = atomicAdd(&p.out_count[o], 1u);
                if (pos < p.cap) p.outbox[(unsigned long long)o * p.cap + pos] = make_uint4(w, nx, t, 0u);
                break;
            }
            u = next;
        }
        if (finished) {
            fin_here++;
            if (a.lengths) a.lengths[i] = t;
            if (a.paths && a.L != BINGO_NO_CAP)
                for (uint32_t s2 = t + 1; s2 <= a.L; s2++) __stcs(&a.paths[(size_t)s2 * a.W + i], 0xFFFFFFFFu);
        }
        }
        __syncwarp();
    }
    const unsigned long long f = warp_sum(fin_here);
    if (lane == 0 && f) atomicAdd(p.done, f);
}

extern "C" bingo_status bingo_walk_partition(bingo_graph *g, const bingo_walk_desc *desc, uint32_t num_walkers,
                                             const uint32_t *bounds, uint32_t parts, uint32_t me, const void *inbox,
                                             uint32_t n_in, void *outbox, uint64_t out_cap, uint32_t *out_count,
                                             uint32_t *paths_or_null, uint32_t *lengths_or_null,
                                             uint64_t *finished_host, void *stream) {
    if (!g || !desc || !bounds || !out_count || (n_in && !inbox) || !outbox || parts == 0 || me >= parts ||
        !finished_host || out_cap < n_in)
        return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    bingo_sq_quiesce(g, (cudaStream_t)stream);
    if (g->radix_log2) return BINGO_E_INVAL;
    if (!(desc->app == BINGO_DEEPWALK || desc->app == BINGO_PPR) || g->float_mode) return BINGO_E_INVAL;
    if (desc->flags || (desc->app == BINGO_PPR && desc->stop_den == 0)) return BINGO_E_INVAL;
    if (desc->length == BINGO_NO_CAP && (paths_or_null || desc->app != BINGO_PPR)) return BINGO_E_INVAL;
    cudaStream_t s = (cudaStream_t)stream;
    PartArgs p;
    memset(&p, 0, sizeof(p));
    WalkArgs &a = p.a;
    a.thdr = g->thdr;
    a.hdr = g->hdr;
    a.bkt = g->bkt;
    a.arc = g->arc;
    a.mdst = g->mdst;
    a.visit = g->visit;
    a.perm = g->perm;
    a.inv = g->inv;
    a.paths = paths_or_null;
    a.lengths = lengths_or_null;
    a.W = num_walkers;
    a.V = g->V;
    a.L = desc->length;
    a.first_walker = desc->first_walker_id;
    a.k0 = (uint32_t)desc->seed;
    a.k1 = (uint32_t)(desc->seed >> 32);
    stop_threshold(desc->stop_num, desc->stop_den, &a.stop_thr, &a.stop_always);
    p.inbox = reinterpret_cast<const uint4 *>(inbox);
    p.n_in = n_in;
    p.outbox = reinterpret_cast<uint4 *>(outbox);
    p.cap = out_cap;
    p.out_count = out_count;
    p.bounds = bounds;
    p.parts = parts;
    p.me = me;
    unsigned long long *dc = (unsigned long long *)bingo_dev_alloc(g, 2 * sizeof(unsigned long long));
    if (!dc) return BINGO_E_NOMEM;
    p.done = dc + 1;
    cudaError_t e = cudaMemsetAsync(dc, 0, 2 * sizeof(unsigned long long), s);
    if (e == cudaSuccess && n_in) {
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (desc->app == BINGO_PPR) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_walk_part<BINGO_PPR>, BINGO_WALK_TPB, 0);
            const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_in + BINGO_WALK_TPB - 1) / BINGO_WALK_TPB,
                                                                                      (uint64_t)sms * std::max(per_sm, 1)));
            k_walk_part<BINGO_PPR><<<grid, BINGO_WALK_TPB, 0, s>>>(p, dc);
        } else {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_walk_part<BINGO_DEEPWALK>, BINGO_WALK_TPB, 0);
            const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_in + BINGO_WALK_TPB - 1) / BINGO_WALK_TPB,
                                                                                      (uint64_t)sms * std::max(per_sm, 1)));
            k_walk_part<BINGO_DEEPWALK><<<grid, BINGO_WALK_TPB, 0, s>>>(p, dc);
        }
        bingo_count_launch();
        e = cudaGetLastError();
    }
    unsigned long long fh = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&fh, dc + 1, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    *finished_host = fh;
    bingo_dev_free(g, dc);
    if (e != cudaSuccess) {
        fprintf(stderr, "libbingo: partitioned walk failed: %s\n", cudaGetErrorString(e));
        g->poisoned = 1;
        return BINGO_E_CUDA;
    }
    return BINGO_OK;
}

// counts in external vertex order: out[u] = visit[inv[u]]
__global__ void k_visit_gather(uint32_t V, const uint32_t *__restrict__ inv, const unsigned long long *__restrict__ visit,
                               unsigned long long *__restrict__ out) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < V; u += gridDim.x * blockDim.x) {
        const uint32_t j = inv ? inv[u] : u;
#ifdef BINGO_VISIT_REC
        out[u] = visit[visit_slot(j)];
#else
        unsigned long long c = visit[visit_slot(j)];
        if (j < BINGO_VISIT_PAD)
            for (uint32_t r = 1; r < BINGO_VISIT_COPIES; r++) c += visit[visit_slot_r(j, r)];
        out[u] = c;
#endif
    }
}

extern "C" bingo_status bingo_visit_counts(bingo_graph *g, uint64_t *counts, int reset, uint32_t flags, void *stream) {
    if (!g) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    bingo_sq_quiesce(g, (cudaStream_t)stream);
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    const size_t bytes = sizeof(uint64_t) * g->V;
    if (counts && g->V) {
        unsigned long long *dst = reinterpret_cast<unsigned long long *>(counts);
        if (flags & BINGO_COUNTS_HOST) {   // gather into the walk staging buffer, then D2H
            if (g->wscratch_bytes < bytes) {
                bingo_dev_free(g, g->wscratch);
                g->wscratch = bingo_dev_alloc(g, bytes);
                g->wscratch_bytes = g->wscratch ? bytes : 0;
                if (!g->wscratch) return BINGO_E_NOMEM;
            }
            dst = (unsigned long long *)g->wscratch;
        }
        k_visit_gather<<<(unsigned)std::min<uint64_t>((g->V + 255) / 256, 148ull * 16), 256, 0, s>>>(g->V, g->inv,
                                                                                                   g->visit, dst);
        bingo_count_launch();
        e = cudaGetLastError();
        if (e == cudaSuccess && (flags & BINGO_COUNTS_HOST))
            e = cudaMemcpyAsync(counts, dst, bytes, cudaMemcpyDeviceToHost, s);
    }
    if (e == cudaSuccess && reset && g->V) e = cudaMemsetAsync(g->visit, 0, 8 * visit_words(g->V), s);
    if (e == cudaSuccess && (flags & BINGO_COUNTS_HOST)) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        g->poisoned = 1;
        return BINGO_E_CUDA;
    }
    return BINGO_OK;
}
