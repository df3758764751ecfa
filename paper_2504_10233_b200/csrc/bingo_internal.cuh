// bingo_internal.cuh -- device data layout and shared device helpers of libbingo.
//
// HBM layout.  Everything is structure-of-arrays inside
// a few pools addressed by OFFSETS (never raw pointers), so a pool can grow by
// reallocation + one memcpy without fix-ups.
//
// Walker-facing (read by every step):
//  thdr  [V]        ThinHdr, 8 B: bucket offset + group count n.  38 MB at
//                   4.7M vertices -> L2-resident (pinned with an access-policy
//                   window), so a step's first load is not a DRAM access.
//  bkt   pool       Bucket, 32 B (one 256-bit load), one per nonempty radix
//                   group in ascending k: alias bucket b = group b (A-13).  It
//                   holds lim = ceil(thr * 2^64 / T), the alias threshold
//                   rescaled so the walker's coin test needs no T (R-4'), the
//                   sampling view (kind, k, count/degree, member or adjacency
//                   base, or the one-element dst) of group b AND of its alias
//                   partner, so the inter-group stage (Eq.5) is one load.
//  mdst  pool       u32 dst of every member of a REGULAR/SPARSE group (the
//                   walker reads only this 4 B array: twice the entries per
//                   byte of L2 than an {index, dst} pair).  Group arrays start
//                   at 16 B units of 4 entries (u32 unit offsets).
//  arc   pool       uint2 {dst, bias} per arc; dense groups sample it directly
//                   (P:465).  Adjacency blocks are 4-arc (32 B) aligned.
// Update-side (canonical state, not read by walkers):
//  hdr   [V]        VHdr, 32 B: T, adjacency offset/capacity, bucket offset and
//                   capacity, degree d, n.
//  gcan  pool       GCan, 16 B per bucket: integer Vose threshold thr, |G_k|,
//                   member capacity or the one-element member's arc index.
//  midx  pool       u32 adjacency INDEX of every member (groups store
//                   neighbour indices), parallel to mdst.
//  arc_epoch pool   u32 epoch per arc (R-9).
//
// A walker step is thdr (L2) -> Bucket -> member (REGULAR/SPARSE), thdr ->
// Bucket (ONE), or thdr -> Bucket -> arc per dense attempt.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "bingo.h"

#include "float_bias.cuh"

namespace bingo {

enum : uint32_t { K_EMPTY = 0, K_ONE = 1, K_DENSE = 2, K_SPARSE = 3, K_REGULAR = 4 };

struct __align__(32) VHdr {
    uint64_t T;        // sum of biases = sum_k W(p_k)
    uint64_t adj_off;  // arc pool index of adj[0]
    uint32_t bkt_off;  // bucket pool index of bucket 0
    uint32_t d;        // out-degree (live arcs)
    uint8_t n;         // nonempty groups (alias buckets)
    uint8_t ncap;      // bucket capacity at bkt_off
    uint16_t pad;
    uint32_t adj_cap;  // arc capacity at adj_off
};
static_assert(sizeof(VHdr) == 32, "VHdr must be one sector");

struct __align__(8) ThinHdr {
    uint32_t bkt_off;  // bucket pool index of bucket 0
    uint8_t n;         // nonempty groups (0: dead end)
    uint8_t flags;     // bit 0: hot buckets, bit 1: hot member arrays (L2 evict_last)
    uint16_t pad1;
};
static_assert(sizeof(ThinHdr) == 8, "ThinHdr is 8 B");

// kk byte: bits 0..4 = k, bits 5..7 = kind.
// Group view (x, y): REGULAR/SPARSE (c, member offset in 16 B units);
// ONE (unused, dst of the member); DENSE (d, adjacency offset / 4).
struct __align__(32) Bucket {
    uint64_t lim;   // coin R (64-bit) < lim -> this group, else the alias partner
    uint32_t px, py;
    uint32_t ax, ay;
    uint8_t kk;     // this group
    uint8_t a_kk;   // alias partner
    uint8_t alias;  // alias partner bucket index
    uint8_t pad;
    uint32_t spare;
};
static_assert(sizeof(Bucket) == 32, "Bucket must be one sector");

struct __align__(16) GCan {
    uint64_t thr;   // integer Vose threshold in [0, T] (canonical, R-4)
    uint32_t c;     // |G_k|
    uint32_t aux;   // REGULAR/SPARSE: member capacity (entries); ONE: the member's arc index
};
static_assert(sizeof(GCan) == 16, "GCan is 16 B");

__host__ __device__ inline uint32_t kk_k(uint8_t kk) { return kk & 31u; }
__host__ __device__ inline uint32_t kk_kind(uint8_t kk) { return (uint32_t)kk >> 5; }
__host__ __device__ inline uint8_t make_kk(uint32_t k, uint32_t kind) { return (uint8_t)(k | (kind << 5)); }

// Eq.9 with the R-3 precedence (one-element first) and strict
// inequalities (R-3 boundaries).  bs: the all-regular baseline.
__host__ __device__ inline uint32_t classify(uint32_t c, uint32_t d, uint32_t alpha, uint32_t beta, bool bs) {
    if (c == 0) return K_EMPTY;
    if (bs) return K_REGULAR;
    if (c == 1) return K_ONE;
    if ((uint64_t)100 * c > (uint64_t)alpha * d) return K_DENSE;
    if ((uint64_t)100 * c < (uint64_t)beta * d) return K_SPARSE;
    return K_REGULAR;
}
__host__ __device__ inline bool is_list(uint32_t kind) { return kind == K_REGULAR || kind == K_SPARSE; }

// ---------------------------------------------------------------- Philox4x32-10
// Counter-based generator (R-1).  Written from the Salmon et al. round
// definition; pinned by the published known-answer vectors in the tests.
struct P4 { uint32_t x, y, z, w; };

__device__ __forceinline__ P4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return P4{c0, c1, c2, c3};
}

__device__ __forceinline__ uint64_t join64(uint32_t hi, uint32_t lo) { return ((uint64_t)hi << 32) | lo; }

// The draw of (outer attempt, inner attempt, tag) (R-1): counter word 2 = (outer << 16) + inner,
// word 3 = tag + ((outer >> 16) << 8), so node2vec outer attempts past 65535 never repeat a counter.
__device__ __forceinline__ P4 draw_oi(uint32_t w, uint32_t t, uint32_t outer, uint32_t inner, uint32_t tag,
                                      uint32_t k0, uint32_t k1) {
    return philox10(w, t, (outer << 16) + inner, tag + ((outer >> 16) << 8), k0, k1);
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() { return (1u << lane_id()) - 1u; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace bingo

// PPR visit counters, indexed by internal id: the hottest VISIT_PAD vertices (ids
// 0..VISIT_PAD-1 after the hot-first relabelling) get a 256 B slot each so their
// atomics spread over the L2 slices (packed, the top hubs' counters shared a few
// lines and serialised in one slice: c4 PPR 403 ms packed, 164 ms padded); the
// rest are packed u64 (hot-first, so within the TLB reach; padding 2^18 vertices
// was slower again, 252 ms).
// graphs with at least this many vertices are relabelled hot-first
#ifndef BINGO_RELABEL_MIN_V
#define BINGO_RELABEL_MIN_V (1u << 23)
#endif
#ifndef BINGO_VISIT_PAD
#define BINGO_VISIT_PAD 4096u
#endif
#ifndef BINGO_VISIT_STRIDE
#define BINGO_VISIT_STRIDE 32u   // u64 words per padded counter slot (256 B)
#endif
#ifdef BINGO_VISIT_REC
// A/B layout: every counter sits beside a copy of its vertex's thin header in one 16 B record
// {header, count}, so a PPR step's header read and its visit increment share a sector (and a
// page); the copies are refreshed from thdr at every PPR launch (k_visit_hdr)
__host__ __device__ inline uint64_t visit_rec(uint32_t j) {
    return j < BINGO_VISIT_PAD ? (uint64_t)j * BINGO_VISIT_STRIDE
                               : (uint64_t)BINGO_VISIT_PAD * BINGO_VISIT_STRIDE + 2ull * (j - BINGO_VISIT_PAD);
}
__host__ __device__ inline uint64_t visit_slot(uint32_t j) { return visit_rec(j) + 1; }
__host__ __device__ inline uint64_t visit_words(uint32_t V) { return visit_rec(V); }
#else
// A/B switch: the hottest vertices' counters split into BINGO_VISIT_COPIES sub-counters, each
// in its own 256 B slot of a different copy of the padded region (copy r of vertex j at
// (r * PAD + j) * STRIDE), a warp adding to copy (warp id mod COPIES) and the export summing
// them.  Measured slower (more counter lines in L2 beats less same-line serialisation), so 1.
// visit_slot(j) is copy 0, which every other writer uses.
#ifndef BINGO_VISIT_COPIES
#define BINGO_VISIT_COPIES 1u   // A/B (profiles/r02_visit_copies_ab.txt): 4 copies +5%, 8 +10%, 32 +51% walk time
#endif
__host__ __device__ inline uint64_t visit_slot_r(uint32_t j, uint32_t r) {
    return j < BINGO_VISIT_PAD ? ((uint64_t)r * BINGO_VISIT_PAD + j) * BINGO_VISIT_STRIDE
                               : (uint64_t)BINGO_VISIT_COPIES * BINGO_VISIT_PAD * BINGO_VISIT_STRIDE + (j - BINGO_VISIT_PAD);
}
__host__ __device__ inline uint64_t visit_slot(uint32_t j) { return visit_slot_r(j, 0); }
__host__ __device__ inline uint64_t visit_words(uint32_t V) {
    return V <= BINGO_VISIT_PAD ? (uint64_t)BINGO_VISIT_COPIES * BINGO_VISIT_PAD * BINGO_VISIT_STRIDE
                                : visit_slot(V);
}
#endif

// walker-claim counters: each walk launch takes the next of these slots (zeroed on its
// stream), so up to BINGO_WALK_SLOTS launches may run concurrently on one graph.
#define BINGO_WALK_SLOTS 64

// ---------------------------------------------------------------- graph object
struct bingo_graph {
    uint32_t V = 0;
    uint32_t alpha = 40, beta = 10, flags = 0;
    uint32_t epoch = 0;
    int poisoned = 0;
    uint64_t num_arcs = 0;

    // allocator
    void *(*alloc)(size_t, void *) = nullptr;
    void (*free_)(void *, void *) = nullptr;
    void *alloc_ctx = nullptr;
    double arc_slack = 0.25, member_slack = 0.25, pool_reserve = 0.1;

    uint32_t *perm = nullptr;          // [V] internal id -> external id (hot-first relabelling), or
    uint32_t *inv = nullptr;           // [V] external id -> internal id; both null: ids are external
    bingo::VHdr *hdr = nullptr;        // [V] indexed by internal id, like every per-vertex array
    uint2 *arc = nullptr;              // [arc_cap]
    uint32_t *arc_epoch = nullptr;     // [arc_cap]
    uint64_t *arc_dval = nullptr;      // [arc_cap] float mode: decimal part D of each arc (R-15/R-16)
    const uint64_t *cur_dins = nullptr; // float mode, during bingo_apply_updates_f64: D of each record
    uint64_t arc_cap = 0;
    bingo::ThinHdr *thdr = nullptr;    // [V]
    bingo::Bucket *bkt = nullptr;      // [bkt_cap]
    bingo::GCan *gcan = nullptr;       // [bkt_cap]
    uint64_t bkt_cap = 0;
    size_t persist_bytes = 0;          // L2 persisting set-aside granted to this process
    uint32_t hot_bkt_degree = 0xFFFFFFFFu; // d >= this: buckets loaded evict_last
    uint32_t hot_mem_degree = 0xFFFFFFFFu; // d >= this: member dsts loaded evict_last
    uint32_t *mdst = nullptr;          // [mem_cap] member dst (walker side)
    uint32_t *midx = nullptr;          // [mem_cap] member adjacency index (canonical)
    bool float_mode = false;
    uint32_t radix_log2 = 0;           // 0: Bingo base 2 with adaptive groups; b >= 1: base-2^b structure (radix.cu)
    uint64_t *rb_meta = nullptr;       // radix graphs: [V] first member unit, [V] (bucket cap << 32 | unit cap)
    bingo::DecRec *dec = nullptr;      // [V] decimal-group records (float mode)
    uint4 *dmem = nullptr;             // decimal members {idx, dst, D lo, D hi}
    uint64_t dmem_cap = 0;
    uint32_t *nbt = nullptr;           // [4 * arc_cap] neighbour hash sets (node2vec), optional
    uint64_t *nbo = nullptr;           // [V] hash-set base | log2 size << 48
    uint32_t *nbtomb = nullptr;        // [V] tombstones in each hash set (incremental updates)
    // hub delete index (update-side, derived; hub_index.cuh): per large vertex a
    // destination -> position multimap, so deletes locate their arcs without a scan
    uint64_t *hixo = nullptr;          // [V] table word offset | log2 entries << 48; 0 = none
    uint32_t *hixt = nullptr;          // [V] tombstones per table
    uint32_t *hix = nullptr;           // pool of tables, 2 words per entry {dst + 1 (0 empty), position}
    uint64_t hix_cap = 0;              // words; bump pointer counters[5]
    uint64_t *gixo = nullptr;          // [V] group index (group_index.cuh): table offset | log2 size << 48, 0 = none
    uint32_t *gixt = nullptr;          // [V] its tombstones
    uint32_t *gix = nullptr;           // table pool (zeroed words), bump pointer counters[6]
    uint64_t gix_cap = 0;              // words
    uint32_t gix_min = 1024;           // vertices with more arcs may get a table
    bool gix_full = false;             // the pool could not grow: no new tables
    uint32_t hix_min = 0xFFFFFFFFu;    // vertices with more arcs than this have tables
    uint64_t mem_cap = 0;              // entries
    unsigned long long *counters = nullptr;  // device bump pointers: [0] arc, [1] bkt, [2] mem units, [3..] scratch
    unsigned long long *visit = nullptr;     // [V] PPR visit counts
    unsigned int *visit32 = nullptr;         // BINGO_VISIT32 A/B: per-launch u32 counts, folded into visit
    unsigned long long *walk_ctr = nullptr;  // [BINGO_WALK_SLOTS] walker-claim counters (counters + 16)
    uint32_t walk_slot = 0;                  // next claim-counter slot (host, atomic increment)
    int *dev_flag = nullptr;                 // device error flag

    // update-side scratch (grown on demand)
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    void *hscratch = nullptr;                // pinned host staging
    size_t hscratch_bytes = 0;
    void *wscratch = nullptr;                // walk staging for HOST_OUTPUT
    size_t wscratch_bytes = 0;
    void *vscratch = nullptr;                // per-touched-vertex delete scratch
    size_t vscratch_bytes = 0;
    void *bscratch = nullptr;                // bulk-synchronous update: per-vertex state + chunk items
    size_t bscratch_bytes = 0;
    void *iscratch = nullptr;                // bulk-synchronous update: per-chunk-item counts
    size_t iscratch_bytes = 0;
    uint64_t isc_sel = 0, isc_grp = 0;       // chunk-item capacities carved from iscratch
    void *uhost = nullptr;                   // pinned staging of the one-sync update route
    uint32_t *vslot = nullptr;               // [V] per-vertex claim slots of the update segmentation (EMPTY between batches)
    bool radix_front = false;                // this batch re-segments with the radix sort (a segment too long)
    uint64_t n_sync_reruns = 0;              // one-sync batches re-run on the synchronous route
    uint32_t *fast_scr = nullptr;            // small-batch fast path scratch (device)
    cudaStream_t aux_stream = nullptr;       // side stream for hub mutations
    cudaStream_t copy_stream = nullptr;      // D2H of walk chunks (HOST_OUTPUT)
    cudaEvent_t ev_walk[2] = {nullptr, nullptr}, ev_copy[2] = {nullptr, nullptr};
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    void *fast_out_host = nullptr;           // mapped pinned status/stats of the fast path
    void *fast_out_dev = nullptr;
    // streaming queue (bingo_stream_update): mapped pinned ring + persistent kernel
    void *sq_host = nullptr;                 // StreamQ (update.cu), host view
    void *sq_dev = nullptr;                  // its device view
    bool sq_running = false;                 // a k_stream_upd generation may be live on sq_stream
    uint32_t sq_gen = 0, sq_seq = 0;         // last generation launched, next record number
    cudaStream_t sq_stream = nullptr;        // the stream it was launched on
    cudaEvent_t sq_ev = nullptr;             // recorded after the launch: completes when it exits
};

// stops a running streaming-queue kernel and orders `s` after its exit (update.cu); every
// entry point that touches the graph calls it first (the epoch fence of the streaming queue)
void bingo_sq_quiesce(bingo_graph *g, cudaStream_t s);
// arbitrary radix base (radix.cu)
bingo_status build_radix(bingo_graph *g, const bingo_build_desc *desc, uint32_t b, cudaStream_t s);
bingo_status launch_walk_radix(bingo_graph *g, const bingo_walk_desc *desc, const uint32_t *starts, uint32_t W,
                               uint32_t *paths, uint32_t *lengths, cudaStream_t s);
bingo_status export_radix(bingo_graph *g, uint8_t *buf, size_t cap, size_t *size_out, cudaStream_t s);
void bingo_sq_release(bingo_graph *g);

// process-wide count of kernel launches issued by libbingo (api.cu)
void bingo_count_launch(unsigned n = 1);

// allocation helpers (api.cu)
void *bingo_dev_alloc(bingo_graph *g, size_t bytes);
void bingo_dev_free(bingo_graph *g, void *p);
