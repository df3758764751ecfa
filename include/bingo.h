/*
 * bingo.h -- C-ABI of the B200-native Bingo hot path (libbingo.so).
 *
 * Bingo (arXiv 2504.10233) samples the next hop of a random walk from a
 * per-vertex radix factorisation of integer edge biases: every bias w_i is
 * split into its set bits (Eq.3), each set bit k puts the edge in
 * group k whose weight is W(p_k) = c_k 2^k (Eq.4), a walker picks
 * a group through an alias table over the group weights (Eq.5) and
 * then an edge uniformly inside the group (Eq.6).  Groups use the
 * dense / one-element / sparse / regular layouts of Eq.9.
 * Batched insert/delete keeps all of it consistent between walk batches
 * (S5.2).  "P:n" = line n of PAPER.md; "R-n" = reading n of
 * DESIGN.md section 3 (the canonical semantics where the paper is silent).
 *
 * Conventions for every call:
 *  - Pointers are DEVICE pointers unless the call's flags say HOST.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Work is enqueued on it; calls that must report sizes or
 *    statistics synchronise that stream before returning (stated per call).
 *  - Caller-owned buffers must stay valid until the stream passes the call.
 *  - No exception crosses the ABI; every call returns a bingo_status.
 *  - After a CUDA error the graph is poisoned: every later call on it
 *    returns BINGO_E_STATE (bingo_destroy still frees it).
 *  - Vertex ids crossing the ABI (CSR, starts, update records, paths, visit
 *    counts, exports) are always the caller's; an internal relabelling
 *    (large graphs) is invisible.
 *  - Concurrency: one writer or many readers per graph; the caller orders
 *    bingo_apply_updates against bingo_walk on one stream (P:523 (ii)).
 */
#ifndef BINGO_H
#define BINGO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bingo_graph bingo_graph; /* opaque; owns all of its HBM */

typedef enum {
    BINGO_OK = 0,
    BINGO_E_INVAL = 1,    /* bad argument / invalid batch record (nothing mutated)   */
    BINGO_E_NOMEM = 2,    /* device memory exhausted (nothing mutated)              */
    BINGO_E_CUDA = 3,     /* CUDA runtime error (graph poisoned)                    */
    BINGO_E_OVERFLOW = 4, /* n * T >= 2^64 or degree >= 2^32 - 1 (nothing mutated)  */
    BINGO_E_STATE = 5     /* graph poisoned by an earlier CUDA error                */
} bingo_status;

/* Group kinds of Eq.9 as they appear in exports (R-3). */
enum { BINGO_KIND_EMPTY = 0, BINGO_KIND_ONE = 1, BINGO_KIND_DENSE = 2, BINGO_KIND_SPARSE = 3,
       BINGO_KIND_REGULAR = 4 };

/* ---------------------------------------------------------------------------
 * bingo_build -- sampling-space construction (S4.1 "Sampling space
 * construction"; Eq.9 kinds P:436-492; inter-group alias P:292).
 *
 * Input is a CSR snapshot in DEVICE memory:
 *   row_offsets [V+1] u64, non-decreasing, row_offsets[0] = 0;
 *   dst [A] u32 < V; bias [A] u32 >= 1.  CSR order is the canonical adjacency
 *   order (R-2); every arc gets epoch 0.
 * alpha_pct / beta_pct: Eq.9 thresholds (paper: 40 / 10).
 * flags: BINGO_BUILD_BS_MODE forces the paper's all-regular baseline (
 *   alpha = 100, beta = 0, no one-element groups).  BINGO_BUILD_NEIGHBOR_INDEX
 *   keeps a per-vertex hash set of destination ids (derived state, rebuilt for
 *   touched vertices by every update) so node2vec's "arc prev -> v exists?"
 *   test (Eq.1, A-17) is one probe instead of a scan of adj(prev).
 *   BINGO_BUILD_FLOAT_BIAS takes real biases from bias_f64 (S4.3):
 *   per vertex lambda = the smallest 10^j (j <= 9) with W_D/(W_I+W_D) < 1/d
 *   (P:377), integer parts floor(w lambda) form the radix groups, fractional
 *   parts (fixed point, 2^-52) form the decimal group sampled by rejection;
 *   sampled probabilities are within 1e-6 relative of w/sum(w) (R-15).
 *   lambda stays fixed per vertex after the build; updates of float
 *   graphs go through bingo_apply_updates_f64 (R-16).  Exports append a
 *   per-vertex decimal trailer (R-11).
 *   Layout (a performance choice only, invisible in every result and export):
 *   by default the pools are laid out hot-first (descending out-degree) and,
 *   for V >= 2^23, the vertices are also relabelled internally by that order
 *   (BINGO_BUILD_RELABEL forces it); BINGO_BUILD_ID_LAYOUT keeps vertex-id
 *   order for everything.
 * arc_slack / member_slack: fraction of extra per-vertex capacity reserved
 *   for growth (Hornet-style dynamic arrays + memory pool);
 *   pool_reserve: extra fraction of every pool for relocations.
 * alloc/free/alloc_ctx: optional device allocator (e.g. PyTorch's caching
 *   allocator); NULL -> cudaMalloc/cudaFree.
 * Errors: EINVAL (V = 0 with A > 0, dst >= V, bias = 0, bad offsets: checked
 *   on the device), EOVERFLOW (a vertex with n*T >= 2^64 or d >= 2^32-1),
 *   NOMEM, CUDA.  Synchronises `stream`.  *out receives the new graph.
 * ------------------------------------------------------------------------- */
#define BINGO_BUILD_BS_MODE 1u
#define BINGO_BUILD_NEIGHBOR_INDEX 2u /* keep per-vertex neighbour hash sets: O(1) node2vec distance test */
#define BINGO_BUILD_FLOAT_BIAS 4u     /* biases come from bias_f64 (S4.3 floating-point extension, R-15) */
#define BINGO_BUILD_ID_LAYOUT 8u      /* pools in vertex-id order (default: hot-first) */
#define BINGO_BUILD_RELABEL 16u       /* relabel vertices hot-first internally at any V (default: V >= 2^23) */
/* Arbitrary radix base B = 2^b, b in [1, 5] (reading R-17): group B^i holds
 * the arcs whose base-B digit i is nonzero, split into subgroups by digit value with an
 * inter-subgroup alias; walks take group -> subgroup -> member.  Every subgroup a member list,
 * vertex-id layout: DeepWalk and PPR walks (step-major paths), bingo_export in the radix dump
 * format (R-18), bingo_visit_counts, and bingo_apply_updates (reading R-19: the adjacency as
 * below, then each touched vertex's nested structure rebuilt from it; statistics without kind
 * transitions; EOVERFLOW when (T + inserted bias) * ceil(32 / b) >= 2^64 or d + inserts >=
 * 2^32 - 1); the other calls (node2vec, float biases, streaming queue, traces, partitions)
 * return EINVAL.  0 (default): the paper's base-2 Bingo with Eq.9 groups. */
#define BINGO_BUILD_RADIX_LOG2(b) ((uint32_t)(b) << 8)
#define BINGO_BUILD_RADIX_MASK 0xF00u

typedef void *(*bingo_alloc_fn)(size_t bytes, void *ctx);
typedef void (*bingo_free_fn)(void *ptr, void *ctx);

typedef struct {
    uint32_t num_vertices;
    uint64_t num_arcs;
    const uint64_t *row_offsets; /* device [V+1] */
    const uint32_t *dst;         /* device [A]   */
    const uint32_t *bias;        /* device [A]   */
    uint32_t alpha_pct, beta_pct;
    uint32_t flags;
    double arc_slack;    /* e.g. 0.25 */
    double member_slack; /* e.g. 0.25 */
    double pool_reserve; /* e.g. 0.10 */
    bingo_alloc_fn alloc;
    bingo_free_fn free;
    void *alloc_ctx;
    const double *bias_f64; /* device [A], > 0 and finite; used with BINGO_BUILD_FLOAT_BIAS */
} bingo_build_desc;

bingo_status bingo_build(const bingo_build_desc *desc, void *stream, bingo_graph **out);

/* Frees every device buffer the graph owns.  Safe on NULL. */
void bingo_destroy(bingo_graph *g);

/* ---------------------------------------------------------------------------
 * bingo_apply_updates -- batched edge insert/delete (S5.2; single
 * records are the streaming case of S4.2).
 *
 * batch: n arc-level records {op, src, dst, bias}, op 0 = insert (bias >= 1),
 *   op 1 = delete (bias ignored).  An undirected edge update is two records.
 *   DEVICE pointer, or HOST pointer with BINGO_UPD_HOST_BATCH (the library
 *   copies it H2D on `stream`).
 * Semantics (R-7 .. R-10): epoch e = number of successful calls so far + 1.
 *   Per touched vertex: all inserts in batch order (append; groups that are
 *   REGULAR/SPARSE before the batch append the new index), then all deletes
 *   (each removes the live instance of (src,dst) with the smallest
 *   (epoch, position) not yet taken; two-phase delete-and-swap,
 *   P:514-516, on groups and adjacency, renaming moved indices), then one
 *   rebuild (Eq.9 reclassification, member materialisation on kind change,
 *   integer Vose alias).  Untouched vertices are not modified.
 *   A delete with no live instance is counted in missing_deletes, not an
 *   error (R-8).
 * Errors (nothing is mutated, epoch unchanged): EINVAL for op > 1, src or
 *   dst >= V, an insert with bias 0, or a float-bias graph (use
 *   bingo_apply_updates_f64); EOVERFLOW if for a touched vertex
 *   (T + inserted bias) * popc(mask | inserted biases) >= 2^64 or
 *   d + inserts >= 2^32 - 1; NOMEM if the pools cannot grow.
 * stats_or_null (HOST) receives counts and the 5x5 kind-transition matrix
 *   [old kind][new kind] over every (touched vertex, k) with a nonempty side
 *   (cf. Table trans).  Synchronises `stream`.
 * ------------------------------------------------------------------------- */
#define BINGO_UPD_HOST_BATCH 1u

typedef struct {
    uint32_t op, src, dst, bias;
} bingo_update;

typedef struct {
    uint64_t inserted, deleted, missing_deletes, touched_vertices;
    uint64_t kind_transitions[5][5];
    uint64_t epoch;
} bingo_update_stats;

bingo_status bingo_apply_updates(bingo_graph *g, const bingo_update *batch, uint64_t n, uint32_t flags,
                                 bingo_update_stats *stats_or_null, void *stream);

/* ---------------------------------------------------------------------------
 * bingo_apply_updates_f64 -- the same batched update for a graph built with
 * BINGO_BUILD_FLOAT_BIAS (floating-point biases, S4.3-4.4 P:344-377; R-16).
 *
 * batch: as for bingo_apply_updates; the records' bias fields are ignored.
 * bias_f64: n doubles, same memory space as batch (HOST with
 *   BINGO_UPD_HOST_BATCH, else DEVICE); entry i is the real bias of insert
 *   record i (> 0, finite, <= 1e300), ignored for deletes.
 * Semantics: each vertex keeps the lambda chosen at its build.  An
 *   insert (u, v, w) computes s = fl(w * lambda_u) (IEEE binary64), appends an
 *   arc with radix bias I = floor(s) (I = 0 is allowed: the arc joins no radix
 *   group) and decimal part D = floor((s - I) * 2^52); inserts, deletes and the
 *   radix rebuild are those of bingo_apply_updates; then every touched
 *   vertex's decimal group is rebuilt from its live arcs (ascending index),
 *   with thrD = floor(W_D 2^64 / (W_I 2^52 + W_D)) and flag bit 0 set iff the
 *   P:377 constraint (d-1) W_D < W_I 2^52 no longer holds.
 * Errors (nothing mutated): EINVAL as bingo_apply_updates, for a non-float
 *   graph, or a bias that is not > 0 and finite; EOVERFLOW if some s >= 2^32
 *   or as bingo_apply_updates; NOMEM.  Synchronises `stream`.
 * ------------------------------------------------------------------------- */
bingo_status bingo_apply_updates_f64(bingo_graph *g, const bingo_update *batch, const double *bias_f64, uint64_t n,
                                     uint32_t flags, bingo_update_stats *stats_or_null, void *stream);

/* bingo_stream_update -- one arc record applied through the persistent streaming queue
 * (streaming updates, P:126 / P:316-336).  Same semantics, statistics, epoch and
 * errors as bingo_apply_updates(g, rec, 1, BINGO_UPD_HOST_BATCH, ...) -- rec is HOST memory,
 * the call returns when the record is applied -- but without a kernel launch per record: a
 * one-warp kernel stays resident on `stream` and polls a ring in mapped pinned host memory;
 * its results come back the same way.  It exits when any other call on the graph needs the
 * graph (that call is ordered after it: the epoch fence), after 2 ms without a record (a
 * caller synchronising `stream` waits at most that long), or on a record that needs pool
 * growth or touches a vertex above 8192 arcs (that record then takes the batched pipeline).
 * Integer-bias graphs only (EINVAL for float graphs). */
bingo_status bingo_stream_update(bingo_graph *g, const bingo_update *rec, bingo_update_stats *stats_or_null,
                                 void *stream);

/* ---------------------------------------------------------------------------
 * bingo_walk -- the batched walker step (S3 "random walk query", P:215;
 * Eq.5/Eq.6 two-stage sample; dense rejection P:465; applications S6.1
 * P:535-536).
 *
 * desc->app: BINGO_DEEPWALK: exactly `length` steps (path of length+1
 *   vertices, R-13);  BINGO_NODE2VEC: second-order walk, first step
 *   first-order, later steps propose with the first-order sampler and accept
 *   with f(prev, v) / f_max, f = 1/p, 1, 1/q by distance 0/1/2 (Eq.1,
 *   P:160-170; KnightKing rejection);  BINGO_PPR: after every step stop
 *   with probability stop_num/stop_den, `length` caps the steps
 *   (0xFFFFFFFF = no cap); visit counts (start included) accumulate in the
 *   graph (read them with bingo_visit_counts).
 * Walker i (0 <= i < num_walkers) has global id first_walker_id + i and
 *   starts at starts[i], or at (first_walker_id + i) mod V if starts is NULL
 *   (one walker per vertex).  Its randomness is Philox4x32-10 keyed by
 *   seed with counter (walker id, step, (outer << 16) + inner,
 *   tag + ((outer >> 16) << 8)) (R-1), so a sharded run (first_walker_id)
 *   reproduces the unsharded one bit for bit, and node2vec's rejection
 *   attempts never repeat a counter (expected proposals per step <= f_max/f_min).
 * A walker at a vertex of out-degree 0 stops (truncation).
 * paths_or_null: step-major u32 [(length+1) x num_walkers], entry
 *   [t * num_walkers + i] = vertex after t steps; 0xFFFFFFFF after truncation.
 *   With BINGO_WALK_WALKER_MAJOR the layout is [num_walkers x (length+1)],
 *   entry [i * (length+1) + t] (one contiguous walk per walker).
 *   Required NULL for PPR without a cap.  lengths_or_null: u32 [num_walkers]
 *   steps actually taken.  DEVICE pointers, or HOST with
 *   BINGO_WALK_HOST_OUTPUT (the library stages through device scratch and
 *   copies D2H on `stream`; `starts` is then HOST too).
 * Errors: EINVAL (bad app / p, q <= 0 / stop_den == 0 / NULL paths with
 *   no cap / node2vec with a ratio f/f_max < 2^-64, whose class could never
 *   be accepted).  Asynchronous unless HOST_OUTPUT (then synchronises `stream`).
 * ------------------------------------------------------------------------- */
enum { BINGO_DEEPWALK = 0, BINGO_NODE2VEC = 1, BINGO_PPR = 2 };
#define BINGO_WALK_HOST_OUTPUT 1u
#define BINGO_WALK_WALKER_MAJOR 2u /* paths walker-major: entry [i * (length+1) + t] */
#define BINGO_NO_CAP 0xFFFFFFFFu

typedef struct {
    uint32_t app;
    uint32_t length;
    double p, q;                 /* node2vec hyper-parameters (0.5, 2) */
    uint32_t stop_num, stop_den; /* PPR termination probability (1/80) */
    uint64_t seed;
    uint32_t first_walker_id;
    uint32_t flags;
} bingo_walk_desc;

bingo_status bingo_walk(bingo_graph *g, const bingo_walk_desc *desc, const uint32_t *starts_or_null,
                        uint32_t num_walkers, uint32_t *paths_or_null, uint32_t *lengths_or_null,
                        void *stream);

/* ---------------------------------------------------------------------------
 * bingo_visit_counts -- PPR visit frequencies ("use the visit frequency
 * of each vertex"): u64 [V] counts accumulated by BINGO_PPR walks since the
 * last reset (start vertices included, R-15).  counts: DEVICE [V] (or HOST
 * with BINGO_COUNTS_HOST; then synchronises).  reset != 0 zeroes the graph's
 * counters after the copy (counts may be NULL to only reset).
 * ------------------------------------------------------------------------- */
#define BINGO_COUNTS_HOST 1u
bingo_status bingo_visit_counts(bingo_graph *g, uint64_t *counts, int reset, uint32_t flags, void *stream);

/* ---------------------------------------------------------------------------
 * Inspection (parity and reporting; not on the hot path).
 * bingo_export: canonical dump (R-11) into a HOST buffer: for each vertex u
 *   ascending: u32 d; d x {u32 dst, u32 bias, u32 epoch}; u32 n; n x {u32 k,
 *   u32 c, u32 kind, u64 thr, u32 alias, REG/SPARSE: c x u32 member index,
 *   ONE: u32 member index}; u64 T.  Little-endian, unaligned.  *size_out
 *   receives the byte count; nothing is written if host_buf is NULL or cap is
 *   too small.  Synchronises `stream`.
 * bingo_digests: per-vertex FNV-1a-64 of the same per-vertex bytes, computed
 *   on the device into DEVICE u64 [V].
 * bingo_info: sizes and pool usage (HOST struct).
 * ------------------------------------------------------------------------- */
bingo_status bingo_export(bingo_graph *g, uint8_t *host_buf, size_t cap, size_t *size_out, void *stream);
bingo_status bingo_digests(bingo_graph *g, uint64_t *digests, void *stream);

typedef struct {
    uint32_t num_vertices;
    uint32_t epoch;
    uint64_t num_arcs;
    uint64_t arc_pool_used, arc_pool_cap;       /* arcs   */
    uint64_t bucket_pool_used, bucket_pool_cap; /* 32 B buckets */
    uint64_t member_pool_used, member_pool_cap; /* 8 B entries */
    uint64_t device_bytes;
    uint64_t kernel_launches;  /* process-wide count of libbingo kernel launches so far */
    uint64_t l2_persist_bytes; /* L2 persisting set-aside in effect (walker hot set) */
    uint64_t hot_degree;       /* low 32 bits: degree from which buckets are L2 evict_last; high 32: member arrays */
    uint64_t update_reruns;    /* batches of the one-sync update route that found a pool or scratch short,
                                  mutated nothing, and were re-applied on the synchronous route */
} bingo_info;
bingo_status bingo_get_info(bingo_graph *g, bingo_info *info, void *stream);

/* bingo_walk_profile: bingo_walk (DEVICE buffers only) that also counts, into
 * counters_host[8] (HOST u64), the records every walker step loaded:
 * [0] steps taken, [1] vertex headers, [2] alias buckets, [3] group members,
 * [4] adjacency arcs (dense attempts), [5] node2vec probe sectors, [6] PPR
 * visit-count increments, [7] walkers.  Same walks as bingo_walk (bit for
 * bit).  Used to compute the algorithmic bytes behind the roofline.
 * Synchronises `stream`. */
bingo_status bingo_walk_profile(bingo_graph *g, const bingo_walk_desc *desc, const uint32_t *starts_or_null,
                                uint32_t num_walkers, uint32_t *paths_or_null, uint32_t *lengths_or_null,
                                uint64_t *counters_host, void *stream);

/* bingo_walk_partition -- one round of the 1-D partitioned walk with walker transfer
 * (SURVEY f3).  The graph g is this rank's partition: built over the full vertex
 * id space with only the arcs of the vertices it owns, the external ids in
 * [bounds[me], bounds[me + 1]) (bounds: DEVICE u32 [parts + 1], ascending, bounds[0] = 0).
 * inbox: DEVICE records {walker id, current vertex (external id), steps taken, flags bit 0 =
 * fresh} of n_in walkers standing on owned vertices; a fresh walker writes path entry 0 and
 * (PPR) counts its start.  Each walker takes steps exactly as bingo_walk would (same
 * counters, same results) while its vertex is owned; one that steps onto another rank's
 * vertex is appended to outbox[owner * out_cap + k] (DEVICE, 16 B records, out_cap >= n_in;
 * out_count[owner] DEVICE u32, zeroed by the caller, counts them) with its steps so far.
 * Paths / lengths (DEVICE, layouts of bingo_walk for num_walkers walkers, index = walker id -
 * desc->first_walker_id) receive the entries of the steps taken here; the rank where a
 * walker finishes writes its length and sentinels.  PPR visit counts accumulate on the rank
 * that took the step (sum them over ranks).  DeepWalk and PPR, integer biases.
 * *finished_host: walkers that finished in this round.  Synchronises `stream`. */
bingo_status bingo_walk_partition(bingo_graph *g, const bingo_walk_desc *desc, uint32_t num_walkers,
                                  const uint32_t *bounds, uint32_t parts, uint32_t me, const void *inbox,
                                  uint32_t n_in, void *outbox, uint64_t out_cap, uint32_t *out_count,
                                  uint32_t *paths_or_null, uint32_t *lengths_or_null, uint64_t *finished_host,
                                  void *stream);

/* bingo_walk_trace / bingo_walk_replay -- measurement only (the walk's roofline,
 * DESIGN.md 6.1): the "achievable random-gather bandwidth" for the walk's own footprint and
 * skew.  bingo_walk_trace runs the same walks as bingo_walk (DeepWalk or PPR, integer
 * biases, step-major, no paths; counters_host as bingo_walk_profile) and records for every
 * step t < lengths[i] of walker i one 16 B record of the loads it made at
 * trace[rec_off[i] + t]: {vertex whose header was read, bucket index | keep << 31, member
 * or dense attempt 0, dense attempt 1} (intra-group codes: 0xFFFFFFFF none, else
 * arc << 31 | keep << 30 | 16 B member granule or 32 B arc sector).
 * rec_off: DEVICE u64 [num_walkers + 1], the exclusive prefix sum of the walkers' lengths (from an earlier launch with the same desc);
 * trace: DEVICE, 16 B x n_records.  EINVAL for node2vec, float graphs, flags, arc or
 * member pools of 2^32 entries or bucket pools of 2^31.  Synchronises `stream`.
 * bingo_walk_replay issues exactly the recorded loads (same addresses, widths, cache
 * policies and fetch hints), one walker per thread like the walk but with 2^(flags & 3)
 * steps' loads in flight and no dependency between them, on (flags >> 8 & 255 or 8) x SMs
 * blocks of 256 threads.  counts_host[4] (HOST u64): headers, buckets, members, arcs
 * loaded.  Time it with events on `stream`; synchronises `stream`. */
bingo_status bingo_walk_trace(bingo_graph *g, const bingo_walk_desc *desc, const uint32_t *starts_or_null,
                              uint32_t num_walkers, const uint64_t *rec_off, void *trace, uint64_t n_records,
                              uint64_t *counters_host, void *stream);
bingo_status bingo_walk_replay(bingo_graph *g, const void *trace, const uint64_t *rec_off, uint32_t num_walkers,
                               uint32_t flags, uint64_t *counts_host, void *stream);

/* ---------------------------------------------------------------------------
 * bingo_export_vertices / bingo_import_vertices -- per-vertex state exchange between
 * replicas (replicated regime): sharded update application.  Updates are
 * independent per source vertex, so with P replicas rank r applies (with
 * bingo_apply_updates) only the records whose source it owns, exports the post-batch state
 * of those touched vertices, and imports every other rank's exports; every replica then
 * holds the canonical state of the single-graph run (R-11: adjacency with epochs, groups,
 * kinds, integer-Vose tables, member order, T).
 *
 * export: ids = DEVICE array of n vertex ids (the caller's ids, < V, each at most once).
 *   offsets (DEVICE, n + 1 u64) receives the record offsets in u32 words, offsets[n] the
 *   total, also written to *words_out (HOST).  buf == NULL: sizes only.  Else buf (DEVICE,
 *   cap_words u32) receives the records: u, d, n, T (2 words), d x (dst, bias, epoch), then
 *   per nonempty group k, kind, c, thr (2 words), alias and its payload (list groups: the c
 *   member adjacency indices in list order; one-element groups: the arc index), all ids
 *   internal (replicas share the build's relabelling).  Errors: EINVAL (an id >= V, a
 *   float-bias, radix-base or neighbour-index graph), EOVERFLOW (cap_words too small).
 * import: buf / offsets (DEVICE) as an export of a replica of the same graph produced them
 *   (n records).  Each record's vertex is rewritten in place where its adjacency, buckets or
 *   a same-k member list fit, else in fresh pool space; its hub / group indices are dropped
 *   (rebuilt lazily).  The epoch does not change.  Errors: EINVAL as above, NOMEM if a pool
 *   cannot grow (nothing written).  Both synchronise `stream`.
 * ------------------------------------------------------------------------- */
bingo_status bingo_export_vertices(bingo_graph *g, const uint32_t *ids, uint32_t n, uint32_t *buf,
                                   uint64_t cap_words, uint64_t *offsets, uint64_t *words_out, void *stream);
bingo_status bingo_import_vertices(bingo_graph *g, const uint32_t *buf, const uint64_t *offsets, uint32_t n,
                                   void *stream);

const char *bingo_status_str(bingo_status s);

#ifdef __cplusplus
}
#endif
#endif /* BINGO_H */
