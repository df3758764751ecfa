/*
 * oracle/bingo_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle of the Bingo hot path
 * (arXiv 2504.10233, "Bingo: Radix-based Bias Factorization for Random Walk on
 * Dynamic Graphs").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product
 * path (paper_2504_10233_b200/) never links, imports or calls it, and this
 * file shares no code, header, table or helper with the CUDA path.
 *
 * Citations: "P:n" = line n of PAPER.md (the paper's LaTeX source);
 * "R-n" = reading n in DESIGN.md section 3 (the canonical semantics we fix
 * where the paper is silent; both sides implement them independently).
 *
 * Every function below follows the paper's definitions in the paper's order:
 *   Eq.3  D(w_i) = {2^k : w_i AND 2^k != 0}
 *   Eq.4  W(p_k) = sum_i (w_i AND 2^k) = c_k * 2^k
 *   Eq.5  P(p_k) = W(p_k) / sum_j W(p_j)  -- alias table
 *   Eq.6  P(v_i | p_k) = uniform over the members of group k
 *   Eq.9  dense / one-element / sparse / regular classification
 *   S4.2  insertion (append), deletion (swap with tail)
 *   S5.2  batched: per vertex insert -> delete -> rebuild
 *   Eq.1  node2vec factor; KnightKing rejection
 *   S6.1  DeepWalk length 80, PPR termination 1/80
 *
 * Parity status: every function here is pinned by a -m "not gpu" test in
 * tests/test_oracle_*.py ("Pins").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define O_EMPTY 0u
#define O_ONE 1u
#define O_DENSE 2u
#define O_SPARSE 3u
#define O_REGULAR 4u

#define O_FLAG_BS_MODE 1u /* R-3: the paper's "regular format for all groups" baseline */

#define O_OK 0
#define O_EINVAL 1
#define O_ENOMEM 2
#define O_EOVERFLOW 4

#define O_NONE 0xFFFFFFFFu

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11).  R-1: the paper is silent on  */
/* the RNG; we fix a counter-based generator so walks are reproducible */
/* ------------------------------------------------------------------ */
void ora_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* floor(a * b / 2^64): maps a uniform 64-bit draw a onto [0, b)  (R-1) */
static uint64_t mulhi64(uint64_t a, uint64_t b)
{
    return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
}

/* ------------------------------------------------------------------ */
/* Graph state (R-2): per vertex an adjacency list of (dst, bias,      */
/* epoch) and its nonempty radix groups in ascending k.  Bucket b of   */
/* the inter-group alias table is group b of that list (A-13).         */
/* ------------------------------------------------------------------ */
typedef struct {
    uint32_t dst, bias, epoch;
    uint64_t dval;     /* float mode: D = floor(frac(w lambda) 2^52) of this arc (R-15); 0 otherwise */
} o_arc;

typedef struct {
    uint32_t k;        /* radix position: the group holds sub-bias 2^k */
    uint32_t c;        /* |G_k| = number of arcs whose bias has bit k   */
    uint32_t kind;     /* Eq.9 kind                                     */
    uint32_t one;      /* ONE: the member's adjacency index             */
    uint32_t *mem;     /* REGULAR/SPARSE: member adjacency indices      */
    uint32_t cap;
    uint64_t thr;      /* alias bucket threshold (integer Vose, R-4)    */
    uint32_t alias;    /* alias bucket partner                          */
} o_group;

typedef struct {
    uint32_t d, cap;
    o_arc *adj;
    uint32_t n;        /* number of nonempty groups */
    o_group *grp;      /* n groups, ascending k     */
    uint64_t T;        /* sum_k W(p_k) = sum_i w_i  */
    /* floating-point bias mode (S4.3; reading R-15) */
    uint32_t lam;      /* lambda = 10^lam                                   */
    uint32_t fflags;   /* bit 0: constraint unmet, bit 1: integer part empty */
    uint32_t dcnt;     /* decimal group: arcs with a nonzero decimal part   */
    uint32_t *didx;    /* their adjacency indices, ascending                */
    uint64_t *dval;    /* D_i = floor(frac(w_i lambda) 2^52)                */
    uint64_t dmax;
    uint64_t thrD;     /* decimal iff 64-bit draw < thrD                    */
} o_vertex;

typedef struct ora_graph {
    uint32_t V;
    int float_mode;
    /* lazy mode (test infrastructure for BASELINE-scale parity): a vertex is built
     * from the caller's CSR on its first access; the result is the same as an
     * eager build, only untouched vertices are never materialised */
    int lazy;
    uint8_t *built;
    const uint64_t *lro;
    const uint32_t *ldst, *lbias;
    uint32_t alpha, beta, flags;
    uint32_t epoch;
    o_vertex *v;
} ora_graph;

static void *xrealloc(void *p, size_t n)
{
    void *q = realloc(p, n ? n : 1);
    if (!q) abort();
    return q;
}

static void build_vertex(const ora_graph *G, o_vertex *x);
static int g_dump_float = 0;
typedef struct o_out_s o_out;
static void dump_vertex(const o_vertex *x, o_out *o);

/* vertex accessor: materialises lazily-built vertices on first use.
 * built[u]: 0 = not built, 1 = being built by one thread, 2 = built.  The thread that
 * moves it 0 -> 1 builds the vertex and publishes it with a release store of 2; every
 * reader acquires 2 before touching the vertex (other builders of the same vertex wait),
 * so distinct vertices build in parallel and no read races a write. */
static o_vertex *vx(const ora_graph *Gc, uint32_t u)
{
    ora_graph *G = (ora_graph *)Gc;
    o_vertex *x = &G->v[u];
    if (!G->lazy || __atomic_load_n(&G->built[u], __ATOMIC_ACQUIRE) == 2) return x;
    uint8_t expect = 0;
    if (__atomic_compare_exchange_n(&G->built[u], &expect, 1, 0, __ATOMIC_ACQ_REL, __ATOMIC_ACQUIRE)) {
        x->d = (uint32_t)(G->lro[u + 1] - G->lro[u]);
        x->cap = x->d;
        x->adj = (o_arc *)malloc(sizeof(o_arc) * (x->cap ? x->cap : 1));
        for (uint32_t i = 0; i < x->d; i++) {
            x->adj[i].dst = G->ldst[G->lro[u] + i];
            x->adj[i].bias = G->lbias[G->lro[u] + i];
            x->adj[i].epoch = 0;
            x->adj[i].dval = 0;
        }
        build_vertex(G, x);
        __atomic_store_n(&G->built[u], 2, __ATOMIC_RELEASE);
    } else {
        while (__atomic_load_n(&G->built[u], __ATOMIC_ACQUIRE) != 2) {
        }
    }
    return x;
}

/* ---------------- Eq.9 classification (R-3) ---------------- */
uint32_t ora_classify(uint32_t c, uint32_t d, uint32_t alpha, uint32_t beta, uint32_t flags)
{
    if (c == 0) return O_EMPTY;
    if (flags & O_FLAG_BS_MODE) return O_REGULAR;              /* all-regular baseline */
    if (c == 1) return O_ONE;                                  /* |G| = 1 (checked first, R-3) */
    if ((uint64_t)100 * c > (uint64_t)alpha * d) return O_DENSE;  /* |G|/d > alpha% */
    if ((uint64_t)100 * c < (uint64_t)beta * d) return O_SPARSE;  /* |G|/d < beta%  */
    return O_REGULAR;
}

/* ---------------- integer Vose alias over the group weights (R-4) ----
 * s_b = n * W_b, T = sum W.  While a small (s < T) and a large (s >= T)
 * unassigned bucket exist: l = lowest small, h = lowest large,
 * thr[l] = s_l, alias[l] = h, s_h -= T - s_l.  Remaining buckets: thr = T,
 * alias = self.  Exact: no rounding anywhere. */
void ora_alias_build(uint32_t n, const uint64_t *W, uint64_t *thr, uint32_t *alias)
{
    uint64_t T = 0;
    uint64_t s[32];
    int assigned[32];
    for (uint32_t b = 0; b < n; b++) T += W[b];
    for (uint32_t b = 0; b < n; b++) {
        s[b] = (uint64_t)n * W[b];
        assigned[b] = 0;
    }
    for (;;) {
        int l = -1, h = -1;
        for (uint32_t b = 0; b < n; b++)
            if (!assigned[b] && s[b] < T) { l = (int)b; break; }
        for (uint32_t b = 0; b < n; b++)
            if (!assigned[b] && s[b] >= T) { h = (int)b; break; }
        if (l < 0 || h < 0) break;
        thr[l] = s[l];
        alias[l] = (uint32_t)h;
        assigned[l] = 1;
        s[h] -= T - s[l];
    }
    for (uint32_t b = 0; b < n; b++)
        if (!assigned[b]) { thr[b] = T; alias[b] = b; }
}

/* Rebuild the group list of x from per-k working arrays and build the alias.
 * kind[k], c[k]; REG/SPARSE members in mem[k] (ownership moves into x). */
static void install_groups(o_vertex *x, const uint32_t *c, const uint32_t *kind,
                           uint32_t **mem, const uint32_t *mcap, const uint32_t *one)
{
    uint32_t n = 0;
    for (int k = 0; k < 32; k++) if (c[k]) n++;
    o_group *g = n ? (o_group *)calloc(n, sizeof(o_group)) : NULL;
    if (n && !g) abort();
    uint64_t W[32], thr[32];
    uint32_t al[32];
    uint64_t T = 0;
    uint32_t b = 0;
    for (int k = 0; k < 32; k++) {
        if (!c[k]) continue;
        g[b].k = (uint32_t)k;
        g[b].c = c[k];
        g[b].kind = kind[k];
        g[b].one = (kind[k] == O_ONE) ? one[k] : O_NONE;
        g[b].mem = (kind[k] == O_SPARSE || kind[k] == O_REGULAR) ? mem[k] : NULL;
        g[b].cap = g[b].mem ? mcap[k] : 0;
        if (!g[b].mem && mem[k]) free(mem[k]);
        W[b] = (uint64_t)c[k] << k;                 /* Eq.4: W(p_k) = c_k * 2^k */
        T += W[b];
        b++;
    }
    for (int k = 0; k < 32; k++) if (!c[k] && mem[k]) free(mem[k]);
    ora_alias_build(n, W, thr, al);
    for (b = 0; b < n; b++) { g[b].thr = thr[b]; g[b].alias = al[b]; }
    free(x->grp);
    x->grp = g;
    x->n = n;
    x->T = T;
}

/* Scan the adjacency for the arcs whose bias has bit k (Eq.3), ascending. */
static uint32_t *scan_members(const o_vertex *x, int k, uint32_t c, uint32_t *cap_out)
{
    uint32_t cap = c ? c : 1;
    uint32_t *m = (uint32_t *)malloc(sizeof(uint32_t) * cap);
    uint32_t j = 0;
    for (uint32_t i = 0; i < x->d; i++)
        if ((x->adj[i].bias >> k) & 1u) m[j++] = i;
    *cap_out = cap;
    return m;
}

static uint32_t find_one(const o_vertex *x, int k)
{
    for (uint32_t i = 0; i < x->d; i++)
        if ((x->adj[i].bias >> k) & 1u) return i;
    return O_NONE;
}

/* Sampling-space construction for one vertex. */
static void build_vertex(const ora_graph *G, o_vertex *x)
{
    uint32_t c[32] = {0}, kind[32] = {0}, mcap[32] = {0}, one[32];
    uint32_t *mem[32] = {0};
    for (uint32_t i = 0; i < x->d; i++)
        for (int k = 0; k < 32; k++)
            if ((x->adj[i].bias >> k) & 1u) c[k]++;           /* Eq.3/Eq.4 */
    for (int k = 0; k < 32; k++) {
        one[k] = O_NONE;
        kind[k] = ora_classify(c[k], x->d, G->alpha, G->beta, G->flags);
        if (kind[k] == O_REGULAR || kind[k] == O_SPARSE) mem[k] = scan_members(x, k, c[k], &mcap[k]);
        else if (kind[k] == O_ONE) one[k] = find_one(x, k);
    }
    install_groups(x, c, kind, mem, mcap, one);
}

/* ------------------------------------------------------------------ */
/* Build from a CSR (R-2: CSR order is the canonical adjacency order,  */
/* epoch 0).                                                           */
/* ------------------------------------------------------------------ */
int ora_build(uint32_t V, const uint64_t *row_offsets, const uint32_t *dst, const uint32_t *bias,
              uint32_t alpha, uint32_t beta, uint32_t flags, ora_graph **out)
{
    *out = NULL;
    for (uint32_t u = 0; u < V; u++) {
        if (row_offsets[u + 1] < row_offsets[u]) return O_EINVAL;
        if (row_offsets[u + 1] - row_offsets[u] >= 0xFFFFFFFFull) return O_EOVERFLOW;
    }
    uint64_t A = row_offsets[V];
    for (uint64_t a = 0; a < A; a++)
        if (dst[a] >= V || bias[a] == 0) return O_EINVAL;
    for (uint32_t u = 0; u < V; u++) {
        unsigned __int128 T = 0;
        uint32_t mask = 0;
        for (uint64_t a = row_offsets[u]; a < row_offsets[u + 1]; a++) { T += bias[a]; mask |= bias[a]; }
        if (T * (unsigned __int128)__builtin_popcount(mask) >= ((unsigned __int128)1 << 64)) return O_EOVERFLOW;
    }
    ora_graph *G = (ora_graph *)calloc(1, sizeof(ora_graph));
    G->V = V;
    G->alpha = (flags & O_FLAG_BS_MODE) ? 100 : alpha;
    G->beta = (flags & O_FLAG_BS_MODE) ? 0 : beta;
    G->flags = flags;
    G->epoch = 0;
    G->v = (o_vertex *)calloc(V ? V : 1, sizeof(o_vertex));
    for (uint32_t u = 0; u < V; u++) {
        o_vertex *x = &G->v[u];
        x->d = (uint32_t)(row_offsets[u + 1] - row_offsets[u]);
        x->cap = x->d;
        x->adj = (o_arc *)xrealloc(NULL, sizeof(o_arc) * (x->cap ? x->cap : 1));
        for (uint32_t i = 0; i < x->d; i++) {
            x->adj[i].dst = dst[row_offsets[u] + i];
            x->adj[i].bias = bias[row_offsets[u] + i];
            x->adj[i].epoch = 0;
            x->adj[i].dval = 0;
        }
        build_vertex(G, x);
    }
    *out = G;
    return O_OK;
}

void ora_free(ora_graph *G);

/* ------------------------------------------------------------------ */
/* Floating-point biases (S4.3 P:344-363, S4.4 P:368-377; R-15).       */
/* For lambda = 10^j, j = 0..9: s_i = fl(w_i lambda) (IEEE binary64),  */
/* I_i = floor(s_i) must be < 2^32, D_i = floor((s_i - I_i) 2^52).      */
/* W_I = sum I_i, W_D = sum D_i (units of 2^-52).  lambda = the        */
/* smallest with W_D / (W_I 2^52 + W_D) < 1/d, i.e. (d-1) W_D < W_I 2^52;*/
/* none -> the largest valid j, flag "constraint unmet".  Integer radix */
/* groups are built over I_i (Eq.3-4, Eq.9); the decimal group holds    */
/* the arcs with D_i > 0.  Inter-group: decimal with            */
/* probability W_D / (W_I 2^52 + W_D) (64-bit threshold), else the      */
/* integer alias.  Decimal intra-group: rejection with bound max D_i.   */
/* ------------------------------------------------------------------ */
static const double POW10[10] = {1e0, 1e1, 1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8, 1e9};

static int scale_one(double w, int j, uint32_t *I, uint64_t *D)
{
    double s = w * POW10[j];
    if (!(s < 4294967296.0)) return 0;
    double fl = floor(s);
    *I = (uint32_t)fl;
    *D = (uint64_t)floor((s - fl) * 4503599627370496.0);   /* 2^52, exact scaling */
    return 1;
}

/* floor(a * 2^64 / b) for a < b (binary long division, exact) */
static uint64_t frac64(unsigned __int128 a, unsigned __int128 b)
{
    uint64_t q = 0;
    for (int i = 0; i < 64; i++) {
        a <<= 1;
        q <<= 1;
        if (a >= b) { a -= b; q |= 1; }
    }
    return q;
}

/* The decimal group of a float-mode vertex from its arcs (R-15): the arcs with
 * D_i > 0 in ascending adjacency index, W_I = sum I_i (= T), W_D = sum D_i,
 * thrD = floor(W_D 2^64 / (W_I 2^52 + W_D)) (always decimal when W_I = 0),
 * flag bit 0 = the lambda constraint (d - 1) W_D < W_I 2^52 does not
 * hold, bit 1 = the integer part is empty.  Used by the build and, with the
 * vertex's lambda fixed, after every batch that touches the vertex. */
static void decimal_group(o_vertex *x)
{
    unsigned __int128 WI = 0, WD = 0;
    free(x->didx);
    free(x->dval);
    x->dcnt = 0;
    x->dmax = 0;
    x->didx = (uint32_t *)malloc(sizeof(uint32_t) * (x->d ? x->d : 1));
    x->dval = (uint64_t *)malloc(sizeof(uint64_t) * (x->d ? x->d : 1));
    for (uint32_t i = 0; i < x->d; i++) {
        const uint64_t D = x->adj[i].dval;
        WI += x->adj[i].bias;
        WD += D;
        if (D) {
            x->didx[x->dcnt] = i;
            x->dval[x->dcnt] = D;
            x->dcnt++;
            if (D > x->dmax) x->dmax = D;
        }
    }
    x->fflags = 0;
    if (x->d && !((unsigned __int128)(x->d - 1) * WD < (WI << 52))) x->fflags |= 1u;
    if (WI == 0 && x->d) x->fflags |= 2u;
    if (WD == 0) x->thrD = 0;
    else if (WI == 0) x->thrD = ~0ull;                 /* always decimal (flag bit 1) */
    else x->thrD = frac64(WD, (WI << 52) + WD);
}

static int build_float_vertex(const ora_graph *G, o_vertex *x, const double *w)
{
    int chosen = -1, last_valid = -1;
    for (int j = 0; j < 10; j++) {
        unsigned __int128 WI = 0, WD = 0;
        int valid = 1;
        for (uint32_t i = 0; i < x->d; i++) {
            uint32_t I = 0;
            uint64_t D = 0;
            if (!scale_one(w[i], j, &I, &D)) { valid = 0; break; }
            WI += I;
            WD += D;
        }
        if (!valid) break;             /* larger lambda only grows s_i */
        last_valid = j;
        if ((unsigned __int128)(x->d ? x->d - 1 : 0) * WD < (WI << 52)) { chosen = j; break; }
    }
    if (last_valid < 0 && x->d > 0) return O_EOVERFLOW;
    if (chosen < 0) chosen = last_valid < 0 ? 0 : last_valid;   /* constraint unmet: flagged below */
    if (x->d == 0) chosen = 0;   /* R-15: P:377's constraint is vacuous for d = 0 -> the smallest lambda */
    x->lam = (uint32_t)chosen;
    for (uint32_t i = 0; i < x->d; i++) {
        uint32_t I = 0;
        uint64_t D = 0;
        scale_one(w[i], chosen, &I, &D);
        x->adj[i].bias = I;            /* the integer part is the radix-decomposed bias */
        x->adj[i].dval = D;
    }
    decimal_group(x);
    (void)G;
    return O_OK;
}

int ora_build_float(uint32_t V, const uint64_t *row_offsets, const uint32_t *dst, const double *wf,
                    uint32_t alpha, uint32_t beta, uint32_t flags, ora_graph **out)
{
    *out = NULL;
    for (uint32_t u = 0; u < V; u++)
        if (row_offsets[u + 1] < row_offsets[u] || row_offsets[u + 1] - row_offsets[u] >= 0xFFFFFFFFull)
            return O_EINVAL;
    uint64_t A = row_offsets[V];
    for (uint64_t a = 0; a < A; a++)
        if (dst[a] >= V || !(wf[a] > 0.0) || wf[a] != wf[a] || wf[a] > 1e300) return O_EINVAL;
    ora_graph *G = (ora_graph *)calloc(1, sizeof(ora_graph));
    G->V = V;
    G->float_mode = 1;
    G->alpha = (flags & O_FLAG_BS_MODE) ? 100 : alpha;
    G->beta = (flags & O_FLAG_BS_MODE) ? 0 : beta;
    G->flags = flags;
    G->v = (o_vertex *)calloc(V ? V : 1, sizeof(o_vertex));
    for (uint32_t u = 0; u < V; u++) {
        o_vertex *x = &G->v[u];
        x->d = (uint32_t)(row_offsets[u + 1] - row_offsets[u]);
        x->cap = x->d;
        x->adj = (o_arc *)xrealloc(NULL, sizeof(o_arc) * (x->cap ? x->cap : 1));
        for (uint32_t i = 0; i < x->d; i++) {
            x->adj[i].dst = dst[row_offsets[u] + i];
            x->adj[i].epoch = 0;
            x->adj[i].dval = 0;
        }
        int rc = build_float_vertex(G, x, wf + row_offsets[u]);
        if (rc == O_OK) {
            unsigned __int128 T = 0;
            uint32_t mask = 0;
            for (uint32_t i = 0; i < x->d; i++) { T += x->adj[i].bias; mask |= x->adj[i].bias; }
            if (T * (unsigned __int128)__builtin_popcount(mask) >= ((unsigned __int128)1 << 64)) rc = O_EOVERFLOW;
        }
        if (rc != O_OK) {
            G->V = u + 1;
            ora_free(G);
            return rc;
        }
        build_vertex(G, x);
    }
    *out = G;
    return O_OK;
}

void ora_free(ora_graph *G)
{
    if (!G) return;
    for (uint32_t u = 0; u < G->V; u++) {
        o_vertex *x = &G->v[u];
        for (uint32_t b = 0; b < x->n; b++) free(x->grp[b].mem);
        free(x->grp);
        free(x->adj);
        free(x->didx);
        free(x->dval);
    }
    free(G->v);
    free(G->built);
    free(G);
}

uint32_t ora_epoch(const ora_graph *G) { return G->epoch; }
uint32_t ora_num_vertices(const ora_graph *G) { return G->V; }
uint32_t ora_degree(const ora_graph *G, uint32_t u) { return vx(G, u)->d; }

/* Lazy build: the CSR arrays must outlive the graph.  Validation is done per
 * vertex on first access by the caller's contract (inputs are generated). */
int ora_build_lazy(uint32_t V, const uint64_t *row_offsets, const uint32_t *dst, const uint32_t *bias,
                   uint32_t alpha, uint32_t beta, uint32_t flags, ora_graph **out)
{
    ora_graph *G = (ora_graph *)calloc(1, sizeof(ora_graph));
    G->V = V;
    G->alpha = (flags & O_FLAG_BS_MODE) ? 100 : alpha;
    G->beta = (flags & O_FLAG_BS_MODE) ? 0 : beta;
    G->flags = flags;
    G->lazy = 1;
    G->built = (uint8_t *)calloc(V ? V : 1, 1);
    G->lro = row_offsets;
    G->ldst = dst;
    G->lbias = bias;
    G->v = (o_vertex *)calloc(V ? V : 1, sizeof(o_vertex));
    *out = G;
    return O_OK;
}

/* ------------------------------------------------------------------ */
/* Two-phase parallel delete-and-swap (pairing R-6).        */
/* arr has len entries; del[0..N) are the slots to delete, ascending.  */
/* Phase (i): stage the last N entries, drop the gamma of them that    */
/* are themselves deleted.  Phase (ii): move the N-gamma survivors, in */
/* ascending order, into the N-gamma front holes, in ascending order.  */
/* moved_from/moved_to (optional) receive the (old, new) pairs.        */
/* Returns the new length len - N.                                     */
/* ------------------------------------------------------------------ */
static uint32_t two_phase_delete(void *arr, size_t esz, uint32_t len, const uint32_t *del, uint32_t N,
                                 uint32_t *moved_from, uint32_t *moved_to, uint32_t *n_moved)
{
    char *a = (char *)arr;
    uint32_t newlen = len - N;
    /* phase (i): survivors of the tail window [len-N, len) */
    uint32_t *surv = (uint32_t *)malloc(sizeof(uint32_t) * (N ? N : 1));
    uint32_t ns = 0;
    for (uint32_t t = newlen; t < len; t++) {
        int deleted = 0;
        for (uint32_t j = 0; j < N; j++) if (del[j] == t) { deleted = 1; break; }
        if (!deleted) surv[ns++] = t;
    }
    /* phase (ii): holes in the front region [0, len-N), ascending */
    uint32_t nh = 0;
    for (uint32_t j = 0; j < N; j++) {
        if (del[j] < newlen) {
            uint32_t hole = del[j];
            memcpy(a + (size_t)hole * esz, a + (size_t)surv[nh] * esz, esz);
            if (moved_from) { moved_from[nh] = surv[nh]; moved_to[nh] = hole; }
            nh++;
        }
    }
    if (n_moved) *n_moved = nh;
    free(surv);
    return newlen;
}

/* Exported for the S:340 / P:514 worked-example pin. */
uint32_t ora_two_phase_u32(uint32_t *arr, uint32_t len, const uint32_t *del_sorted, uint32_t N)
{
    return two_phase_delete(arr, sizeof(uint32_t), len, del_sorted, N, NULL, NULL, NULL);
}


/* stats layout (u64): [0] inserted [1] deleted [2] missing_deletes
 * [3] touched_vertices [4..28] kind_transitions[5][5] [29] epoch */
#define ST_INS 0
#define ST_DEL 1
#define ST_MISS 2
#define ST_TOUCH 3
#define ST_TRANS 4
#define ST_EPOCH 29

/* Batched update of one vertex: insert -> delete -> rebuild. */
static void update_vertex(ora_graph *G, o_vertex *x, const uint32_t *recs, const uint64_t *dv, const uint64_t *idx,
                          uint64_t m, uint32_t e, uint64_t *st)
{
    /* expand the pre-batch groups into per-k working arrays */
    uint32_t kind0[32] = {0}, c[32] = {0}, len[32] = {0}, mcap[32] = {0}, one[32];
    uint32_t *mem[32] = {0};
    for (int k = 0; k < 32; k++) one[k] = O_NONE;
    for (uint32_t b = 0; b < x->n; b++) {
        o_group *g = &x->grp[b];
        kind0[g->k] = g->kind;
        c[g->k] = g->c;
        one[g->k] = g->one;
        if (g->mem) {
            mem[g->k] = g->mem;
            len[g->k] = g->c;
            mcap[g->k] = g->cap;
            g->mem = NULL;
        }
    }
    /* (1) insertions, in batch order: append the arc to the
     * adjacency; each set bit k counts into c_k; a group that is REGULAR or
     * SPARSE before the batch gets the new index appended; DENSE does nothing;
     * ONE/EMPTY groups are re-derived at the rebuild (R-7). */
    for (uint64_t r = 0; r < m; r++) {
        const uint32_t *rec = recs + 4 * idx[r];
        if (rec[0] != 0) continue;
        if (x->d == x->cap) {
            x->cap = x->cap ? 2 * x->cap : 4;
            x->adj = (o_arc *)xrealloc(x->adj, sizeof(o_arc) * x->cap);
        }
        uint32_t i = x->d++;
        x->adj[i].dst = rec[2];
        x->adj[i].bias = rec[3];
        x->adj[i].epoch = e;
        x->adj[i].dval = dv ? dv[idx[r]] : 0;   /* float mode: the inserted arc's decimal part */
        for (int k = 0; k < 32; k++) {
            if (!((rec[3] >> k) & 1u)) continue;
            c[k]++;
            if (kind0[k] == O_REGULAR || kind0[k] == O_SPARSE) {
                if (len[k] == mcap[k]) {
                    mcap[k] = mcap[k] ? 2 * mcap[k] : 4;
                    mem[k] = (uint32_t *)xrealloc(mem[k], sizeof(uint32_t) * mcap[k]);
                }
                mem[k][len[k]++] = i;
            }
        }
        st[ST_INS]++;
    }
    /* (2) deletions.  Each delete(u,v) takes the
     * live instance of (u,v) with the smallest (epoch, position) not already
     * taken by an earlier delete of this batch (R-8); none -> missing. */
    uint32_t L = x->d;
    uint8_t *taken = (uint8_t *)calloc(L ? L : 1, 1);
    uint32_t N = 0;
    for (uint64_t r = 0; r < m; r++) {
        const uint32_t *rec = recs + 4 * idx[r];
        if (rec[0] != 1) continue;
        uint32_t best = O_NONE;
        for (uint32_t p = 0; p < L; p++) {
            if (taken[p] || x->adj[p].dst != rec[2]) continue;
            if (best == O_NONE || x->adj[p].epoch < x->adj[best].epoch) best = p;
        }
        if (best == O_NONE) { st[ST_MISS]++; continue; }
        taken[best] = 1;
        N++;
        st[ST_DEL]++;
    }
    if (N) {
        uint32_t *P = (uint32_t *)malloc(sizeof(uint32_t) * N);
        uint32_t np = 0;
        for (uint32_t p = 0; p < L; p++) if (taken[p]) P[np++] = p;   /* ascending */
        /* (2a) groups: sub-biases of each deleted arc leave their groups */
        for (uint32_t j = 0; j < N; j++)
            for (int k = 0; k < 32; k++)
                if ((x->adj[P[j]].bias >> k) & 1u) c[k]--;
        for (int k = 0; k < 32; k++) {
            if (!(kind0[k] == O_REGULAR || kind0[k] == O_SPARSE)) continue;
            uint32_t *Q = (uint32_t *)malloc(sizeof(uint32_t) * (len[k] ? len[k] : 1));
            uint32_t nq = 0;
            for (uint32_t s = 0; s < len[k]; s++) if (taken[mem[k][s]]) Q[nq++] = s;
            len[k] = two_phase_delete(mem[k], sizeof(uint32_t), len[k], Q, nq, NULL, NULL, NULL);
            free(Q);
        }
        /* (2b) the adjacency itself, same two-phase delete-and-swap */
        uint32_t *from = (uint32_t *)malloc(sizeof(uint32_t) * N);
        uint32_t *to = (uint32_t *)malloc(sizeof(uint32_t) * N);
        uint32_t nm = 0;
        x->d = two_phase_delete(x->adj, sizeof(o_arc), L, P, N, from, to, &nm);
        /* (2c) rename moved arcs in every group that references them */
        for (int k = 0; k < 32; k++) {
            if (!(kind0[k] == O_REGULAR || kind0[k] == O_SPARSE)) continue;
            for (uint32_t s = 0; s < len[k]; s++)
                for (uint32_t j = 0; j < nm; j++)
                    if (mem[k][s] == from[j]) { mem[k][s] = to[j]; break; }
        }
        free(from);
        free(to);
        free(P);
    }
    free(taken);
    /* (3) rebuild: reclassify with the post-batch degree;
     * REG/SPARSE -> REG/SPARSE keeps its member order; any other kind ->
     * REG/SPARSE rescans the adjacency ascending; ONE takes the unique arc;
     * DENSE / EMPTY drop their members.  Then the alias once. */
    uint32_t kind1[32];
    for (int k = 0; k < 32; k++) {
        kind1[k] = ora_classify(c[k], x->d, G->alpha, G->beta, G->flags);
        if (kind0[k] != O_EMPTY || kind1[k] != O_EMPTY) st[ST_TRANS + 5 * kind0[k] + kind1[k]]++;
        int was_list = (kind0[k] == O_REGULAR || kind0[k] == O_SPARSE);
        int is_list = (kind1[k] == O_REGULAR || kind1[k] == O_SPARSE);
        if (is_list && !was_list) {
            free(mem[k]);
            mem[k] = scan_members(x, k, c[k], &mcap[k]);
        } else if (!is_list && mem[k]) {
            free(mem[k]);
            mem[k] = NULL;
        }
        one[k] = (kind1[k] == O_ONE) ? find_one(x, k) : O_NONE;
    }
    install_groups(x, c, kind1, mem, mcap, one);
    if (G->float_mode) decimal_group(x);   /* R-16: lambda fixed, decimal group from the live arcs */
    st[ST_TOUCH]++;
}

/* Batched updates.  recs: n records of 4 x u32 {op, src, dst, bias},
 * op 0 = insert, 1 = delete.  Whole-batch validation before any mutation.
 * Float-mode graphs (R-16) take the inserted biases from wf[n] (the records'
 * bias fields are ignored): with the source vertex's lambda fixed at build
 * (S:229), s = fl(w lambda), the arc's integer bias I = floor(s) (must be
 * < 2^32, else EOVERFLOW; I = 0 is allowed: the arc joins no radix group) and
 * its decimal part D = floor((s - I) 2^52). */
static int apply_updates_int(ora_graph *G, const uint32_t *recs, const uint64_t *dv, uint64_t n, uint64_t *st);

int ora_apply_updates_f(ora_graph *G, const uint32_t *recs, const double *wf, uint64_t n, uint64_t *stats)
{
    uint64_t st[30];
    memset(st, 0, sizeof(st));
    if (G->float_mode != (wf != NULL) && n) return O_EINVAL;
    for (uint64_t r = 0; r < n; r++) {
        const uint32_t *rec = recs + 4 * r;
        if (rec[0] > 1 || rec[1] >= G->V || rec[2] >= G->V) return O_EINVAL;
        if (!G->float_mode && rec[0] == 0 && rec[3] == 0) return O_EINVAL;
        if (G->float_mode && rec[0] == 0 && (!(wf[r] > 0.0) || wf[r] != wf[r] || wf[r] > 1e300)) return O_EINVAL;
    }
    uint32_t *frecs = NULL;
    uint64_t *dv = NULL;
    if (G->float_mode && n) {
        frecs = (uint32_t *)malloc(sizeof(uint32_t) * 4 * n);
        dv = (uint64_t *)calloc(n, sizeof(uint64_t));
        memcpy(frecs, recs, sizeof(uint32_t) * 4 * n);
        for (uint64_t r = 0; r < n; r++) {
            if (frecs[4 * r] != 0) { frecs[4 * r + 3] = 0; continue; }
            uint32_t I = 0;
            if (!scale_one(wf[r], (int)vx(G, frecs[4 * r + 1])->lam, &I, &dv[r])) {
                free(frecs); free(dv);
                return O_EOVERFLOW;
            }
            frecs[4 * r + 3] = I;
        }
        recs = frecs;
    }
    int rc = apply_updates_int(G, recs, dv, n, st);
    free(frecs);
    free(dv);
    if (rc == O_OK && stats) memcpy(stats, st, sizeof(st));
    return rc;
}

int ora_apply_updates(ora_graph *G, const uint32_t *recs, uint64_t n, uint64_t *stats)
{
    return ora_apply_updates_f(G, recs, NULL, n, stats);
}

static int apply_updates_int(ora_graph *G, const uint32_t *recs, const uint64_t *dv, uint64_t n, uint64_t *st)
{
    /* stable partition of the batch by src ("put the graph updates of
     * the same vertex together") -- a counting sort keeps batch order */
    uint64_t *cnt = (uint64_t *)calloc((size_t)G->V + 1, sizeof(uint64_t));
    for (uint64_t r = 0; r < n; r++) cnt[recs[4 * r + 1] + 1]++;
    for (uint32_t u = 0; u < G->V; u++) cnt[u + 1] += cnt[u];
    uint64_t *idx = (uint64_t *)malloc(sizeof(uint64_t) * (n ? n : 1));
    uint64_t *fill = (uint64_t *)malloc(sizeof(uint64_t) * ((size_t)G->V + 1));
    memcpy(fill, cnt, sizeof(uint64_t) * ((size_t)G->V + 1));
    for (uint64_t r = 0; r < n; r++) idx[fill[recs[4 * r + 1]]++] = r;
    free(fill);
    /* overflow check (R-10): per touched vertex (T + inserted) * popc(mask) < 2^64,
     * and d + inserted < 2^32 - 1 */
    for (uint32_t u = 0; u < G->V; u++) {
        if (cnt[u + 1] == cnt[u]) continue;
        const o_vertex *x = vx(G, u);
        unsigned __int128 T = x->T;
        uint32_t mask = 0;
        uint64_t ins = 0;
        for (uint32_t b = 0; b < x->n; b++) mask |= 1u << x->grp[b].k;
        for (uint64_t j = cnt[u]; j < cnt[u + 1]; j++) {
            const uint32_t *rec = recs + 4 * idx[j];
            if (rec[0] == 0) { T += rec[3]; mask |= rec[3]; ins++; }
        }
        if (T * (unsigned __int128)__builtin_popcount(mask) >= ((unsigned __int128)1 << 64) ||
            (uint64_t)x->d + ins >= 0xFFFFFFFFull) {
            free(cnt); free(idx);
            return O_EOVERFLOW;
        }
    }
    uint32_t e = ++G->epoch;   /* R-9: epoch = call number, build = 0 */
    for (uint32_t u = 0; u < G->V; u++) {
        if (cnt[u + 1] == cnt[u]) continue;
        update_vertex(G, vx(G, u), recs, dv, idx + cnt[u], cnt[u + 1] - cnt[u], e, st);
    }
    st[ST_EPOCH] = e;
    free(cnt);
    free(idx);
    return O_OK;
}

/* ------------------------------------------------------------------ */
/* Sampling.                             */
/* counter = (walker, step, (outer << 16) + inner, tag + (outer >> 16 << 8)), key = seed. */
/* ------------------------------------------------------------------ */
static void draw(uint64_t seed, uint32_t w, uint32_t t, uint32_t c2, uint32_t tag, uint32_t r[4])
{
    uint32_t ctr[4] = {w, t, c2, tag};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    ora_philox4x32_10(ctr, key, r);
}

/* The draw of (outer attempt, inner attempt, tag): counter word 2 = (outer << 16) + inner,
 * word 3 = tag + ((outer >> 16) << 8) -- outer attempts past 65535 carry their high bits
 * into the tag word, so node2vec's rejection draws never repeat (R-1). */
static void draw_oi(uint64_t seed, uint32_t w, uint32_t t, uint32_t outer, uint32_t inner, uint32_t tag,
                    uint32_t r[4])
{
    draw(seed, w, t, (outer << 16) + inner, tag + ((outer >> 16) << 8), r);
}

/* One first-order sample at vertex u (d > 0): inter-group alias (Eq.5),
 * then intra-group (Eq.6) with the group's Eq.9 layout.  Returns the arc
 * index; *attempts receives the number of dense-rejection attempts. */
static uint32_t sample_arc(const o_vertex *x, uint64_t seed, uint32_t w, uint32_t t, uint32_t outer,
                           uint32_t *attempts)
{
    uint32_t r[4];
    *attempts = 0;
    if (x->thrD) {
        /* float mode (R-15): the decimal group with probability thrD / 2^64 */
        int dec = 1;
        if (!(x->fflags & 2u)) {
            draw_oi(seed, w, t, outer, 0, 5, r);
            dec = (((uint64_t)r[0] << 32) | r[1]) < x->thrD;
        }
        if (dec) {
            for (uint32_t a = 0;; a++) {
                draw_oi(seed, w, t, outer, a, 4, r);
                uint64_t j = mulhi64(((uint64_t)r[0] << 32) | r[1], x->dcnt);
                if (mulhi64(((uint64_t)r[2] << 32) | r[3], x->dmax) < x->dval[j]) return x->didx[j];
            }
        }
    }
    draw_oi(seed, w, t, outer, 0, 0, r);
    /* stage (i): inter-group alias */
    uint32_t b = (uint32_t)(((uint64_t)r[0] * x->n) >> 32);
    uint64_t coin = mulhi64(((uint64_t)r[1] << 32) | r[2], x->T);
    uint32_t gsel = (coin < x->grp[b].thr) ? b : x->grp[b].alias;
    const o_group *g = &x->grp[gsel];
    /* stage (ii): intra-group */
    if (g->kind == O_ONE) return g->one;
    if (g->kind == O_REGULAR || g->kind == O_SPARSE) {
        draw_oi(seed, w, t, outer, 0, 1, r);
        uint64_t j = mulhi64(((uint64_t)r[0] << 32) | r[1], g->c);
        return g->mem[j];
    }
    /* DENSE: rejection over the whole adjacency, accept iff bias AND 2^k != 0 */
    for (uint32_t a = 0;; a++) {
        draw_oi(seed, w, t, outer, a, 1, r);
        uint64_t j = mulhi64(((uint64_t)r[0] << 32) | r[1], x->d);
        *attempts = a + 1;
        if ((x->adj[j].bias >> g->k) & 1u) return (uint32_t)j;
    }
}

uint32_t ora_sample(const ora_graph *G, uint32_t u, uint64_t seed, uint32_t w, uint32_t t, uint32_t outer)
{
    uint32_t att;
    const o_vertex *x = vx(G, u);
    if (x->d == 0) return O_NONE;
    return x->adj[sample_arc(x, seed, w, t, outer, &att)].dst;
}

/* node2vec distance class (Eq.1): 0 if v == prev, 1 if a live arc prev->v
 * exists, 2 otherwise. */
static int n2v_class(const ora_graph *G, uint32_t prev, uint32_t v)
{
    if (v == prev) return 0;
    const o_vertex *y = vx(G, prev);
    for (uint32_t i = 0; i < y->d; i++)
        if (y->adj[i].dst == v) return 1;
    return 2;
}

/* app: 0 DeepWalk, 1 node2vec, 2 PPR.
 * n2v_thr[3] / n2v_always[3]: per distance class, accept iff draw < thr, or
 * always (ratio 1).  stop_thr / stop_always: PPR termination.
 * paths: step-major [(L+1) x W] or NULL; lengths [W] or NULL; counts [V] or NULL. */
void ora_walk(const ora_graph *G, uint32_t app, uint32_t L, uint64_t seed, uint32_t first_walker,
              const uint32_t *starts, uint32_t W, uint32_t *paths, uint32_t *lengths,
              unsigned long long *counts, const uint64_t *n2v_thr, const uint32_t *n2v_always,
              uint64_t stop_thr, uint32_t stop_always, int nthreads, uint64_t *dense_attempts_out)
{
    uint64_t dense_total = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static) reduction(+ : dense_total)
#endif
    for (int64_t i = 0; i < (int64_t)W; i++) {
        uint32_t w = first_walker + (uint32_t)i;
        uint32_t u = starts ? starts[i] : (uint32_t)(((uint64_t)first_walker + (uint64_t)i) % G->V);
        uint32_t steps = 0, prev = O_NONE;
        if (paths) paths[(size_t)i] = u;
        if (counts && app == 2) {
#ifdef _OPENMP
#pragma omp atomic
#endif
            counts[u]++;
        }
        for (uint32_t t = 0; L == 0xFFFFFFFFu || t < L; t++) {
            const o_vertex *x = vx(G, u);
            if (x->d == 0) break;                       /* dead end: truncate */
            uint32_t att, next;
            if (app == 1 && t >= 1) {
                /* KnightKing-style rejection */
                for (uint32_t o = 0;; o++) {
                    uint32_t i_arc = sample_arc(x, seed, w, t, o, &att);
                    dense_total += att;
                    next = x->adj[i_arc].dst;
                    int cls = n2v_class(G, prev, next);
                    if (n2v_always[cls]) break;
                    uint32_t r[4];
                    draw_oi(seed, w, t, o, 0, 2, r);
                    if ((((uint64_t)r[0] << 32) | r[1]) < n2v_thr[cls]) break;
                }
            } else {
                next = x->adj[sample_arc(x, seed, w, t, 0, &att)].dst;
                dense_total += att;
            }
            steps++;
            if (paths) paths[(size_t)(t + 1) * W + (size_t)i] = next;
            prev = u;
            u = next;
            if (app == 2) {
                if (counts) {
#ifdef _OPENMP
#pragma omp atomic
#endif
                    counts[u]++;
                }
                if (stop_always) break;
                uint32_t r[4];
                draw(seed, w, t, 0, 3, r);
                if ((((uint64_t)r[0] << 32) | r[1]) < stop_thr) break;
            }
        }
        if (lengths) lengths[i] = steps;
        if (paths && L != 0xFFFFFFFFu)
            for (uint32_t t = steps + 1; t <= L; t++) paths[(size_t)t * W + (size_t)i] = O_NONE;
    }
    if (dense_attempts_out) *dense_attempts_out = dense_total;
}

/* ------------------------------------------------------------------ */
/* Canonical dump (R-11): per vertex u ascending,                      */
/*   u32 d; d x {u32 dst, u32 bias, u32 epoch}; u32 n;                 */
/*   n x {u32 k, u32 c, u32 kind, u64 thr, u32 alias,                  */
/*        REG/SPARSE: c x u32 member; ONE: u32 member}; u64 T.         */
/* little-endian.  Returns the byte count; writes only if cap allows.  */
/* ------------------------------------------------------------------ */
struct o_out_s { uint8_t *buf; size_t cap, pos; };

static void put32(o_out *o, uint32_t v)
{
    if (o->buf && o->pos + 4 <= o->cap) memcpy(o->buf + o->pos, &v, 4);
    o->pos += 4;
}
static void put64(o_out *o, uint64_t v)
{
    if (o->buf && o->pos + 8 <= o->cap) memcpy(o->buf + o->pos, &v, 8);
    o->pos += 8;
}

static void dump_vertex(const o_vertex *x, o_out *o)
{
    put32(o, x->d);
    for (uint32_t i = 0; i < x->d; i++) {
        put32(o, x->adj[i].dst);
        put32(o, x->adj[i].bias);
        put32(o, x->adj[i].epoch);
    }
    put32(o, x->n);
    for (uint32_t b = 0; b < x->n; b++) {
        const o_group *g = &x->grp[b];
        put32(o, g->k);
        put32(o, g->c);
        put32(o, g->kind);
        put64(o, g->thr);
        put32(o, g->alias);
        if (g->kind == O_REGULAR || g->kind == O_SPARSE)
            for (uint32_t s = 0; s < g->c; s++) put32(o, g->mem[s]);
        else if (g->kind == O_ONE)
            put32(o, g->one);
    }
    put64(o, x->T);
    if (g_dump_float) {
        put32(o, x->lam);
        put32(o, x->fflags);
        put64(o, x->dmax);
        put64(o, x->thrD);
        put32(o, x->dcnt);
        for (uint32_t j = 0; j < x->dcnt; j++) {
            put32(o, x->didx[j]);
            put64(o, x->dval[j]);
        }
    }
}

size_t ora_dump(const ora_graph *G, uint8_t *buf, size_t cap)
{
    g_dump_float = G->float_mode;
    o_out o = {buf, cap, 0};
    for (uint32_t u = 0; u < G->V; u++) dump_vertex(vx(G, u), &o);
    return o.pos;
}

/* Per-vertex FNV-1a 64 digest of the vertex's canonical dump bytes. */
void ora_digests(const ora_graph *G, uint64_t *dig)
{
    g_dump_float = G->float_mode;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1024)
#endif
    for (int64_t u = 0; u < (int64_t)G->V; u++) {
        o_out o = {NULL, 0, 0};
        dump_vertex(vx(G, (uint32_t)u), &o);
        uint8_t *tmp = (uint8_t *)malloc(o.pos);
        o_out o2 = {tmp, o.pos, 0};
        dump_vertex(vx(G, (uint32_t)u), &o2);
        uint64_t h = 0xcbf29ce484222325ull;
        for (size_t i = 0; i < o.pos; i++) { h ^= tmp[i]; h *= 0x100000001b3ull; }
        dig[u] = h;
        free(tmp);
    }
}

/* Per-vertex canonical dump bytes of one vertex (for sampled parity at scale). */
size_t ora_dump_vertex(const ora_graph *G, uint32_t u, uint8_t *buf, size_t cap)
{
    o_out o = {buf, cap, 0};
    g_dump_float = G->float_mode;
    dump_vertex(vx(G, u), &o);
    return o.pos;
}

/* ------------------------------------------------------------------ */
/* Arbitrary radix base B = 2^b (S "Bingo with Arbitrary Radix Bases", */
/* P:910-928; reading R-17).  Static structure: build + sampling.      */
/*   w = sum_i d_i B^i, digits d_i in [0, B).  Group B^i holds the arcs */
/*   with d_i != 0, weight W_i = B^i sum_j j c_ij; inside it subgroup j */
/*   holds the arcs with d_i = j (c_ij of them, ascending adjacency     */
/*   index) -- the neighbours of a group no longer share one bias       */
/*   (P:917), so a second, inter-subgroup alias over the weights        */
/*   j c_ij picks the subgroup, then a member uniformly.    */
/*   P(a) = sum_i (W_i/T)(d_i(a) c_{i,d_i(a)} B^i / W_i)(1/c_{i,d_i(a)}) */
/*        = w(a)/T (Theorem 1, base B).  Both alias tables are the      */
/*   integer Vose of R-4 (ora_alias_build).                             */
/* ------------------------------------------------------------------ */
typedef struct {
    uint32_t j, c;
    uint64_t thr;
    uint32_t alias;
    uint32_t *mem;            /* adjacency indices with digit j, ascending */
} r_sub;

typedef struct {
    uint32_t i;               /* digit position: group B^i */
    uint64_t W, S;            /* W = B^i S, S = sum_j j c_ij */
    uint64_t thr;
    uint32_t alias, ns;
    r_sub *sub;
} r_group;

typedef struct {
    uint32_t d, n;
    uint32_t *dst, *bias;     /* into the CSR copies, or the vertex's own arrays once updated */
    uint32_t *epoch;          /* NULL: every arc from the build (epoch 0) */
    uint32_t cap;             /* capacity of the own arrays (0: CSR-backed) */
    r_group *grp;
    uint64_t T;
} r_vertex;

typedef struct ora_radix {
    uint32_t V, b;
    uint32_t *dst, *bias;     /* owned copies of the CSR arrays */
    r_vertex *v;
    uint32_t epoch;           /* successful ora_radix_apply_updates calls (R-9) */
} ora_radix;

static uint32_t digit(uint32_t w, uint32_t i, uint32_t b)
{
    const uint32_t sh = i * b;
    return sh >= 32 ? 0u : (w >> sh) & ((1u << b) - 1u);
}

static void radix_free_groups(r_vertex *x)
{
    for (uint32_t g = 0; g < x->n; g++) {
        for (uint32_t s = 0; s < x->grp[g].ns; s++) free(x->grp[g].sub[s].mem);
        free(x->grp[g].sub);
    }
    free(x->grp);
    x->grp = NULL;
    x->n = 0;
}

void ora_radix_free(ora_radix *G)
{
    if (!G) return;
    for (uint32_t u = 0; u < G->V; u++) {
        r_vertex *x = &G->v[u];
        radix_free_groups(x);
        if (x->cap) { free(x->dst); free(x->bias); free(x->epoch); }
    }
    free(G->v);
    free(G->dst);
    free(G->bias);
    free(G);
}

static int radix_build_vertex(r_vertex *x, uint32_t b);

/* b in [1, 5]: B = 2^b <= 32, so a group has at most 31 subgroups. */
int ora_build_radix(uint32_t V, const uint64_t *ro, const uint32_t *dst, const uint32_t *bias, uint32_t b,
                    ora_radix **out)
{
    if (b < 1 || b > 5) return O_EINVAL;
    /* B = 2^b <= 32, K = ceil(32 / b) digit positions: see radix_build_vertex */
    ora_radix *G = (ora_radix *)calloc(1, sizeof(ora_radix));
    const uint64_t A = ro[V];
    G->V = V;
    G->b = b;
    G->dst = (uint32_t *)xrealloc(NULL, sizeof(uint32_t) * (A ? A : 1));
    G->bias = (uint32_t *)xrealloc(NULL, sizeof(uint32_t) * (A ? A : 1));
    memcpy(G->dst, dst, sizeof(uint32_t) * A);
    memcpy(G->bias, bias, sizeof(uint32_t) * A);
    G->v = (r_vertex *)calloc(V ? V : 1, sizeof(r_vertex));
    for (uint32_t u = 0; u < V; u++) {
        r_vertex *x = &G->v[u];
        x->d = (uint32_t)(ro[u + 1] - ro[u]);
        x->dst = G->dst + ro[u];
        x->bias = G->bias + ro[u];
        for (uint32_t a = 0; a < x->d; a++)
            if (x->bias[a] == 0) { ora_radix_free(G); return O_EINVAL; }
        if (radix_build_vertex(x, b) != O_OK) { ora_radix_free(G); return O_EOVERFLOW; }
    }
    *out = G;
    return O_OK;
}

/* The nested structure of one vertex from its adjacency (x->dst, x->bias, x->d), replacing
 * any previous one: groups in ascending i, subgroups in ascending j, members ascending. */
static int radix_build_vertex(r_vertex *x, uint32_t b)
{
    const uint32_t B = 1u << b, K = (32 + b - 1) / b;
    radix_free_groups(x);
    {
        x->T = 0;
        for (uint32_t a = 0; a < x->d; a++) x->T += x->bias[a];
        /* groups in ascending i, subgroups in ascending j */
        x->grp = (r_group *)calloc(K, sizeof(r_group));
        for (uint32_t i = 0; i < K; i++) {
            uint32_t c[32] = {0};
            for (uint32_t a = 0; a < x->d; a++) c[digit(x->bias[a], i, b)]++;
            uint64_t S = 0;
            uint32_t ns = 0;
            for (uint32_t j = 1; j < B; j++) {
                S += (uint64_t)j * c[j];
                ns += c[j] ? 1u : 0u;
            }
            if (!ns) continue;
            r_group *g = &x->grp[x->n++];
            g->i = i;
            g->S = S;
            g->W = S << (i * b);          /* B^i S < 2^32 d: no overflow for d < 2^32 */
            g->sub = (r_sub *)calloc(ns, sizeof(r_sub));
            uint64_t sw[32];
            for (uint32_t j = 1; j < B; j++) {
                if (!c[j]) continue;
                r_sub *sb = &g->sub[g->ns];
                sb->j = j;
                sb->c = c[j];
                sb->mem = (uint32_t *)xrealloc(NULL, sizeof(uint32_t) * c[j]);
                uint32_t k = 0;
                for (uint32_t a = 0; a < x->d; a++)
                    if (digit(x->bias[a], i, b) == j) sb->mem[k++] = a;
                sw[g->ns] = (uint64_t)j * c[j];
                g->ns++;
            }
            uint64_t thr[32];
            uint32_t al[32];
            ora_alias_build(g->ns, sw, thr, al);    /* inter-subgroup alias */
            for (uint32_t s = 0; s < g->ns; s++) { g->sub[s].thr = thr[s]; g->sub[s].alias = al[s]; }
        }
        if (x->n) {
            if ((unsigned __int128)x->T * x->n >= ((unsigned __int128)1 << 64)) return O_EOVERFLOW;
            uint64_t W[32], thr[32];
            uint32_t al[32];
            for (uint32_t g = 0; g < x->n; g++) W[g] = x->grp[g].W;
            ora_alias_build(x->n, W, thr, al);      /* inter-group alias (Eq.5) */
            for (uint32_t g = 0; g < x->n; g++) { x->grp[g].thr = thr[g]; x->grp[g].alias = al[g]; }
        }
    }
    return O_OK;
}

/* Updates of a radix graph (reading R-19; the paper leaves nested dynamic structures to
 * future work).  The adjacency follows exactly the base-2 readings: whole-batch
 * validation (op 0/1, ids < V, insert bias > 0: a radix arc needs a nonzero digit), epoch =
 * the number of the successful call (R-9), records grouped by source in batch order,
 * inserts appended in batch order (R-7), each delete takes the live instance with the smallest
 * (epoch, position) (R-8), the adjacency compacted by the two-phase delete-and-swap (R-6).
 * Then every touched vertex's nested structure is rebuilt from its adjacency exactly as the
 * build does (groups, subgroups, members ascending, both integer-Vose tables), so the structure
 * stays a function of the adjacency.  Overflow (whole batch, nothing mutated): d + inserts >=
 * 2^32 - 1, or (T + inserted biases) x ceil(32 / b) >= 2^64.  stats as ora_apply_updates
 * ([0] inserted [1] deleted [2] missing [3] touched, [29] epoch; no kind transitions). */
static void radix_own(r_vertex *x, uint32_t need)
{
    if (x->cap >= need && x->cap) return;
    uint32_t cap = x->cap ? x->cap : 4;
    while (cap < need) cap *= 2;
    uint32_t *nd = (uint32_t *)malloc(sizeof(uint32_t) * cap), *nb = (uint32_t *)malloc(sizeof(uint32_t) * cap),
             *ne = (uint32_t *)calloc(cap, sizeof(uint32_t));
    memcpy(nd, x->dst, sizeof(uint32_t) * x->d);
    memcpy(nb, x->bias, sizeof(uint32_t) * x->d);
    if (x->epoch) memcpy(ne, x->epoch, sizeof(uint32_t) * x->d);
    if (x->cap) { free(x->dst); free(x->bias); free(x->epoch); }
    x->dst = nd;
    x->bias = nb;
    x->epoch = ne;
    x->cap = cap;
}

int ora_radix_apply_updates(ora_radix *G, const uint32_t *recs, uint64_t n, uint64_t *stats)
{
    uint64_t st[30];
    memset(st, 0, sizeof(st));
    const uint32_t K = (32 + G->b - 1) / G->b;
    for (uint64_t r = 0; r < n; r++) {
        const uint32_t *rec = recs + 4 * r;
        if (rec[0] > 1 || rec[1] >= G->V || rec[2] >= G->V) return O_EINVAL;
        if (rec[0] == 0 && rec[3] == 0) return O_EINVAL;
    }
    /* stable grouping by source (counting sort keeps batch order) */
    uint64_t *cnt = (uint64_t *)calloc((size_t)G->V + 1, sizeof(uint64_t));
    for (uint64_t r = 0; r < n; r++) cnt[recs[4 * r + 1] + 1]++;
    for (uint32_t u = 0; u < G->V; u++) cnt[u + 1] += cnt[u];
    uint64_t *idx = (uint64_t *)malloc(sizeof(uint64_t) * (n ? n : 1));
    uint64_t *pos = (uint64_t *)malloc(sizeof(uint64_t) * ((size_t)G->V + 1));
    memcpy(pos, cnt, sizeof(uint64_t) * ((size_t)G->V + 1));
    for (uint64_t r = 0; r < n; r++) idx[pos[recs[4 * r + 1]]++] = r;
    free(pos);
    /* overflow checks for every touched vertex before anything changes */
    for (uint32_t u = 0; u < G->V; u++) {
        if (cnt[u + 1] == cnt[u]) continue;
        const r_vertex *x = &G->v[u];
        uint64_t ins = 0, m = 0;
        for (uint64_t k = cnt[u]; k < cnt[u + 1]; k++) {
            const uint32_t *rec = recs + 4 * idx[k];
            if (rec[0] == 0) { ins += rec[3]; m++; }
        }
        if ((uint64_t)x->d + m >= 0xFFFFFFFFull ||
            (unsigned __int128)(x->T + ins) * K >= ((unsigned __int128)1 << 64)) {
            free(cnt); free(idx);
            return O_EOVERFLOW;
        }
    }
    const uint32_t e = ++G->epoch;
    for (uint32_t u = 0; u < G->V; u++) {
        if (cnt[u + 1] == cnt[u]) continue;
        r_vertex *x = &G->v[u];
        uint32_t m = 0;
        for (uint64_t k = cnt[u]; k < cnt[u + 1]; k++) m += recs[4 * idx[k]] == 0 ? 1u : 0u;
        radix_own(x, x->d + m);
        /* (1) inserts, batch order (R-7) */
        for (uint64_t k = cnt[u]; k < cnt[u + 1]; k++) {
            const uint32_t *rec = recs + 4 * idx[k];
            if (rec[0] != 0) continue;
            x->dst[x->d] = rec[2];
            x->bias[x->d] = rec[3];
            x->epoch[x->d] = e;
            x->d++;
            st[ST_INS]++;
        }
        /* (2) deletes, batch order: smallest (epoch, position) live instance (R-8) */
        const uint32_t L = x->d;
        uint8_t *taken = (uint8_t *)calloc(L ? L : 1, 1);
        uint32_t N = 0;
        for (uint64_t k = cnt[u]; k < cnt[u + 1]; k++) {
            const uint32_t *rec = recs + 4 * idx[k];
            if (rec[0] != 1) continue;
            uint32_t best = O_NONE;
            for (uint32_t p = 0; p < L; p++) {
                if (taken[p] || x->dst[p] != rec[2]) continue;
                if (best == O_NONE || x->epoch[p] < x->epoch[best]) best = p;
            }
            if (best == O_NONE) { st[ST_MISS]++; continue; }
            taken[best] = 1;
            N++;
            st[ST_DEL]++;
        }
        /* (3) two-phase delete-and-swap of the adjacency (R-6): dst, bias and epoch move together */
        if (N) {
            uint32_t *P = (uint32_t *)malloc(sizeof(uint32_t) * N);
            uint32_t np = 0;
            for (uint32_t p = 0; p < L; p++) if (taken[p]) P[np++] = p;
            two_phase_delete(x->dst, sizeof(uint32_t), L, P, N, NULL, NULL, NULL);
            two_phase_delete(x->bias, sizeof(uint32_t), L, P, N, NULL, NULL, NULL);
            two_phase_delete(x->epoch, sizeof(uint32_t), L, P, N, NULL, NULL, NULL);
            x->d = L - N;
            free(P);
        }
        free(taken);
        /* (4) the nested structure from the new adjacency (cannot overflow: checked above) */
        radix_build_vertex(x, G->b);
        st[ST_TOUCH]++;
    }
    free(cnt);
    free(idx);
    st[ST_EPOCH] = e;
    if (stats) memcpy(stats, st, sizeof(st));
    return O_OK;
}

/* The adjacency of vertex u: d, then (dst, bias, epoch) of each arc into out[3 * d]
 * (out may be NULL to query d). */
uint32_t ora_radix_adj(const ora_radix *G, uint32_t u, uint32_t *out)
{
    const r_vertex *x = &G->v[u];
    if (out)
        for (uint32_t a = 0; a < x->d; a++) {
            out[3 * a] = x->dst[a];
            out[3 * a + 1] = x->bias[a];
            out[3 * a + 2] = x->epoch ? x->epoch[a] : 0u;
        }
    return x->d;
}

/* three-stage sample (R-17): tag 0 group (bucket, coin vs thr over T), tag 6 subgroup
 * (bucket, coin vs thr over S_i), tag 1 member floor(X c / 2^64).  Returns the dst. */
uint32_t ora_radix_sample(const ora_radix *G, uint32_t u, uint64_t seed, uint32_t w, uint32_t t)
{
    const r_vertex *x = &G->v[u];
    if (x->d == 0) return O_NONE;
    uint32_t r[4];
    draw_oi(seed, w, t, 0, 0, 0, r);
    uint32_t bk = (uint32_t)(((uint64_t)r[0] * x->n) >> 32);
    uint64_t coin = mulhi64(((uint64_t)r[1] << 32) | r[2], x->T);
    const r_group *g = &x->grp[coin < x->grp[bk].thr ? bk : x->grp[bk].alias];
    draw_oi(seed, w, t, 0, 0, 6, r);
    bk = (uint32_t)(((uint64_t)r[0] * g->ns) >> 32);
    coin = mulhi64(((uint64_t)r[1] << 32) | r[2], g->S);
    const r_sub *sb = &g->sub[coin < g->sub[bk].thr ? bk : g->sub[bk].alias];
    draw_oi(seed, w, t, 0, 0, 1, r);
    const uint64_t j = mulhi64(((uint64_t)r[0] << 32) | r[1], sb->c);
    return x->dst[sb->mem[j]];
}

/* DeepWalk (app 0) and PPR (app 2) over a radix structure, as ora_walk (R-13). */
void ora_radix_walk(const ora_radix *G, uint32_t app, uint32_t L, uint64_t seed, uint32_t first_walker,
                    const uint32_t *starts, uint32_t W, uint32_t *paths, uint32_t *lengths, uint64_t *counts,
                    uint64_t stop_thr, uint32_t stop_always, int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < (int64_t)W; i++) {
        const uint32_t w = first_walker + (uint32_t)i;
        uint32_t u = starts ? starts[i] : (uint32_t)(((uint64_t)first_walker + (uint64_t)i) % G->V);
        uint32_t steps = 0;
        if (paths) paths[(size_t)i] = u;
        if (counts && app == 2) {
#ifdef _OPENMP
#pragma omp atomic
#endif
            counts[u]++;
        }
        for (uint32_t t = 0; L == 0xFFFFFFFFu || t < L; t++) {
            if (G->v[u].d == 0) break;
            const uint32_t next = ora_radix_sample(G, u, seed, w, t);
            steps++;
            if (paths) paths[(size_t)(t + 1) * W + (size_t)i] = next;
            u = next;
            if (app == 2) {
                if (counts) {
#ifdef _OPENMP
#pragma omp atomic
#endif
                    counts[u]++;
                }
                if (stop_always) break;
                uint32_t r[4];
                draw(seed, w, t, 0, 3, r);
                if ((((uint64_t)r[0] << 32) | r[1]) < stop_thr) break;
            }
        }
        if (lengths) lengths[i] = steps;
        if (paths && L != 0xFFFFFFFFu)
            for (uint32_t t = steps + 1; t <= L; t++) paths[(size_t)t * W + (size_t)i] = O_NONE;
    }
}

/* canonical dump (R-18), per vertex: u32 d; u32 n; n x {u32 i, u64 thr, u32 alias, u32 ns,
 * ns x {u32 j, u32 c, u64 thr, u32 alias, c x u32 dst}}; u64 T. */
size_t ora_radix_dump(const ora_radix *G, uint8_t *buf, size_t cap)
{
    o_out o = {buf, cap, 0};
    for (uint32_t u = 0; u < G->V; u++) {
        const r_vertex *x = &G->v[u];
        put32(&o, x->d);
        put32(&o, x->n);
        for (uint32_t g = 0; g < x->n; g++) {
            const r_group *gr = &x->grp[g];
            put32(&o, gr->i);
            put64(&o, gr->thr);
            put32(&o, gr->alias);
            put32(&o, gr->ns);
            for (uint32_t s = 0; s < gr->ns; s++) {
                const r_sub *sb = &gr->sub[s];
                put32(&o, sb->j);
                put32(&o, sb->c);
                put64(&o, sb->thr);
                put32(&o, sb->alias);
                for (uint32_t k = 0; k < sb->c; k++) put32(&o, x->dst[sb->mem[k]]);
            }
        }
        put64(&o, x->T);
    }
    return o.pos;
}

/* Materialise the listed vertices of a lazy graph (parallel; no effect on an eager one):
 * measurement support, so timed operations are not billed for first-touch builds. */
void ora_touch(const ora_graph *G, const uint32_t *ids, uint64_t n, int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
    for (int64_t k = 0; k < (int64_t)n; k++)
        if (ids[k] < G->V) (void)vx(G, ids[k]);
}
