// exchange.cuh -- per-vertex state export / import between replicas (replicated
// regime): sharded update application.  Included by update.cu (pool growth helpers).
//
// With P replicas, rank r applies only the records whose source it owns, exports the full
// post-batch state of those touched vertices, and installs every other rank's exports, so the
// replicas end with identical canonical state (per-vertex independent updates).  A
// vertex record (u32 words, internal ids -- replicas share the build's relabelling):
//   u, d, n, T lo, T hi,
//   d x (dst, bias, epoch)                                   (adjacency in order, R-2)
//   n x (k, kind, c, thr lo, thr hi, alias, payload...)      (nonempty groups, ascending k)
//     payload: REGULAR / SPARSE: the c member adjacency indices in list order; ONE: its arc index
// exactly the canonical state of the dump (R-11), so installing it reproduces every result.
// Import rewrites a vertex in place where its arcs, buckets or a same-k member list fit, else
// in fresh pool space (with the usual slack); hub / group indices of imported vertices are
// dropped (rebuilt lazily, like any other route that touches them).
namespace bingo {

struct ExArgs {
    const VHdr *hdr;
    const uint2 *arc;
    const uint32_t *ep;
    const Bucket *bkt;
    const GCan *gcan;
    const uint32_t *midx;
    const uint32_t *inv;      // external -> internal (relabelled graphs), else null
    const uint32_t *ids;      // [n] external ids
    uint32_t n, V;
    uint64_t *words;          // [n + 1] sizes, then (scanned) offsets
    uint32_t *buf;
};

__global__ void k_check_ids(const uint32_t *ids, uint32_t n, uint32_t V, int *bad) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (ids[i] >= V) atomicOr(bad, 1);
}

__global__ void k_ex_sizes(const ExArgs a) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        const uint32_t x = a.ids[i];
        const uint32_t u = x < a.V ? (a.inv ? a.inv[x] : x) : 0u;
        const VHdr h = a.hdr[u];
        uint64_t w = 5 + 3ull * h.d;
        for (uint32_t b = 0; b < h.n; b++) {
            const uint32_t kind = kk_kind(load_bucket(a.bkt + h.bkt_off + b).kk);
            const GCan G = load_gcan(a.gcan + h.bkt_off + b);
            w += 6 + (is_list(kind) ? G.c : (kind == K_ONE ? 1u : 0u));
        }
        a.words[i] = w;
    }
}

// one warp per vertex
__global__ void __launch_bounds__(256) k_ex_fill(const ExArgs a) {
    const uint32_t lane = lane_id();
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < a.n; i += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t x = a.ids[i];
        const uint32_t u = a.inv ? a.inv[x] : x;
        const VHdr h = a.hdr[u];
        uint32_t *r = a.buf + a.words[i];
        if (lane == 0) {
            r[0] = u;
            r[1] = h.d;
            r[2] = h.n;
            r[3] = (uint32_t)h.T;
            r[4] = (uint32_t)(h.T >> 32);
        }
        for (uint32_t p = lane; p < h.d; p += 32) {
            const uint2 e = a.arc[h.adj_off + p];
            r[5 + 3 * p] = e.x;
            r[6 + 3 * p] = e.y;
            r[7 + 3 * p] = a.ep[h.adj_off + p];
        }
        uint64_t pos = 5 + 3ull * h.d;
        for (uint32_t b = 0; b < h.n; b++) {
            const Bucket B = load_bucket(a.bkt + h.bkt_off + b);
            const GCan G = load_gcan(a.gcan + h.bkt_off + b);
            const uint32_t kind = kk_kind(B.kk);
            if (lane == 0) {
                r[pos] = kk_k(B.kk);
                r[pos + 1] = kind;
                r[pos + 2] = G.c;
                r[pos + 3] = (uint32_t)G.thr;
                r[pos + 4] = (uint32_t)(G.thr >> 32);
                r[pos + 5] = B.alias;
                if (kind == K_ONE) r[pos + 6] = G.aux;
            }
            if (is_list(kind))
                for (uint32_t j = lane; j < G.c; j += 32) r[pos + 6 + j] = a.midx[(uint64_t)B.py * 4 + j];
            pos += 6 + (is_list(kind) ? G.c : (kind == K_ONE ? 1u : 0u));
        }
    }
}

struct ImArgs {
    const uint32_t *buf;
    const uint64_t *off;      // [n + 1] record offsets (words)
    uint32_t n;
    VHdr *hdr;
    ThinHdr *thdr;
    uint2 *arc;
    uint32_t *ep;
    Bucket *bkt;
    GCan *gcan;
    uint32_t *midx, *mdst;
    uint64_t *hixo, *gixo;
    uint32_t V;
    double arc_slack, mem_slack;
    uint32_t hot_b, hot_m;
    uint64_t *need;           // [3][n + 1]: fresh arcs, buckets, member units (then scanned)
    const uint64_t *pref;     // [3][n + 1] exclusive prefixes of need
    uint64_t bump[3];         // pool bump pointers at this import
    long long *darcs;         // sum of (new d - old d)
    int *bad;                 // a record that does not parse (bounds)
};

// lane b < n reads incoming group b's header; returns its payload start (words from r)
__device__ __forceinline__ void im_group(const uint32_t *r, uint32_t d, uint32_t n, uint32_t &k, uint32_t &kind,
                                         uint32_t &c, uint64_t &thr, uint32_t &alias, uint64_t &pay) {
    const uint32_t lane = lane_id();
    // group b starts after the payloads of groups < b: a lane-serial walk (n <= 32)
    uint64_t pos = 5 + 3ull * d;
    k = kind = c = alias = 0;
    thr = 0;
    pay = 0;
    for (uint32_t b = 0; b < n; b++) {
        const uint32_t kb = r[pos + 1], cb = r[pos + 2];
        if (lane == b) {
            k = r[pos];
            kind = kb;
            c = cb;
            thr = (uint64_t)r[pos + 3] | ((uint64_t)r[pos + 4] << 32);
            alias = r[pos + 5];
            pay = pos + 6;
        }
        pos += 6 + (is_list(kb) ? cb : (kb == K_ONE ? 1u : 0u));
    }
}

// the local vertex's list group with digit k (member offset and capacity), if any
__device__ __forceinline__ bool im_local_list(const ImArgs &a, const VHdr &h, uint32_t k, uint32_t &moff,
                                              uint32_t &cap) {
    for (uint32_t b = 0; b < h.n; b++) {
        const Bucket B = load_bucket(a.bkt + h.bkt_off + b);
        if (kk_k(B.kk) != k) continue;
        if (!is_list(kk_kind(B.kk))) return false;
        moff = B.py;
        cap = load_gcan(a.gcan + h.bkt_off + b).aux;
        return true;
    }
    return false;
}

// fresh pool space record i needs (0 where it fits in place): one warp per record
__global__ void __launch_bounds__(256) k_im_plan(const ImArgs a) {
    const uint32_t lane = lane_id();
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < a.n; i += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t *r = a.buf + a.off[i];
        const uint64_t len = a.off[i + 1] - a.off[i];
        // a record must parse: vertex < V, at most 32 groups, every group inside the record,
        // kinds / digits / member indices in range (EINVAL before anything is written)
        bool ok = len >= 5 && r[0] < a.V && r[2] <= 32 && 5 + 3ull * r[1] <= len;
        if (ok) {
            uint64_t pos = 5 + 3ull * r[1];
            for (uint32_t b = 0; ok && b < r[2]; b++) {
                ok = pos + 6 <= len && r[pos] < 32 && r[pos + 1] <= K_REGULAR;
                if (!ok) break;
                const uint32_t kb = r[pos + 1], cb = r[pos + 2];
                const uint64_t pl = is_list(kb) ? cb : (kb == K_ONE ? 1u : 0u);
                ok = pos + 6 + pl <= len;
                for (uint64_t j = lane; ok && j < pl; j += 32)
                    if (r[pos + 6 + j] >= r[1]) atomicOr(a.bad, 1);
                pos += 6 + pl;
            }
            ok = ok && pos == len;
        }
        if (!ok) {
            if (lane == 0) atomicOr(a.bad, 1);
            continue;
        }
        const uint32_t u = r[0], d = r[1], n = r[2];
        const VHdr h = a.hdr[u];
        uint32_t k, kind, c, alias;
        uint64_t thr, pay;
        im_group(r, d, n, k, kind, c, thr, alias, pay);
        uint64_t units = 0;
        if (lane < n && is_list(kind)) {
            uint32_t mo, cap;
            if (!(im_local_list(a, h, k, mo, cap) && cap >= c)) units = member_units(c, a.mem_slack);
        }
        units = warp_sum(units);
        if (lane == 0) {
            a.need[i] = h.adj_cap >= d ? 0ull : arc_capacity(d, a.arc_slack);
            a.need[(a.n + 1) + i] = h.ncap >= n ? 0ull : bucket_capacity(n);
            a.need[2 * (a.n + 1) + i] = units;
        }
    }
}

__global__ void __launch_bounds__(256) k_im_install(const ImArgs a) {
    const uint32_t lane = lane_id();
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < a.n; i += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t *r = a.buf + a.off[i];
        const uint32_t u = r[0], d = r[1], n = r[2];
        const uint64_t T = (uint64_t)r[3] | ((uint64_t)r[4] << 32);
        const VHdr h = a.hdr[u];
        uint32_t k, kind, c, alias;
        uint64_t thr, pay;
        im_group(r, d, n, k, kind, c, thr, alias, pay);
        // destinations: in place where the vertex's space fits, else the fresh space of the plan
        const bool fa = h.adj_cap < d, fb = h.ncap < n;
        const uint64_t aoff = fa ? a.bump[0] + a.pref[i] : h.adj_off;
        const uint32_t acap = fa ? (uint32_t)arc_capacity(d, a.arc_slack) : h.adj_cap;
        const uint64_t bo = fb ? a.bump[1] + a.pref[(a.n + 1) + i] : h.bkt_off;
        const uint32_t ncap = fb ? bucket_capacity(n) : h.ncap;
        // member lists: the local same-k list if it is large enough (read before any bucket is
        // overwritten), else fresh units in group order
        uint32_t moff = 0, mcap = 0;
        bool fresh = false;
        if (lane < n && is_list(kind)) {
            uint32_t mo, cap;
            if (im_local_list(a, h, k, mo, cap) && cap >= c) {
                moff = mo;
                mcap = cap;
            } else {
                fresh = true;
                mcap = member_units(c, a.mem_slack) * 4;
            }
        }
        {   // fresh member units: exclusive prefix over the lanes
            const uint32_t v = fresh ? mcap / 4 : 0u;
            uint32_t incl = v;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (uint32_t)o) incl += y;
            }
            if (fresh) moff = (uint32_t)(a.bump[2] + a.pref[2 * (a.n + 1) + i] + (incl - v));
        }
        __syncwarp();
        const long long dold = h.d;
        // adjacency
        for (uint32_t p = lane; p < d; p += 32) {
            a.arc[aoff + p] = make_uint2(r[5 + 3 * p], r[6 + 3 * p]);
            a.ep[aoff + p] = r[7 + 3 * p];
        }
        // members: list groups one at a time, lanes over the entries
        for (uint32_t b = 0; b < n; b++) {
            const uint32_t kb = __shfl_sync(0xffffffffu, kind, b);
            if (!is_list(kb)) continue;
            const uint32_t cb = __shfl_sync(0xffffffffu, c, b), mb = __shfl_sync(0xffffffffu, moff, b);
            const uint64_t pb = __shfl_sync(0xffffffffu, pay, b);
            for (uint32_t j = lane; j < cb; j += 32) {
                const uint32_t idx = r[pb + j];
                a.midx[(uint64_t)mb * 4 + j] = idx;
                a.mdst[(uint64_t)mb * 4 + j] = r[5 + 3 * idx];
            }
        }
        // buckets (walker views, R-4' limits) and headers
        uint32_t one = 0, onedst = 0;
        if (lane < n && kind == K_ONE) {
            one = r[pay];
            onedst = r[5 + 3 * one];
        }
        uint32_t x, y;
        group_view(kind, c, moff, onedst, d, aoff, x, y);
        const uint32_t aux = is_list(kind) ? mcap : (kind == K_ONE ? one : 0u);
        write_buckets(a.bkt, a.gcan, bo, n, lane, k, kind, c, x, y, aux, thr, alias, T);
        if (lane == 0) {
            VHdr nh;
            nh.T = T;
            nh.adj_off = aoff;
            nh.bkt_off = (uint32_t)bo;
            nh.d = d;
            nh.n = (uint8_t)n;
            nh.ncap = (uint8_t)ncap;
            nh.pad = 0;
            nh.adj_cap = acap;
            a.hdr[u] = nh;
            ThinHdr th;
            th.bkt_off = (uint32_t)bo;
            th.n = (uint8_t)n;
            th.flags = (d >= a.hot_b ? 1 : 0) | (d >= a.hot_m ? 2 : 0);
            th.pad1 = 0;
            a.thdr[u] = th;
            if (a.hixo) a.hixo[u] = 0;   // indices of imported vertices: rebuilt lazily
            if (a.gixo) a.gixo[u] = 0;
            atomicAdd(reinterpret_cast<unsigned long long *>(a.darcs), (unsigned long long)((long long)d - dold));
        }
    }
}

}  // namespace bingo
