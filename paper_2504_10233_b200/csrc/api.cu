// api.cu -- allocation, lifetime, inspection (export / digests / info) of libbingo.
#include <cstdio>
#include <cstring>
#include <vector>

#include "bingo.h"
#include "bingo_internal.cuh"
#include "build_common.cuh"

using namespace bingo;

#include <atomic>
static std::atomic<unsigned long long> g_launch_count{0};
void bingo_count_launch(unsigned n) { g_launch_count += n; }

void *bingo_dev_alloc(bingo_graph *g, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (g && g->alloc) return g->alloc(bytes, g->alloc_ctx);
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void bingo_dev_free(bingo_graph *g, void *p) {
    if (!p) return;
    if (g && g->free_) g->free_(p, g->alloc_ctx);
    else cudaFree(p);
}

extern "C" void bingo_destroy(bingo_graph *g) {
    if (!g) return;
    bingo_sq_release(g);
    void *bufs[] = {g->perm, g->inv, g->hdr, g->thdr, g->gcan, g->arc, g->arc_epoch, g->arc_dval, g->bkt, g->mdst, g->midx, g->nbt, g->nbo, g->nbtomb, g->hixo, g->hixt, g->hix, g->dec, g->dmem, g->counters, g->visit, g->dev_flag,
                    g->scratch, g->wscratch, g->vscratch, g->bscratch, g->iscratch, g->fast_scr, g->vslot, g->gixo, g->gixt, g->gix, g->visit32, g->rb_meta};
    for (void *p : bufs) bingo_dev_free(g, p);
    if (g->hscratch) cudaFreeHost(g->hscratch);
    if (g->uhost) cudaFreeHost(g->uhost);
    if (g->fast_out_host) cudaFreeHost(g->fast_out_host);
    if (g->aux_stream) cudaStreamDestroy(g->aux_stream);
    if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
    for (int i = 0; i < 2; i++) {
        if (g->ev_walk[i]) cudaEventDestroy(g->ev_walk[i]);
        if (g->ev_copy[i]) cudaEventDestroy(g->ev_copy[i]);
    }
    if (g->ev_fork) cudaEventDestroy(g->ev_fork);
    if (g->ev_join) cudaEventDestroy(g->ev_join);
    delete g;
}

extern "C" const char *bingo_status_str(bingo_status s) {
    switch (s) {
        case BINGO_OK: return "ok";
        case BINGO_E_INVAL: return "invalid argument";
        case BINGO_E_NOMEM: return "out of device memory";
        case BINGO_E_CUDA: return "CUDA error";
        case BINGO_E_OVERFLOW: return "overflow (n*T >= 2^64 or degree >= 2^32-1)";
        case BINGO_E_STATE: return "graph poisoned by an earlier CUDA error";
    }
    return "unknown status";
}

extern "C" bingo_status bingo_get_info(bingo_graph *g, bingo_info *info, void *stream) {
    if (g) bingo_sq_quiesce(g, (cudaStream_t)stream);
    if (!g || !info) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    unsigned long long c[4];
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemcpyAsync(c, g->counters, sizeof(c), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        g->poisoned = 1;
        return BINGO_E_CUDA;
    }
    info->num_vertices = g->V;
    info->epoch = g->epoch;
    info->num_arcs = g->num_arcs;
    info->arc_pool_used = c[0];
    info->arc_pool_cap = g->arc_cap;
    info->bucket_pool_used = c[1];
    info->bucket_pool_cap = g->bkt_cap;
    info->member_pool_used = 4 * c[2];
    info->member_pool_cap = g->mem_cap;
    info->kernel_launches = g_launch_count.load();
    info->l2_persist_bytes = g->persist_bytes;
    info->hot_degree = ((uint64_t)g->hot_mem_degree << 32) | g->hot_bkt_degree;
    info->update_reruns = g->n_sync_reruns;
    info->device_bytes = (sizeof(VHdr) + sizeof(ThinHdr)) * (uint64_t)g->V + (sizeof(uint2) + 4) * g->arc_cap +
                         (sizeof(Bucket) + sizeof(GCan)) * g->bkt_cap + (g->radix_log2 ? 4ull : 8ull) * g->mem_cap +
                         8ull * g->V +
                         g->scratch_bytes + g->wscratch_bytes + g->vscratch_bytes + g->bscratch_bytes +
                         g->iscratch_bytes;
    return BINGO_OK;
}

// ---------------------------------------------------------------- canonical dump (R-11)
namespace {
struct Out {
    uint8_t *buf;
    size_t cap, pos;
    void u32(uint32_t v) {
        if (buf && pos + 4 <= cap) memcpy(buf + pos, &v, 4);
        pos += 4;
    }
    void u64(uint64_t v) {
        if (buf && pos + 8 <= cap) memcpy(buf + pos, &v, 8);
        pos += 8;
    }
};
}  // namespace

extern "C" bingo_status bingo_export(bingo_graph *g, uint8_t *host_buf, size_t cap, size_t *size_out, void *stream) {
    if (g) bingo_sq_quiesce(g, (cudaStream_t)stream);
    if (!g || !size_out) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    cudaStream_t s = (cudaStream_t)stream;
    if (g->radix_log2) {   // the radix structure's own dump (R-18)
        const bingo_status rs = export_radix(g, host_buf, cap, size_out, s);
        if (rs == BINGO_E_CUDA) g->poisoned = 1;
        return rs;
    }
    unsigned long long c[4];
    std::vector<VHdr> hdr(g->V);
    std::vector<uint32_t> perm(g->V), inv(g->V);   // dumps are in external ids and order (R-11)
    cudaError_t e = cudaMemcpyAsync(c, g->counters, sizeof(c), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && g->V)
        e = cudaMemcpyAsync(hdr.data(), g->hdr, sizeof(VHdr) * g->V, cudaMemcpyDeviceToHost, s);
    for (uint32_t x = 0; x < g->V; x++) perm[x] = inv[x] = x;   // identity unless relabelled
    if (e == cudaSuccess && g->V && g->perm)
        e = cudaMemcpyAsync(perm.data(), g->perm, sizeof(uint32_t) * g->V, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && g->V && g->inv)
        e = cudaMemcpyAsync(inv.data(), g->inv, sizeof(uint32_t) * g->V, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { g->poisoned = 1; return BINGO_E_CUDA; }
    std::vector<uint2> arc(c[0]);
    std::vector<uint32_t> ep(c[0]);
    std::vector<Bucket> bkt(c[1]);
    std::vector<GCan> gc(c[1]);
    std::vector<uint32_t> mem(4 * c[2]);
    std::vector<DecRec> dec(g->float_mode ? g->V : 0);
    std::vector<uint4> dmem(g->float_mode ? g->dmem_cap : 0);
    if (c[0]) e = cudaMemcpyAsync(arc.data(), g->arc, sizeof(uint2) * c[0], cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && c[0]) e = cudaMemcpyAsync(ep.data(), g->arc_epoch, 4 * c[0], cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && c[1]) e = cudaMemcpyAsync(bkt.data(), g->bkt, sizeof(Bucket) * c[1], cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && c[1]) e = cudaMemcpyAsync(gc.data(), g->gcan, sizeof(GCan) * c[1], cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && c[2]) e = cudaMemcpyAsync(mem.data(), g->midx, sizeof(uint32_t) * 4 * c[2], cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && g->float_mode && g->V)
        e = cudaMemcpyAsync(dec.data(), g->dec, sizeof(DecRec) * g->V, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && g->float_mode)
        e = cudaMemcpyAsync(dmem.data(), g->dmem, sizeof(uint4) * g->dmem_cap, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { g->poisoned = 1; return BINGO_E_CUDA; }
    Out o{(host_buf && cap) ? host_buf : nullptr, cap, 0};
    for (uint32_t x = 0; x < g->V; x++) {
        const uint32_t u = inv[x];
        const VHdr &h = hdr[u];
        o.u32(h.d);
        for (uint32_t i = 0; i < h.d; i++) {
            o.u32(perm[arc[h.adj_off + i].x]);
            o.u32(arc[h.adj_off + i].y);
            o.u32(ep[h.adj_off + i]);
        }
        o.u32(h.n);
        for (uint32_t b = 0; b < h.n; b++) {
            const Bucket &B = bkt[(size_t)h.bkt_off + b];
            const GCan &G = gc[(size_t)h.bkt_off + b];
            const uint32_t kind = kk_kind(B.kk);
            o.u32(kk_k(B.kk));
            o.u32(G.c);
            o.u32(kind);
            o.u64(G.thr);
            o.u32(B.alias);
            if (is_list(kind))
                for (uint32_t j = 0; j < G.c; j++) o.u32(mem[(size_t)B.py * 4 + j]);
            else if (kind == K_ONE)
                o.u32(G.aux);
        }
        o.u64(h.T);
        if (g->float_mode) {
            const DecRec &r = dec[u];
            o.u32(r.lam);
            o.u32(r.flags);
            o.u64(r.dmax);
            o.u64(r.thrD);
            o.u32(r.dcnt);
            for (uint32_t j = 0; j < r.dcnt; j++) {
                const uint4 &m = dmem[(size_t)r.doff + j];
                o.u32(m.x);
                o.u64(((uint64_t)m.w << 32) | m.z);
            }
        }
    }
    *size_out = o.pos;
    if (host_buf && o.pos > cap) return BINGO_E_INVAL;
    return BINGO_OK;
}

// ---------------------------------------------------------------- device digests
namespace bingo {
__device__ __forceinline__ uint64_t fnv32(uint64_t h, uint32_t v) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
        h ^= (v >> (8 * i)) & 0xffu;
        h *= 0x100000001b3ull;
    }
    return h;
}
__device__ __forceinline__ uint64_t fnv64(uint64_t h, uint64_t v) {
    h = fnv32(h, (uint32_t)v);
    return fnv32(h, (uint32_t)(v >> 32));
}

__global__ void k_digests(uint32_t V, const VHdr *__restrict__ hdr, const uint2 *__restrict__ arc,
                          const uint32_t *__restrict__ ep, const Bucket *__restrict__ bkt,
                          const GCan *__restrict__ gcan, const uint32_t *__restrict__ midx,
                          const DecRec *__restrict__ dec, const uint4 *__restrict__ dmem, const uint32_t *__restrict__ perm,
                          const uint32_t *__restrict__ inv, uint64_t *__restrict__ out) {
    for (uint32_t xu = blockIdx.x * blockDim.x + threadIdx.x; xu < V; xu += gridDim.x * blockDim.x) {
        const uint32_t u = inv ? inv[xu] : xu;   // digest of external vertex xu over its canonical (external-id) bytes
        const VHdr h = hdr[u];
        uint64_t x = 0xcbf29ce484222325ull;
        x = fnv32(x, h.d);
        for (uint32_t i = 0; i < h.d; i++) {
            const uint2 a = arc[h.adj_off + i];
            x = fnv32(x, perm ? perm[a.x] : a.x);
            x = fnv32(x, a.y);
            x = fnv32(x, ep[h.adj_off + i]);
        }
        x = fnv32(x, h.n);
        for (uint32_t b = 0; b < h.n; b++) {
            const Bucket B = load_bucket(bkt + h.bkt_off + b);
            const GCan G = load_gcan(gcan + h.bkt_off + b);
            const uint32_t kind = kk_kind(B.kk);
            x = fnv32(x, kk_k(B.kk));
            x = fnv32(x, G.c);
            x = fnv32(x, kind);
            x = fnv64(x, G.thr);
            x = fnv32(x, B.alias);
            if (is_list(kind))
                for (uint32_t j = 0; j < G.c; j++) x = fnv32(x, midx[(uint64_t)B.py * 4 + j]);
            else if (kind == K_ONE)
                x = fnv32(x, G.aux);
        }
        x = fnv64(x, h.T);
        if (dec) {
            const DecRec r = dec[u];
            x = fnv32(x, r.lam);
            x = fnv32(x, r.flags);
            x = fnv64(x, r.dmax);
            x = fnv64(x, r.thrD);
            x = fnv32(x, r.dcnt);
            for (uint32_t j = 0; j < r.dcnt; j++) {
                const uint4 m = dmem[(uint64_t)r.doff + j];
                x = fnv32(x, m.x);
                x = fnv64(x, ((uint64_t)m.w << 32) | m.z);
            }
        }
        out[xu] = x;
    }
}
}  // namespace bingo

extern "C" bingo_status bingo_digests(bingo_graph *g, uint64_t *digests, void *stream) {
    if (g) bingo_sq_quiesce(g, (cudaStream_t)stream);
    if (g && g->radix_log2) return BINGO_E_INVAL;
    if (!g || !digests) return BINGO_E_INVAL;
    if (g->poisoned) return BINGO_E_STATE;
    if (!g->V) return BINGO_OK;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned blocks = (unsigned)std::min<uint64_t>(((uint64_t)g->V + 255) / 256, 148ull * 16);
    k_digests<<<blocks, 256, 0, s>>>(g->V, g->hdr, g->arc, g->arc_epoch, g->bkt, g->gcan, g->midx,
                                                 g->float_mode ? g->dec : nullptr, g->dmem, g->perm, g->inv, digests);
    bingo_count_launch();
    if (cudaGetLastError() != cudaSuccess) { g->poisoned = 1; return BINGO_E_CUDA; }
    return BINGO_OK;
}
