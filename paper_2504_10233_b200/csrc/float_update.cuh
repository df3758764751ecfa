// float_update.cuh -- batched updates of floating-point-bias graphs (reading R-16; included by
// update.cu).  Each vertex keeps the lambda of its build.  An inserted real bias w
// becomes the arc's radix bias I = floor(fl(w lambda)) (Eq.3-9 unchanged; I = 0 joins no radix
// group) and its decimal part D = floor((fl(w lambda) - I) 2^52), stored per arc in arc_dval and
// moved with the arc by every relocation and delete-and-swap of the integer pipeline.  After the
// integer pipeline, the decimal group of every touched vertex is recomputed from its live arcs in
// ascending adjacency order (members, W_D, D_max, thrD, flags), exactly as the build does.
#pragma once

namespace bingo {

// per record: the integer part into the record's bias field, D into dins (inserts only)
__global__ void k_float_scale(uint4 *__restrict__ recs, const double *__restrict__ wf, uint64_t n, uint32_t V,
                              const DecRec *__restrict__ dec, uint64_t *__restrict__ dins, UpdCounters *cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 r = recs[i];
        uint64_t D = 0;
        if (r.x == 0u && r.y < V) {
            const double w = wf[i];
            uint32_t I = 0;
            if (!(w > 0.0) || !(w <= 1e300)) atomicOr(&cnt->flag, 1);          // EINVAL
            else if (!scale_one(w, dec[r.y].lam, I, D)) atomicOr(&cnt->flag, 4);   // EOVERFLOW: I >= 2^32
            r.w = I;
        } else {
            r.w = 0;
        }
        recs[i] = r;
        dins[i] = D;
    }
}

// per touched vertex: decimal-member capacity for the batch (an upper bound: members before the
// batch + inserts with D > 0); a vertex that outgrows its region moves to a new one from the
// decimal-member bump pointer (counters[3]); the host grows the pool before anything is mutated
__global__ void k_float_plan(const uint4 *__restrict__ recs, const uint32_t *__restrict__ sval,
                             const uint32_t *__restrict__ seg, const uint32_t *__restrict__ tv, uint64_t ntouch,
                             const uint64_t *__restrict__ dins, const DecRec *__restrict__ dec,
                             unsigned long long *bump, uint32_t *__restrict__ fdoff, uint32_t *__restrict__ fdcap) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntouch; t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t add = 0;
        for (uint32_t p = seg[t]; p < seg[t + 1]; p++) {
            const uint32_t ri = sval[p];
            if (recs[ri].x == 0u && dins[ri]) add++;
        }
        const DecRec r = dec[tv[t]];
        const uint32_t need = r.dcnt + add;
        if (need > r.pad2) {
            const uint32_t cap = dec_capacity(need);
            fdoff[t] = (uint32_t)atomicAdd(&bump[3], (unsigned long long)cap);
            fdcap[t] = cap;
        } else {
            fdoff[t] = r.doff;
            fdcap[t] = r.pad2;
        }
    }
}

// per touched vertex (warp): the decimal group from the post-batch arcs (R-15/R-16)
__global__ void k_float_fixup(const uint32_t *__restrict__ tv, uint64_t ntouch, const VHdr *__restrict__ hdr,
                              const uint2 *__restrict__ arc, const uint64_t *__restrict__ arc_dval,
                              const uint32_t *__restrict__ fdoff, const uint32_t *__restrict__ fdcap,
                              DecRec *__restrict__ dec, uint4 *__restrict__ dmem) {
    const uint32_t lane = lane_id();
    const uint64_t warps = ((uint64_t)blockDim.x >> 5) * gridDim.x;
    for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntouch; t += warps) {
        const uint32_t u = tv[t];
        const VHdr h = hdr[u];
        const uint32_t base = fdoff[t];
        unsigned __int128 wd = 0;
        uint64_t dmax = 0;
        uint32_t run = 0;
        for (uint32_t c0 = 0; c0 < h.d; c0 += 32) {
            const uint32_t i = c0 + lane;
            uint64_t D = 0;
            uint32_t v = 0;
            if (i < h.d) {
                D = arc_dval[h.adj_off + i];
                v = arc[h.adj_off + i].x;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, D != 0);
            if (D) dmem[(uint64_t)base + run + __popc(bal & lanemask_lt())] = make_uint4(i, v, (uint32_t)D, (uint32_t)(D >> 32));
            run += __popc(bal);
            wd += D;
            dmax = D > dmax ? D : dmax;
        }
        wd = warp_sum128(wd);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t m = __shfl_xor_sync(0xffffffffu, dmax, o);
            dmax = m > dmax ? m : dmax;
        }
        if (lane == 0) {
            const unsigned __int128 wi = h.T;    // sum of the integer parts (Eq.4)
            DecRec r = dec[u];
            uint32_t fl = 0;
            if (h.d && !((unsigned __int128)(h.d - 1) * wd < (wi << 52))) fl |= 1u;   // P:377 constraint unmet
            if (wi == 0 && h.d) fl |= 2u;                                              // integer part empty
            r.thrD = wd == 0 ? 0ull : (wi == 0 ? ~0ull : frac64(wd, (wi << 52) + wd));
            r.dmax = dmax;
            r.doff = base;
            r.dcnt = run;
            r.flags = (uint8_t)fl;
            r.pad2 = fdcap[t];
            dec[u] = r;
        }
    }
}

}  // namespace bingo
