// pool.cuh — HEAP_HYBRID: bitmask object pools below a page in front of a TLSF heap.
//
// The paper's §5.3 hybrid: "object buffers to manage object pools for
// allocations smaller than a page (<4kB), and segregated lists for larger allocations", with the
// pools managed by bitmasks (§3.2: a bit per object, allocation finds set
// bits, free sets them back, "coalescence is implicit").  Reading C26 fixes what the
// paper leaves open: pool j holds objects of align*2^j bytes (align*2^j <= 4096), the first half
// of the arena is split evenly between the J pools (each share S a whole number of pages), a
// request of 0 < s < 4096 bytes takes the LOWEST free slot of the smallest pool that holds it,
// a full pool (or any other request) goes to the TLSF heap on [J*S, arena).
//
// Batch semantics stay the canonical ones (frees against the batch-start state, allocs in
// request order), and on the pools they are exactly parallel: within an alloc batch a pool only
// hands out slots, so the k-th request of pool j takes the k-th lowest free slot of the
// batch-start bitmap; requests past the pool's free count, and every other request, keep their
// request order in the TLSF heap's sub-batch.
//
// Layout: one u32 word per 32 slots (bit = 1: free), each pool's words padded to a multiple of
// 32 words so that a 1024-slot superblock never straddles two pools; sbcnt[] holds the free
// count of every superblock (maintained by free and select), so the slots of a batch are found
// by a scan over superblock counts and one warp per touched superblock.
#pragma once
#include "common.cuh"

namespace pool {

constexpr u64 PAGE = 4096;
constexpr int MAXJ = 13;   // align 1 B .. 4096 B

struct Geom {              // passed by value
    int J, alog2;
    u64 S, pool_end, nwords, nsb;
    u64 nslots[MAXJ];
    u64 wbase[MAXJ + 1];   // first word of pool j (multiple of 32)
};

struct Ctr {               // pool-side counters (device)
    u64 nreq;              // n of the current batch (device copy for the count-driven kernels)
    u64 nsb;               // superblock count (scan length)
    u64 frees_null, frees_ok, frees_invalid, frees_double, allocs_ok;
    u64 live_n, live_b, hwm;
    u64 pfree[MAXJ];       // free slots per pool
    u64 take[MAXJ];        // slots the pools hand out in the current alloc batch
    u64 n_tl;              // requests of the current batch handed to the TLSF heap
    u64 runs, nlive_out;   // export / stats scratch
    u64 scan_total;
    u64 nwords;            // word count (scan length of the export)
};

__device__ __forceinline__ int pool_of_word(const Geom &G, u64 w) {
    int j = 0;
    while (j + 1 < G.J && w >= G.wbase[j + 1]) j++;
    return j;
}
// valid-slot mask of word w of pool j (bits past the pool's last slot are never free)
__device__ __forceinline__ u32 valid_mask(const Geom &G, int j, u64 w) {
    const u64 first = (w - G.wbase[j]) * 32;
    if (first >= G.nslots[j]) return 0;
    const u64 left = G.nslots[j] - first;
    return left >= 32 ? 0xFFFFFFFFu : ((1u << left) - 1);
}

// every slot free, superblock counts, per-pool free counts
__global__ void k_init(Geom G, u32 *bits, u32 *sbcnt, Ctr *c) {
    PDL_ENTRY();
    const u64 nth = (u64)gridDim.x * blockDim.x;
    for (u64 w = (u64)blockIdx.x * blockDim.x + threadIdx.x; w < G.nwords; w += nth) {   // nwords % 32 == 0
        const u32 m = valid_mask(G, pool_of_word(G, w), w);
        bits[w] = m;
        const u32 tot = __reduce_add_sync(FULLMASK, (u32)__popc(m));
        if (lane_id() == 0) sbcnt[w >> 5] = tot;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c->nsb = G.nsb;
        c->nwords = G.nwords;
        for (int j = 0; j < G.J; j++) c->pfree[j] = G.nslots[j];
    }
}

// ---- free batch: classify every copy against the batch-start state; pool frees set their bit
// (atomicOr: exactly one copy of an allocated slot sees it clear); the rest go to the TLSF heap
__global__ void __launch_bounds__(256) k_free(const u64 *__restrict__ offs, u64 n, const u64 *n_in, Geom G, u32 *bits,
                                              u32 *sbcnt, Ctr *c, u32 *__restrict__ flags, u64 *__restrict__ toff) {
    PDL_ENTRY();
    __shared__ u64 s_cnt[5 + 2 * MAXJ];      // null, ok, invalid, double, live_b, pfree[J]
    if (n_in) n = *n_in;
    for (int t = threadIdx.x; t < 5 + 2 * MAXJ; t += blockDim.x) s_cnt[t] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) c->nreq = n;
    __syncthreads();
    u64 nnull = 0, nok = 0, ninv = 0, ndbl = 0, lb = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 o = offs[i];
        u32 tl = 0;
        if (o == HEAP_NULL_U64) nnull++;
        else if (o >= G.pool_end) { tl = 1; toff[i] = o - G.pool_end; }
        else {
            const int j = (int)(o / G.S);
            const u64 rel = o - (u64)j * G.S;
            const int sh = G.alog2 + j;
            if (rel & ((1ull << sh) - 1)) ninv++;
            else {
                const u64 t = rel >> sh, w = G.wbase[j] + (t >> 5);
                const u32 bit = 1u << (t & 31);
                const u32 old = atomicOr(&bits[w], bit);
                if (old & bit) ndbl++;
                else {
                    nok++;
                    lb += 1ull << sh;
                    atomicAdd(&sbcnt[w >> 5], 1u);
                    atomicAdd((unsigned long long *)&s_cnt[5 + j], 1ull);
                }
            }
        }
        flags[i] = tl;
    }
    nnull = warp_sum64(nnull); nok = warp_sum64(nok); ninv = warp_sum64(ninv); ndbl = warp_sum64(ndbl); lb = warp_sum64(lb);
    if (lane_id() == 0) {
        if (nnull) atomicAdd((unsigned long long *)&s_cnt[0], nnull);
        if (nok) atomicAdd((unsigned long long *)&s_cnt[1], nok);
        if (ninv) atomicAdd((unsigned long long *)&s_cnt[2], ninv);
        if (ndbl) atomicAdd((unsigned long long *)&s_cnt[3], ndbl);
        if (lb) atomicAdd((unsigned long long *)&s_cnt[4], lb);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_cnt[0]) atomicAdd(&c->frees_null, s_cnt[0]);
        if (s_cnt[1]) {
            atomicAdd(&c->frees_ok, s_cnt[1]);
            atomicAdd(&c->live_n, (u64)0 - s_cnt[1]);
            atomicAdd(&c->live_b, (u64)0 - s_cnt[4]);
        }
        if (s_cnt[2]) atomicAdd(&c->frees_invalid, s_cnt[2]);
        if (s_cnt[3]) atomicAdd(&c->frees_double, s_cnt[3]);
        for (int j = 0; j < G.J; j++)
            if (s_cnt[5 + j]) atomicAdd(&c->pfree[j], s_cnt[5 + j]);
    }
}

// ---- alloc batch ----
// key = pool class j for 0 < s < PAGE (smallest pool whose objects hold s), J for the TLSF heap
__global__ void k_keys(const u64 *__restrict__ sizes, u64 n, const u64 *n_in, Geom G, u32 *__restrict__ key,
                       u32 *__restrict__ val, Ctr *c) {
    PDL_ENTRY();
    if (n_in) n = *n_in;
    if (blockIdx.x == 0 && threadIdx.x == 0) c->nreq = n;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 s = sizes[i];
        u32 k = (u32)G.J;
        if (s > 0 && s < PAGE && G.J > 0) {
            const int cl = (s <= 1) ? 0 : 64 - __clzll(s - 1);     // ceil(log2 s)
            k = (u32)(cl > G.alog2 ? cl - G.alog2 : 0);
        }
        key[i] = k;
        val[i] = (u32)i;
    }
}

// how many requests each pool serves: min(requests of class j, free slots of pool j)
__global__ void k_take(const u32 *__restrict__ coff, Geom G, Ctr *c) {
    PDL_ENTRY();
    u64 ok = 0, lb = 0;
    for (int j = 0; j < G.J; j++) {
        const u64 m = coff[j + 1] - coff[j];
        const u64 t = m < c->pfree[j] ? m : c->pfree[j];
        c->take[j] = t;
        c->pfree[j] -= t;
        ok += t;
        lb += t << (G.alog2 + j);
    }
    c->allocs_ok += ok;
    c->live_n += ok;
    c->live_b += lb;
}

// one warp per superblock: the pool's k-th lowest free slot goes to its k-th request (ranks from
// the exclusive scan of superblock free counts); taken bits are cleared in place
__global__ void __launch_bounds__(256) k_select(Geom G, u32 *bits, u32 *sbcnt, const u32 *__restrict__ sbpre,
                                                const u32 *__restrict__ coff, const u32 *__restrict__ sval,
                                                Ctr *c, u64 *__restrict__ out) {
    PDL_ENTRY();
    const u32 lane = lane_id();
    const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((u64)gridDim.x * blockDim.x) >> 5;
    u64 hw = 0;
    for (u64 sb = gw; sb < G.nsb; sb += nw) {
        const u64 w = sb * 32 + lane;
        const int j = pool_of_word(G, sb * 32);
        const u64 rank0 = (u64)sbpre[sb] - sbpre[G.wbase[j] >> 5];
        const u64 take = c->take[j];
        if (rank0 >= take || sbcnt[sb] == 0) continue;          // warp-uniform
        u32 word = bits[w];
        const u32 pc = __popc(word);
        const u32 ex = warp_incl_scan(pc) - pc;
        u64 rank = rank0 + ex;
        u32 mine = 0;
        const int sh = G.alog2 + j;
        u32 m = word;
        while (m && rank < take) {
            const u32 b = __ffs(m) - 1;
            m &= m - 1;
            const u64 slot = (w - G.wbase[j]) * 32 + b;
            const u64 off = (u64)j * G.S + (slot << sh);
            out[sval[coff[j] + rank]] = off;
            word &= ~(1u << b);
            hw = off + (1ull << sh);
            mine++;
            rank++;
        }
        if (mine) bits[w] = word;
        const u32 tot = __reduce_add_sync(FULLMASK, mine);
        if (lane == 0 && tot) sbcnt[sb] -= tot;
    }
    hw = warp_max64(hw);
    if (lane == 0 && hw) atomicMax(&c->hwm, hw);
}

// requests the pools do not serve, flagged by request index (class J, or rank past the take)
__global__ void k_tl_flags(const u32 *__restrict__ skey, const u32 *__restrict__ sval, const u32 *__restrict__ coff,
                           const u64 *n_dev, Geom G, const Ctr *c, u32 *__restrict__ flags) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (u64)gridDim.x * blockDim.x) {
        const u32 k = skey[p];
        flags[sval[p]] = (k >= (u32)G.J || p - coff[k] >= c->take[k]) ? 1u : 0u;
    }
}
// compact the TLSF share of the requests (request order kept) with their request index
__global__ void k_tl_compact(const u64 *__restrict__ sizes, const u32 *__restrict__ flags, const u32 *__restrict__ pos,
                             const u64 *n_dev, u64 *__restrict__ tsz, u32 *__restrict__ tidx) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        if (flags[i]) { tsz[pos[i]] = sizes[i]; tidx[pos[i]] = (u32)i; }
}
// TLSF results back to request order, shifted by the pools' extent
__global__ void k_tl_scatter(const u64 *__restrict__ tout, const u32 *__restrict__ tidx, const u64 *n_dev, u64 base,
                             u64 *__restrict__ out) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (u64)gridDim.x * blockDim.x) {
        const u64 o = tout[k];
        out[tidx[k]] = (o == HEAP_NULL_U64) ? HEAP_NULL_U64 : o + base;
    }
}

// ---- stats / export ----
// bit masks of run starts / run ends / live slots of word w (runs never cross a pool boundary)
__device__ __forceinline__ void word_marks(const Geom &G, const u32 *bits, u64 w, u32 &st, u32 &en, u32 &lv) {
    const int j = pool_of_word(G, w);
    const u32 b = bits[w];
    const bool first = (w == G.wbase[j]), last = (w + 1 == G.wbase[j + 1]);
    const u32 prev_top = first ? 0u : (bits[w - 1] >> 31);
    const u32 next_low = last ? 0u : (bits[w + 1] & 1u);
    st = b & ~((b << 1) | prev_top);
    en = b & ~((b >> 1) | (next_low << 31));
    lv = ~b & valid_mask(G, j, w);
}
// per-word counts (runs, live slots) for the scans; grand totals into c->runs / c->nlive_out
__global__ void k_marks(Geom G, const u32 *bits, u32 *__restrict__ nrun, u32 *__restrict__ nlive, Ctr *c) {
    PDL_ENTRY();
    u64 r = 0, l = 0;
    for (u64 w = (u64)blockIdx.x * blockDim.x + threadIdx.x; w < G.nwords; w += (u64)gridDim.x * blockDim.x) {
        u32 st, en, lv;
        word_marks(G, bits, w, st, en, lv);
        if (nrun) { nrun[w] = __popc(st); nlive[w] = __popc(lv); }
        r += __popc(st);
        l += __popc(lv);
    }
    r = warp_sum64(r);
    l = warp_sum64(l);
    if (lane_id() == 0 && (r || l)) { atomicAdd(&c->runs, r); atomicAdd(&c->nlive_out, l); }
}
// export: run k -> (start, end) then (start, size); live slot -> (offset, object size)
__global__ void k_emit(Geom G, const u32 *bits, const u32 *__restrict__ prun, const u32 *__restrict__ plive,
                       u64 *fpairs, u64 cap_f, u64 *lpairs, u64 cap_l) {
    PDL_ENTRY();
    for (u64 w = (u64)blockIdx.x * blockDim.x + threadIdx.x; w < G.nwords; w += (u64)gridDim.x * blockDim.x) {
        u32 st, en, lv;
        word_marks(G, bits, w, st, en, lv);
        const int j = pool_of_word(G, w);
        const int sh = G.alog2 + j;
        const u64 base = (u64)j * G.S + (((w - G.wbase[j]) * 32) << sh);
        u64 k = prun[w];
        for (u32 m = st; m; m &= m - 1, k++)
            if (fpairs && k < cap_f) fpairs[2 * k] = base + ((u64)(__ffs(m) - 1) << sh);
        // the k-th end closes the k-th run; a run entering this word from the previous one was
        // counted among the starts before w
        k = prun[w] - ((w != G.wbase[j] && (bits[w - 1] >> 31) && (bits[w] & 1u)) ? 1 : 0);
        for (u32 m = en; m; m &= m - 1, k++)
            if (fpairs && k < cap_f) fpairs[2 * k + 1] = base + ((u64)__ffs(m) << sh);
        k = plive[w];
        for (u32 m = lv; m; m &= m - 1, k++)
            if (lpairs && k < cap_l) { lpairs[2 * k] = base + ((u64)(__ffs(m) - 1) << sh); lpairs[2 * k + 1] = 1ull << sh; }
    }
}
__global__ void k_end_to_size(u64 *fpairs, u64 n) {
    PDL_ENTRY();
    for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (u64)gridDim.x * blockDim.x)
        fpairs[2 * k + 1] -= fpairs[2 * k];
}
__global__ void k_shift_pairs(u64 *pairs, u64 n, u64 base) {
    PDL_ENTRY();
    for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (u64)gridDim.x * blockDim.x)
        pairs[2 * k] += base;
}
// heap_stats of the hybrid: pools + the TLSF heap's own stats (reading C26: largest_free is the
// TLSF heap's; the pools' free runs count as free blocks)
__global__ void k_stats(const heap_stats_t *sub, const Ctr *c, Geom G, u64 arena, u64 align, u64 meta,
                        heap_stats_t *out) {
    PDL_ENTRY();
    const u64 live = c->live_b + sub->live_bytes;
    out->arena_bytes = arena;
    out->align = align;
    out->live_bytes = live;
    out->free_bytes = arena - live;
    out->n_live = c->live_n + sub->n_live;
    out->n_free = c->runs + sub->n_free;
    out->largest_free = sub->largest_free;
    const u64 shw = sub->high_water_end ? sub->high_water_end + G.pool_end : 0;
    out->high_water_end = c->hwm > shw ? c->hwm : shw;
    out->allocs_ok = c->allocs_ok + sub->allocs_ok;
    out->allocs_failed = sub->allocs_failed;
    out->frees_ok = c->frees_ok + sub->frees_ok;
    out->frees_invalid = c->frees_invalid + sub->frees_invalid;
    out->frees_double = c->frees_double + sub->frees_double;
    out->frees_null = c->frees_null + sub->frees_null;
    out->metadata_bytes = meta;
    out->error_flags = sub->error_flags;
}

}  // namespace pool
