// buddy.cuh — binary buddy as level-by-level scans.
//
// State: for each order t (block = 2^t units) the free block starts, sorted, stored back to
// back with offsets ctr->bud_off[t] (a CSR by order).
//
// Free phase (merge): for t = 0..K the order-t free set is the merge of the
// resident order-t blocks, the freed order-t blocks and the blocks promoted from order t-1.
// In that sorted list two buddies (a, a + 2^t with bit t of a clear) are adjacent; each such
// pair is removed and its parent a is promoted to order t+1.  What stays is final for order t.
// The result is the canonical set of maximal aligned free blocks (lemma L2), i.e. the same
// set the one-by-one merge of the oracle produces.
//
// Alloc phase (split, "the first is split further"), lemma L6:
//   bottom-up, order t: demands D_t = time-ordered merge of the order-t requests and the
//   borrows from order t-1.  The first n_t demands take the batch-start order-t blocks in
//   address order; excess demand x (0-based) is served by borrow floor(x/2) from order t+1:
//   the low half for even x, +2^t for odd x.  Order t issues ceil(x_t/2) borrows, each
//   carrying the time of the demand that triggered it.  Demands the top order cannot serve
//   fail, and failure propagates down (it is absorbing: once orders >= t are empty they stay
//   empty for the rest of the batch).
//   top-down, order t = K..0: addresses flow from each demand to its request or borrow.
//   Leftover: if x_t is odd and its last borrow succeeded, that borrow's high half stays free.
// Both passes run in one CTA per heap (levels are dependent; the work per level is spread
// over 1024 threads with merge-path partitions).
#pragma once
#include "common.cuh"

namespace buddy {

constexpr int NT = 1024;
constexpr int FREE_CAP = 16384;     // per-level staging capacity (units) of k_free_levels
constexpr size_t FREE_SMEM = 3 * FREE_CAP * sizeof(u32);
constexpr int ALLOC_CAP = 49152;    // per-level staging capacity (u32 words) of k_alloc_levels
constexpr size_t ALLOC_SMEM = ALLOC_CAP * sizeof(u32);
constexpr u32 BORROW = 0x80000000u;
constexpr u64 FAIL = 0xFFFFFFFFFFFFFFFFull;
#ifndef BUDDY_TIMING
#define BUDDY_TIMING 0
#endif

// CTA-wide copy global -> shared with 8 independent loads per thread in flight (a plain
// strided loop would serialise one global round trip per element)
template <typename TS, typename TD>
__device__ __forceinline__ void cta_copy(TD *dst, const TS *src, u64 n64) {
    const u32 n = (u32)n64, wb = threadIdx.x & ~31u;
    if (n <= NT) {                                   // one element per thread at most (most levels)
        if (threadIdx.x < n) dst[threadIdx.x] = (TD)src[threadIdx.x];
        return;
    }
    for (u32 base = 0; base < n; base += 8 * NT) {
        // warp-uniform step count: warps past the end skip the unrolled steps instead of running
        // them predicated off (the kernel is issue-bound on its one SM)
        if (base + wb >= n) break;                  // warp-uniform: nothing left for this warp
        const u32 kw = min(8u, (n - base - wb + NT - 1) / NT);
        TS v[8];
#pragma unroll
        for (u32 k = 0; k < 8; k++) {
            const u32 i = base + k * NT + threadIdx.x;
            if (k < kw) v[k] = i < n ? src[i] : (TS)0;
        }
#pragma unroll
        for (u32 k = 0; k < 8; k++) {
            const u32 i = base + k * NT + threadIdx.x;
            if (k < kw && i < n) dst[i] = (TD)v[k];
        }
    }
}

// CTA-wide merge of two sorted arrays (ties: a first) into out; all threads call.
template <typename TA, typename TO>
__device__ void cta_merge(const TA *a, u64 na, const TA *b, u64 nb, TO *out) {
    const u64 n = na + nb;
    const u64 per = (n + NT - 1) / NT;
    u64 diag = (u64)threadIdx.x * per;
    if (diag < n) {
        u64 lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
        while (lo < hi) {
            u64 mid = (lo + hi) >> 1;
            if (a[mid] <= b[diag - mid - 1]) lo = mid + 1; else hi = mid;
        }
        u64 i = lo, j = diag - lo;
        for (u64 k = 0; k < per && diag + k < n; k++) {
            bool ta = (j >= nb) || (i < na && a[i] <= b[j]);
            out[diag + k] = (TO)(ta ? a[i++] : b[j++]);
        }
    }
}

// CTA-wide merge of two sorted u64 arrays (ties: a first) into out; all threads call.
__device__ void cta_merge_u64(const u64 *a, u64 na, const u64 *b, u64 nb, u64 *out) {
    const u64 n = na + nb;
    const u64 per = (n + NT - 1) / NT;
    u64 diag = (u64)threadIdx.x * per;
    if (diag < n) {
        u64 lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
        while (lo < hi) {
            u64 mid = (lo + hi) >> 1;
            if (a[mid] <= b[diag - mid - 1]) lo = mid + 1; else hi = mid;
        }
        u64 i = lo, j = diag - lo;
        for (u64 k = 0; k < per && diag + k < n; k++) {
            bool ta = (j >= nb) || (i < na && a[i] <= b[j]);
            out[diag + k] = ta ? a[i++] : b[j++];
        }
    }
}

// CTA-wide merge by time of (tm, src) pairs
__device__ void cta_merge_tm(const u32 *at, const u32 *as, u64 na, const u32 *bt, const u32 *bsrc, u64 nb,
                             u32 *ot, u32 *os) {
    const u64 n = na + nb;
    const u64 per = (n + NT - 1) / NT;
    u64 diag = (u64)threadIdx.x * per;
    if (diag < n) {
        u64 lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
        while (lo < hi) {
            u64 mid = (lo + hi) >> 1;
            if (at[mid] <= bt[diag - mid - 1]) lo = mid + 1; else hi = mid;
        }
        u64 i = lo, j = diag - lo;
        for (u64 k = 0; k < per && diag + k < n; k++) {
            bool ta = (j >= nb) || (i < na && at[i] <= bt[j]);
            if (ta) { ot[diag + k] = at[i]; os[diag + k] = as[i]; i++; }
            else { ot[diag + k] = bt[j]; os[diag + k] = bsrc[j]; j++; }
        }
    }
}

// CTA-wide stream compaction helper: each thread handles a contiguous chunk; returns the
// number of kept elements.  keep(i) decides, emit(i, pos) writes.
template <typename Keep, typename Emit>
__device__ u64 cta_compact(u64 n, Keep keep, Emit emit, u32 *sm) {
    const u64 per = (n + NT - 1) / NT;
    const u64 b = (u64)threadIdx.x * per;
    u32 cnt = 0;
    for (u64 k = 0; k < per && b + k < n; k++) cnt += keep(b + k) ? 1 : 0;
    u32 tot;
    u32 pos = block_excl_scan<NT>(cnt, sm, &tot);
    for (u64 k = 0; k < per && b + k < n; k++)
        if (keep(b + k)) emit(b + k, (u64)pos++);
    return tot;
}

// ------------------------------------------------------------------ free phase ----
// freed blocks: fr_start (units) grouped by order via fr_off[t] (sorted within order)
__global__ void __launch_bounds__(NT) k_free_levels(const u64 *__restrict__ old_list, u64 *__restrict__ new_list,
                                                    const u64 *__restrict__ fr, const u32 *__restrict__ fr_off,
                                                    u64 *bufA, u64 *bufB, u64 *promo, int K, DevCtr *ctr) {
    PDL_ENTRY();
    __shared__ u32 sm[33];
    __shared__ u64 ooff[41];
    __shared__ u64 s_np, s_out;
    __shared__ u32 foff[42];
    if (threadIdx.x <= (unsigned)K + 1) {
        ooff[threadIdx.x] = ctr->bud_off[threadIdx.x];
        foff[threadIdx.x] = fr_off[threadIdx.x];
    }
    if (threadIdx.x == 0) { s_np = 0; s_out = 0; }
    __syncthreads();
    extern __shared__ u32 stage[];      // 3 x FREE_CAP units (addresses < 2^32 units)
    u32 *X = stage, *Y = stage + FREE_CAP, *Z = stage + 2 * FREE_CAP;
    for (int t = 0; t <= K; t++) {
        const u64 *old_t = old_list + ooff[t];
        const u64 n_old = ooff[t + 1] - ooff[t];
        const u64 *fr_t = fr + foff[t];
        const u64 n_fr = foff[t + 1] - foff[t];
        const u64 n_pr = s_np;
        const u64 n = n_old + n_fr + n_pr;
        const u64 bit = 1ull << t;
        const u64 out0 = s_out;
        if (n == 0) {                    // empty level: nothing to merge, keep the offsets
            if (threadIdx.x == 0) { ctr->bud_off[t] = out0; ctr->bud_cnt[t] = 0; }
            continue;
        }
        u64 ns, np;
        if (n <= (u64)FREE_CAP) {
            // stage the level in shared memory (coalesced), merge there: binary searches at
            // shared-memory latency instead of global
            cta_copy(X, old_t, n_old);                     // 8 independent loads in flight per thread
            cta_copy(X + n_old, fr_t, n_fr);
            cta_copy(X + n_old + n_fr, promo, n_pr);
            __syncthreads();
            cta_merge(X, n_old, X + n_old, n_fr, Y);
            __syncthreads();
            cta_merge(Y, n_old + n_fr, X + n_old + n_fr, n_pr, Z);
            __syncthreads();
            // one fused pass: flags for survivors and promotions (bit masks over this thread's
            // contiguous chunk of <= 16 elements), one packed block scan, then the writes
            const u32 nn = (u32)n, per = (nn + NT - 1) / NT, b0 = threadIdx.x * per;
            const u32 bt = (u32)bit;
            const bool top = (t >= K);
            u32 ms = 0, mp = 0;
            for (u32 k = 0; k < per; k++) {
                const u32 i = b0 + k;
                if (i >= nn) break;
                const u32 zi = Z[i];
                const bool lo = !top && !(zi & bt) && i + 1 < nn && Z[i + 1] == zi + bt;
                const bool hi = !top && (zi & bt) && i > 0 && Z[i - 1] == zi - bt;
                if (!lo && !hi) ms |= 1u << k;
                if (lo) mp |= 1u << k;
            }
            u32 tot;
            const u32 pos = block_excl_scan<NT>(__popc(ms) | (__popc(mp) << 16), sm, &tot);
            u32 ps = pos & 0xFFFF, pp = pos >> 16;
            for (u32 k = 0; k < per; k++) {
                const u32 i = b0 + k;
                if ((ms >> k) & 1) new_list[out0 + ps++] = Z[i];
                if ((mp >> k) & 1) promo[pp++] = Z[i];
            }
            ns = tot & 0xFFFF;
            np = tot >> 16;
            __syncthreads();
        } else {
            cta_merge_u64(old_t, n_old, fr_t, n_fr, bufA);
            __syncthreads();
            cta_merge_u64(bufA, n_old + n_fr, promo, n_pr, bufB);
            __syncthreads();
            auto paired_lo = [&](u64 i) { return t < K && !(bufB[i] & bit) && i + 1 < n && bufB[i + 1] == bufB[i] + bit; };
            auto paired_hi = [&](u64 i) { return t < K && (bufB[i] & bit) && i > 0 && bufB[i - 1] == bufB[i] - bit; };
            // survivors -> new list (order t)
            ns = cta_compact(n, [&](u64 i) { return !paired_lo(i) && !paired_hi(i); },
                             [&](u64 i, u64 p) { new_list[out0 + p] = bufB[i]; }, sm);
            __syncthreads();
            // promotions -> promo (read by the next level; bufB still holds this level)
            np = cta_compact(n, [&](u64 i) { return paired_lo(i); },
                             [&](u64 i, u64 p) { promo[p] = bufB[i]; }, sm);
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            ctr->bud_off[t] = out0;
            ctr->bud_cnt[t] = ns;
            s_out = out0 + ns;
            s_np = np;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ctr->bud_off[K + 1] = s_out;
        ctr->bud_total = s_out;
    }
}

// ------------------------------------------------ free phase, parallel form (default) ----
// The buddy free set is the set of maximal free nodes of the buddy trees (lemma L2): every node
// whose whole span is free and whose parent's is not.  Inside a maximal run of free space [x, y)
// those nodes are exactly the greedy decomposition — at x the largest 2^s with x % 2^s == 0 and
// x + 2^s <= y, repeat — and it never crosses a root boundary (the roots are the binary digits of
// the arena, largest first, so each root start is a multiple of twice its size and every later
// root is smaller).  So the merge that k_free_levels does level by level (27 dependent levels at
// config 4) is computed in one pass of independent steps: the free set, kept in address order
// beside the per-order lists (bq: start << 6 | order, maintained by both phases), merged with the
// freed blocks, coalesced into maximal runs (the fits path's kernels), each run decomposed, the
// result grouped by order (stable one-pass sort) for the alloc phase.
__device__ __forceinline__ int bud_step(u64 x, u64 y) {   // order of the greedy block at x in [x, y)
    const int a = x ? __ffsll((long long)x) - 1 : 63;
    const int b = 63 - __clzll(y - x);
    return a < b ? a : b;
}
// merge of the address-ordered free set (packed start << 6 | order) with the freed blocks
// (start, end), both sorted by start (disjoint), into (start, end) arrays (merge path)
constexpr int QSH = 6;
__global__ void __launch_bounds__(256) k_bud_merge(const u64 *__restrict__ q, const DevCtr *ctr,
                                                   const u64 *__restrict__ bs, const u64 *__restrict__ be,
                                                   const u64 *nb_dev, u64 *__restrict__ os, u64 *__restrict__ oe,
                                                   u64 *total) {
    PDL_ENTRY();
    const u64 na = ctr->bud_qn, nb = *nb_dev, n = na + nb;
    if (blockIdx.x == 0 && threadIdx.x == 0) *total = n;
    constexpr int IPT = 8;
    const u64 nchunks = (n + IPT - 1) / IPT;
    for (u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += (u64)gridDim.x * blockDim.x) {
        const u64 diag = c * IPT;
        u64 lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
        while (lo < hi) {
            const u64 mid = (lo + hi) >> 1;
            if ((q[mid] >> QSH) <= bs[diag - mid - 1]) lo = mid + 1; else hi = mid;
        }
        u64 i = lo, j = diag - lo;
#pragma unroll
        for (int k = 0; k < IPT; k++) {
            const u64 o = diag + k;
            if (o >= n) break;
            const u64 qa = i < na ? q[i] : 0;
            const bool ta = (j >= nb) || (i < na && (qa >> QSH) <= bs[j]);
            if (ta) { os[o] = qa >> QSH; oe[o] = (qa >> QSH) + (1ull << (qa & 63)); i++; }
            else { os[o] = bs[j]; oe[o] = be[j]; j++; }
        }
    }
}
// after an alloc phase: the surviving blocks of the address-ordered set (each order lost a prefix:
// keep iff start >= the order's first surviving start), then the leftovers inserted in place
__global__ void k_bud_qflags(const u64 *__restrict__ q, const DevCtr *ctr, u32 *__restrict__ flags) {
    PDL_ENTRY();
    const u64 n = ctr->bud_qn;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 v = q[i];
        flags[i] = (v >> QSH) >= ctr->bud_thr[v & 63] ? 1u : 0u;
    }
}
__global__ void k_bud_qwrite(const u64 *__restrict__ q, const u32 *__restrict__ flags, const u32 *__restrict__ pos,
                             const u64 *kept_dev, int K, u64 *__restrict__ out, DevCtr *ctr) {
    PDL_ENTRY();
    __shared__ u64 lv[48];
    __shared__ int nl;
    if (threadIdx.x == 0) {
        int c = 0;
        for (int t = 0; t <= K; t++)
            if (ctr->bud_left[t] != FAIL) lv[c++] = (ctr->bud_left[t] << QSH) | (u64)t;
        nl = c;
    }
    __syncthreads();
    const u64 n = ctr->bud_qn, kept = *kept_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        if (!flags[i]) continue;
        const u64 v = q[i];
        u64 d = 0;
        for (int c = 0; c < nl; c++) d += (lv[c] >> QSH) < (v >> QSH) ? 1 : 0;
        out[pos[i] + d] = v;
    }
    if (blockIdx.x == 0 && threadIdx.x < (unsigned)nl) {
        const u64 v = lv[threadIdx.x], st = v >> QSH;
        u64 lo = 0, hi = n;                  // kept blocks below it: pos at the first start >= st
        while (lo < hi) { const u64 m = (lo + hi) >> 1; if ((q[m] >> QSH) < st) lo = m + 1; else hi = m; }
        const u64 kb = lo < n ? pos[lo] : kept;
        u64 d = 0;
        for (int c = 0; c < nl; c++) d += (lv[c] >> QSH) < st ? 1 : 0;
        out[kb + d] = v;
    }
    // the new length is published by the last CTA to finish: every CTA reads the old one at its
    // start, and a CTA scheduled after block 0 had finished would otherwise see the new length
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&ctr->bud_qdone, 1u) == gridDim.x - 1) {
            ctr->bud_qn = kept + (u64)nl;
            ctr->bud_qdone = 0;
        }
    }
}

// blocks of each maximal run's greedy decomposition
__global__ void k_bud_count(const u64 *__restrict__ rs, const u64 *__restrict__ re, const u64 *R_dev,
                            u32 *__restrict__ cnt) {
    PDL_ENTRY();
    const u64 R = *R_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += (u64)gridDim.x * blockDim.x) {
        u64 x = rs[i];
        const u64 y = re[i];
        u32 c = 0;
        while (x < y) { x += 1ull << bud_step(x, y); c++; }
        cnt[i] = c;
    }
}
// write the decomposition in address order: start (units) and the order as the sort key
// (launched with prims::OS_NT threads: it also counts the order digits of what it writes — the
// one-pass onesweep sort by order that follows needs no histogram launch)
__global__ void __launch_bounds__(256) k_bud_write(const u64 *__restrict__ rs, const u64 *__restrict__ re,
                                                   const u64 *R_dev, const u32 *__restrict__ pos,
                                                   u64 *__restrict__ ostart, u32 *__restrict__ okey,
                                                   u32 *__restrict__ oval, u64 *__restrict__ oq, u64 cap, DevCtr *ctr) {
    PDL_ENTRY();
    __shared__ u32 hh[1][256];
    hh[0][threadIdx.x] = 0;
    __syncthreads();
    const u64 R = *R_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += (u64)gridDim.x * blockDim.x) {
        u64 x = rs[i];
        const u64 y = re[i];
        u64 o = pos[i];
        while (x < y) {
            const int t = bud_step(x, y);
            if (o < cap) {
                ostart[o] = x; okey[o] = (u32)t; oval[o] = (u32)o; oq[o] = (x << QSH) | (u64)t;
                atomicAdd(&hh[0][t], 1u);
            } else atomicOr(&ctr->error_flags, (u64)ERR_CAP_FREE);
            x += 1ull << t;
            o++;
        }
    }
    prims::os_hist_finish(hh, 1, ctr);
}
// order-grouped (stable: address order inside an order) -> the new per-order lists
// (block 0 also writes the per-order offsets and counts: the keys were just sorted by one 8-bit
// onesweep pass, whose digit-histogram scan is still in ctr->os_gbase[0] — the first position with
// order >= t is its entry t)
__global__ void k_bud_lists(const u32 *__restrict__ idx, const u64 *n_dev, const u64 *__restrict__ start,
                            u64 *__restrict__ out, int K, DevCtr *ctr) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (u64)gridDim.x * blockDim.x)
        out[p] = start[idx[p]];
    if (blockIdx.x == 0) {
        const int t = threadIdx.x;
        if (t <= K + 1) ctr->bud_off[t] = (t <= K) ? (u64)ctr->os_gbase[0][t] : n;
        __syncthreads();
        if (t <= K) ctr->bud_cnt[t] = ctr->bud_off[t + 1] - ctr->bud_off[t];
        if (t == 0) { ctr->bud_total = n; ctr->bud_qn = n; }
    }
}

// freed (start, end) -> sort key = order, payload = index
__global__ void k_free_orders(const u64 *__restrict__ vs, const u64 *__restrict__ ve, const u64 *nv_dev,
                              u32 *__restrict__ key, u32 *__restrict__ val) {
    PDL_ENTRY();
    const u64 nv = *nv_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (u64)gridDim.x * blockDim.x) {
        key[i] = (u32)flog2(ve[i] - vs[i]);
        val[i] = (u32)i;
    }
}
__global__ void k_gather_u64(const u64 *__restrict__ src, const u32 *__restrict__ idx, const u64 *n_dev,
                             u64 *__restrict__ dst) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

// ------------------------------------------------------------------ alloc phase ----
// r -> order key (K+1 = fail bucket)
// (launched with prims::OS_NT threads: it also counts the order digits — the one-pass onesweep sort
// that follows needs no histogram launch)
__global__ void __launch_bounds__(256) k_alloc_orders(const u64 *__restrict__ sizes, u64 n, const u64 *n_in, int alog2,
                                                      u64 A_u, int K, u32 *__restrict__ key, u32 *__restrict__ val,
                                                      u64 *n_dev, DevCtr *ctr) {
    PDL_ENTRY();
    __shared__ u32 hh[1][256];
    hh[0][threadIdx.x] = 0;
    __syncthreads();
    if (n_in) n = *n_in;
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_dev = n;
    const u64 amask = (1ull << alog2) - 1;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 s = sizes[i];
        u64 r = (s >> alog2) + ((s & amask) != 0);
        u32 k = (u32)K + 1;
        if (s != 0 && r <= A_u) {
            u32 kk = (r <= 1) ? 0u : (u32)(flog2(r - 1) + 1);   // ceil(log2 r)
            if (kk <= (u32)K && (1ull << kk) <= A_u) k = kk;
        }
        key[i] = k;
        val[i] = (u32)i;
        atomicAdd(&hh[0][k], 1u);
    }
    prims::os_hist_finish(hh, 1, ctr);
}

// Bottom-up + top-down L6 in one CTA.
//   req_t/req_off: request indices sorted by (order, time); blocks: old per-order lists.
//   dtm/dsrc: pool for the demand streams, daddr: their addresses; baddr: borrow addresses.
__global__ void __launch_bounds__(NT) k_alloc_levels(const u32 *__restrict__ req, const u32 *__restrict__ req_off,
                                                     const u64 *__restrict__ old_list, u64 *__restrict__ new_list,
                                                     u32 *dtm, u32 *dsrc, u64 *daddr, u64 *baddr,
                                                     u32 *btm, u32 *bsrc, u64 *__restrict__ out_u, int K,
                                                     DevCtr *ctr) {
    PDL_ENTRY();
    extern __shared__ __align__(16) u32 astage_td[];   // the staging area, reused by the top-down
    __shared__ u64 ooff[41];
    __shared__ u64 doff[42], boff[42];
    __shared__ u32 ro[42];
    if (threadIdx.x <= (unsigned)K + 1) ooff[threadIdx.x] = ctr->bud_off[threadIdx.x];
    // request offsets by order: req_off, or (nullptr) the digit-histogram scan of the one-pass order
    // sort that just ran (ctr->os_gbase[0]) with the request count in ctr->tmp[0]
    if (threadIdx.x <= (unsigned)K + 2)
        ro[threadIdx.x] = req_off ? req_off[threadIdx.x]
                                  : (threadIdx.x <= (unsigned)K + 1 ? ctr->os_gbase[0][threadIdx.x] : (u32)ctr->tmp[0]);
    __syncthreads();
    // requests of the fail bucket
    for (u64 i = ro[K + 1] + threadIdx.x; i < ro[K + 2]; i += NT) out_u[req[i]] = FAIL;
#if BUDDY_TIMING
    long long tb0 = clock64();
#endif
    // ---- bottom-up ----
    // The level scalars (borrows in, demand / borrow offsets) are uniform: every thread keeps them
    // in registers, so a level costs two barriers (staged inputs, merged demands) and a level with
    // no demand none.
    u64 nb = 0, dacc = 0, bacc = 0;
    for (int t = 0; t <= K; t++) {
        const u64 n_t = ooff[t + 1] - ooff[t];
        const u64 nr = ro[t + 1] - ro[t];
        const u64 nd = nr + nb;
        const u64 x = nd > n_t ? nd - n_t : 0;
        const u64 nbor = (t < K) ? (x + 1) / 2 : 0;
        if (threadIdx.x == 0) { doff[t] = dacc; boff[t] = bacc; }
#if BUDDY_TIMING == 2
        if (threadIdx.x == 0 && t > 0) { const long long t1 = clock64(); ctr->eng[t - 1] += t1 - tb0; tb0 = t1; }
#endif
        if (nd == 0) { nb = 0; continue; }
        const u32 *rq = req + ro[t];
        u32 *Dt = dtm + dacc, *Ds = dsrc + dacc;
        // direct requests: time = request index, src = request index; merged by time with the
        // borrows from t-1 (btm, bsrc); staged in shared memory when the level fits, and then the
        // merge itself writes the borrows to t+1: borrow j carries the time of demand n_t + 2j
        if (nb == 0 || nr == 0) {
            // one stream only (level 0 has no borrows, the levels above the largest request order
            // have no requests): the demands are that stream, no merge.  Requests: time = src =
            // request index; borrows from t-1: (btm, bsrc), read before this level rewrites them
            const u32 nd_ = (u32)nd, nt_ = (u32)n_t, nbor_ = (u32)nbor;
            const u32 *tin = nb == 0 ? rq : btm, *sin = nb == 0 ? rq : bsrc;
            for (u32 o = threadIdx.x; o < nd_; o += NT) { Dt[o] = tin[o]; Ds[o] = sin[o]; }
            __syncthreads();                       // (btm may be rewritten below: read Dt instead)
            for (u32 jb = threadIdx.x; jb < nbor_; jb += NT) { btm[jb] = Dt[nt_ + 2 * jb]; bsrc[jb] = jb | BORROW; }
            __syncthreads();
        } else if (nd >= 2048 && 3 * nr + 4 * nb <= (u64)ALLOC_CAP) {
            // large level: inputs and the merged demands both in shared memory — the merge-path
            // threads own contiguous output chunks, so their stores are staged and written out
            // coalesced (level 0 of config 4: 31.6k -> 12.0k cycles)
            extern __shared__ u32 astage[];
            u32 *sr = astage, *st = astage + nr, *ss = astage + nr + nb;
            u32 *ot = ss + nb, *os = ot + nd;
            cta_copy(sr, rq, nr);
            cta_copy(st, btm, nb);
            cta_copy(ss, bsrc, nb);
            __syncthreads();
            const u32 nd_ = (u32)nd, nr_ = (u32)nr, nb_ = (u32)nb, nt_ = (u32)n_t, nbor_ = (u32)nbor;
            const u32 per = (nd_ + NT - 1) / NT;
            const u32 diag = threadIdx.x * per;
            if (diag < nd_) {
                u32 lo = diag > nb_ ? diag - nb_ : 0, hi = diag < nr_ ? diag : nr_;
                while (lo < hi) {
                    const u32 mid = (lo + hi) >> 1;
                    if (sr[mid] <= st[diag - mid - 1]) lo = mid + 1; else hi = mid;
                }
                u32 i = lo, j = diag - lo;
                const u32 oe = min(diag + per, nd_);
                for (u32 o = diag; o < oe; o++) {
                    const bool ta = (j >= nb_) || (i < nr_ && sr[i] <= st[j]);
                    ot[o] = ta ? sr[i] : st[j];
                    os[o] = ta ? sr[i] : ss[j];
                    if (ta) i++; else j++;
                }
            }
            __syncthreads();
            for (u32 o = threadIdx.x; o < nd_; o += NT) { Dt[o] = ot[o]; Ds[o] = os[o]; }
            // borrow j carries the time of demand n_t + 2j (btm / bsrc were staged: free to rewrite)
            for (u32 jb = threadIdx.x; jb < nbor_; jb += NT) { btm[jb] = ot[nt_ + 2 * jb]; bsrc[jb] = jb | BORROW; }
            __syncthreads();
        } else if (nr + 2 * nb <= (u64)ALLOC_CAP) {
            // small level: staged inputs, the merge writes the demands and the borrows directly
            extern __shared__ u32 astage[];
            u32 *sr = astage, *st = astage + nr, *ss = astage + nr + nb;
            cta_copy(sr, rq, nr);
            cta_copy(st, btm, nb);
            cta_copy(ss, bsrc, nb);
            __syncthreads();
            const u32 nd_ = (u32)nd, nr_ = (u32)nr, nb_ = (u32)nb, nt_ = (u32)n_t, nbor_ = (u32)nbor;
            const u32 per = (nd_ + NT - 1) / NT;
            const u32 diag = threadIdx.x * per;
            if (diag < nd_) {
                u32 lo = diag > nb_ ? diag - nb_ : 0, hi = diag < nr_ ? diag : nr_;
                while (lo < hi) {
                    const u32 mid = (lo + hi) >> 1;
                    if (sr[mid] <= st[diag - mid - 1]) lo = mid + 1; else hi = mid;
                }
                u32 i = lo, j = diag - lo;
                const u32 oe = min(diag + per, nd_);
                for (u32 o = diag; o < oe; o++) {
                    const bool ta = (j >= nb_) || (i < nr_ && sr[i] <= st[j]);
                    const u32 tm = ta ? sr[i] : st[j];
                    const u32 sc = ta ? sr[i] : ss[j];
                    if (ta) i++; else j++;
                    Dt[o] = tm;
                    Ds[o] = sc;
                    if (o >= nt_ && !((o - nt_) & 1)) {
                        const u32 bj = (o - nt_) >> 1;
                        if (bj < nbor_) { btm[bj] = tm; bsrc[bj] = bj | BORROW; }
                    }
                }
            }
            __syncthreads();
        } else {
            cta_merge_tm(rq, rq, nr, btm, bsrc, nb, Dt, Ds);
            __syncthreads();
            for (u64 base = 0; base < nbor; base += 8 * NT) {
                u32 v[8];
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const u64 j = base + (u64)k * NT + threadIdx.x;
                    v[k] = j < nbor ? Dt[n_t + 2 * j] : 0u;
                }
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const u64 j = base + (u64)k * NT + threadIdx.x;
                    if (j < nbor) { btm[j] = v[k]; bsrc[j] = (u32)j | BORROW; }
                }
            }
            __syncthreads();
        }
        dacc += nd;
        bacc += nbor;
        nb = nbor;
    }
    if (threadIdx.x == 0) { doff[K + 1] = dacc; boff[K + 1] = bacc; ctr->bud_nd = dacc; }
    __syncthreads();
#if BUDDY_TIMING
    if (threadIdx.x == 0) { const long long t1 = clock64(); ctr->eng[20] += t1 - tb0; tb0 = t1; }
#endif
    // ---- top-down ----
    // Borrow addresses of adjacent orders live in shared memory (ping-pong, the staging area is free
    // now) when the largest order's borrows fit; a level's own loads (its demands' sources and
    // resident blocks) do not depend on the level above, so they are issued before the barrier that
    // publishes the level above's borrow addresses: per level one barrier and shared-memory
    // latency instead of a global round trip.
    __shared__ u64 s_left[41], s_cnt[41];
    __shared__ u64 s_maxb;
    if (threadIdx.x == 0) {
        u64 m = 0;
        for (int t = 0; t <= K; t++) m = max(m, boff[t + 1] - boff[t]);
        s_maxb = m;
    }
    __syncthreads();
    const u64 maxb = s_maxb;
    const bool bsm = 2 * maxb * sizeof(u64) <= ALLOC_SMEM;
    u64 *sbuf = reinterpret_cast<u64 *>(astage_td);
    for (int t = K; t >= 0; t--) {
        const u64 n_t = ooff[t + 1] - ooff[t];
        const u64 nd = doff[t + 1] - doff[t];
#if BUDDY_TIMING == 3
        if (threadIdx.x == 0) { const long long t1 = clock64(); ctr->eng[t < 20 ? t : 19] += t1 - tb0; tb0 = t1; ctr->eng[23 + (t < 8 ? t : 7)] += nd; }
#endif
        if (nd == 0) {                      // no demand: the level keeps its blocks, nothing moves
            if (threadIdx.x == 0) { s_left[t] = FAIL; s_cnt[t] = n_t; }
            continue;
        }
        const u64 *blk = old_list + ooff[t];
        const u32 *Ds = dsrc + doff[t];
        const u64 nbor = boff[t + 1] - boff[t];
        const u64 *bad = bsm ? sbuf + (t & 1) * maxb : baddr + boff[t];     // borrows of order t (served by t+1)
        u64 *bad_lo = (t > 0) ? (bsm ? sbuf + ((t - 1) & 1) * maxb : baddr + boff[t - 1]) : nullptr;   // of t-1
        const u32 nd_ = (u32)nd, nt_ = (u32)n_t, nbor_ = (u32)nbor, wb = threadIdx.x & ~31u;
        const u64 dbase = doff[t];
        if (nd_ <= NT) {                                   // one demand per thread at most (most levels)
            const u32 p = threadIdx.x;
            u32 sc = 0;
            u64 a = FAIL;
            if (p < nd_) {
                sc = Ds[p];
                if (p < nt_) a = blk[p];
            }
            __syncthreads();                               // the level above has written bad[]
            if (p < nd_) {
                if (p >= nt_) {
                    const u32 xx = p - nt_, j = xx >> 1;
                    const u64 bj = j < nbor_ ? bad[j] : FAIL;
                    a = (bj != FAIL) ? bj + ((xx & 1) ? (1ull << t) : 0) : FAIL;
                }
                if (sc & BORROW) bad_lo[sc & ~BORROW] = a;
                else if (daddr) daddr[dbase + p] = a;
                else out_u[sc] = a;
            }
        } else
        for (u32 base = 0; base < nd_; base += 8 * NT) {    // 8 independent elements per thread
            const u32 kw = base + wb < nd_ ? min(8u, (nd_ - base - wb + NT - 1) / NT) : 0u;   // warp-uniform
            u64 a[8];
            u32 s[8];
            if (kw) {
#pragma unroll
                for (u32 k = 0; k < 8; k++) {              // level-local loads
                    const u32 p = base + k * NT + threadIdx.x;
                    if (k < kw) {
                        s[k] = p < nd_ ? Ds[p] : 0u;
                        a[k] = (p < nd_ && p < nt_) ? blk[p] : FAIL;
                    }
                }
            }
            if (base == 0) __syncthreads();                // the level above has written bad[]
            if (!kw) continue;                             // idle warp: nothing of this level
#pragma unroll
            for (u32 k = 0; k < 8; k++) {
                const u32 p = base + k * NT + threadIdx.x;
                if (k < kw && p < nd_ && p >= nt_) {
                    const u32 xx = p - nt_, j = xx >> 1;
                    const u64 bj = j < nbor_ ? bad[j] : FAIL;
                    a[k] = (bj != FAIL) ? bj + ((xx & 1) ? (1ull << t) : 0) : FAIL;
                }
            }
#pragma unroll
            for (u32 k = 0; k < 8; k++) {
                const u32 p = base + k * NT + threadIdx.x;
                if (k >= kw || p >= nd_) continue;
                if (s[k] & BORROW) bad_lo[s[k] & ~BORROW] = a[k];
                else if (daddr) daddr[dbase + p] = a[k];   // in demand order (coalesced); k_bud_scatter
                else out_u[s[k]] = a[k];
            }
        }
        if (threadIdx.x == 0) {
            const u64 last_bad = nbor > 0 ? bad[nbor - 1] : FAIL;
            u64 x = nd > n_t ? nd - n_t : 0;
            u64 left = FAIL;
            if ((x & 1) && nbor > 0 && last_bad != FAIL) left = last_bad + (1ull << t);
            s_left[t] = left;
            s_cnt[t] = (nd < n_t ? n_t - nd : 0) + (left != FAIL ? 1 : 0);
        }
    }
    __syncthreads();
#if BUDDY_TIMING
    if (threadIdx.x == 0) { const long long t1 = clock64(); ctr->eng[21] += t1 - tb0; tb0 = t1; }
#endif
    // for the address-ordered set (k_bud_qflags / k_bud_qwrite): per order the first surviving
    // start (the first nd blocks were consumed) and the leftover
    if (threadIdx.x <= (unsigned)K) {
        const int t = threadIdx.x;
        const u64 n_t = ooff[t + 1] - ooff[t], nd = doff[t + 1] - doff[t];
        ctr->bud_thr[t] = nd == 0 ? 0ull : (nd < n_t ? old_list[ooff[t] + nd] : FAIL);
        ctr->bud_left[t] = s_left[t];
    }
    // ---- new per-order lists: surviving batch-start blocks, or the one leftover ----
    __shared__ u64 noff[42];
    if (threadIdx.x == 0) {
        u64 o = 0;
        for (int t = 0; t <= K; t++) { noff[t] = o; o += s_cnt[t]; }
        noff[K + 1] = o;
    }
    __syncthreads();
    // the surviving batch-start blocks of each order are copied by the whole grid (k_bud_scatter);
    // this CTA records what to copy and writes the single leftovers
    if (threadIdx.x <= (unsigned)K) {
        const int t = threadIdx.x;
        const u64 n_t = ooff[t + 1] - ooff[t];
        const u64 nd = doff[t + 1] - doff[t];
        ctr->bud_csrc[t] = ooff[t] + nd;
        ctr->bud_ccnt[t] = nd < n_t ? n_t - nd : 0;
        if (nd >= n_t && s_left[t] != FAIL) new_list[noff[t]] = s_left[t];
    }
    __syncthreads();
    if (threadIdx.x <= (unsigned)K + 1) {
        ctr->bud_off[threadIdx.x] = noff[threadIdx.x];
        if (threadIdx.x <= (unsigned)K) ctr->bud_cnt[threadIdx.x] = s_cnt[threadIdx.x];
    }
    if (threadIdx.x == 0) ctr->bud_total = noff[K + 1];
#if BUDDY_TIMING
    if (threadIdx.x == 0) { const long long t1 = clock64(); ctr->eng[22] += t1 - tb0; }
#endif
}

// The request demands' addresses, written by k_alloc_levels in demand order (one CTA: its stores
// are coalesced), scattered to request order by the whole grid — one CTA issuing ~n scattered
// 8-byte stores (one L2 transaction each) is what bounded the top-down pass.
__global__ void k_bud_scatter(const u32 *__restrict__ dsrc, const u64 *__restrict__ daddr, const DevCtr *ctr,
                              u64 *__restrict__ out_u, const u64 *__restrict__ old_list, u64 *__restrict__ new_list,
                              int K) {
    PDL_ENTRY();
    const u64 nd = ctr->bud_nd;
    for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < nd; g += (u64)gridDim.x * blockDim.x) {
        const u32 sc = dsrc[g];
        if (!(sc & BORROW)) out_u[sc] = daddr[g];
    }
    // ... and the surviving batch-start blocks of every order into the new per-order lists
    __shared__ u64 pre[50];
    if (threadIdx.x == 0) {
        u64 a = 0;
        for (int t = 0; t <= K; t++) { pre[t] = a; a += ctr->bud_ccnt[t]; }
        pre[K + 1] = a;
    }
    __syncthreads();
    const u64 tot = pre[K + 1];
    for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < tot; g += (u64)gridDim.x * blockDim.x) {
        int lo = 0, hi = K + 1;                   // the order t with pre[t] <= g < pre[t+1]
        while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (pre[mid] <= g) lo = mid; else hi = mid; }
        const u64 q = g - pre[lo];
        new_list[ctr->bud_off[lo] + q] = old_list[ctr->bud_csrc[lo] + q];
    }
}

// buddy results: order -> units = 2^k; reuse fits::k_alloc_finish by materialising r
__global__ void k_alloc_r(const u32 *__restrict__ key_by_req, u64 n, const u64 *n_in, int K, u64 *__restrict__ r) {
    PDL_ENTRY();
    if (n_in) n = *n_in;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u32 k = key_by_req[i];
        r[i] = (k <= (u32)K) ? (1ull << k) : 0;
    }
}

__device__ __forceinline__ bool is_free_start(const u64 *list, const DevCtr *ctr, int K, u64 key) {
    for (int t = 0; t <= K; t++) {
        u64 lo = ctr->bud_off[t], hi = ctr->bud_off[t + 1];
        while (lo < hi) {
            u64 mid = (lo + hi) >> 1;
            if (list[mid] < key) lo = mid + 1; else hi = mid;
        }
        if (lo < ctr->bud_off[t + 1] && list[lo] == key) return true;
    }
    return false;
}

}  // namespace buddy
