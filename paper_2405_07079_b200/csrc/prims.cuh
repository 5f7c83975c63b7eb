// prims.cuh — device-wide primitives with device-resident element counts: single-pass exclusive
// scan, onesweep LSD radix sort (8-bit digits, stable), merge path.
//
// Every kernel reads its element count from a u64 in device memory (tiles are claimed
// dynamically or walked with a grid-stride loop), so the host never has to synchronise to size a
// launch.
#pragma once
#include "common.cuh"

namespace prims {

constexpr int NT = 256;        // threads per CTA
constexpr int IPT = 8;         // items per thread
constexpr int TILE = NT * IPT; // 2048 elements per tile

__host__ __device__ inline u64 ntiles_of(u64 n) { return (n + TILE - 1) / TILE; }

// ------------------------------------------------ onesweep radix sort (8-bit digits) ----
// A stable LSD sort whose passes each take ONE launch: k_os_hist computes the digit histograms of
// every pass in one read of the keys (global atomics; the last CTA turns them into the digits'
// first output positions and zeroes them again), then per pass k_os_scatter claims 4096-key tiles
// in launch order, ranks its keys per warp (match + per-warp digit counters, index order kept), gets
// each digit's offset from the tiles before it by decoupled lookback (one 64-bit word per (tile,
// digit): epoch | status | count, no separate scan), stages the tile in shared memory in sorted
// order and writes it out as runs of consecutive addresses per digit.
constexpr int OS_NT = 256, OS_IPT = 16, OS_TILE = OS_NT * OS_IPT, OS_W = OS_NT / 32;
constexpr u32 LB_AGG = 1u, LB_INC = 2u;

__host__ __device__ inline u64 os_ntiles(u64 n) { return (n + OS_TILE - 1) / OS_TILE; }

__device__ __forceinline__ void lb_store(u64 *p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 lb_load(const u64 *p) {
    u64 v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Decoupled lookback for one value: publish `agg` for tile t, return the sum of all tiles before t,
// publish the inclusive sum.  flags: one word per tile (stride apart); tag = epoch of this call.
// The predecessors' words are read LB_W at a time (independent loads in flight), newest first, so a
// walk back over many tiles that published only their aggregate takes 1/LB_W of the round trips.
constexpr int LB_W = 8;
__device__ __forceinline__ u32 lookback(u64 *flags, u64 stride, u64 t, u32 tag, u32 agg) {
    const u64 hi = (u64)tag << 32;
    if (t == 0) {
        lb_store(flags, hi | ((u64)LB_INC << 30) | agg);
        return 0;
    }
    lb_store(flags + t * stride, hi | ((u64)LB_AGG << 30) | agg);
    u32 prefix = 0;
    u64 tt = t;                                   // tiles [tt, t) are summed into prefix
    for (;;) {
        u64 v[LB_W];
#pragma unroll
        for (int j = 0; j < LB_W; j++) v[j] = (tt > (u64)j) ? lb_load(flags + (tt - 1 - j) * stride) : 0ull;
        bool done = false;
        int j = 0;
        for (; j < LB_W && tt > (u64)j; j++) {
            const u32 st = (u32)(v[j] >> 30) & 3u;
            if ((u32)(v[j] >> 32) != tag || st == 0) break;     // not published yet: re-read from here
            prefix += (u32)v[j] & 0x3FFFFFFFu;
            if (st == LB_INC) { done = true; break; }
        }
        if (done) break;
        tt -= (u64)j;                             // j words consumed (all aggregates)
    }
    lb_store(flags + t * stride, hi | ((u64)LB_INC << 30) | (prefix + agg));
    return prefix;
}

// The end of a histogram pass (OS_NT threads per CTA; h = this CTA's digit counts in shared
// memory): the counts go to the global histograms, the last CTA turns them into digit start offsets
// (os_gbase), re-zeroes them and resets the onesweep tile counters / bumps the epoch.  Shared by
// k_os_hist and by producers that count their keys' digits while writing them (a fused histogram).
__device__ __forceinline__ void os_hist_finish(u32 (*h)[256], int passes, DevCtr *ctr) {
    __shared__ u32 s_last, sm[33];
    __syncthreads();
    for (int p = 0; p < passes; p++)
        if (h[p][threadIdx.x]) atomicAdd(&ctr->os_gh[p][threadIdx.x], h[p][threadIdx.x]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&ctr->os_done, 1u) == gridDim.x - 1) ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int p = 0; p < passes; p++) {
        const u32 c = atomicExch(&ctr->os_gh[p][threadIdx.x], 0u);   // read and re-zero
        u32 tot;
        ctr->os_gbase[p][threadIdx.x] = block_excl_scan<OS_NT>(c, sm, &tot);
    }
    if (threadIdx.x < 8) ctr->os_tile[threadIdx.x] = 0;
    if (threadIdx.x == 0) { ctr->os_epoch += 1; ctr->os_done = 0; }
}

template <typename K>
__global__ void __launch_bounds__(OS_NT) k_os_hist(const K *__restrict__ keys, const u64 *n_dev, int passes,
                                                   DevCtr *ctr) {
    PDL_ENTRY();
    __shared__ u32 h[8][256];
    __shared__ u32 s_last, sm[33];
    const u64 n = *n_dev;
    for (int p = 0; p < passes; p++) h[p][threadIdx.x] = 0;
    __syncthreads();
    for (u64 i = (u64)blockIdx.x * OS_NT + threadIdx.x; i < n; i += (u64)gridDim.x * OS_NT) {
        const K k = keys[i];
        for (int p = 0; p < passes; p++) atomicAdd(&h[p][(u32)(k >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
    for (int p = 0; p < passes; p++)
        if (h[p][threadIdx.x]) atomicAdd(&ctr->os_gh[p][threadIdx.x], h[p][threadIdx.x]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&ctr->os_done, 1u) == gridDim.x - 1) ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int p = 0; p < passes; p++) {
        const u32 c = atomicExch(&ctr->os_gh[p][threadIdx.x], 0u);   // read and re-zero
        u32 tot;
        ctr->os_gbase[p][threadIdx.x] = block_excl_scan<OS_NT>(c, sm, &tot);
    }
    if (threadIdx.x < 8) ctr->os_tile[threadIdx.x] = 0;
    if (threadIdx.x == 0) { ctr->os_epoch += 1; ctr->os_done = 0; }
}

template <typename K, bool HV>
constexpr size_t os_smem() { return OS_TILE * sizeof(K) + (HV ? OS_TILE * sizeof(u32) : 0); }

template <typename K, bool HV>
__global__ void __launch_bounds__(OS_NT) k_os_scatter(const K *__restrict__ kin, const u32 *__restrict__ vin,
                                                      K *__restrict__ kout, u32 *__restrict__ vout,
                                                      const u64 *n_dev, int pass, u64 *flags, DevCtr *ctr) {
    PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char os_dyn[];   // os_smem<K, HV>() bytes
    K *ks = reinterpret_cast<K *>(os_dyn);
    u32 *vs = reinterpret_cast<u32 *>(os_dyn + OS_TILE * sizeof(K));
    __shared__ u32 wc[OS_W][256];
    __shared__ u32 lstart[256], gpos[256];
    __shared__ u32 s_tile, sm[33];
    const u64 n = *n_dev, nt = os_ntiles(n);
    const u32 tag = ctr->os_epoch * 8u + (u32)pass;
    const int shift = 8 * pass;
    const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->os_tile[pass], 1u);
#pragma unroll
        for (int i = 0; i < 8; i++) wc[w][lane + 32 * i] = 0;
        __syncthreads();
        const u64 t = s_tile;
        if (t >= nt) break;
        const u64 base = t * OS_TILE + (u64)w * (32 * OS_IPT);
        K key[OS_IPT];
        u32 val[OS_IPT], dig[OS_IPT], lr[OS_IPT];
#pragma unroll
        for (int j = 0; j < OS_IPT; j++) {
            const u64 idx = base + (u64)j * 32 + lane;
            const bool v = idx < n;
            key[j] = v ? kin[idx] : (K)0;
            val[j] = (HV && v) ? vin[idx] : 0u;
            dig[j] = v ? ((u32)(key[j] >> shift) & 255u) : 256u;
        }
        // per-warp ranks in index order (j, then lane)
#pragma unroll
        for (int j = 0; j < OS_IPT; j++) {
            const u32 peers = __match_any_sync(FULLMASK, dig[j]);
            const u32 c0 = dig[j] < 256u ? wc[w][dig[j]] : 0u;
            __syncwarp();
            if (dig[j] < 256u && (peers & lanemask_lt()) == 0) wc[w][dig[j]] = c0 + __popc(peers);
            __syncwarp();
            lr[j] = c0 + __popc(peers & lanemask_lt());
        }
        __syncthreads();
        // thread d: exclusive offsets of digit d over the warps, the tile's count of d, and its place
        {
            const u32 d = threadIdx.x;
            u32 c = 0;
#pragma unroll
            for (int q = 0; q < OS_W; q++) { const u32 x = wc[q][d]; wc[q][d] = c; c += x; }
            u32 tot;
            const u32 ls = block_excl_scan<OS_NT>(c, sm, &tot);
            lstart[d] = ls;
            const u32 prefix = lookback(flags + d, 256, t, tag, c);
            gpos[d] = ctr->os_gbase[pass][d] + prefix - ls;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < OS_IPT; j++)
            if (dig[j] < 256u) {
                const u32 lp = lstart[dig[j]] + wc[w][dig[j]] + lr[j];
                ks[lp] = key[j];
                if (HV) vs[lp] = val[j];
            }
        __syncthreads();
        const u32 tn = (u32)min((u64)OS_TILE, n - t * OS_TILE);
        for (u32 i = threadIdx.x; i < tn; i += OS_NT) {
            const K k = ks[i];
            const u32 pos = gpos[(u32)(k >> shift) & 255u] + i;
            kout[pos] = k;
            if (HV) vout[pos] = vs[i];
        }
        __syncthreads();
    }
}

// ------------------------------------------------ single-pass exclusive scan (u32) ----
// One launch: tiles of 4096 claimed in launch order, block scan, decoupled lookback for the tile's
// offset; the CTA holding the last tile writes the grand total; the last CTA to leave resets the
// tile counter and bumps the epoch for the next call.  in == out is allowed.
__global__ void __launch_bounds__(OS_NT) k_scan_1p(const u32 *in, u32 *out, const u64 *n_dev, u64 *total,
                                                   u64 *flags, DevCtr *ctr) {
    PDL_ENTRY();
    __shared__ u32 sm[33];
    __shared__ u32 s_tile, s_pre;
    const u64 n = *n_dev, nt = os_ntiles(n);
    const u32 tag = ctr->sc_epoch;
    if (nt == 0 && blockIdx.x == 0 && threadIdx.x == 0) *total = 0;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->sc_tile, 1u);
        __syncthreads();
        const u64 t = s_tile;
        if (t >= nt) break;
        const u64 base = t * OS_TILE + (u64)threadIdx.x * OS_IPT;   // 16 consecutive items per thread
        u32 v[OS_IPT], s = 0;
#pragma unroll
        for (int j = 0; j < OS_IPT; j++) { v[j] = base + j < n ? in[base + j] : 0u; s += v[j]; }
        u32 tot;
        const u32 ex = block_excl_scan<OS_NT>(s, sm, &tot);
        if (threadIdx.x == 0) s_pre = lookback(flags, 1, t, tag, tot);
        __syncthreads();
        u32 run = s_pre + ex;
#pragma unroll
        for (int j = 0; j < OS_IPT; j++) { if (base + j < n) out[base + j] = run; run += v[j]; }
        if (t == nt - 1 && threadIdx.x == 0) *total = (u64)s_pre + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&ctr->sc_done, 1u) == gridDim.x - 1) {
            ctr->sc_tile = 0;
            ctr->sc_done = 0;
            ctr->sc_epoch += 1;
        }
    }
}

// ------------------------------------------------------------ merge path ----
// Merge two start-sorted SoA arrays (start, end) of lengths *na, *nb into out (length
// na + nb).  Starts are distinct (disjoint blocks), ties go to a.
constexpr int MIPT = 8;
__global__ void __launch_bounds__(NT) k_merge(const u64 *__restrict__ as, const u64 *__restrict__ ae,
                                              const u64 *na_dev, const u64 *__restrict__ bs,
                                              const u64 *__restrict__ be, const u64 *nb_dev,
                                              u64 *__restrict__ os, u64 *__restrict__ oe, u64 *total,
                                              const u32 *__restrict__ at = nullptr,
                                              const u32 *__restrict__ bt = nullptr, u32 *__restrict__ ot = nullptr) {
    PDL_ENTRY();
    // at/bt/ot: optional per-block payload merged alongside (push stamps of SEGFIT_LIFO)
    const u64 na = *na_dev, nb = *nb_dev, n = na + nb;
    if (blockIdx.x == 0 && threadIdx.x == 0 && total) *total = n;
    const u64 nchunks = (n + MIPT - 1) / MIPT;
    for (u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += (u64)gridDim.x * blockDim.x) {
        u64 diag = c * MIPT;
        u64 lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
        while (lo < hi) {
            u64 mid = (lo + hi) >> 1;
            if (as[mid] <= bs[diag - mid - 1]) lo = mid + 1; else hi = mid;
        }
        u64 i = lo, j = diag - lo;
#pragma unroll
        for (int k = 0; k < MIPT; k++) {
            u64 o = diag + k;
            if (o >= n) break;
            bool take_a = (j >= nb) || (i < na && as[i] <= bs[j]);
            if (take_a) { os[o] = as[i]; oe[o] = ae[i]; if (ot) ot[o] = at[i]; i++; }
            else { os[o] = bs[j]; oe[o] = be[j]; if (ot) ot[o] = bt[j]; j++; }
        }
    }
}

}  // namespace prims
