// common.cuh — shared device helpers for libheap (sm_100a).
//
// All kernels are grid-stride / persistent: the grid is a multiple of the SM count
// (148 on B200) and element counts are read from device memory, so a batch never needs
// a host round trip to learn how many free blocks, valid frees, ... there are.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef unsigned int u32;

#define HEAP_NULL_U64 0xFFFFFFFFFFFFFFFFull
#define NIL32 0xFFFFFFFFu
#define FULLMASK 0xFFFFFFFFu

// Device counters (one struct in the workspace).  Counts are u64 so that they can be
// read as element counts by the grid-stride kernels.
struct DevCtr {
    u64 F;              // free-block count of the current free array (fits policies)
    u64 n_live;         // live blocks
    u64 live_units;     // sum of live sizes (units)
    u64 allocs_ok, allocs_failed, frees_ok, frees_invalid, frees_double, frees_null;
    u64 high_water_units;
    u64 error_flags;
    u64 tbl_used;       // non-EMPTY table slots (live + tombstones)
    u64 tbl_tombs;
    // per-batch scratch counts
    u64 nk;             // candidate free keys after classification
    u64 nv;             // valid frees
    u64 M;              // merged element count
    u64 scan_total;
    u64 n_hist;         // radix histogram length (256 * tiles)
    u64 nsort;          // element count for a sort
    u64 tmp[8];
    u64 rb_n;           // table rebuild: live slots collected (k_rb_clear -> k_rb_insert)
    u32 bud_qdone, bud_pad;   // k_bud_qwrite: CTAs finished (the last one publishes bud_qn)
    // buddy: per-order counts of the current per-order free lists and their offsets (binary
    // buddies use K + 1 <= 33 orders, Fibonacci buddies K + 1 <= 46 classes: fib::MAXC = 48)
    u64 bud_cnt[48];
    u64 bud_off[49];
    u64 bud_total;
    // buddy free set in address order (buddy.cuh parallel form): its length, and from the last
    // alloc phase per order the first surviving start (consumed blocks are a prefix) and leftover
    u64 bud_qn;
    u64 bud_thr[48], bud_left[48];
    u64 bud_csrc[48], bud_ccnt[48];   // alloc phase: per order, the surviving batch-start blocks to copy
                                      // (first index in the old list, count) — k_bud_scatter copies them
    u64 eng[32];        // alloc engine diagnostics (engine_tlsf.cuh)
    u64 lifo_clock;     // SEGFIT_LIFO logical push clock (fits.cuh)
    u64 req_n;          // request count of a graph-launched batch (heap.cu graph path)
    u64 rover;          // NEXT_FIT: unit address where the next search starts (reading C27)
    u64 wild_n;         // TLSF/SEGFIT wilderness split: request count when active, else 0
    u64 wild_start;     // the wilderness piece's start at the batch start (units)
    u64 wild_total;     // units the batch took from it
    u64 wild_acc[2];    // k_alloc_prep: units of all requests, max search class of a valid one
    u32 wild[2];        // {class Kw, piece f} of the wilderness, {NONE, NONE} when inactive
    // single-pass sort / scan control (prims.cuh; zero at creation, self-resetting)
    u32 os_tile[8];     // onesweep radix sort: dynamic tile counter per pass
    u32 os_epoch;       // bumped once per sort call (tags the lookback flags)
    u32 os_done;        // histogram kernel: CTAs finished
    u32 sc_tile, sc_done, sc_epoch, sc_pad;   // single-pass scan: tile counter, CTAs done, epoch
    u32 os_gh[8][256];  // digit histograms of the current sort (zeroed again by the last CTA)
    u32 os_gbase[8][256];   // their exclusive scans: first output position of each digit
    u64 bud_nd;         // buddy alloc: total demands of the last batch's levels (k_bud_scatter)
};

enum { ERR_CAP_LIVE = 1, ERR_TABLE_FULL = 2, ERR_CAP_FREE = 4, ERR_ENGINE = 8, ERR_LIVEMAP = 16 };

// Programmatic dependent launch (heap.cu LAUNCH): every kernel lets the next kernel of the stream
// be scheduled as soon as all of its own CTAs have started, then waits until the previous kernel
// has completed and its memory is visible before touching anything.  Consecutive launches of a
// batch thus overlap their launch latency, never their data (griddepcontrol.wait is a full
// completion wait; without the launch attribute both instructions are no-ops).
#define PDL_ENTRY()                                                          \
    do {                                                                     \
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");     \
        asm volatile("griddepcontrol.wait;" ::: "memory");                  \
    } while (0)

__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ u32 lanemask_lt() {
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// floor(log2 u), u >= 1
__device__ __forceinline__ int flog2(u64 u) { return 63 - __clzll(u); }

// inclusive warp scan (u32)
__device__ __forceinline__ u32 warp_incl_scan(u32 v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 t = __shfl_up_sync(FULLMASK, v, o);
        if (lane_id() >= (u32)o) v += t;
    }
    return v;
}
__device__ __forceinline__ u64 warp_incl_scan64(u64 v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u64 t = __shfl_up_sync(FULLMASK, v, o);
        if (lane_id() >= (u32)o) v += t;
    }
    return v;
}
__device__ __forceinline__ u64 warp_sum64(u64 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    return v;
}
__device__ __forceinline__ u64 warp_max64(u64 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { u64 t = __shfl_xor_sync(FULLMASK, v, o); v = t > v ? t : v; }
    return v;
}

// block-wide exclusive scan of one u32 per thread; returns exclusive prefix, *total = sum.
// smem must hold >= 33 u32.  All threads of the block must call it.
template <int NT>
__device__ __forceinline__ u32 block_excl_scan(u32 v, u32 *smem, u32 *total) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    u32 inc = warp_incl_scan(v);
    if (l == 31) smem[w] = inc;
    __syncthreads();
    if (w == 0) {
        u32 x = (l < NT / 32) ? smem[l] : 0;
        u32 xi = warp_incl_scan(x);
        if (l < NT / 32) smem[l] = xi - x;
        if (l == NT / 32 - 1) smem[32] = xi;
    }
    __syncthreads();
    u32 r = smem[w] + inc - v;
    *total = smem[32];
    __syncthreads();
    return r;
}

template <int NT>
__device__ __forceinline__ u64 block_sum64(u64 v, u64 *smem) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    v = warp_sum64(v);
    if (l == 0) smem[w] = v;
    __syncthreads();
    u64 r = 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NT / 32; i++) r += smem[i];
        smem[0] = r;
    }
    __syncthreads();
    r = smem[0];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------------
// TLSF class mapping (C10; the same definition the oracle implements, written
// independently): classes below 2^L units are exact; above, fl = m - L + 1 with
// m = floor(log2 u) and sl = the L bits after the leading one.  L = 0 gives the paper's
// power-of-two bins (Alg. 4 floor/ceil log2) shifted by one.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ u32 cls_insert(u64 u, int L) {
    if (u < (1ull << L)) return (u32)u;
    int m = flog2(u);
    return (u32)(((u64)(m - L + 1) << L) + ((u >> (m - L)) - (1ull << L)));
}
// smallest block size (units) of class c
__device__ __forceinline__ u64 cls_lo(u32 c, int L) {
    u32 fl = c >> L, sl = c & ((1u << L) - 1);
    return fl == 0 ? (u64)sl : ((u64)((1u << L) + sl) << (fl - 1));
}
__device__ __forceinline__ u32 cls_search(u64 u, int L) {
    if (u < (1ull << L)) return (u32)u;
    int m = flog2(u);
    return cls_insert(u + (1ull << (m - L)) - 1, L);
}

#define CUDA_TRY(x)                                   \
    do {                                              \
        cudaError_t _e = (x);                         \
        if (_e != cudaSuccess) return HEAP_ECUDA;     \
    } while (0)
