// partial.cuh — partial (tail) deallocation, policy flag HEAP_PARTIAL_FREE (sm_100a).
//
// The paper's dealloc looks the address up in the used list with a containing-block search
// (Alg. 2, `search(used_list, addr)`), so "freeing the last 2kB of a 10kB
// block" shrinks the in-use block.  The block table (table.cuh) is keyed by
// exact start, so a containing-block query needs an ordered view of the live starts.  On the
// GPU that view is a hierarchical bitmap over arena units — one bit per unit that starts a
// live block, and above it one bit per nonzero word of the level below up to a single word —
// so "the live block holding unit u" is a predecessor query: the highest set bit <= u, found by
// climbing to the first level with a set bit below the path and descending by
// count-leading-zeros (at most 2 x levels dependent 4-byte loads; 7 levels at 2^32 units).
//
// Exactness: a summary bit is set iff its child word is nonzero at every kernel boundary.  The
// free phase only clears bits (the thread whose atomicAnd empties a word clears the parent
// bit, recursively), the alloc phase only sets them; queries run in a separate kernel.
//
// A free batch with the flag (reading C29): after the address sort, every key u is
// resolved read-only (k_resolve): a = pred(u); if a exists and u < a + size(a) the key lies in
// live block a.  Keys inside one live block are contiguous in sorted order, so the first of
// them is the block's winner (the lowest offset frees; the whole block when u = a) and the rest
// are double frees (k_apply).  Only a winner writes its block's table slot (tombstone, or the
// shrunk size u - a) and its bitmap bit, so the two kernels need no further synchronisation.
#pragma once
#include "common.cuh"
#include "table.cuh"

namespace partial {

constexpr int MAXLEV = 8;
constexpr u32 NONE32 = 0xFFFFFFFFu;
enum { K_INVALID = 0, K_DOUBLE = 1, K_INSIDE = 2 };

struct Lbm {
    u32 *w;                 // all levels, level l at w + off[l]
    u64 off[MAXLEV];
    int nlev;
};

// host: level offsets for A_u units; returns total words
inline u64 lbm_layout(u64 A_u, Lbm *b) {
    u64 n = (A_u + 31) / 32, o = 0;
    b->nlev = 0;
    for (;;) {
        b->off[b->nlev++] = o;
        o += n;
        if (n == 1 || b->nlev == MAXLEV) break;
        n = (n + 31) / 32;
    }
    return o;
}

// highest live start <= x, or NONE32
__device__ __forceinline__ u32 pred(const Lbm &b, u64 x) {
    u64 p = x;
    int l = 0;
    for (;;) {
        const u32 w = b.w[b.off[l] + (p >> 5)];
        const u32 bit = (u32)(p & 31);
        // level 0: bits <= x; above: bits strictly below the child word already searched
        const u32 m = (l == 0) ? (w & (0xFFFFFFFFu >> (31 - bit))) : (w & ((1u << bit) - 1u));
        if (m) { p = ((p >> 5) << 5) + 31 - __clz(m); break; }
        if (l == b.nlev - 1) return NONE32;
        p >>= 5;
        l++;
    }
    while (l > 0) {
        l--;
        const u32 w = b.w[b.off[l] + p];
        p = (p << 5) + 31 - __clz(w);
    }
    return (u32)p;
}

// set the live-start bit of every successful allocation (alloc phase: sets only)
__global__ void k_set_bits(const u64 *__restrict__ out_u, u64 n, const u64 *n_in, Lbm b) {
    PDL_ENTRY();
    if (n_in) n = *n_in;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 p = out_u[i];
        if (p == HEAP_NULL_U64) continue;
        for (int l = 0; l < b.nlev; l++) {
            const u32 old = atomicOr(&b.w[b.off[l] + (p >> 5)], 1u << (p & 31));
            if (old) break;          // the word was nonzero: its parent bit is (being) set
            p >>= 5;
        }
    }
}

// clear the live-start bit of unit p (free phase: clears only)
__device__ __forceinline__ void clear_bit(const Lbm &b, u64 p) {
    for (int l = 0; l < b.nlev; l++) {
        const u32 m = 1u << (p & 31);
        const u32 old = atomicAnd(&b.w[b.off[l] + (p >> 5)], ~m);
        if (old & ~m) break;         // the word stays nonzero
        p >>= 5;
    }
}

__device__ __forceinline__ bool bsearch_free(const u64 *a, u64 n, u64 key) {
    u64 lo = 0, hi = n;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo < n && a[lo] == key;
}

// Read-only resolution of every sorted key (one table tile per key, as table::lookup).
// kind[i]: K_INSIDE (own[i] = the live block's start, endu[i] = its end), K_DOUBLE (start of a
// free block), K_INVALID (free memory that is not a block start).
__global__ void __launch_bounds__(256) k_resolve(const u32 *__restrict__ keys, const u64 *nk_dev,
                                                 u64 *__restrict__ slots, u64 tmask, u64 max_lines, Lbm b,
                                                 const u64 *__restrict__ fstart, const u64 *F_dev,
                                                 u32 *__restrict__ kind, u32 *__restrict__ own,
                                                 u64 *__restrict__ endu, DevCtr *ctr) {
    PDL_ENTRY();
    const u64 nk = *nk_dev, F = *F_dev;
    const u32 lane = lane_id(), g = lane / table::TILE_LANES, sub = lane % table::TILE_LANES;
    const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
    for (u64 base = gw * table::KPW; base < nk; base += nwarps * table::KPW) {
        const u64 idx = base + g;
        const bool in = idx < nk;
        const u32 u = in ? keys[idx] : 0;
        const u32 a = in ? pred(b, u) : NONE32;
        const bool has = in && a != NONE32;
        const u64 s = table::lookup(slots, tmask, has ? a : 0, has, table::EMPTY, max_lines);
        if (in && sub == 0) {
            u32 k = K_INVALID;
            u64 e = 0;
            if (has) {
                if (s == table::EMPTY) atomicOr(&ctr->error_flags, (u64)ERR_LIVEMAP);  // bitmap/table disagree
                else {
                    e = (u64)a + table::slot_size(s);
                    if ((u64)u < e) k = K_INSIDE;
                }
            }
            if (k != K_INSIDE && bsearch_free(fstart, F, u)) k = K_DOUBLE;
            kind[idx] = k;
            own[idx] = (k == K_INSIDE) ? a : NONE32;
            endu[idx] = e;
        }
    }
}

// Winners free [u, end): the whole block (u = a: tombstone, clear its bit) or its tail (the
// slot's size becomes u - a).  vflag / vs / ve feed the merge + coalesce steps of fits.
// endu and vs may alias (each index is read before it is written, by the same lane).
__global__ void __launch_bounds__(256) k_apply(const u32 *__restrict__ keys, const u64 *nk_dev,
                                               const u32 *__restrict__ kind, const u32 *__restrict__ own,
                                               const u64 *endu, u64 *__restrict__ slots, u64 tmask,
                                               u64 max_lines, Lbm b, u32 *__restrict__ vflag, u64 *vs,
                                               u64 *__restrict__ ve, DevCtr *ctr) {
    PDL_ENTRY();
    __shared__ u64 sm[33];
    const u64 nk = *nk_dev;
    const u32 lane = lane_id(), g = lane / table::TILE_LANES, sub = lane % table::TILE_LANES;
    const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
    u64 c_ok = 0, c_dbl = 0, c_inv = 0, c_units = 0, c_whole = 0;
    for (u64 base = gw * table::KPW; base < nk; base += nwarps * table::KPW) {
        const u64 idx = base + g;
        const bool in = idx < nk;
        const u32 k = in ? kind[idx] : K_INVALID;
        const u32 a = in ? own[idx] : NONE32;
        const u64 e = in ? endu[idx] : 0;
        const u32 u = in ? keys[idx] : 0;
        const bool win = in && k == K_INSIDE && (idx == 0 || kind[idx - 1] != K_INSIDE || own[idx - 1] != a);
        const bool whole = win && u == a;
        const u64 repl = whole ? table::TOMB : table::pack(a, (u64)u - a);
        table::lookup(slots, tmask, win ? a : 0, win, repl, max_lines);
        if (in && sub == 0) {
            if (win) {
                if (whole) { clear_bit(b, a); c_whole++; }
                c_ok++;
                c_units += e - u;
                vs[idx] = u;
                ve[idx] = e;
            } else if (k == K_INVALID) {
                c_inv++;
            } else {
                c_dbl++;
            }
            vflag[idx] = win ? 1u : 0u;
        }
    }
    const u64 x0 = block_sum64<256>(c_ok, sm), x1 = block_sum64<256>(c_dbl, sm);
    const u64 x2 = block_sum64<256>(c_inv, sm), x3 = block_sum64<256>(c_units, sm);
    const u64 x4 = block_sum64<256>(c_whole, sm);
    if (threadIdx.x == 0) {
        if (x0) atomicAdd(&ctr->frees_ok, x0);
        if (x1) atomicAdd(&ctr->frees_double, x1);
        if (x2) atomicAdd(&ctr->frees_invalid, x2);
        if (x3) atomicAdd(&ctr->live_units, (u64)0 - x3);
        if (x4) { atomicAdd(&ctr->n_live, (u64)0 - x4); atomicAdd(&ctr->tbl_tombs, x4); }
    }
}

}  // namespace partial
