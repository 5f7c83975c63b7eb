// fits.cuh — batched free and alloc phases for the non-buddy policies
// (FIRST_FIT, BEST_FIT, SEGFIT, TLSF).
//
// State between batches: the free blocks as an address-sorted, fully coalesced SoA array
// (start, end) in units (the role of the paper's address-sorted HAL free list, §3.1,
// PAPER.md:166-168), plus the block table (table.cuh).
//
// Free phase (canonical order: every offset classified against the batch-start state, then
// valid frees applied as if one by one in ascending address order, Alg. 2 / Alg. 5):
//   classify -> compact -> radix sort of keys -> table lookup+delete (dedup, double/invalid)
//   -> compact valid -> merge path with the free array -> coalesce by head flags + scan.
// The result is the set of maximal free runs (lemma L2: the free set is a function of the
// live set), so applying the frees "one by one" and "all at once" coincide.
//
// Alloc phase: requests are normalised in parallel, then matched by an exact engine that
// walks them in request order (the paper's per-request semantics, C25 reading A).
// Key fact used by every engine: during an alloc phase each batch-start free block f holds
// at most ONE free piece, [start_f, end_f), which only shrinks from its low end (Alg. 1
// splits at the low end and nothing is freed during the phase).  So the engine state is just
// start_f per block, and address order among pieces is the order of f.
#pragma once
#include "common.cuh"
#include "prims.cuh"
#include "table.cuh"
#include "buddy.cuh"

namespace fits {

// ------------------------------------------------------------------ free phase ----
// (also counts the digits of the candidate keys for the address sort that follows — the compaction
// in between keeps exactly the candidates — so that sort needs no histogram launch; prims::NT threads)
__global__ void __launch_bounds__(256) k_free_classify(const u64 *__restrict__ offs, u64 n, const u64 *n_in, int alog2,
                                                       u64 A_u, u32 *__restrict__ keys, u32 *__restrict__ flags,
                                                       u64 *n_dev, DevCtr *ctr, int passes) {
    PDL_ENTRY();
    __shared__ u64 sm[33];
    __shared__ u32 hh[4][256];
    for (int p = 0; p < passes; p++) hh[p][threadIdx.x] = 0;
    __syncthreads();
    if (n_in) n = *n_in;   // count on the device (a hybrid heap's TLSF share)
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_dev = n;
    u64 nnull = 0, ninv = 0;
    const u64 amask = (1ull << alog2) - 1;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    const u64 nround = (n + stride - 1) / stride;
    for (u64 r = 0; r < nround; r++) {
        u64 i = r * stride + (u64)blockIdx.x * blockDim.x + threadIdx.x;
        if (i < n) {
            u64 o = offs[i];
            u32 f = 0, key = 0;
            if (o == HEAP_NULL_U64) nnull++;
            else if ((o & amask) || (o >> alog2) >= A_u) ninv++;
            else {
                f = 1;
                key = (u32)(o >> alog2);
                for (int p = 0; p < passes; p++) atomicAdd(&hh[p][(key >> (8 * p)) & 255u], 1u);
            }
            flags[i] = f;
            keys[i] = key;
        }
    }
    u64 a = block_sum64<prims::NT>(nnull, sm);
    u64 b = block_sum64<prims::NT>(ninv, sm);
    if (threadIdx.x == 0) {
        if (a) atomicAdd(&ctr->frees_null, a);
        if (b) atomicAdd(&ctr->frees_invalid, b);
    }
    prims::os_hist_finish(hh, passes, ctr);
}

template <typename T>
__global__ void k_compact(const T *__restrict__ in, const u32 *__restrict__ flags,
                          const u32 *__restrict__ pos, const u64 *n_dev, T *__restrict__ out) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        if (flags[i]) out[pos[i]] = in[i];
}

// two arrays compacted by the same flags / positions in one launch
template <typename T>
__global__ void k_compact2(const T *__restrict__ a, const T *__restrict__ b, const u32 *__restrict__ flags,
                           const u32 *__restrict__ pos, const u64 *n_dev, T *__restrict__ oa, T *__restrict__ ob) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        if (flags[i]) { const u32 p = pos[i]; oa[p] = a[i]; ob[p] = b[i]; }
}

__device__ __forceinline__ bool bsearch_u64(const u64 *a, u64 n, u64 key) {
    u64 lo = 0, hi = n;
    while (lo < hi) {
        u64 mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo < n && a[lo] == key;
}

// Per sorted key: the first copy of each run of equal keys looks the key up in the block
// table (deleting it if live); the run's other copies are classified from that result.
// Live -> 1 ok + (copies-1) double; start of a free block -> all double; else all invalid.
__global__ void __launch_bounds__(256) k_free_lookup(const u32 *__restrict__ keys, const u64 *nk_dev,
                                                     u64 *__restrict__ slots, u64 tmask, u64 max_lines,
                                                     const u64 *__restrict__ fstart, const u64 *F_dev,
                                                     const u64 *__restrict__ bud_list, int K,
                                                     u32 *__restrict__ vflag, u64 *__restrict__ vs,
                                                     u64 *__restrict__ ve, DevCtr *ctr) {
    PDL_ENTRY();
    __shared__ u64 sm[33];
    const u64 nk = *nk_dev, F = F_dev ? *F_dev : 0;
    const u32 lane = lane_id(), g = lane / table::TILE_LANES, sub = lane % table::TILE_LANES;
    const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
    u64 c_ok = 0, c_dbl = 0, c_inv = 0, c_units = 0;
    for (u64 base = gw * table::KPW; base < nk; base += nwarps * table::KPW) {
        u64 idx = base + g;
        bool in = idx < nk;
        u32 key = in ? keys[idx] : 0;
        bool first = in && (idx == 0 || keys[idx - 1] != key);
        u64 s = table::lookup(slots, tmask, key, first, table::TOMB, max_lines);
        if (in && sub == 0) {
            u32 f = 0;
            if (first) {
                u64 ndup = 0;
                for (u64 j = idx + 1; j < nk && keys[j] == key; j++) ndup++;
                if (s != table::EMPTY) {
                    u64 z = table::slot_size(s);
                    f = 1;
                    vs[idx] = key;
                    ve[idx] = (u64)key + z;
                    c_ok++; c_dbl += ndup; c_units += z;
                } else if (bud_list ? buddy::is_free_start(bud_list, ctr, K, key)
                                    : bsearch_u64(fstart, F, key)) {
                    c_dbl += 1 + ndup;
                } else {
                    c_inv += 1 + ndup;
                }
            }
            vflag[idx] = f;
        }
    }
    u64 a = block_sum64<256>(c_ok, sm), b = block_sum64<256>(c_dbl, sm);
    u64 c = block_sum64<256>(c_inv, sm), d = block_sum64<256>(c_units, sm);
    if (threadIdx.x == 0) {
        if (a) { atomicAdd(&ctr->frees_ok, a); atomicAdd(&ctr->n_live, (u64)0 - a); atomicAdd(&ctr->tbl_tombs, a); }
        if (b) atomicAdd(&ctr->frees_double, b);
        if (c) atomicAdd(&ctr->frees_invalid, c);
        if (d) atomicAdd(&ctr->live_units, (u64)0 - d);
    }
}

// head flag: element i starts a new maximal run unless the previous block ends where it starts
__global__ void k_coal_flags(const u64 *__restrict__ ms, const u64 *__restrict__ me, const u64 *M_dev,
                             u32 *__restrict__ head) {
    PDL_ENTRY();
    const u64 M = *M_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (u64)gridDim.x * blockDim.x)
        head[i] = (i == 0 || me[i - 1] != ms[i]) ? 1u : 0u;
}

// heads write the run start, tails the run end (the coalesced block is [first start, last end))
__global__ void k_coal_write(const u64 *__restrict__ ms, const u64 *__restrict__ me, const u64 *M_dev,
                             const u32 *__restrict__ head, const u32 *__restrict__ pos,
                             u64 *__restrict__ os, u64 *__restrict__ oe, u64 cap, DevCtr *ctr) {
    PDL_ENTRY();
    const u64 M = *M_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (u64)gridDim.x * blockDim.x) {
        u32 h = head[i];
        u64 run = pos[i] + h - 1;
        if (run >= cap) { atomicOr(&ctr->error_flags, (u64)ERR_CAP_FREE); continue; }
        if (h) os[run] = ms[i];
        if (i + 1 == M || head[i + 1]) oe[run] = me[i];
    }
}

// ---------------------------------------------------------- SEGFIT_LIFO push stamps ----
// The paper's segregated fit keeps each bin as a stack (Alg. 4/5: every free and every split
// remainder is pushed at the head of its bin).  A block's position in its bin is its push time
// on a logical clock ctr->lifo_clock: the valid frees of a batch are pushed in ascending address
// order (clock + rank), an alloc's remainder at clock + request index.
__global__ void k_free_stamps(const u64 *nv_dev, const DevCtr *ctr, u32 *__restrict__ vstamp) {
    PDL_ENTRY();
    const u64 nv = *nv_dev, t0 = ctr->lifo_clock;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (u64)gridDim.x * blockDim.x)
        vstamp[i] = (u32)(t0 + i);
}
__global__ void k_clock_add(DevCtr *ctr, const u64 *n_dev, u64 n_host) {
    PDL_ENTRY();
    ctr->lifo_clock += n_dev ? *n_dev : n_host;
    if (ctr->lifo_clock >= 0xFFFFFFF0ull) ctr->error_flags |= ERR_CAP_LIVE;   // u32 stamps exhausted
}
// a coalesced run is pushed when its last free happens: its stamp is the largest in the run
// (freed stamps exceed every resident stamp); heads wrote their own stamp, the rest max into it
__global__ void k_coal_stamp(const u32 *__restrict__ mt, const u64 *M_dev, const u32 *__restrict__ head,
                             const u32 *__restrict__ pos, u32 *__restrict__ ot, u64 cap) {
    PDL_ENTRY();
    const u64 M = *M_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (u64)gridDim.x * blockDim.x) {
        const u64 run = pos[i] + head[i] - 1;
        if (!head[i] && run < cap) atomicMax(&ot[run], mt[i]);
    }
}
__global__ void k_coal_stamp_head(const u32 *__restrict__ mt, const u64 *M_dev, const u32 *__restrict__ head,
                                  const u32 *__restrict__ pos, u32 *__restrict__ ot, u64 cap) {
    PDL_ENTRY();
    const u64 M = *M_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (u64)gridDim.x * blockDim.x)
        if (head[i] && pos[i] < cap) ot[pos[i]] = mt[i];
}
// CSR key for SEGFIT_LIFO pieces: class major, newest push first
__global__ void k_lifo_keys(const u64 *__restrict__ fs, const u64 *__restrict__ fe, const u32 *__restrict__ ft,
                            const u64 *F_dev, u64 *__restrict__ key, u32 *__restrict__ val) {
    PDL_ENTRY();
    const u64 F = *F_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < F; i += (u64)gridDim.x * blockDim.x) {
        key[i] = ((u64)cls_insert(fe[i] - fs[i], 0) << 32) | (u64)(~ft[i]);
        val[i] = (u32)i;
    }
}
__global__ void k_u64_hi(const u64 *__restrict__ key, const u64 *n_dev, u32 *__restrict__ out) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = (u32)(key[i] >> 32);
}

// ------------------------------------------------------------------ alloc phase ----
// r = ceil(s / align) units (0 = fail: size 0 or larger than the arena), c = search class
// acc (optional, zeroed before): acc[0] += sum of r, acc[1] = max search class of a valid request
__global__ void k_alloc_prep(const u64 *__restrict__ sizes, u64 n, const u64 *n_in, int alog2, u64 A_u, int L,
                             int want_cls, u64 *__restrict__ r_out, u32 *__restrict__ c_out, u64 *acc) {
    PDL_ENTRY();
    if (n_in) n = *n_in;
    const u64 amask = (1ull << alog2) - 1;
    u64 t = 0, cm = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 s = sizes[i];
        u64 r = (s >> alog2) + ((s & amask) != 0);
        if (s == 0 || r > A_u) r = 0;
        r_out[i] = r;
        if (want_cls) {
            const u32 c = r ? cls_search(r, L) : 0xFFFFFFFFu;
            c_out[i] = c;
            t += r;
            if (r) cm = max(cm, (u64)c);
        }
    }
    if (acc) {
        for (int o = 16; o > 0; o >>= 1) {
            t += __shfl_xor_sync(FULLMASK, t, o);
            cm = max(cm, __shfl_xor_sync(FULLMASK, cm, o));
        }
        if (lane_id() == 0 && (t || cm)) {
            atomicAdd(&acc[0], t);
            atomicMax((unsigned long long *)&acc[1], (unsigned long long)cm);
        }
    }
}

__global__ void k_zero2(u64 *p) {
    PDL_ENTRY(); p[0] = 0; p[1] = 0; }

// piece survives iff it still has units
__global__ void k_piece_flags(const u64 *__restrict__ fs, const u64 *__restrict__ fe, const u64 *F_dev,
                              u32 *__restrict__ flags) {
    PDL_ENTRY();
    const u64 F = *F_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < F; i += (u64)gridDim.x * blockDim.x)
        flags[i] = fs[i] < fe[i] ? 1u : 0u;
}

// write results, insert the new live blocks into the block table, update counters
__global__ void __launch_bounds__(256) k_alloc_finish(const u64 *__restrict__ r, const u64 *__restrict__ out_u,
                                                      u64 n, const u64 *n_in, int alog2, u64 *__restrict__ out_bytes,
                                                      u64 *__restrict__ slots, u64 tmask, u64 max_lines,
                                                      DevCtr *ctr, u64 max_live,
                                                      const u32 *__restrict__ order = nullptr) {
    // order != nullptr (binary buddies): the request's units are 2^order[i] (r unused)
    PDL_ENTRY();
    __shared__ u64 sm[33];
    if (n_in) n = *n_in;
    const u32 lane = lane_id(), g = lane / table::TILE_LANES, sub = lane % table::TILE_LANES;
    const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
    u64 c_ok = 0, c_fail = 0, c_units = 0, c_used = 0, c_tomb = 0, c_full = 0, hw = 0;
    for (u64 base = gw * table::KPW; base < n; base += nwarps * table::KPW) {
        u64 i = base + g;
        bool in = i < n;
        u64 o = in ? out_u[i] : HEAP_NULL_U64;
        bool ok = in && o != HEAP_NULL_U64;
        u64 ri = ok ? (order ? (1ull << order[i]) : r[i]) : 0;
        int rc = table::insert(slots, tmask, o, ri, ok, max_lines);
        if (rc == 1) c_used++;
        if (rc == -1) c_tomb++;
        if (rc == 2) c_full++;
        if (in && sub == 0) {
            out_bytes[i] = ok ? (o << alog2) : HEAP_NULL_U64;
            if (ok) { c_ok++; c_units += ri; hw = max(hw, o + ri); }
            else c_fail++;
        }
    }
    u64 a = block_sum64<256>(c_ok, sm), b = block_sum64<256>(c_fail, sm), c = block_sum64<256>(c_units, sm);
    u64 d = block_sum64<256>(c_used, sm), e = block_sum64<256>(c_tomb, sm), f = block_sum64<256>(c_full, sm);
    hw = warp_max64(hw);
    __shared__ u64 hwm;
    if (threadIdx.x == 0) hwm = 0;
    __syncthreads();
    if (lane == 0 && hw) atomicMax(&hwm, hw);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (a) {
            atomicAdd(&ctr->allocs_ok, a);
            u64 nl = atomicAdd(&ctr->n_live, a) + a;
            if (nl > max_live) atomicOr(&ctr->error_flags, (u64)ERR_CAP_LIVE);
        }
        if (b) atomicAdd(&ctr->allocs_failed, b);
        if (c) atomicAdd(&ctr->live_units, c);
        if (d) atomicAdd(&ctr->tbl_used, d);
        if (e) atomicAdd(&ctr->tbl_tombs, (u64)0 - e);
        if (f) atomicOr(&ctr->error_flags, (u64)ERR_TABLE_FULL);
        if (hwm) atomicMax(&ctr->high_water_units, hwm);
    }
}

// ---------------------------------------------------------------- TLSF / SEGFIT ----
// Per batch the free blocks are grouped by their class (stable radix sort of (class, f)),
// giving each class an address-ordered CSR range consumed as a prefix (engine_tlsf.cuh reads it
// as 16-byte records).  A block whose carved remainder drops to a lower class k' joins k' in the
// engine's shared-memory head cache or, past the cache, in k''s overflow bitmap over f (a block
// is in one class at a time).  Class emptiness is kept in two-level bitmaps (one u32 word per
// first level, 32 second-level classes = one word), searched with ffs.
// (prims::NT threads: also counts the key digits of the `passes` sort passes that follow)
__global__ void __launch_bounds__(256) k_cls_keys(const u64 *__restrict__ fs, const u64 *__restrict__ fe,
                                                  const u64 *F_dev, int L, u32 *__restrict__ key, u32 *__restrict__ val,
                                                  DevCtr *ctr, int passes) {
    PDL_ENTRY();
    __shared__ u32 hh[4][256];
    for (int p = 0; p < passes; p++) hh[p][threadIdx.x] = 0;
    __syncthreads();
    const u64 F = *F_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < F; i += (u64)gridDim.x * blockDim.x) {
        const u32 k = cls_insert(fe[i] - fs[i], L);
        key[i] = k;
        val[i] = (u32)i;
        for (int p = 0; p < passes; p++) atomicAdd(&hh[p][(k >> (8 * p)) & 255u], 1u);
    }
    prims::os_hist_finish(hh, passes, ctr);
}

// off[k] = first position in the class-sorted order whose class >= k, for k = 0..NC
__global__ void k_cls_off(const u32 *__restrict__ key, const u64 *F_dev, int NC, u32 *__restrict__ off) {
    PDL_ENTRY();
    const u64 F = *F_dev;
    const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x, nth = (u64)gridDim.x * blockDim.x;
    if (F == 0) {
        for (u64 k = tid; k <= (u64)NC; k += nth) off[k] = 0;
        return;
    }
    for (u64 i = tid; i <= F; i += nth) {
        u32 lo = (i == 0) ? 0 : key[i - 1] + 1;
        u32 hi = (i == F) ? (u32)NC : key[i];
        for (u32 k = lo; k <= hi; k++) off[k] = (u32)i;
    }
}

constexpr int MAX_NC = 1024;   // class-offset array bound (TLSF classes of 2^32 units: 897)

// ------------------------------------------------------------------- FIRST FIT ----
// A 32-ary max tree over piece sizes: the first block with size >= r is found by one ballot
// per level (warp-cooperative descent), then the carved piece's ancestors are refreshed.
// Level l has ceil(F / 32^l) entries; levels are stored back to back at lvl_off[l].
__global__ void k_ff_leaves(const u64 *__restrict__ fs, const u64 *__restrict__ fe, const u64 *F_dev,
                            u64 *__restrict__ lv0) {
    PDL_ENTRY();
    const u64 F = *F_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < F; i += (u64)gridDim.x * blockDim.x)
        lv0[i] = fe[i] - fs[i];
}

__global__ void k_ff_level(const u64 *__restrict__ below, u64 *__restrict__ above, const u64 *F_dev, int l) {
    PDL_ENTRY();
    u64 nb = *F_dev;
    for (int i = 1; i < l; i++) nb = (nb + 31) >> 5;
    const u64 na = (nb + 31) >> 5;
    const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((u64)gridDim.x * blockDim.x) >> 5;
    for (u64 j = gw; j < na; j += nw) {
        u64 idx = j * 32 + lane_id();
        u64 v = idx < nb ? below[idx] : 0;
        v = warp_max64(v);
        if (lane_id() == 0) above[j] = v;
    }
}

constexpr int FF_MAX_LEVELS = 8;

// NEXT_FIT (rover != nullptr, reading C27): the search starts at the first piece whose start is
// >= the rover — walk up from that leaf checking only later siblings, descend into the first
// subtree holding a fit — and wraps to the plain first-fit search from piece 0 when nothing at
// or after the rover fits.  Pieces only shrink from their low end during the phase, so after a
// carve of piece f the rover (its new start) is again at index f.
__global__ void __launch_bounds__(32) k_ff_engine(u64 *tree, const u64 *__restrict__ lvl_off, int nlev,
                                                  u64 *fs, const u64 *F_dev, const u64 *__restrict__ r, u64 n,
                                                  const u64 *n_in, u64 *__restrict__ out_u, u64 *rover) {
    PDL_ENTRY();
    const u32 lane = lane_id();
    if (n_in) n = *n_in;
    u64 sz[FF_MAX_LEVELS];
    u64 F = *F_dev;
    sz[0] = F;
    for (int l = 1; l < nlev; l++) sz[l] = (sz[l - 1] + 31) >> 5;
    int top = 0;
    while (top + 1 < nlev && sz[top] > 32) top++;
    u64 f0 = 0;                  // rover as a piece index
    bool moved = false;
    if (rover) {
        const u64 R = *rover;
        u64 lo = 0, hi = F;      // first piece with start >= R
        while (hi - lo > 32) {
            const u64 step = (hi - lo + 31) >> 5;
            u64 idx = lo + (u64)(lane + 1) * step - 1;
            if (idx >= hi) idx = hi - 1;
            const u32 b = __ballot_sync(FULLMASK, fs[idx] >= R);
            if (!b) { lo = hi; break; }
            const u32 fl = __ffs(b) - 1;
            const u64 nlo = lo + (u64)fl * step, nhi = lo + (u64)(fl + 1) * step;
            lo = nlo;
            hi = nhi < hi ? nhi : hi;
        }
        if (lo < hi) {
            const u32 b = __ballot_sync(FULLMASK, lo + lane < hi && fs[lo + lane] >= R);
            lo = b ? lo + __ffs(b) - 1 : hi;
        }
        f0 = lo;
    }
    for (u64 i = 0; i < n; i++) {
        u64 ri = r[i];
        if (ri == 0 || F == 0) { if (lane == 0) out_u[i] = HEAP_NULL_U64; continue; }
        u64 f = ~0ull;
        if (rover && f0 < F) {
            // leaves of f0's group at or after f0
            u64 g = f0 >> 5, idx = g * 32 + lane;
            u64 v = (idx < sz[0] && idx >= f0) ? tree[lvl_off[0] + idx] : 0;
            u32 b = __ballot_sync(FULLMASK, v >= ri);
            if (b) f = g * 32 + __ffs(b) - 1;
            u64 node = g;
            for (int l = 1; l <= top && f == ~0ull; l++) {
                g = node >> 5;
                idx = g * 32 + lane;
                v = (idx < sz[l] && idx > node) ? tree[lvl_off[l] + idx] : 0;
                b = __ballot_sync(FULLMASK, v >= ri);
                if (b) {
                    u64 j = g * 32 + __ffs(b) - 1;
                    for (int ll = l - 1; ll >= 0; ll--) {
                        idx = j * 32 + lane;
                        v = idx < sz[ll] ? tree[lvl_off[ll] + idx] : 0;
                        j = j * 32 + __ffs(__ballot_sync(FULLMASK, v >= ri)) - 1;
                    }
                    f = j;
                }
                node = g;
            }
        }
        if (f == ~0ull) {        // first fit from piece 0 (also the wrap-around of next fit)
            u64 j = 0;           // node index at the current level (level top has one node: 0)
            bool fail = false;
            for (int l = top; l >= 0; l--) {
                u64 idx = j * 32 + lane;
                u64 v = idx < sz[l] ? tree[lvl_off[l] + idx] : 0;
                u32 b = __ballot_sync(FULLMASK, v >= ri);
                if (!b) { fail = true; break; }
                j = j * 32 + __ffs(b) - 1;
            }
            if (fail) { if (lane == 0) out_u[i] = HEAP_NULL_U64; continue; }
            f = j;
        }
        f0 = f;
        moved = true;
        if (lane == 0) {
            u64 s = fs[f];
            out_u[i] = s;
            fs[f] = s + ri;
            tree[lvl_off[0] + f] -= ri;
        }
        __syncwarp();
        u64 node = f;
        for (int l = 1; l <= top; l++) {
            u64 p = node >> 5;
            u64 idx = p * 32 + lane;
            u64 v = idx < sz[l - 1] ? tree[lvl_off[l - 1] + idx] : 0;
            v = warp_max64(v);
            if (lane == 0) tree[lvl_off[l] + p] = v;
            __syncwarp();
            node = p;
        }
    }
    if (rover && moved && lane == 0) *rover = fs[f0];   // the end of the last allocation
}

// -------------------------------------------------------------------- BEST FIT ----
// Pieces sorted by key = (size << FB) | f, i.e. by (size, address).  Per request a 32-ary
// warp search finds the first key >= (r << FB): the smallest fitting block, lowest address on
// ties (Alg. 3 with reading C3).  The carved piece moves down to its new rank (warp shift).
// The array lives in shared memory when it fits, otherwise in global memory.
// (prims::NT threads: also counts the key digits of the `passes` sort passes that follow)
__global__ void __launch_bounds__(256) k_bf_keys(const u64 *__restrict__ fs, const u64 *__restrict__ fe,
                                                 const u64 *F_dev, int FB, u64 *__restrict__ key, DevCtr *ctr,
                                                 int passes) {
    PDL_ENTRY();
    __shared__ u32 hh[8][256];
    for (int p = 0; p < passes; p++) hh[p][threadIdx.x] = 0;
    __syncthreads();
    const u64 F = *F_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < F; i += (u64)gridDim.x * blockDim.x) {
        const u64 k = ((fe[i] - fs[i]) << FB) | i;
        key[i] = k;
        for (int p = 0; p < passes; p++) atomicAdd(&hh[p][(u32)(k >> (8 * p)) & 255u], 1u);
    }
    prims::os_hist_finish(hh, passes, ctr);
}

__device__ __forceinline__ u64 warp_lower_bound(const u64 *a, u64 lo, u64 hi, u64 target) {
    const u32 lane = lane_id();
    while (hi - lo > 32) {
        u64 step = (hi - lo + 31) >> 5;
        u64 idx = lo + (u64)(lane + 1) * step - 1;
        if (idx >= hi) idx = hi - 1;
        u32 b = __ballot_sync(FULLMASK, a[idx] >= target);
        if (!b) return hi;
        u32 fl = __ffs(b) - 1;
        u64 nlo = lo + (u64)fl * step;
        u64 nhi = lo + (u64)(fl + 1) * step;
        if (nhi > hi) nhi = hi;
        lo = nlo;
        hi = nhi;   // answer in [lo, hi]: a[hi-1] >= target
    }
    u64 idx = lo + lane;
    u32 b = __ballot_sync(FULLMASK, idx < hi && a[idx] >= target);
    return b ? lo + __ffs(b) - 1 : hi;
}

// the flat engine: one sorted key array (shared or global memory), warp shift per request
__device__ void bf_flat(u64 *keys, u64 nb, int FB, u64 *fs, const u64 *__restrict__ r, u64 n,
                        u64 *__restrict__ out_u) {
    const u32 lane = lane_id();
    const u64 fmask = (1ull << FB) - 1;
    for (u64 i = 0; i < n; i++) {
        u64 ri = r[i];
        if (ri == 0) { if (lane == 0) out_u[i] = HEAP_NULL_U64; continue; }
        u64 p = warp_lower_bound(keys, 0, nb, ri << FB);
        if (p >= nb) { if (lane == 0) out_u[i] = HEAP_NULL_U64; continue; }
        u64 key = keys[p];
        u64 z = key >> FB, f = key & fmask;
        if (lane == 0) {
            u64 s = fs[f];
            out_u[i] = s;
            fs[f] = s + ri;
        }
        u64 z2 = z - ri;
        if (z2) {
            u64 nkey = (z2 << FB) | f;
            u64 q = warp_lower_bound(keys, 0, p, nkey);
            // shift [q, p) up by one, highest chunk first
            for (u64 hi = p; hi > q;) {
                u64 lo = hi >= q + 32 ? hi - 32 : q;
                u64 idx = lo + lane;
                u64 v = idx < hi ? keys[idx] : 0;
                __syncwarp();
                if (idx < hi) keys[idx + 1] = v;
                __syncwarp();
                hi = lo;
            }
            if (lane == 0) keys[q] = nkey;
        } else {
            for (u64 lo = p + 1; lo < nb; lo += 32) {
                u64 idx = lo + lane;
                u64 v = idx < nb ? keys[idx] : 0;
                __syncwarp();
                if (idx < nb) keys[idx - 1] = v;
                __syncwarp();
            }
            nb--;
        }
        __syncwarp();
    }
}

// The blocked engine: the same key order kept as a list of chunks of <= 32 keys (one per lane) in
// shared memory, with the chunks' maxima in position order.  A request costs one 32-ary search over
// the maxima, one ballot inside a chunk, and one-step shifts inside at most two chunks (delete the
// chosen key, insert the carved piece's new key), instead of a shift across up to F keys.  Results
// are those of bf_flat (same keys, same order).  Chunks only split (a full chunk into two of 16):
// with phi = sum over chunks of max(0, count - 16), an insert raises phi by at most 1, a split
// lowers it by 16, and phi starts at 8 per chunk, so there are at most nc0/2 + n/16 splits
// (nc0 = ceil(F/BF_FILL)); batches that could exceed BF_NCH chunks use bf_flat on the global array.
constexpr u32 BF_NCH = 640, BF_FILL = 24;
struct BfSmem {
    u64 K[BF_NCH * 32];     // chunk id c holds K[c*32 .. c*32 + cnt[c])
    u64 mx[BF_NCH];         // largest key of the chunk at position i
    unsigned short ord[BF_NCH], fl[BF_NCH];   // chunk id at position i; free chunk ids
    unsigned char cnt[BF_NCH];
    u32 nch, nfl;
};

__device__ __forceinline__ void bf_pos_insert(BfSmem &S, u32 i, u32 c, u64 m) {   // new position i
    const u32 lane = lane_id();
    const int n0 = (int)S.nch;
    for (int hi = n0; hi > (int)i;) {                    // shift [i, nch) right, top chunk first
        const int lo = hi - 32 > (int)i ? hi - 32 : (int)i;
        const int idx = lo + (int)lane;
        unsigned short o = 0;
        u64 v = 0;
        if (idx < hi) { o = S.ord[idx]; v = S.mx[idx]; }
        __syncwarp();
        if (idx < hi) { S.ord[idx + 1] = o; S.mx[idx + 1] = v; }
        __syncwarp();
        hi = lo;
    }
    __syncwarp();                                        // every lane has read nch
    if (lane == 0) { S.ord[i] = (unsigned short)c; S.mx[i] = m; S.nch = (u32)n0 + 1; }
    __syncwarp();
}

__device__ __forceinline__ void bf_pos_remove(BfSmem &S, u32 i) {
    const u32 lane = lane_id();
    const u32 n = S.nch;
    for (u32 lo = i + 1; lo < n; lo += 32) {
        const u32 idx = lo + lane;
        unsigned short o = 0;
        u64 v = 0;
        if (idx < n) { o = S.ord[idx]; v = S.mx[idx]; }
        __syncwarp();
        if (idx < n) { S.ord[idx - 1] = o; S.mx[idx - 1] = v; }
        __syncwarp();
    }
    __syncwarp();
    if (lane == 0) S.nch = n - 1;
    __syncwarp();
}

__device__ void bf_blocked(BfSmem &S, u64 *gkeys, const u64 *F_dev, int FB, u64 *fs, const u64 *__restrict__ r, u64 n,
                           u64 *__restrict__ out_u) {
    const u32 lane = lane_id();
    const u64 nb = *F_dev;
    const u64 nc0_ = (nb + BF_FILL - 1) / BF_FILL;
    if (nc0_ + (nc0_ + 1) / 2 + (n + 15) / 16 + 2 > BF_NCH) {   // could outgrow the chunk pool
        bf_flat(gkeys, nb, FB, fs, r, n, out_u);
        return;
    }
    // build: chunks of BF_FILL keys in order
    const u32 nc0 = (u32)((nb + BF_FILL - 1) / BF_FILL);
    for (u32 c = 0; c < nc0; c++) {
        const u64 b = (u64)c * BF_FILL, e = min(b + BF_FILL, nb);
        if (lane < e - b) S.K[c * 32 + lane] = gkeys[b + lane];
        if (lane == 0) { S.cnt[c] = (unsigned char)(e - b); S.ord[c] = (unsigned short)c; S.mx[c] = gkeys[e - 1]; }
    }
    for (u32 c = nc0 + lane; c < BF_NCH; c += 32) S.fl[BF_NCH - 1 - c] = (unsigned short)c;   // pop from the end: lowest id first
    if (lane == 0) { S.nch = nc0; S.nfl = BF_NCH - nc0; }
    __syncwarp();
    const u64 fmask = (1ull << FB) - 1;
    u64 r_next = n ? r[0] : 0;                     // the next request's size, loaded one step ahead
    for (u64 i = 0; i < n; i++) {
        const u64 ri = r_next;
        if (i + 1 < n) r_next = r[i + 1];
        if (ri == 0) { if (lane == 0) out_u[i] = HEAP_NULL_U64; continue; }
        const u64 target = ri << FB;
        const u32 nch = S.nch;
        const u32 p = (u32)warp_lower_bound(S.mx, 0, nch, target);
        if (p >= nch) { if (lane == 0) out_u[i] = HEAP_NULL_U64; continue; }
        u32 c = S.ord[p];
        u32 m = S.cnt[c];
        u64 v = lane < m ? S.K[c * 32 + lane] : ~0ull;
        const u32 j = __ffs(__ballot_sync(FULLMASK, lane < m && v >= target)) - 1;   // exists: mx[p] >= target
        const u64 key = __shfl_sync(FULLMASK, v, j);
        const u64 z = key >> FB, f = key & fmask;
        // the piece's start: its load overlaps the chunk updates below, the stores come last
        const u64 s0 = lane == 0 ? fs[f] : 0;
        // delete key j of chunk c (position p)
        __syncwarp();
        if (lane > j && lane < m) S.K[c * 32 + lane - 1] = v;
        if (lane == 0) S.cnt[c] = (unsigned char)(m - 1);
        __syncwarp();
        if (m == 1) {
            bf_pos_remove(S, p);
            if (lane == 0) S.fl[S.nfl++] = (unsigned short)c;
        } else if (j == m - 1) {
            if (lane == 0) S.mx[p] = S.K[c * 32 + m - 2];
        }
        __syncwarp();
        // insert the carved piece's new key
        const u64 z2 = z - ri;
        if (!z2) {
            if (lane == 0) { out_u[i] = s0; fs[f] = s0 + ri; }
            continue;
        }
        const u64 x = (z2 << FB) | f;
        const u32 nch1 = S.nch;
        u32 q = nch1 ? (u32)warp_lower_bound(S.mx, 0, nch1, x) : 0;
        __syncwarp();
        if (nch1 == 0) {
            if (lane == 0) { const u32 c0 = S.fl[--S.nfl]; S.cnt[c0] = 0; S.ord[0] = (unsigned short)c0; S.mx[0] = 0; S.nch = 1; }
            __syncwarp();
        } else if (q == nch1) {
            q = nch1 - 1;                            // above every key: the last chunk
        }
        c = S.ord[q];
        m = S.cnt[c];
        if (m == 32) {                               // split: upper half to a new chunk at q + 1
            u32 c2 = 0;
            if (lane == 0) c2 = S.fl[--S.nfl];
            c2 = __shfl_sync(FULLMASK, c2, 0);
            const u64 w = S.K[c * 32 + lane];
            if (lane >= 16) S.K[c2 * 32 + lane - 16] = w;
            const u64 top = __shfl_sync(FULLMASK, w, 31), mid = __shfl_sync(FULLMASK, w, 15);
            __syncwarp();                            // every lane has read cnt[c] and mx
            if (lane == 0) { S.cnt[c] = 16; S.cnt[c2] = 16; S.mx[q] = mid; }
            __syncwarp();
            bf_pos_insert(S, q + 1, c2, top);
            if (x > mid) { q = q + 1; c = c2; }
            m = 16;
        }
        v = lane < m ? S.K[c * 32 + lane] : 0;
        const u32 at = __popc(__ballot_sync(FULLMASK, lane < m && v < x));
        __syncwarp();
        if (lane >= at && lane < m) S.K[c * 32 + lane + 1] = v;
        if (lane == 0) {
            S.K[c * 32 + at] = x;
            S.cnt[c] = (unsigned char)(m + 1);
            if (at == m) S.mx[q] = x;
            out_u[i] = s0;
            fs[f] = s0 + ri;
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(32) k_bf_engine(u64 *gkeys, const u64 *F_dev, int FB, u64 *fs,
                                                  const u64 *__restrict__ r, u64 n, const u64 *n_in,
                                                  u64 *__restrict__ out_u) {
    PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char bf_raw[];
    if (n_in) n = *n_in;
    bf_blocked(*reinterpret_cast<BfSmem *>(bf_raw), gkeys, F_dev, FB, fs, r, n, out_u);
}

// ------------------------------------------------------ BEST FIT, class-indexed ----
// The same key order (size << FB | f ascending = (size, address), Alg. 3 with reading C3) kept as a
// doubly linked list of chunks of <= 32 keys in shared memory, with a TLSF-style class index over
// it (the two-level class of the size, used here only as an index): per class its
// member count and the chunk holding its smallest key, and a two-level bitmap of the nonempty
// classes.  The smallest key >= (r << FB) is either in r's own class or the smallest key of the
// first nonempty class above it (every size in a higher class exceeds r), so a search is one ffs on
// the bitmap (first nonempty class >= cls(r)), one chunk load at that class's start chunk and one
// ballot — a walk to the next chunk only when the class's members below r fill the rest of the
// chunk.  No 32-ary search over chunk maxima, no position array to shift when a chunk splits or
// empties.  Piece starts are kept in shared memory (u32 units) for the batch.  Results are those of
// bf_blocked and bf_flat (same keys, same order).  Chunk budget: as bf_blocked (fill 24, splits
// 32 -> 16 + 16, at most nc0/2 + n/16 splits); heaps beyond it, beyond BC_FS pieces or with unit
// addresses >= 2^32 run bf_blocked.
#ifndef BF_TIMING
#define BF_TIMING 0   // phase clocks of k_bf_cls_engine into ctr->eng[0..5] (tools/micro/bf_probe.py)
#endif
constexpr u32 BC_CH = 512, BC_FILL = 24, BC_FS = 12288, BC_NC = 928;
constexpr unsigned short BC_NIL = 0xFFFF;
struct BcSmem {
    u64 K[BC_CH * 32];                         // chunk c holds K[c*32 .. c*32 + cnt[c]), ascending
    u32 fsm[BC_FS];                            // piece starts (units)
    u32 ccnt[BC_NC];                           // members per class
    unsigned short cch[BC_NC];                 // chunk holding the class's smallest key (ccnt > 0)
    unsigned short nxt[BC_CH], prv[BC_CH], fl[BC_CH];
    unsigned char cnt[BC_CH];
    u32 cw[32];                                // nonempty classes, one bit per class
};
constexpr size_t BF_ENGINE_SMEM = sizeof(BcSmem) > sizeof(BfSmem) ? sizeof(BcSmem) : sizeof(BfSmem);

__device__ __forceinline__ u32 bc_cls(u64 key, int FB) { return cls_insert(key >> FB, 5); }

// first nonempty class >= c (NIL32 if none); sw = one bit per nonzero bitmap word
__device__ __forceinline__ u32 bc_first_ge(const BcSmem &S, u32 sw, u32 c) {
    if (c >= BC_NC) return NIL32;
    const u32 w = c >> 5;
    const u32 m = S.cw[w] & (0xFFFFFFFFu << (c & 31));
    if (m) return (w << 5) + __ffs(m) - 1;
    const u32 sm = (w >= 31) ? 0u : (sw & (0xFFFFFFFFu << (w + 1)));
    if (!sm) return NIL32;
    const u32 w2 = __ffs(sm) - 1;
    return (w2 << 5) + __ffs(S.cw[w2]) - 1;
}

// the first key >= t: chunk c (BC_NIL: none), slot j, chunk count m, each lane's key v of chunk c.
// kt = cls(t): keys of classes below kt are < t, so the walk starts at the first nonempty class >= kt.
__device__ __forceinline__ void bc_find(const BcSmem &S, u32 sw, u32 kt, u64 t, u32 &c, u32 &j, u32 &m, u64 &v) {
    const u32 lane = lane_id();
    const u32 k1 = bc_first_ge(S, sw, kt);
    c = (k1 == NIL32) ? (u32)BC_NIL : (u32)S.cch[k1];
    j = 0;
    m = 0;
    v = 0;
    while (c != BC_NIL) {
        m = S.cnt[c];
        v = lane < m ? S.K[c * 32 + lane] : 0ull;
        const u32 b = __ballot_sync(FULLMASK, lane < m && v >= t);
        if (b) { j = __ffs(b) - 1; return; }
        c = S.nxt[c];
    }
}

__device__ void bf_classes(unsigned char *bf_raw, u64 *gkeys, const u64 *F_dev, int FB, u64 *fs,
                           const u64 *__restrict__ r, u64 n, u64 *__restrict__ out_u, int cls_ok, u64 *dbg) {
    const u32 lane = lane_id();
    const u64 F = *F_dev;
    const u64 nc0 = (F + BC_FILL - 1) / BC_FILL;
#if BF_TIMING
    long long tq = clock64(), tph[6] = {0, 0, 0, 0, 0, 0};
#define BF_T(k) do { const long long _t = clock64(); tph[k] += _t - tq; tq = _t; } while (0)
#else
#define BF_T(k) do { } while (0)
#endif
    if (!cls_ok || F > BC_FS || nc0 + (nc0 + 1) / 2 + (n + 15) / 16 + 2 > BC_CH) {
        bf_blocked(*reinterpret_cast<BfSmem *>(bf_raw), gkeys, F_dev, FB, fs, r, n, out_u);
        return;
    }
    BcSmem &S = *reinterpret_cast<BcSmem *>(bf_raw);
    const u64 fmask = (1ull << FB) - 1;
    // ---- build: chunks of BC_FILL keys in order, class starts and counts, bitmap ----
    for (u32 k = lane; k < BC_NC; k += 32) S.ccnt[k] = 0;
    for (u64 x = lane; x < F; x += 32) {
        S.K[(x / BC_FILL) * 32 + x % BC_FILL] = gkeys[x];
        S.fsm[x] = (u32)fs[x];
    }
    for (u32 c = lane; c < (u32)nc0; c += 32) {
        S.cnt[c] = (unsigned char)min((u64)BC_FILL, F - (u64)c * BC_FILL);
        S.nxt[c] = (unsigned short)(c + 1 < nc0 ? c + 1 : BC_NIL);
        S.prv[c] = (unsigned short)(c ? c - 1 : BC_NIL);
    }
    for (u32 c = (u32)nc0 + lane; c < BC_CH; c += 32) S.fl[BC_CH - 1 - c] = (unsigned short)c;   // lowest id popped first
    u32 nfl = BC_CH - (u32)nc0;
    __syncwarp();
    for (u64 x = lane; x < F; x += 32) {                 // class starts: chunk of the first key, start index
        const u32 k = bc_cls(gkeys[x], FB);
        if (x == 0 || bc_cls(gkeys[x - 1], FB) != k) { S.cch[k] = (unsigned short)(x / BC_FILL); S.ccnt[k] = (u32)x; }
    }
    __syncwarp();
    for (u64 x = lane; x < F; x += 32) {                 // class ends: count
        const u32 k = bc_cls(gkeys[x], FB);
        if (x + 1 == F || bc_cls(gkeys[x + 1], FB) != k) S.ccnt[k] = (u32)x - S.ccnt[k] + 1;
    }
    __syncwarp();
    for (u32 w = 0; w < 32; w++) {
        const u32 k = w * 32 + lane;
        const u32 b = __ballot_sync(FULLMASK, k < BC_NC && S.ccnt[k] > 0);
        if (lane == 0) S.cw[w] = b;
    }
    __syncwarp();
    u32 sw = __ballot_sync(FULLMASK, S.cw[lane] != 0u);
    u32 tail = nc0 ? (u32)nc0 - 1 : (u32)BC_NIL;      // last chunk (the list's head is never needed)
    BF_T(0);
    // ---- requests in order ----
    for (u64 i0 = 0; i0 < n; i0 += 32) {
        const u64 il = i0 + lane;
        const u64 rl = il < n ? r[il] : 0ull;
        const u32 kl = rl ? cls_insert(rl, 5) : 0u;      // r <= A_u < 2^32
        const u32 nj = (n - i0) < 32 ? (u32)(n - i0) : 32u;
        for (u32 jj = 0; jj < nj; jj++) {
            const u64 ri = __shfl_sync(FULLMASK, rl, jj);
            const u32 kr = __shfl_sync(FULLMASK, kl, jj);
            const u64 i = i0 + jj;
            if (ri == 0) { if (lane == 0) out_u[i] = HEAP_NULL_U64; continue; }
            u32 c, j, m;
            u64 v;
            bc_find(S, sw, kr, ri << FB, c, j, m, v);
            if (c == BC_NIL) { if (lane == 0) out_u[i] = HEAP_NULL_U64; continue; }
            BF_T(1);
            const u64 key = __shfl_sync(FULLMASK, v, j);
            const u64 pv = __shfl_sync(FULLMASK, v, j ? j - 1 : 0);
            const u64 z = key >> FB;
            const u32 f = (u32)(key & fmask);
            const u32 k = cls_insert(z, 5);
            const u32 s0 = S.fsm[f];
            const bool first = S.cch[k] == c && (j == 0 || bc_cls(pv, FB) != k);
            const u32 cc = S.ccnt[k] - 1;
            const u32 cn = S.nxt[c], cp = S.prv[c];
            const u32 cwk = S.cw[k >> 5];
            __syncwarp();
            // ---- delete slot j of chunk c ----
            const u32 m1 = m - 1;
            if (lane > j && lane < m) S.K[c * 32 + lane - 1] = v;
            if (lane == 0) {
                S.cnt[c] = (unsigned char)m1;
                S.ccnt[k] = cc;
                if (cc == 0) S.cw[k >> 5] = cwk & ~(1u << (k & 31));
                else if (first) S.cch[k] = (unsigned short)((j < m1) ? c : cn);
                if (m1 == 0) {                               // chunk emptied: unlink, free
                    if (cp != BC_NIL) S.nxt[cp] = (unsigned short)cn;
                    if (cn != BC_NIL) S.prv[cn] = (unsigned short)cp;
                    S.fl[nfl] = (unsigned short)c;
                }
            }
            if (cc == 0 && (cwk & ~(1u << (k & 31))) == 0u) sw &= ~(1u << (k >> 5));
            if (m1 == 0) {
                if (cn == BC_NIL) tail = cp;
                nfl++;
            }
            __syncwarp();
            BF_T(2);
            // ---- the remainder (z - r, f) joins its class ----
            const u64 z2 = z - ri;
            if (z2) {
                const u64 x = (z2 << FB) | f;
                const u32 k2 = cls_insert(z2, 5);
                u32 c2, j2, m2;
                u64 v2;
                bc_find(S, sw, k2, x, c2, j2, m2, v2);
                BF_T(3);
                if (c2 == BC_NIL) {                          // above every key: append to the tail chunk
                    if (tail == BC_NIL) {                    // the list is empty: a fresh chunk
                        c2 = S.fl[--nfl];
                        __syncwarp();
                        if (lane == 0) { S.nxt[c2] = BC_NIL; S.prv[c2] = BC_NIL; S.cnt[c2] = 0; }
                        tail = c2;
                        m2 = 0;
                        v2 = 0;
                    } else {
                        c2 = tail;
                        m2 = S.cnt[c2];
                        v2 = lane < m2 ? S.K[c2 * 32 + lane] : 0ull;
                    }
                    j2 = m2;
                }
                if (m2 == 32) {                              // split: upper half to a new chunk after c2
                    const u32 cN = S.fl[--nfl];
                    const u32 c2n = S.nxt[c2];
                    const u64 pl = __shfl_sync(FULLMASK, v2, lane ? lane - 1 : 0);
                    __syncwarp();
                    if (lane >= 16) {
                        S.K[cN * 32 + lane - 16] = v2;
                        const u32 kv = bc_cls(v2, FB);
                        if (kv != bc_cls(pl, FB)) S.cch[kv] = (unsigned short)cN;   // class starts that moved
                    }
                    if (lane == 0) {
                        S.cnt[c2] = 16;
                        S.cnt[cN] = 16;
                        S.nxt[cN] = (unsigned short)c2n;
                        S.prv[cN] = (unsigned short)c2;
                        S.nxt[c2] = (unsigned short)cN;
                        if (c2n != BC_NIL) S.prv[c2n] = (unsigned short)cN;
                    }
                    if (c2n == BC_NIL) tail = cN;
                    const u64 hi = __shfl_sync(FULLMASK, v2, (lane + 16) & 31);
                    if (j2 > 16) { c2 = cN; j2 -= 16; v2 = hi; }
                    m2 = 16;
                    __syncwarp();
                }
                // is x the smallest member of class k2?  (its predecessor in key order is of a lower class)
                u64 pk;
                bool haspk = true;
                if (j2 > 0) pk = __shfl_sync(FULLMASK, v2, j2 - 1);
                else {
                    const u32 p = S.prv[c2];
                    if (p == BC_NIL) { haspk = false; pk = 0; }
                    else pk = S.K[p * 32 + S.cnt[p] - 1];
                }
                const bool first2 = !haspk || bc_cls(pk, FB) != k2;
                const u32 cc2 = S.ccnt[k2];
                const u32 cwk2 = S.cw[k2 >> 5];
                __syncwarp();
                if (lane >= j2 && lane < m2) S.K[c2 * 32 + lane + 1] = v2;
                if (lane == 0) {
                    S.K[c2 * 32 + j2] = x;
                    S.cnt[c2] = (unsigned char)(m2 + 1);
                    S.ccnt[k2] = cc2 + 1;
                    if (cc2 == 0) S.cw[k2 >> 5] = cwk2 | (1u << (k2 & 31));
                    if (first2) S.cch[k2] = (unsigned short)c2;
                }
                sw |= 1u << (k2 >> 5);
                BF_T(4);
            }
            if (lane == 0) {
                out_u[i] = s0;
                S.fsm[f] = s0 + (u32)ri;
            }
            __syncwarp();
        }
    }
    __syncwarp();
    for (u64 x = lane; x < F; x += 32) fs[x] = S.fsm[x];
#if BF_TIMING
    BF_T(5);
    if (lane == 0) for (int k = 0; k < 6; k++) dbg[16 + k] += (u64)tph[k];
#endif
#undef BF_T
}

__global__ void __launch_bounds__(32) k_bf_cls_engine(u64 *gkeys, const u64 *F_dev, int FB, u64 *fs,
                                                      const u64 *__restrict__ r, u64 n, const u64 *n_in,
                                                      u64 *__restrict__ out_u, int cls_ok, u64 *dbg) {
    PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char bf_raw[];
    if (n_in) n = *n_in;
    bf_classes(bf_raw, gkeys, F_dev, FB, fs, r, n, out_u, cls_ok, dbg);
}

// ------------------------------------------------- BEST FIT, speculative chunks ----
// One warp serves the requests in chunks of up to 32 (lane = request order) against the
// chunk-start key array A (sorted (size, address) keys in shared memory, as bf_flat):
//   * each lane finds p = the first key >= (r << FB) by binary search; lanes with the same p are
//     ranked in time order and take A[p + rank] (q);
//   * lane i is *dirty* if an earlier lane of another group took an index in [p_i, q_i] (its
//     choice is then not the smallest untaken key), or an earlier lane's remainder x_j (the carved
//     piece's new key) lies in [r_i << FB, A[q_i]) (a better fit appeared).  Up to the first dirty
//     lane the choices are exactly the sequential best fit (Alg. 3, reading C3): at request i the
//     free set is A minus the earlier choices plus their remainders, the first untaken index
//     >= p_i is q_i, and no remainder lies below A[q_i] and at or above the request;
//   * the committed prefix writes its results, and A is rebuilt into the other buffer: the
//     taken keys removed (a bitmap over indices), the remainders merged in (each one's insertion
//     point in A by binary search, a bitmap over insertion points; its rank among the remainders
//     by ballots), every key moved by popcounts over the two bitmaps, 4 tiles of 32 in flight.
// Lane 0 is never dirty, so every chunk commits at least one request.  Measured commit rate on
// config 2: ~17-19 requests per 32-request chunk (tools/research/bestfit_chunk_model.cpp).
constexpr u32 BS_N = 8192, BS_RB = 512;
struct BsSmem {
    u64 A[2][BS_N];
    u32 fsm[BS_N];
    u64 rb[BS_RB];
    u64 dx[32], sX[32];
    uint2 dqp[32];                     // per lane: (p, q or NONE)
    u32 rmb[BS_N / 32 + 4];            // removed-index bitmap of the chunk (zero between chunks)
    u32 lbm[BS_N / 32 + 4];            // remainders' insertion points (zero between chunks)
};
constexpr size_t BF_ENGINE_SMEM2 = sizeof(BsSmem) > BF_ENGINE_SMEM ? sizeof(BsSmem) : BF_ENGINE_SMEM;

// #(A[i] < t) over a sorted A[0, N): fixed power-of-two steps (the same trip count on every lane,
// so several searches of one thread interleave instead of diverging)
template <typename T>
__device__ __forceinline__ u32 bs_lower_bound(const T *A, u32 N, T t) {
    u32 lo = 0;
    for (u32 step = N ? 1u << (31 - __clz(N)) : 0u; step; step >>= 1)
        if (lo + step <= N && A[lo + step - 1] < t) lo += step;
    return lo;
}
__global__ void __launch_bounds__(32) k_bf_spec_engine(u64 *gkeys, const u64 *F_dev, int FB, u64 *fs,
                                                       const u64 *__restrict__ r, u64 n, const u64 *n_in,
                                                       u64 *__restrict__ out_u, int cls_ok, u64 *dbg) {
    PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char bf_raw[];
    if (n_in) n = *n_in;
    const u32 lane = lane_id();
    const u64 F = *F_dev;
    if (!cls_ok || F > BS_N) {
        bf_classes(bf_raw, gkeys, F_dev, FB, fs, r, n, out_u, cls_ok, dbg);
        return;
    }
    BsSmem &S = *reinterpret_cast<BsSmem *>(bf_raw);
    const u64 fmask = (1ull << FB) - 1;
    for (u32 x = lane; x < (u32)F; x += 32) {
        S.A[0][x] = gkeys[x];
        S.fsm[x] = (u32)fs[x];
    }
    for (u32 x = lane; x < BS_N / 32 + 4; x += 32) { S.rmb[x] = 0u; S.lbm[x] = 0u; }
    u32 N = (u32)F, cur = 0;
    u64 rb0 = 0, rb1 = 0;             // staged request window [rb0, rb1)
    u64 pos = 0, n_chunks = 0;
#if BF_TIMING
    long long tq = clock64(), tph[6] = {0, 0, 0, 0, 0, 0};
#define BS_T(k) do { const long long _t = clock64(); tph[k] += _t - tq; tq = _t; } while (0)
#else
#define BS_T(k) do { } while (0)
#endif
    __syncwarp();
    while (pos < n) {
        n_chunks++;
        if (pos + 32 > rb1 && rb1 < n) {                 // stage the next requests
            __syncwarp();
            rb0 = pos;
            rb1 = pos + BS_RB < n ? pos + BS_RB : n;
            for (u64 j = lane; j < rb1 - rb0; j += 32) S.rb[j] = r[rb0 + j];
            __syncwarp();
        }
        const u32 limit = (n - pos) < 32 ? (u32)(n - pos) : 32u;
        const bool act = lane < limit;
        const u64 ri = act ? S.rb[pos + lane - rb0] : 0ull;
        const bool valid = act && ri != 0;
        const u64 t = ri << FB;
        const u64 *A = S.A[cur];
        const u32 p = valid ? bs_lower_bound<u64>(A, N, t) : 0u;
        const u32 peers = __match_any_sync(FULLMASK, valid ? p : (0x80000000u | lane));
        const u32 q = p + (u32)__popc(peers & lanemask_lt());
        const bool has = valid && q < N;
        const u64 K = has ? A[q] : ~0ull;
        const u64 z = K >> FB;
        const u64 rem = (has && z > ri) ? (((z - ri) << FB) | (K & fmask)) : ~0ull;
        BS_T(0);
        S.dqp[lane] = make_uint2(p, has ? q : 0xFFFFFFFFu);
        S.dx[lane] = rem;
        __syncwarp();
        bool bad = false;
#pragma unroll
        for (u32 j = 0; j < 31; j++) {                   // earlier lanes (independent broadcast loads)
            const uint2 pq = S.dqp[j];
            const u64 xj = S.dx[j];
            const bool e = j < lane && valid;
            bad |= e && pq.y != 0xFFFFFFFFu && pq.x != p && pq.y >= p && pq.y <= q;
            bad |= e && xj != ~0ull && xj >= t && xj < K;
        }
        const u32 badm = __ballot_sync(FULLMASK, bad && act);
        const u32 commit = badm ? (u32)(__ffs(badm) - 1) : limit;
        const bool cm = lane < commit;
        const u64 i = pos + lane;
        BS_T(1);
        if (cm) {
            if (!has) out_u[i] = HEAP_NULL_U64;
            else {
                const u32 f = (u32)(K & fmask);
                const u32 s0 = S.fsm[f];
                out_u[i] = s0;
                S.fsm[f] = s0 + (u32)ri;
            }
        }
        const bool rmv = cm && has, ins = cm && rem != ~0ull;
        const u32 nr = __popc(__ballot_sync(FULLMASK, rmv)), nx = __popc(__ballot_sync(FULLMASK, ins));
        if (nr) {
            u64 *B = S.A[cur ^ 1];
            // each remainder's insertion point in A (#keys below it), its rank among the remainders
            // and #removed indices below its insertion point (one ballot pair per remainder)
            const u32 lb = ins ? bs_lower_bound<u64>(A, N, rem) : 0u;
            const u32 insm = __ballot_sync(FULLMASK, ins);
            u32 rank = 0, rcnt = 0;
            for (u32 mm = insm; mm; mm &= mm - 1) {
                const u32 k = __ffs(mm) - 1;
                const u32 lbk = __shfl_sync(FULLMASK, lb, k);
                const u64 xk = __shfl_sync(FULLMASK, rem, k);
                const u32 r1 = __popc(__ballot_sync(FULLMASK, rmv && q < lbk));
                const u32 r2 = __popc(__ballot_sync(FULLMASK, ins && rem < xk));
                if (lane == k) { rcnt = r1; rank = r2; }
            }
            // one bit per insertion point; two remainders between the same neighbours (rare) make
            // the survivors count the remainders below them by binary search instead
            const u32 dupm = __match_any_sync(FULLMASK, ins ? lb : (0x80000000u | lane));
            const bool dup = __any_sync(FULLMASK, ins && __popc(dupm) > 1);
            if (rmv) atomicOr(&S.rmb[q >> 5], 1u << (q & 31));
            if (ins) {
                S.sX[rank] = rem;
                if (!dup) atomicOr(&S.lbm[lb >> 5], 1u << (lb & 31));
            }
            __syncwarp();
            BS_T(2);
            // survivors, 4 tiles of 32 consecutive keys in flight: key e moves to
            // e - #(removed indices < e) + #(remainders whose insertion point is <= e)
            const u32 lmle = lanemask_lt() | (1u << lane);
            u32 before = 0, xbefore = 0;
            for (u32 base = 0; base < N; base += 128) {
                u64 a[4];
                u32 w[4], v[4], xc[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const u32 e = base + k * 32 + lane;
                    a[k] = e < N ? A[e] : ~0ull;
                    w[k] = S.rmb[(base >> 5) + k];
                    v[k] = dup ? 0u : S.lbm[(base >> 5) + k];
                }
                if (dup) {
#pragma unroll
                    for (int k = 0; k < 4; k++) xc[k] = 0;
#pragma unroll
                    for (u32 step = 16; step; step >>= 1) {
#pragma unroll
                        for (int k = 0; k < 4; k++)
                            if (xc[k] + step <= nx && S.sX[xc[k] + step - 1] < a[k]) xc[k] += step;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 4; k++) { xc[k] = xbefore + __popc(v[k] & lmle); xbefore += __popc(v[k]); }
                }
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const u32 e = base + k * 32 + lane;
                    const bool rm = (w[k] >> lane) & 1u;
                    if (e < N && !rm) B[e - before - __popc(w[k] & lanemask_lt()) + xc[k]] = a[k];
                    before += __popc(w[k]);
                }
            }
            BS_T(3);
            if (ins) B[rank + lb - rcnt] = rem;       // rank among the remainders + survivors below
            __syncwarp();
            if (rmv) S.rmb[q >> 5] = 0u;
            if (ins) S.lbm[lb >> 5] = 0u;
            N = N - nr + nx;
            cur ^= 1;
            __syncwarp();
            BS_T(4);
        }
        pos += commit;
    }
    __syncwarp();
    for (u32 x = lane; x < (u32)F; x += 32) fs[x] = S.fsm[x];
    if (dbg && lane == 0) { dbg[8] += n_chunks; dbg[9] += n; }
#if BF_TIMING
    if (lane == 0) for (int k = 0; k < 5; k++) dbg[16 + k] += (u64)tph[k];
#endif
#undef BS_T
}

// the flat engine with the array in shared memory (small heaps) or global memory
template <bool SMEM>
__global__ void __launch_bounds__(32) k_bf_engine_flat(u64 *gkeys, const u64 *F_dev, int FB, u64 *fs,
                                                       const u64 *__restrict__ r, u64 n, const u64 *n_in,
                                                       u64 *__restrict__ out_u) {
    PDL_ENTRY();
    extern __shared__ u64 skeys[];
    if (n_in) n = *n_in;
    const u32 lane = lane_id();
    const u64 nb = *F_dev;
    u64 *keys = SMEM ? skeys : gkeys;
    if (SMEM) {
        for (u64 i = lane; i < nb; i += 32) skeys[i] = gkeys[i];
        __syncwarp();
    }
    bf_flat(keys, nb, FB, fs, r, n, out_u);
}

}  // namespace fits
