// micro.cuh — the whole batch in ONE launch for small heaps (first / next / best fit, SEGFIT, TLSF).
//
// A heap whose free array can never exceed MICRO_F pieces (max_live < MICRO_F: the free blocks are
// separated by live blocks, so F <= n_live + 1), whose unit addresses fit 32 bits and whose batches
// hold at most MICRO_N requests runs each free batch and each alloc batch as one CTA of 1024 threads
// with the free array in shared memory, instead of the ~30 grid-wide launches of the general path
// (fits.cuh).  The results are the same by construction — the same canonical order (frees
// classified against the batch-start state and applied in ascending address order, Alg. 2; allocs
// served one by one in request order, Alg. 1), the same block table (table.cuh) and the same state
// between batches (address-sorted, coalesced free array + counters) — so micro and general batches
// interleave freely.  The alloc engine is a brute-force exact one run by one warp: per request every
// piece's policy key is computed by the lanes (pieces in shared memory, lane j % 32) and two warp
// REDUX reductions pick the lowest (key, address) — no barrier, no index to maintain, which at these
// sizes is cheaper than any index.
//
// Policy keys: FIRST_FIT (f), NEXT_FIT (f < f0, f) with f0 the rover's piece,
// BEST_FIT (size, f), SEGFIT / TLSF (cls_insert(size), f) over pieces with cls_insert(size) >=
// cls_search(r).  f is the address rank of the piece (address order = f order).
#pragma once
#include "common.cuh"
#include "table.cuh"

namespace micro {

constexpr int MT = 512;                     // threads per CTA
constexpr u32 MICRO_F = 4160;               // pieces (max_live + 1 <= MICRO_F)
// (The engine below costs O(F) per request — brute force — and the first-fit scan O(F / 32) in the
// worst case: the general path's indexes (max tree, blocked sorted list, class caches) win for
// larger free arrays, so the single-launch path stops at a few thousand pieces.)
constexpr u32 MICRO_N = 4096;               // requests per batch
constexpr u32 NONE = 0xFFFFFFFFu;
enum { P_FF = 0, P_NF = 1, P_BF = 2, P_CLS = 3 };
#ifndef PAIR_FF
#define PAIR_FF 1      // first fit on the register path: two requests per step (0: one)
#endif

constexpr size_t FREE_SMEM = (size_t)MICRO_F * 8 + (size_t)MICRO_N * 8 + ((MICRO_F + MICRO_N) / 32 + 64) * 8;
constexpr size_t ALLOC_SMEM = (size_t)MICRO_N * 8 + (size_t)MICRO_F * 8 + (MICRO_F / 32 + 64) * 8;

#ifndef MICRO_TIMING
#define MICRO_TIMING 0
#endif
// phase clocks of thread 0 into the engine diagnostics (tools/micro probes; off in production)
#if MICRO_TIMING
#define MCLK(idx)                                                     \
    if (threadIdx.x == 0) {                                           \
        const long long _t = clock64();                               \
        ctr->eng[idx] += (u64)(_t - t_prev);                          \
        t_prev = _t;                                                  \
    }
#else
#define MCLK(idx)
#endif

// CTA-wide exclusive scan of one u32 per thread; *total = sum
__device__ __forceinline__ u32 cta_scan(u32 v, u32 *sm, u32 *total) { return block_excl_scan<MT>(v, sm, total); }

// ------------------------------------------------------------------------------ free ----
#define MICRO_FREE_PARAMS                                                                                    \
    const u64 *__restrict__ offs, u64 n, const u64 *n_in, int alog2, u64 A_u, const u64 *__restrict__ fs_in,      \
        const u64 *__restrict__ fe_in, u64 *__restrict__ fs_out, u64 *__restrict__ fe_out, u64 *__restrict__ tbl, \
        u64 tmask, u64 max_lines, u64 cap_f, DevCtr *ctr, const u64 *__restrict__ hidx, u64 hlen
#define MICRO_FREE_ARGS offs, n, n_in, alog2, A_u, fs_in, fe_in, fs_out, fe_out, tbl, tmask, max_lines, cap_f, ctr, hidx, hlen
__device__ __forceinline__ void micro_free_body(MICRO_FREE_PARAMS) {
    extern __shared__ __align__(16) unsigned char dyn[];
    u32 *ps = reinterpret_cast<u32 *>(dyn);          // free array (units), F entries
    u32 *pe = ps + MICRO_F;
    u32 *vs = pe + MICRO_F;                          // candidate keys, sorted; then the valid frees
    u32 *ve = vs + MICRO_N;                          // sizes of the valid frees, then their ends
    u32 *hb = ve + MICRO_N;                          // head bits of the merged order
    u32 *wp = hb + (MICRO_F + MICRO_N) / 32 + 32;    // word prefix counts
    __shared__ u32 sm[33];
    __shared__ u64 c_null, c_inv, c_ok, c_dbl, c_units;
    __shared__ u32 s_nk;
    const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if MICRO_TIMING
    long long t_prev = clock64();
#endif
    if (n_in) n = *n_in;
    const u32 F = (u32)ctr->F;
    if (F > MICRO_F || n > MICRO_N) {                // capacity exceeded (live cap broken): report, stop
        if (tid == 0) ctr->error_flags |= ERR_CAP_FREE;
        return;
    }
    if (tid == 0) { c_null = 0; c_inv = 0; c_ok = 0; c_dbl = 0; c_units = 0; s_nk = 0; }
    // handles (heap_free_batch_handles): offset i is offs[hidx[i]] (an index >= hlen frees nothing)
    auto off_at = [&](u32 i) -> u64 {
        if (!hidx) return offs[i];
        const u64 x = hidx[i];
        return x < hlen ? offs[x] : HEAP_NULL_U64;
    };
    // the first MT offsets are loaded together with the free array (one memory round trip)
    const u64 o_first = tid < n ? off_at(tid) : HEAP_NULL_U64;
    for (u32 i = tid; i < F; i += MT) { ps[i] = (u32)fs_in[i]; pe[i] = (u32)fe_in[i]; }
    __syncthreads();
    MCLK(16)
    // 1. classify: HEAP_NULL -> no-op, unaligned / out of range -> invalid, else a candidate key
    const u64 amask = (1ull << alog2) - 1;
    u32 nnull = 0, ninv = 0;
    for (u32 base = 0; base < (u32)n; base += MT) {
        const u32 i = base + tid;
        bool cand = false;
        u32 key = 0;
        if (i < n) {
            const u64 o = base == 0 ? o_first : off_at(i);
            if (o == HEAP_NULL_U64) nnull++;
            else if ((o & amask) || (o >> alog2) >= A_u) ninv++;
            else { cand = true; key = (u32)(o >> alog2); }
        }
        const u32 b = __ballot_sync(FULLMASK, cand);
        u32 wbase = 0;
        if (lane == 0 && b) wbase = atomicAdd(&s_nk, (u32)__popc(b));   // order is irrelevant: sorted next
        wbase = __shfl_sync(FULLMASK, wbase, 0);
        if (cand) vs[wbase + __popc(b & lanemask_lt())] = key;
    }
    if (nnull) atomicAdd(&c_null, (u64)nnull);
    if (ninv) atomicAdd(&c_inv, (u64)ninv);
    __syncthreads();
    const u32 nk = s_nk;
    MCLK(17)
    // 2. bitonic sort of the keys (padded to a power of two with keys that cannot occur)
    u32 P2 = 1;
    while (P2 < nk) P2 <<= 1;
    if (P2 <= 32) {                                   // one warp, in registers (no barriers)
        if (warp == 0) {
            u32 v = lane < nk ? vs[lane] : NONE;
            for (u32 k = 2; k <= 32; k <<= 1)
                for (u32 j = k >> 1; j > 0; j >>= 1) {
                    const u32 o = __shfl_xor_sync(FULLMASK, v, j);
                    const bool up = (lane & k) == 0, lo = (lane & j) == 0;
                    v = (lo == up) ? min(v, o) : max(v, o);
                }
            vs[lane] = v;
        }
        __syncthreads();
    } else {
        for (u32 i = nk + tid; i < P2; i += MT) vs[i] = NONE;
        __syncthreads();
        for (u32 k = 2; k <= P2; k <<= 1)
            for (u32 j = k >> 1; j > 0; j >>= 1) {
                for (u32 i = tid; i < P2; i += MT) {
                    const u32 x = i ^ j;
                    if (x > i) {
                        const u32 a = vs[i], b = vs[x];
                        if (((i & k) == 0) ? (a > b) : (a < b)) { vs[i] = b; vs[x] = a; }
                    }
                }
                __syncthreads();
            }
    }
    MCLK(18)
    // 3. table lookup + delete for the first copy of each key (2-lane tiles, table::KPW keys per warp),
    //    the copies classified from it: live -> 1 ok + copies-1 double; start of a free block ->
    //    all double; otherwise all invalid.  ve[q] = size of the freed block at key q (0: none).
    {
        u64 ok = 0, dbl = 0, inv = 0, units = 0;
        const u32 g = lane / table::TILE_LANES, sub = lane % table::TILE_LANES;
        for (u32 base = warp * table::KPW; base < ((nk + table::KPW - 1) & ~(u32)(table::KPW - 1)); base += (MT / 32) * table::KPW) {
            const u32 q = base + g;
            const bool in = q < nk;
            const u32 key = in ? vs[q] : 0;
            const bool first = in && (q == 0 || vs[q - 1] != key);
            const u64 s = table::lookup(tbl, tmask, key, first, table::TOMB, max_lines);
            if (in && sub == 0) {
                u32 z = 0;
                if (first) {
                    u32 ndup = 0;
                    for (u32 j = q + 1; j < nk && vs[j] == key; j++) ndup++;
                    if (s != table::EMPTY) {
                        z = (u32)table::slot_size(s);
                        ok++; dbl += ndup; units += z;
                    } else {
                        u32 lo = 0, hi = F;                 // start of a free block?
                        while (lo < hi) { const u32 m = (lo + hi) >> 1; if (ps[m] < key) lo = m + 1; else hi = m; }
                        if (lo < F && ps[lo] == key) dbl += 1 + ndup;
                        else inv += 1 + ndup;
                    }
                }
                ve[q] = z;
            }
        }
        ok = warp_sum64(ok); dbl = warp_sum64(dbl); inv = warp_sum64(inv); units = warp_sum64(units);
        if (lane == 0) {
            if (ok) atomicAdd(&c_ok, ok);
            if (dbl) atomicAdd(&c_dbl, dbl);
            if (inv) atomicAdd(&c_inv, inv);
            if (units) atomicAdd(&c_units, units);
        }
    }
    __syncthreads();
    MCLK(19)
    // compact the valid frees (sorted order kept) into vs / ve = (start, end): read, barrier, write
    u32 nv;
    {
        const u32 per = (nk + MT - 1) / MT, b0 = tid * per;     // <= 8
        u32 kk[8], zz[8], cnt = 0;
        for (u32 j = 0; j < per && j < 8; j++) {
            const u32 q = b0 + j;
            kk[j] = q < nk ? vs[q] : 0;
            zz[j] = q < nk ? ve[q] : 0;
            cnt += zz[j] ? 1u : 0u;
        }
        u32 pos = cta_scan(cnt, sm, &nv);
        for (u32 j = 0; j < per && j < 8; j++)
            if (zz[j]) { vs[pos] = kk[j]; ve[pos] = kk[j] + zz[j]; pos++; }
    }
    __syncthreads();
    MCLK(20)
    // 4. merge the freed blocks into the free array and coalesce (Alg. 2): every element's merged
    //    position from one binary search in the other list, a head bit where the previous block of
    //    the merged order does not end at its start, runs numbered by a popcount prefix of the bits
    const u32 M = F + nv, nw = (M + 31) / 32;
    for (u32 i = tid; i < nw + 1; i += MT) hb[i] = 0;
    __syncthreads();
    auto lb = [](const u32 *a, u32 na, u32 key) {
        u32 lo = 0, hi = na;
        while (lo < hi) { const u32 m = (lo + hi) >> 1; if (a[m] < key) lo = m + 1; else hi = m; }
        return lo;
    };
    for (u32 e = tid; e < M; e += MT) {
        u32 st, pos, pend = NONE;
        if (e < F) {
            const u32 i = e;
            st = ps[i];
            const u32 l = lb(vs, nv, st);
            pos = i + l;
            if (l > 0 && (i == 0 || vs[l - 1] > ps[i - 1])) pend = ve[l - 1];
            else if (i > 0) pend = pe[i - 1];
        } else {
            const u32 j = e - F;
            st = vs[j];
            const u32 l = lb(ps, F, st);
            pos = j + l;
            if (j > 0 && (l == 0 || vs[j - 1] > ps[l - 1])) pend = ve[j - 1];
            else if (l > 0) pend = pe[l - 1];
        }
        if (pos == 0 || pend != st) atomicOr(&hb[pos >> 5], 1u << (pos & 31));
    }
    __syncthreads();
    u32 Fn;
    {
        // two words per thread (nw <= (MICRO_F + MICRO_N) / 32 + 1 = 673 <= 2 MT)
        const u32 c0 = 2 * tid < nw ? (u32)__popc(hb[2 * tid]) : 0u;
        const u32 c1 = 2 * tid + 1 < nw ? (u32)__popc(hb[2 * tid + 1]) : 0u;
        const u32 ex = cta_scan(c0 + c1, sm, &Fn);
        if (2 * tid < nw) wp[2 * tid] = ex;
        if (2 * tid + 1 < nw) wp[2 * tid + 1] = ex + c0;
    }
    __syncthreads();
    if (Fn > cap_f) {
        if (tid == 0) atomicOr(&ctr->error_flags, (u64)ERR_CAP_FREE);
    } else {
        for (u32 e = tid; e < M; e += MT) {
            u32 st, en, pos;
            if (e < F) { st = ps[e]; en = pe[e]; pos = e + lb(vs, nv, st); }
            else { const u32 j = e - F; st = vs[j]; en = ve[j]; pos = j + lb(ps, F, st); }
            const u32 w = pos >> 5, bit = 1u << (pos & 31);
            const u32 run = wp[w] + __popc(hb[w] & (bit - 1)) + ((hb[w] & bit) ? 1u : 0u) - 1u;
            if (hb[w] & bit) fs_out[run] = st;
            const u32 p1 = pos + 1;
            if (p1 == M || (hb[p1 >> 5] >> (p1 & 31)) & 1u) fe_out[run] = en;
        }
    }
    MCLK(21)
    if (tid == 0) {
        ctr->F = Fn;
        ctr->nk = nk;
        ctr->nv = nv;
        if (c_null) ctr->frees_null += c_null;
        if (c_inv) ctr->frees_invalid += c_inv;
        if (c_dbl) ctr->frees_double += c_dbl;
        if (c_ok) { ctr->frees_ok += c_ok; ctr->n_live -= c_ok; ctr->tbl_tombs += c_ok; }
        if (c_units) ctr->live_units -= c_units;
    }
}

// ----------------------------------------------------------------------------- alloc ----
template <int POL>
__device__ __forceinline__ u32 pkey(u32 z, u32 r, u32 cs, u32 j, u32 f0, int L) {
    // primary key of piece j (NONE: not a candidate)
    if (POL == P_CLS) {
        if (z == 0) return NONE;
        const u32 c = cls_insert(z, L);
        return c >= cs ? c : NONE;
    }
    if (z < r) return NONE;
    if (POL == P_FF) return 0u;
    if (POL == P_NF) return j < f0 ? 1u : 0u;
    return z;                                        // BEST_FIT
}

#define MICRO_ALLOC_PARAMS                                                                                    \
    const u64 *__restrict__ sizes, u64 n, const u64 *n_in, int alog2, u64 A_u, int L, const u64 *__restrict__ fs_in, \
        const u64 *__restrict__ fe_in, u64 *__restrict__ fs_out, u64 *__restrict__ fe_out, u64 *__restrict__ out_bytes, \
        u64 *__restrict__ tbl, u64 tmask, u64 max_lines, u64 tcap, u64 *__restrict__ scratch, DevCtr *ctr, u64 max_live
#define MICRO_ALLOC_ARGS sizes, n, n_in, alog2, A_u, L, fs_in, fe_in, fs_out, fe_out, out_bytes, tbl, tmask, max_lines, tcap, \
    scratch, ctr, max_live
template <int POL>
__device__ __forceinline__ void micro_alloc_body(MICRO_ALLOC_PARAMS) {
    extern __shared__ __align__(16) unsigned char dyn[];
    u32 *rr = reinterpret_cast<u32 *>(dyn);          // request units (0: fails)
    u32 *res = rr + MICRO_N;                         // result (unit offset) or NONE
    u32 *ps = res + MICRO_N;                         // piece starts / ends (units)
    u32 *pe = ps + MICRO_F;
    u32 *sb = pe + MICRO_F;                          // survivor bits of the pieces
    u32 *sp = sb + MICRO_F / 32 + 32;                // their word prefix counts
    __shared__ u32 sm[33];
    __shared__ u64 c_ok, c_fail, c_units, c_used, c_tomb, c_hw, c_full;
    const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if MICRO_TIMING
    long long t_prev = clock64();
#endif
    if (n_in) n = *n_in;
    const u32 F = (u32)ctr->F;
    if (F > MICRO_F || n > MICRO_N) {                // capacity exceeded (live cap broken): report, stop
        if (tid == 0) ctr->error_flags |= ERR_CAP_FREE;
        return;
    }
    const u64 amask = (1ull << alog2) - 1;
    for (u32 i = tid; i < n; i += MT) {
        const u64 s = sizes[i];
        u64 r = (s >> alog2) + ((s & amask) != 0);
        if (s == 0 || r > A_u) r = 0;
        rr[i] = (u32)r;
    }
    for (u32 j = tid; j < F; j += MT) { ps[j] = (u32)fs_in[j]; pe[j] = (u32)fe_in[j]; }
    for (u32 w = tid; w < MICRO_F / 32 + 32; w += MT) sb[w] = 0;
    if (tid == 0) { c_ok = 0; c_fail = 0; c_units = 0; c_used = 0; c_tomb = 0; c_hw = 0; c_full = 0; }
    __syncthreads();
    MCLK(22)
    if (warp == 0) {
        // NEXT_FIT: f0 = first piece whose start is >= the rover (reading C27)
        u32 f0 = 0;
        if (POL == P_NF) {
            const u64 R = ctr->rover;
            u32 lo = 0, hi = F;
            while (lo < hi) { const u32 m = (lo + hi) >> 1; if (ps[m] < R) lo = m + 1; else hi = m; }
            f0 = lo;
        }
        bool moved = false;
        // pe[] becomes the piece sizes during the engine (carves shrink them), restored after
        for (u32 j = lane; j < F; j += 32) pe[j] -= ps[j];
        __syncwarp();
        if ((POL == P_FF || POL == P_NF) && F <= 128) {
            // small free array, first / next fit: piece lane + 32 q in registers of its lane
            // (q < 4); four independent ballots per request, the winning lane carves in place —
            // no shared-memory round trip on the chain
            u32 z[4], st[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const u32 j = lane + 32 * q;
                z[q] = j < F ? pe[j] : 0u;
                st[q] = j < F ? ps[j] : 0u;
            }
            u32 rn = n ? rr[0] : 0u;
            if (POL == P_FF && PAIR_FF) {
                // first fit, two requests per step: both searches run on the state before the first
                // one's carve (eight independent ballots).  Only the first request's piece fa changed
                // (it shrank), so the second one's speculative choice fb stands unless fb == fa and fa
                // no longer fits it — then it is the next fitting piece after fa in the same masks.
                for (u32 i = 0; i < (u32)n; i += 2) {
                    const u32 ra = rr[i], rb = i + 1 < (u32)n ? rr[i + 1] : 0u;
                    u32 ba[4], bb[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        ba[q] = __ballot_sync(FULLMASK, ra != 0 && z[q] >= ra);
                        bb[q] = __ballot_sync(FULLMASK, rb != 0 && z[q] >= rb);
                    }
                    const u32 fa = ba[0] ? __ffs(ba[0]) - 1 : ba[1] ? 32 + __ffs(ba[1]) - 1
                                 : ba[2] ? 64 + __ffs(ba[2]) - 1 : ba[3] ? 96 + __ffs(ba[3]) - 1 : NONE;
                    u32 fb = bb[0] ? __ffs(bb[0]) - 1 : bb[1] ? 32 + __ffs(bb[1]) - 1
                           : bb[2] ? 64 + __ffs(bb[2]) - 1 : bb[3] ? 96 + __ffs(bb[3]) - 1 : NONE;
                    u32 zsel = 0;                          // this lane's size of piece row fa >> 5, after a
                    if (fa == NONE) {
                        if (lane == 0) res[i] = NONE;
                    } else {
                        const int qa = (int)(fa >> 5);
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            if (k == qa && (fa & 31) == lane) { res[i] = st[k]; st[k] += ra; z[k] -= ra; }
                            if (k == qa) zsel = z[k];
                        }
                    }
                    if (i + 1 >= (u32)n) break;
                    if (fb != NONE && fb == fa) {
                        const u32 zf = __shfl_sync(FULLMASK, zsel, fa & 31);
                        if (zf < rb) {                     // the next fitting piece after fa
                            const int qa = (int)(fa >> 5);
                            u32 m[4];
#pragma unroll
                            for (int k = 0; k < 4; k++)
                                m[k] = k < qa ? 0u : k > qa ? bb[k] : (bb[k] & ~((2u << (fa & 31)) - 1u));
                            fb = m[0] ? __ffs(m[0]) - 1 : m[1] ? 32 + __ffs(m[1]) - 1
                               : m[2] ? 64 + __ffs(m[2]) - 1 : m[3] ? 96 + __ffs(m[3]) - 1 : NONE;
                        }
                    }
                    if (fb == NONE) {
                        if (lane == 0) res[i + 1] = NONE;
                    } else if ((fb & 31) == lane) {
                        const int qb = (int)(fb >> 5);
#pragma unroll
                        for (int k = 0; k < 4; k++)
                            if (k == qb) { res[i + 1] = st[k]; st[k] += rb; z[k] -= rb; }
                    }
                }
            } else
            for (u32 i = 0; i < (u32)n; i++) {
                const u32 r = rn;
                rn = i + 1 < (u32)n ? rr[i + 1] : 0u;      // the next request, off the chain
                u32 f = NONE;
                if (r != 0) {
                    u32 bq[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) bq[q] = __ballot_sync(FULLMASK, z[q] >= r && lane + 32 * q >= f0);
                    const u32 any = bq[0] | bq[1] | bq[2] | bq[3];
                    if (any) {
                        const int q = bq[0] ? 0 : bq[1] ? 1 : bq[2] ? 2 : 3;
                        f = 32 * q + __ffs(bq[q]) - 1;
                    } else if (POL == P_NF && f0 > 0) {  // wrap: first fit from piece 0
#pragma unroll
                        for (int q = 0; q < 4; q++) bq[q] = __ballot_sync(FULLMASK, z[q] >= r);
                        if (bq[0] | bq[1] | bq[2] | bq[3]) {
                            const int q = bq[0] ? 0 : bq[1] ? 1 : bq[2] ? 2 : 3;
                            f = 32 * q + __ffs(bq[q]) - 1;
                        }
                    }
                }
                if (f == NONE) {
                    if (lane == 0) res[i] = NONE;
                } else {
                    if ((f & 31) == lane) {
                        const int q = (int)(f >> 5);
#pragma unroll
                        for (int k = 0; k < 4; k++)
                            if (k == q) { res[i] = st[k]; st[k] += r; z[k] -= r; }
                    }
                    if (POL == P_NF) { f0 = f; moved = true; }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const u32 j = lane + 32 * q;
                if (j < F) { ps[j] = st[q]; pe[j] = z[q]; }
            }
            __syncwarp();
        } else
        for (u32 i = 0; i < (u32)n; i++) {
            const u32 r = rr[i];
            u32 f = NONE;
            if (r != 0 && (POL == P_FF || POL == P_NF)) {
                // first fit (next fit: from the rover's piece, then wrapping): the first eligible
                // piece in address order, one ballot per 32 pieces
                for (u32 b0 = (POL == P_NF) ? (f0 & ~31u) : 0u; b0 < F; b0 += 32) {
                    const u32 j = b0 + lane;
                    const u32 b = __ballot_sync(FULLMASK, j < F && j >= f0 && pe[j] >= r);
                    if (b) { f = b0 + __ffs(b) - 1; break; }
                }
                if (POL == P_NF && f == NONE)
                    for (u32 b0 = 0; b0 < F; b0 += 32) {
                        const u32 j = b0 + lane;
                        const u32 b = __ballot_sync(FULLMASK, j < F && pe[j] >= r);
                        if (b) { f = b0 + __ffs(b) - 1; break; }
                    }
            } else if (r != 0) {
                const u32 cs = (POL == P_CLS) ? cls_search(r, L) : 0u;
                u32 b1 = NONE, b2 = NONE;
                for (u32 j = lane; j < F; j += 32) {
                    const u32 key = pkey<POL>(pe[j], r, cs, j, f0, L);
                    if (key < b1) { b1 = key; b2 = j; }      // j increases: the first j wins ties
                }
                const u32 m1 = __reduce_min_sync(FULLMASK, b1);
                const u32 m2 = __reduce_min_sync(FULLMASK, b1 == m1 ? b2 : NONE);
                f = (m1 == NONE) ? NONE : m2;
            }
            if (lane == 0) {
                if (f == NONE) res[i] = NONE;
                else { res[i] = ps[f]; ps[f] += r; pe[f] -= r; }
            }
            if (POL == P_NF && f != NONE) { f0 = f; moved = true; }
            __syncwarp();
        }
        for (u32 j = lane; j < F; j += 32) pe[j] += ps[j];
        __syncwarp();
        if (POL == P_NF && moved && lane == 0) ctr->rover = ps[f0];   // the end of the last allocation
    }
    __syncthreads();
    MCLK(23)
    // the surviving pieces, compacted in address order
    for (u32 j = tid; j < F; j += MT)
        if (pe[j] > ps[j]) atomicOr(&sb[j >> 5], 1u << (j & 31));
    __syncthreads();
    u32 Fn;
    {
        const u32 nw = (F + 31) / 32;                         // <= 544 <= 2 MT: two words per thread
        const u32 c0 = 2 * tid < nw ? (u32)__popc(sb[2 * tid]) : 0u;
        const u32 c1 = 2 * tid + 1 < nw ? (u32)__popc(sb[2 * tid + 1]) : 0u;
        const u32 ex = cta_scan(c0 + c1, sm, &Fn);
        if (2 * tid < nw) sp[2 * tid] = ex;
        if (2 * tid + 1 < nw) sp[2 * tid + 1] = ex + c0;
    }
    __syncthreads();
    for (u32 j = tid; j < F; j += MT)
        if (pe[j] > ps[j]) {
            const u32 w = j >> 5;
            const u32 q = sp[w] + __popc(sb[w] & ((1u << (j & 31)) - 1u));
            fs_out[q] = ps[j];
            fe_out[q] = pe[j];
        }
    __syncthreads();
    MCLK(24)
    // results, block-table inserts (2-lane tiles), counters
    {
        u64 ok = 0, fail = 0, units = 0, used = 0, tomb = 0, full = 0, hw = 0;
        const u32 g = lane / table::TILE_LANES, sub = lane % table::TILE_LANES;
        for (u32 base = warp * table::KPW; base < (((u32)n + table::KPW - 1) & ~(u32)(table::KPW - 1)); base += (MT / 32) * table::KPW) {
            const u32 i = base + g;
            const bool in = i < n;
            const u32 o = in ? res[i] : NONE;
            const bool okk = in && o != NONE;
            const u64 ri = okk ? rr[i] : 0;
            const int rc = table::insert(tbl, tmask, o, ri, okk, max_lines);
            if (rc == 1) used++;
            if (rc == -1) tomb++;
            if (rc == 2) full++;
            if (in && sub == 0) {
                out_bytes[i] = okk ? ((u64)o << alog2) : HEAP_NULL_U64;
                if (okk) { ok++; units += ri; hw = max(hw, (u64)o + ri); }
                else fail++;
            }
        }
        ok = warp_sum64(ok); fail = warp_sum64(fail); units = warp_sum64(units);
        used = warp_sum64(used); tomb = warp_sum64(tomb); full = warp_sum64(full); hw = warp_max64(hw);
        if (lane == 0) {
            if (ok) atomicAdd(&c_ok, ok);
            if (fail) atomicAdd(&c_fail, fail);
            if (units) atomicAdd(&c_units, units);
            if (used) atomicAdd(&c_used, used);
            if (tomb) atomicAdd(&c_tomb, tomb);
            if (full) atomicAdd(&c_full, full);
            if (hw) atomicMax(&c_hw, hw);
        }
    }
    __syncthreads();
    MCLK(25)
    __shared__ u32 s_rb;
    if (tid == 0) {
        ctr->F = Fn;
        ctr->allocs_ok += c_ok;
        ctr->allocs_failed += c_fail;
        ctr->live_units += c_units;
        ctr->n_live += c_ok;
        if (ctr->n_live > max_live) ctr->error_flags |= ERR_CAP_LIVE;
        ctr->tbl_used += c_used;
        ctr->tbl_tombs -= c_tomb;
        if (c_full) ctr->error_flags |= ERR_TABLE_FULL;
        if (c_hw > ctr->high_water_units) ctr->high_water_units = c_hw;
        // tombstone purge when the table fills (the general path's maybe_rebuild, same threshold)
        s_rb = (ctr->tbl_used > tcap / 4 * 3) ? 1u : 0u;
        ctr->tmp[5] = 0;
    }
    __syncthreads();
    if (!s_rb) return;
    __shared__ u32 s_cnt;
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (u64 i = tid; i < tcap; i += MT) {
        const u64 v = tbl[i];
        if (table::is_live(v)) scratch[atomicAdd(&s_cnt, 1u)] = v;
    }
    __syncthreads();
    for (u64 i = tid; i < tcap; i += MT) tbl[i] = table::EMPTY;
    __syncthreads();
    const u32 nl = s_cnt;
    {
        const u32 g = lane / table::TILE_LANES;
        u64 full = 0;
        for (u32 base = warp * table::KPW; base < ((nl + table::KPW - 1) & ~(u32)(table::KPW - 1)); base += (MT / 32) * table::KPW) {
            const u32 i = base + g;
            const bool in = i < nl;
            const u64 v = in ? scratch[i] : 0;
            const int rc = table::insert(tbl, tmask, in ? table::slot_key(v) : 0, in ? table::slot_size(v) : 1, in,
                                         max_lines);
            if (rc == 2) full++;
        }
        if (full) atomicOr(&ctr->error_flags, (u64)ERR_TABLE_FULL);
    }
    if (tid == 0) { ctr->tbl_used = nl; ctr->tbl_tombs = 0; }
}

__global__ void __launch_bounds__(MT, 1) k_micro_free(MICRO_FREE_PARAMS) {
    PDL_ENTRY();
    micro_free_body(MICRO_FREE_ARGS);
}

template <int POL>
__global__ void __launch_bounds__(MT, 1) k_micro_alloc(MICRO_ALLOC_PARAMS) {
    PDL_ENTRY();
    micro_alloc_body<POL>(MICRO_ALLOC_ARGS);
}

// heap_step on a single-launch heap: the free batch then the alloc batch in ONE launch (the
// canonical batch order; the alloc phase reads the state the free phase wrote, made visible to the
// CTA by the barrier between them).  Dynamic shared memory: max(FREE_SMEM, ALLOC_SMEM).
template <int POL>
__global__ void __launch_bounds__(MT, 1) k_micro_step(const u64 *__restrict__ offs, u64 nf, const u64 *__restrict__ hidx,
                                                      u64 hlen, const u64 *__restrict__ sizes, u64 na,
                                                      u64 *__restrict__ out_bytes, int alog2, u64 A_u, int L,
                                                      u64 *fs0, u64 *fe0, u64 *fs1, u64 *fe1, u64 *__restrict__ tbl,
                                                      u64 tmask, u64 max_lines, u64 tcap, u64 cap_f,
                                                      u64 *__restrict__ scratch, DevCtr *ctr, u64 max_live) {
    PDL_ENTRY();
    if (nf) micro_free_body(offs, nf, nullptr, alog2, A_u, fs0, fe0, fs1, fe1, tbl, tmask, max_lines, cap_f, ctr, hidx, hlen);
    __syncthreads();
    if (na) {
        if (nf) micro_alloc_body<POL>(sizes, na, nullptr, alog2, A_u, L, fs1, fe1, fs0, fe0, out_bytes, tbl, tmask,
                                      max_lines, tcap, scratch, ctr, max_live);
        else micro_alloc_body<POL>(sizes, na, nullptr, alog2, A_u, L, fs0, fe0, fs1, fe1, out_bytes, tbl, tmask,
                                   max_lines, tcap, scratch, ctr, max_live);
    }
}
constexpr size_t STEP_SMEM = FREE_SMEM > ALLOC_SMEM ? FREE_SMEM : ALLOC_SMEM;

}  // namespace micro
