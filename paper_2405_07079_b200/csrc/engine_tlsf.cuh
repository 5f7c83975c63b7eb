// engine_tlsf.cuh — warp-speculative exact engine for SEGFIT / TLSF allocation batches.
//
// Semantics (must equal the oracle): requests are served in request order; request i takes,
// among free pieces whose class is >= its search class c_i, the one with the smallest
// (class, address) key (Alg. 4 + the bitmap/ffs fallback PAPER.md:332-337,440; TLSF two-level
// lookup PAPER.md:449; address order within a class, C9), and carves r_i units off
// its low end (Alg. 1).  Pieces are indexed by f = address rank of their batch-start free block
// (each batch-start block holds at most one piece during the phase; see fits.cuh).
//
// One warp walks the batch in chunks of up to 32 consecutive requests (one per lane):
//   1. every lane finds the first nonempty class >= c_i in the chunk-start two-level bitmap
//      (ffs on the second-level word, then on the first-level summary);
//   2. lanes aiming at the same class are grouped with __match_any_sync and ranked in time
//      order; the group's members come from a per-class head cache in shared memory holding
//      the class's H smallest members with their (start, end) — no global memory on this path;
//   3. each group leader replays its group in time order: a block keeps serving the next
//      request while its remainder stays in the class (head carve), otherwise the next member
//      is used; requests finding the class exhausted are re-aimed at the next nonempty class
//      and the chunk is replayed;
//   4. a request is *dirty* if an earlier request of the chunk dropped a remainder into a
//      class >= its search class with a smaller key than the one it chose, or if its rank
//      fell past the head cache; the chunk commits every request before the first dirty one
//      (exactly the sequential results), updates the class state, and the next chunk starts
//      at the first dirty request.  Request 0 of a chunk is never dirty, so chunks progress.
// Class state: per class a CSR range of batch-start members (address order, consumed as a
// prefix; class-sorted copies of (f, start, end)), a sorted head cache (ring buffer of up to H
// members in shared memory), and an overflow set (three-level bitmap over f, see Heap) of
// remainders that dropped into the class and did not fit the cache.  Invariant: the cache
// holds the n smallest members of the class (n >= min(REFILL_AT, members) after a refill).
// Ablation (measured on B200, config 5 batch 5 / config 3 batch 29): one lane replaying the
// requests strictly one by one on the same state takes 376 ms / 23.6 ms per batch versus
// 238 ms / 8.9 ms for this chunked engine.
#pragma once
#include "common.cuh"

namespace tlsfw {

#ifndef REFILL_AT_DEF
#define REFILL_AT_DEF 6
#endif

// per-phase cycle counters for tools/engine_probe.py (heap_debug_counters): off in the production
// build (measured cost with them: 0.4 %); a diagnostic build passes -DENGINE_TIMING=1
#ifndef ENGINE_TIMING
#define ENGINE_TIMING 0
#endif
#if ENGINE_TIMING
#define ENG_CLK() clock64()
#else
#define ENG_CLK() 0ll
#endif
#ifndef LIGHT_ROUNDS
#define LIGHT_ROUNDS 16
#endif
#ifndef H_DEF
#define H_DEF 8
#endif
constexpr int H = H_DEF;          // head-cache depth of the classes below HOT (power of two)
constexpr int REFILL_AT = REFILL_AT_DEF;      // refill a class's cache when it holds fewer members
#ifndef HOT_DEF
#define HOT_DEF 256
#endif
#ifndef HL_DEF
#define HL_DEF 4
#endif
// Classes at and above HOT (pieces of >= 2^13 units at SL_LOG2 = 5, above every request's search
// class of config 5) are reached only when everything below is empty and hold few members: they
// keep a depth-HL cache.  The shared memory this saves (162 -> 118 KB) goes to the L1 carveout,
// which the chain's global accesses (CSR records, overflow words, piece data) hit: measured +6.4 %
// engine time per 40 KB of extra shared memory; net of the per-class depth arithmetic, HL = 4 is
// 1.3 % faster than one depth for all classes and HL = 2 2 % slower (config 5, batches 10-11).
constexpr int HOT = HOT_DEF;
constexpr int HL = HL_DEF;
__device__ __forceinline__ u32 hbase(u32 k) { return k < (u32)HOT ? k * H : HOT * H + (k - HOT) * HL; }
__device__ __forceinline__ u32 hmask(u32 k) { return k < (u32)HOT ? H - 1 : HL - 1; }
__device__ __forceinline__ u32 hrefill(u32 k) { return k < (u32)HOT ? (u32)REFILL_AT : (u32)HL; }
#ifndef FILL_TO_DEF
#define FILL_TO_DEF H_DEF
#endif
constexpr int FILL_TO = FILL_TO_DEF;          // a refill appends CSR members up to this many cached
constexpr int MAX_NC = 928;       // classes of 2^32 units at SL_LOG2 = 5 (fl <= 28)
#ifndef RB_DEF
#define RB_DEF 512
#endif
constexpr int RB = RB_DEF;        // request staging buffer

constexpr u32 NONE = 0xFFFFFFFFu;
constexpr u32 HEAPBIT = 0x80000000u;
constexpr u32 SAME = 0xFFFFFFFEu; // block stays in its class after the carve
constexpr u32 F_OK = 0, F_OVER = 1, F_MISS = 2;
constexpr u64 NIL64 = ~0ull;
constexpr u64 WILD = 0xFFFFFFFFFFFFFFFEull;   // result marker: served by the wilderness (k_wild_apply)

struct Smem {
    u32 ptr[MAX_NC], endp[MAX_NC], cnt[MAX_NC], root[MAX_NC], slot[MAX_NC];
    u32 nslot;
    u32 ow_i[MAX_NC], ow_v[MAX_NC];   // cached overflow word per class (see Heap)
    uint4 hc[HOT * H + (MAX_NC - HOT) * HL];   // cached member {f (| HEAPBIT when it came from the overflow set),
                                  //  current start, end - 1 (units; ends can be 2^32), 0}
    unsigned char hn[MAX_NC];
    unsigned char hb[MAX_NC];     // ring-buffer base of the cache (entry j at (hb + j) % H)
    u32 cw[32];
    u32 sw;
    u64 rbuf[RB];
    u32 cbuf[RB];
    u32 lor[32 * 32];             // lane of rank q in the group led by lane l: lor[l*32+q]
    u64 res_s[32];
    u32 res_f[32], res_nk[32], res_flag[32], res_e[32];
    u64 ch_i[32], ch_r[32];       // the chunk's requests (index, units), lane = time order
    u32 ch_c[32];
#ifdef SMEM_PAD
    u32 pad_[SMEM_PAD];           // experiment: shared memory taken from the L1 carveout
#endif
    // two-warp engine (non-LIFO): warp 1 applies the arrivals of a chunk while warp 0 updates the
    // classes that lost members; classes touched by both (etag == ctag) stay on warp 0
    u32 etag[MAX_NC];             // chunk tag of the last chunk that popped / carved class k
    u32 atag[MAX_NC];             // three-warp engine: chunk tag of the last chunk with an arrival into class k
    u32 dg[32], dnk[32];          // per lane: its arrival group (dropper mask, 0 if not a leader), class
    u32 rk[32];                   // three-warp engine, per lane: a class that lost members and has no
                                  // arrival in the chunk (warp 1 refills it), else NONE
    u64 w1_delmin;
    u32 ctag, eng_done, broken1;
    // warp 1 also gathers the next chunk's candidates (wilderness mode): carried-over candidates
    // of this chunk first, then requests from g_scan with search class <= g_mx
    u64 nx_i[32], nx_r[32];
    u32 nx_c[32];
    u32 nx_n, g_need, g_commit, g_limit;
    int g_mx;
    u64 nx_scan, g_scan;
    u64 w1_visits, w1_inserts;
    u64 dkey[32];                 // the chunk's droppers in time order: (drop class << 32 | f) ...
    u32 dlane[32];                // ... and their lanes (the dirty check reads them as broadcasts)
};

// Overflow members of a class (remainders that arrived while its head cache was full) live in
// a three-level bitmap over f (a bit per piece, a bit per nonempty word, a bit per nonempty
// second-level word), one bitmap slot per class that needs it.  Keys taken out of a class's
// overflow set only grow (every insert is above the cache, which is above everything already
// taken), so the minimum is tracked in shared memory (root[k]) and extract-min clears the
// minimum's bit (its word is usually cached in shared memory) plus, when the word empties, a walk
// up the summary levels.  Only the engine's warp touches these words and a class's slot is used
// by one lane at a time (phases are separated by __syncwarp), so they are plain L1-cached
// read-modify-writes, not L2 atomics (measured: engine −5 %).  All bits still set when
// the engine finishes belong to pieces sitting in their final class; k_bitheap_clear zeroes
// them for the next batch.
struct Heap {
    u32 *l0, *l1, *l2;       // slot s: l0 + s*w0, ...
    u64 w0, w1, w2;          // words per slot at each level
    u32 *slot;               // smem: slot of class k (NONE = none yet)
    u32 *nslot;              // smem counter
    u32 *ow_i, *ow_v;        // smem: cached level-0 word (index, value) holding class k's minimum
    u64 visits = 0, inserts = 0;
    bool broken = false;
    __device__ __forceinline__ u32 slot_of(u32 k) {
        u32 s = slot[k];
        if (s == NONE) { s = atomicAdd(nslot, 1u); slot[k] = s; }
        return s;
    }
    // add f to class k's overflow set whose current minimum is root; returns the new minimum
    __device__ __forceinline__ u32 insert(u32 k, u32 root, u32 f) {
        const u64 s = slot_of(k);
        inserts++;
        // one warp owns these words (a class's slot is touched by one lane at a time, phases are
        // separated by __syncwarp), so plain L1-cached read-modify-writes replace L2 atomics
        // (a summary bit is set iff the word below it is nonzero, so a nonempty word's summary
        // bits are already set)
        if (ow_i[k] == (f >> 5)) {                 // the cached word holds the minimum: nonzero
            ow_v[k] |= 1u << (f & 31);
            l0[s * w0 + (f >> 5)] = ow_v[k];
        } else {
            u32 *p0 = &l0[s * w0 + (f >> 5)];
            const u32 o0 = *p0;
            *p0 = o0 | (1u << (f & 31));
            if (!o0) {
                u32 *p1 = &l1[s * w1 + (f >> 10)];
                const u32 o1 = *p1;
                *p1 = o1 | (1u << ((f >> 5) & 31));
                if (!o1) l2[s * w2 + (f >> 15)] |= 1u << ((f >> 10) & 31);
            }
        }
        return f < root ? f : root;
    }
    __device__ __forceinline__ static u32 and_fetch(u32 *p, u32 m) { const u32 v = *p & m; *p = v; return v; }
    // remove the minimum h of class k's overflow set; returns the next minimum (NIL32 if empty)
    __device__ u32 extract(u32 k, u32 h) {
        const u64 s = slot[k];
        u32 *a0 = l0 + s * w0, *a1 = l1 + s * w1, *a2 = l2 + s * w2;
        visits++;
        const u32 w = h >> 5;
        u32 rest;
        if (ow_i[k] == w) {                                   // cached word: no atomic round trip
            rest = ow_v[k] & ~(1u << (h & 31));
            ow_v[k] = rest;
            a0[w] = rest;
        } else {
            rest = and_fetch(&a0[w], ~(1u << (h & 31)));
            ow_i[k] = w;
            ow_v[k] = rest;
        }
        if (rest) return (w << 5) + __ffs(rest) - 1;          // bits below h are never set
        ow_i[k] = NONE;
        const u32 v = w >> 5;
        rest = and_fetch(&a1[v], ~(1u << (w & 31)));
        u32 ww;
        if (rest) ww = (v << 5) + __ffs(rest) - 1;
        else {
            const u32 x = v >> 5;
            rest = and_fetch(&a2[x], ~(1u << (v & 31)));
            u32 vv = NONE;
            if (rest) vv = (x << 5) + __ffs(rest) - 1;
            else {
                for (u64 j = x + 1; j < w2; j++) {
                    visits++;
                    const u32 t = a2[j];
                    if (t) { vv = (u32)(j << 5) + __ffs(t) - 1; break; }
                }
                if (vv == NONE) return NIL32;
            }
            const u32 t1 = a1[vv];
            if (!t1) { broken = true; return NIL32; }
            ww = (vv << 5) + __ffs(t1) - 1;
        }
        const u32 t0 = a0[ww];
        if (!t0) { broken = true; return NIL32; }
        ow_i[k] = ww;
        ow_v[k] = t0;
        return (ww << 5) + __ffs(t0) - 1;
    }
};

__device__ __forceinline__ u32 first_ge(const Smem &S, u32 sw, u32 c, int NC) {
    if (c >= (u32)NC) return NONE;
    u32 w = c >> 5;
    u32 m = S.cw[w] & (0xFFFFFFFFu << (c & 31));
    if (m) return (w << 5) + __ffs(m) - 1;
    u32 sm = (w >= 31) ? 0u : (sw & (0xFFFFFFFFu << (w + 1)));
    if (!sm) return NONE;
    u32 w2 = __ffs(sm) - 1;
    return (w2 << 5) + __ffs(S.cw[w2]) - 1;
}

// The first-level summary is not maintained here: each chunk recomputes it from the second-level
// words with one ballot, so the arrivals warp and the class-update warp can set and clear bits of
// the same word concurrently (atomics on cw only).
__device__ __forceinline__ void set_bit(Smem &S, u32 k) { atomicOr(&S.cw[k >> 5], 1u << (k & 31)); }
__device__ __forceinline__ void clear_bit(Smem &S, u32 k) { atomicAnd(&S.cw[k >> 5], ~(1u << (k & 31))); }

struct Csr {
    const uint4 *r4;   // class-sorted {f, batch-start start, end - 1, 0} (one 16-byte record per member)
};

#define RI(j) ((b + (j)) & msk)
// Sorted insertion of v (key f) into class k's ring holding n < H entries: every entry is loaded
// at once (independent loads), the position is a count of smaller keys, and the shift is a set of
// predicated stores — no load-compare-store chain per step.
__device__ __forceinline__ void ring_insert(uint4 *hc, u32 b, u32 msk, u32 n, uint4 v, u32 f) {
    uint4 x[H];
#pragma unroll
    for (int j = 0; j < H - 1; j++) x[j] = hc[RI(j)];
    u32 pos = 0;
#pragma unroll
    for (int j = 0; j < H - 1; j++) pos += ((u32)j < n && (x[j].x & ~HEAPBIT) < f) ? 1u : 0u;
#pragma unroll
    for (int j = H - 1; j >= 1; j--)
        if ((u32)j <= n && (u32)j > pos) hc[RI(j)] = x[j - 1];
    hc[RI(pos)] = v;
}

// Refill of class k's head cache from min(CSR[ptr], overflow root), in two passes that the warp
// runs converged (every leader's CSR part, then every leader's overflow part).
// Pass 1: append the next CSR members.  Returns whether the cache needed members (below
// REFILL_AT); pass 2 runs only then.
__device__ __forceinline__ bool refill_csr(Smem &S, const Csr &csr, u32 k) {
    const u32 n = S.hn[k];
    if (n >= hrefill(k)) return false;
    const u32 p = S.ptr[k], e = S.endp[k];
    if (p >= e) return true;
    uint4 *hc = &S.hc[hbase(k)];
    const u32 msk = hmask(k);
    const u32 b = S.hb[k];                      // ring buffer: entry j lives at (b + j) % depth
    const u32 m = min(min((u32)FILL_TO, msk + 1) - n, e - p);
    uint4 v[H];
#pragma unroll
    for (int j = 0; j < H; j++)
        if ((u32)j < m) v[j] = csr.r4[p + j];   // one round of independent 16-byte loads
#pragma unroll
    for (int j = 0; j < H; j++)
        if ((u32)j < m) hc[RI(n + j)] = v[j];
    S.hn[k] = (unsigned char)(n + m);
    S.ptr[k] = p + m;
    return true;
}
// Pass 2: merge in overflow members smaller than the cache's tail (or filling it to REFILL_AT),
// evicting CSR members back to the CSR range (they are its last consumed entries).  Overflow pulls
// are serial: pull only what correctness needs — members below the tail — plus enough to get back
// to REFILL_AT.
__device__ void refill_ovf(Smem &S, Heap &hp, const u64 *__restrict__ fs, const u64 *__restrict__ fe, u32 k,
                           u64 &delmins) {
    u32 rt = S.root[k];
    if (rt == NIL32) return;
    u32 n = S.hn[k];
    u32 p = S.ptr[k];
    uint4 *hc = &S.hc[hbase(k)];
    const u32 msk = hmask(k), dep = msk + 1, rat = hrefill(k);
    const u32 b = S.hb[k];
    while (rt != NIL32 && (n < rat || rt < (hc[RI(n - 1)].x & ~HEAPBIT))) {
        // issue the extract's accesses and the member's data loads together (independent)
        u32 nxt = hp.extract(k, rt);
        const u32 s0 = (u32)fs[rt], e0 = (u32)(fe[rt] - 1);
        if (n == dep) {                          // evict the tail (it is > rt)
            const u32 ev = hc[RI(dep - 1)].x;
            if (ev & HEAPBIT) nxt = hp.insert(k, nxt, ev & ~HEAPBIT);
            else p--;
            n--;
        }
        ring_insert(hc, b, msk, n, make_uint4(rt | HEAPBIT, s0, e0, 0u), rt);
        n++;
        rt = nxt;
        delmins++;
    }
    S.hn[k] = (unsigned char)n;
    S.ptr[k] = p;
    S.root[k] = rt;
}
__device__ __forceinline__ void refill(Smem &S, Heap &hp, const Csr &csr, const u64 *__restrict__ fs,
                                       const u64 *__restrict__ fe, u32 k, u64 &delmins) {
    if (refill_csr(S, csr, k)) refill_ovf(S, hp, fs, fe, k, delmins);
}

// a remainder piece f = [s, e1 + 1) joins class k
__device__ void arrive(Smem &S, Heap &hp, u32 k, u32 f, u32 s, u32 e1) {
    const u32 before = S.cnt[k]++;
    if (before == 0) set_bit(S, k);
    u32 n = S.hn[k];
    uint4 *hc = &S.hc[hbase(k)];
    const u32 msk = hmask(k), dep = msk + 1;
    const u32 b = S.hb[k];
    // the cache must stay "the n smallest members": f enters it if it is below the cache's
    // tail, or if every member is cached (nothing outside could be smaller)
    const u32 tail = n > 0 ? (hc[RI(n - 1)].x & ~HEAPBIT) : 0u;
    if ((n > 0 && f < tail) || (n < dep && before == n)) {
        if (n == dep) {         // evict the largest cached member
            const u32 ev = hc[RI(dep - 1)].x;
            if (ev & HEAPBIT) S.root[k] = hp.insert(k, S.root[k], ev & ~HEAPBIT);
            else S.ptr[k]--;    // the largest cached CSR member is CSR[ptr-1]
            n = dep - 1;
        } else {
            S.hn[k] = (unsigned char)(n + 1);
        }
        ring_insert(hc, b, msk, n, make_uint4(f | HEAPBIT, s, e1, 0u), f);
    } else {
        S.root[k] = hp.insert(k, S.root[k], f);
    }
}

// ---------------------------------------------------------------- SEGFIT_LIFO ----
// The paper's own segregated fit (Alg. 4/5): each bin is a stack; a class's member order is
// push recency (newest first) instead of address.  Every remainder dropped during the batch is
// the newest member of its class, so it enters the head cache at the FRONT; when the cache is
// full its oldest entry is evicted — a CSR member goes back to the CSR range, an earlier
// remainder onto a per-class spill stack (links in global memory, indexed by f).  Spilled
// remainders are all newer than every CSR member, and the stack top is the newest spilled, so a
// refill pops the stack before touching the CSR range.
struct Lifo {
    u32 *next;          // spill-stack links, indexed by f
    u32 *stamp;         // per-piece push stamp (persisted for the next batch)
    const u64 *clock;   // logical push clock at the start of this alloc batch
};

__device__ void refill_lifo(Smem &S, const Lifo &lf, const Csr &csr, const u64 *__restrict__ fs,
                            const u64 *__restrict__ fe, u32 k, u64 &pops) {
    u32 n = S.hn[k];
    u32 p = S.ptr[k], e = S.endp[k], rt = S.root[k];
    const u32 rat = hrefill(k), msk = hmask(k);
    if (n >= rat || (p >= e && rt == NIL32)) return;
    uint4 *hc = &S.hc[hbase(k)];
    const u32 b = S.hb[k];
    while (rt != NIL32 && n < rat) {                     // spilled remainders first (newer)
        const u32 nx = lf.next[rt];
        hc[RI(n)] = make_uint4(rt | HEAPBIT, (u32)fs[rt], (u32)(fe[rt] - 1), 0u);
        n++;
        rt = nx;
        pops++;
    }
    if (rt == NIL32) {                                   // then the CSR range (oldest members)
        const u32 m = min(msk + 1 - n, e - p);
#pragma unroll
        for (int j = 0; j < H; j++) {
            if ((u32)j < m) hc[RI(n + j)] = csr.r4[p + j];
        }
        n += m;
        p += m;
    }
    S.hn[k] = (unsigned char)n;
    S.ptr[k] = p;
    S.root[k] = rt;
}

// a remainder f = [s, e1 + 1) is pushed at the head of class k (Alg. 4 :350-356)
__device__ void arrive_lifo(Smem &S, const Lifo &lf, u32 k, u32 f, u32 s, u32 e1) {
    if (S.cnt[k]++ == 0) set_bit(S, k);
    u32 n = S.hn[k];
    u32 b = S.hb[k];
    uint4 *hc = &S.hc[hbase(k)];
    const u32 msk = hmask(k);
    if (n == msk + 1) {                                  // evict the oldest cached member
        const u32 ev = hc[RI(msk)].x;
        if (ev & HEAPBIT) {
            const u32 x = ev & ~HEAPBIT;
            lf.next[x] = S.root[k];
            S.root[k] = x;
        } else {
            S.ptr[k]--;
        }
        n--;
    }
    b = (b - 1) & msk;
    S.hb[k] = (unsigned char)b;
    hc[RI(0)] = make_uint4(f | HEAPBIT, s, e1, 0u);
    S.hn[k] = (unsigned char)(n + 1);
}

__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive_n(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Candidates of the next chunk (wilderness mode): the uncommitted candidates [commit, limit) of the
// current chunk first (time order), then requests from `sc` whose search class is at most Mx
// (requests above Mx are WILD or fail — written here, they never enter a chunk; a stale, higher Mx
// only admits candidates the engine then marks itself).  Stages requests through rbuf/cbuf.
// Returns the candidate count; *scan_end = where the scan stopped.
__device__ u32 gather_next(Smem &S, const u64 *__restrict__ R, const u32 *__restrict__ C, u64 n,
                           u64 *__restrict__ out_u, u64 &rb_base, u64 &rb_end, int Mx, u32 commit, u32 limit,
                           u64 sc, u64 *di, u64 *dr, u32 *dc, u64 *scan_end) {
    const u32 lane = lane_id();
    u32 ncand = limit > commit ? limit - commit : 0u;
    {
        u64 a = 0, b = 0;
        u32 c = 0;
        if (lane < ncand) { a = S.ch_i[commit + lane]; b = S.ch_r[commit + lane]; c = S.ch_c[commit + lane]; }
        __syncwarp();
        if (lane < ncand) { di[lane] = a; dr[lane] = b; dc[lane] = c; }
    }
    while (ncand < 32 && sc < n) {
        if (sc < rb_base || sc + 32 > rb_end) {
            __syncwarp();
            rb_base = sc;
            rb_end = sc + RB < n ? sc + RB : n;
            for (u64 j = lane; j < rb_end - rb_base; j += 32) {
                S.rbuf[j] = R[rb_base + j];
                S.cbuf[j] = C[rb_base + j];
            }
            __syncwarp();
        }
        const u64 j = sc + lane;
        const bool v = j < n;
        const u64 rj = v ? S.rbuf[j - rb_base] : 0;
        const u32 cj = v ? S.cbuf[j - rb_base] : NONE;
        const bool cand = v && rj != 0 && (int)cj <= Mx;
        const u32 cmask = __ballot_sync(FULLMASK, cand);
        const u32 take = min((u32)__popc(cmask), 32u - ncand);
        const u32 rk = __popc(cmask & lanemask_lt());
        if (cand && rk < take) { di[ncand + rk] = j; dr[ncand + rk] = rj; dc[ncand + rk] = cj; }
        u64 nsc = sc + 32 < n ? sc + 32 : n;               // scanning stops at the first one not taken
        const u32 firstout = __ballot_sync(FULLMASK, cand && rk == take);
        if (firstout) nsc = sc + __ffs(firstout) - 1;
        if (v && !cand && j < nsc) out_u[j] = rj != 0 ? WILD : HEAP_NULL_U64;
        ncand += take;
        sc = nsc;
    }
    __syncwarp();
    *scan_end = sc;
    return ncand;
}

// Helper warps of the multi-warp engine (nthr = 64 or 96 threads).  Per chunk each waits for warp
// 0's hand-off (named barrier 1), does its share and signals completion (barrier 2):
//   * warp 1 applies the arrival groups of every class warp 0 does not pop / carve in the chunk
//     (classes are disjoint between the warps within a chunk, the availability words are updated
//     with atomics, new overflow slots are numbered atomically); with three warps it also refills
//     the classes that lost members and see no arrival in the chunk (CSR part, then overflow part,
//     converged as on warp 0);
//   * the next chunk's candidate gather (wilderness mode) runs on warp 1 with two warps, on warp 2
//     with three — it reads only the request staging, so it overlaps everything else.
__device__ void helper_worker(Smem &S, Heap hp, const u64 *__restrict__ R, const u32 *__restrict__ C, u64 n,
                              u64 *__restrict__ out_u, const Csr csr, const u64 *__restrict__ fs,
                              const u64 *__restrict__ fe, const int nthr, const int wid) {
    const u32 lane = lane_id();
    u64 rb_base = 0, rb_end = 0;                  // this warp's view of the request staging buffer
    u64 delmin = 0;
    const bool arr = wid == 1, refills = wid == 1 && nthr == 96, gath = (wid == 1 && nthr == 64) || wid == 2;
    for (;;) {
        bar_sync_n(1, nthr);
        if (S.eng_done) break;
        if (arr) {
            const u32 tag = S.ctag, g = S.dg[lane], k = S.dnk[lane];
            if (g && S.etag[k] != tag) {
                u32 mm = g;
                while (mm) {
                    const u32 d = __ffs(mm) - 1;
                    mm &= mm - 1;
                    arrive(S, hp, k, S.res_f[d], (u32)(S.res_s[d] + S.ch_r[d]), S.res_e[d]);
                }
            }
        }
        if (refills) {
            const u32 rk = S.rk[lane];
            __syncwarp();
            const bool rf2 = rk != NONE && refill_csr(S, csr, rk);
            __syncwarp();
            if (rf2) refill_ovf(S, hp, fs, fe, rk, delmin);
        }
        if (arr && hp.broken) S.broken1 = 1;
        if (gath && S.g_need) {                   // the next chunk's candidates
            u64 se = 0;
            const u32 nc = gather_next(S, R, C, n, out_u, rb_base, rb_end, S.g_mx, S.g_commit, S.g_limit, S.g_scan,
                                       S.nx_i, S.nx_r, S.nx_c, &se);
            if (lane == 0) { S.nx_n = nc; S.nx_scan = se; }
        }
        __syncwarp();
        bar_arrive_n(2, nthr);
    }
    if (arr) {
        const u64 v = warp_sum64(hp.visits), ins = warp_sum64(hp.inserts), dm = warp_sum64(delmin);
        if (lane == 0) { S.w1_visits = v; S.w1_inserts = ins; S.w1_delmin = dm; }
    }
    __syncwarp();
    bar_arrive_n(3, nthr);                       // its counters are in
}

template <bool LIFO>
__global__ void __launch_bounds__(96, 1) k_engine(Csr csr, const u32 *__restrict__ off,
                                                  u64 *__restrict__ fs, const u64 *__restrict__ fe,
                                                  const u64 *__restrict__ R, const u32 *__restrict__ C, u64 n,
                                                  u64 *__restrict__ out_u, u32 *bm, u64 w0, u64 w1, u64 w2,
                                                  u32 *slot_map, int NC, int L, u64 *stats, Lifo lf,
                                                  const u64 *n_in, const u32 *wild) {
    PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (n_in) n = *n_in;   // request count on the device (a hybrid heap's TLSF share)
    // wilderness split (k_wild_setup): class Kw's single member is left out of the class state;
    // a valid request finding no class >= its search class is marked WILD and served later by
    // k_wild_apply's prefix sum.  Kw = NONE: every class is in the state (the plain engine).
    const u32 Kw = wild ? wild[0] : NONE;
    const bool wmode = Kw != NONE;
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const u32 lane = lane_id();
    const u64 nslots = (u64)NC;
    Heap hp{bm, bm + nslots * w0, bm + nslots * (w0 + w1), w0, w1, w2, S.slot, &S.nslot, S.ow_i, S.ow_v, 0, false};
    const int nthr = blockDim.x;
    const bool two = !LIFO && nthr >= 64;        // helper warps (helper_worker)
    const bool three = two && nthr == 96;        // warp 1 also refills classes without arrivals, warp 2 gathers
    if (threadIdx.x >= 32) {
        bar_sync_n(4, nthr);                      // warp 0 has built the class state
        if (two) helper_worker(S, hp, R, C, n_in ? *n_in : n, out_u, csr, fs, fe, nthr, threadIdx.x >> 5);
        return;
    }
    if (lane == 0) { S.nslot = 0; S.eng_done = 0; S.broken1 = 0; S.w1_visits = 0; S.w1_inserts = 0; S.w1_delmin = 0; }
    for (int k = lane; k < MAX_NC; k += 32) { S.etag[k] = NONE; S.atag[k] = NONE; }
    // ---- init: CSR ranges, head caches, bitmaps ----
    for (int k = lane; k < NC; k += 32) {
        u32 b = off[k], e = off[k + 1];
        if ((u32)k == Kw) b = e;     // the wilderness is not a member of the class state
        S.slot[k] = NONE;
        S.ow_i[k] = NONE;
        S.cnt[k] = e - b;
        S.hn[k] = 0;
        S.hb[k] = 0;
        S.ptr[k] = b;
        S.endp[k] = e;
        S.root[k] = NIL32;
    }
    __syncwarp();
    u64 n_delmin = 0;
    for (int k = lane; k < NC; k += 32) {
        if constexpr (LIFO) refill_lifo(S, lf, csr, fs, fe, k, n_delmin);
        else refill(S, hp, csr, fs, fe, k, n_delmin);
    }
    const u64 t_alloc = LIFO ? *lf.clock : 0;    // push stamp of request i's remainder: t_alloc + i
    __syncwarp();
    {
        u32 swl = 0;
        for (int w = 0; w < 32; w++) {
            int k = w * 32 + lane;
            u32 b = __ballot_sync(FULLMASK, k < NC && S.cnt[k] > 0);
            if (lane == 0) S.cw[w] = b;
            if (b) swl |= 1u << w;
        }
        if (lane == 0) S.sw = swl;
    }
    __syncwarp();
    if (nthr >= 64) bar_arrive_n(4, nthr);       // releases the helper warps (named barriers: warp-specialised)
    u64 rb_base = 0, rb_end = 0;
    u32 keep = 0;          // wilderness mode: candidates carried over from the previous chunk
    u64 resume = 0;        // ... and where its gather stopped
    bool prefetched = false;   // two-warp wilderness mode: warp 1 gathered this chunk's candidates
    int mx_chunk = 0;          // Mx at this chunk's start (the next gather's bound: never below the truth)
    u64 n_iter = 0, n_retarget = 0, n_rounds = 0, n_qsteps = 0, n_refill = 0;
    long long t_refill = 0;
    long long t_spec = 0, t_dirty = 0, t_cls = 0, t_arr = 0, t_store = 0, t0;
    long long t_pop = 0, t_rcsr = 0, t_rovf = 0;   // class-update sub-phases (warp-level)
    long long t_gather = 0;                        // candidate gather / request staging
    u64 pos = 0;
    while (pos < n) {
        n_iter++;
        const long long tg0 = ENG_CLK();
        // watchdogs: the engine must terminate even if an invariant broke (reported as error)
        if (__any_sync(FULLMASK, hp.broken) || S.broken1 || n_iter > n + 64) {
            if (lane == 0 && stats) stats[2] = (hp.broken || S.broken1) ? 4 : 3;
            break;
        }
        const u32 sw = __ballot_sync(FULLMASK, S.cw[lane] != 0u);   // NC <= 32 * 32
        u64 i = NIL64, ri = 0, scan_end = 0;
        u32 ci = NONE, limit = 0;
        bool act = false;
        if (!wmode) {
            if (pos + 32 > rb_end) {                 // stage requests
                rb_base = pos;
                rb_end = pos + RB < n ? pos + RB : n;
                for (u64 j = lane; j < rb_end - rb_base; j += 32) {
                    S.rbuf[j] = R[rb_base + j];
                    S.cbuf[j] = C[rb_base + j];
                }
                __syncwarp();
            }
            i = pos + lane;
            act = i < n;
            ri = act ? S.rbuf[i - rb_base] : 0;
            ci = act ? S.cbuf[i - rb_base] : NONE;
            limit = (n - pos) < 32 ? (u32)(n - pos) : 32u;
        } else {
            // gather the next 32 candidates: requests whose search class is at most the highest
            // nonempty class Mx.  The highest nonempty class only falls during the phase (pieces
            // only shrink), so a request with c > Mx now finds nothing >= c at its own time
            // either: it is WILD (valid) or fails; it is written here and never enters a chunk.
            int Mx = -1;
            if (sw) {
                const u32 w = 31 - __clz(sw);
                Mx = (int)(w * 32 + 31 - __clz(S.cw[w]));
            }
            mx_chunk = Mx;
            u32 ncand = keep;                        // ch_*[0, keep) already hold candidates
            u64 sc = keep ? resume : pos;
            if (prefetched) {                        // gathered by warp 1 during the last chunk
                ncand = S.nx_n;
                sc = S.nx_scan;
                if (ncand == 0) { pos = sc; continue; }
                act = lane < ncand;
                if (act) { i = S.nx_i[lane]; ri = S.nx_r[lane]; ci = S.nx_c[lane]; }
                S.ch_i[lane] = i;                    // this chunk's candidates, for the next carry-over
                S.ch_c[lane] = ci;
                limit = ncand;
                scan_end = sc;
            } else
            while (ncand < 32 && sc < n) {
                if (sc < rb_base || sc + 32 > rb_end) {   // a retried chunk can start below
                    __syncwarp();
                    rb_base = sc;
                    rb_end = sc + RB < n ? sc + RB : n;
                    for (u64 j = lane; j < rb_end - rb_base; j += 32) {
                        S.rbuf[j] = R[rb_base + j];
                        S.cbuf[j] = C[rb_base + j];
                    }
                    __syncwarp();
                }
                const u64 j = sc + lane;
                const bool v = j < n;
                const u64 rj = v ? S.rbuf[j - rb_base] : 0;
                const u32 cj = v ? S.cbuf[j - rb_base] : NONE;
                const bool cand = v && rj != 0 && (int)cj <= Mx;
                const u32 cmask = __ballot_sync(FULLMASK, cand);
                const u32 nc = __popc(cmask);
                const u32 take = min(nc, 32u - ncand);
                const u32 rk = __popc(cmask & lanemask_lt());
                if (cand && rk < take) { S.ch_i[ncand + rk] = j; S.ch_r[ncand + rk] = rj; S.ch_c[ncand + rk] = cj; }
                // scanning stops at the first candidate not taken
                u64 nsc = sc + 32 < n ? sc + 32 : n;
                const u32 firstout = __ballot_sync(FULLMASK, cand && rk == take);
                if (firstout) nsc = sc + __ffs(firstout) - 1;
                if (v && !cand && j < nsc) out_u[j] = rj != 0 ? WILD : HEAP_NULL_U64;
                ncand += take;
                sc = nsc;
            }
            if (!prefetched) {
                __syncwarp();
                if (ncand == 0) { pos = sc; continue; }
                act = lane < ncand;
                if (act) { i = S.ch_i[lane]; ri = S.ch_r[lane]; ci = S.ch_c[lane]; }
                limit = ncand;
                scan_end = sc;
            }
        }
        __syncwarp();
        S.ch_r[lane] = ri;
        __syncwarp();
        t0 = ENG_CLK();
        t_gather += t0 - tg0;
        const bool fail0 = act && (ri == 0 || ci >= (u32)NC);
        u32 k = (act && !fail0) ? first_ge(S, sw, ci, NC) : NONE;
        // light pre-rounds (count model): a lane ranked at or past its class's member count is
        // moved to the next nonempty class before the full round.  The model ignores head carves
        // (a member serving several requests), so a moved lane is checked after the full round:
        // if a class it skipped saw a head carve, the lane is dirty (see the dirty phase).
        const u32 k0 = k;
        u32 pm_fin = 0;                              // grouping of the final light round
        bool have_pm = false;
#pragma unroll 1
        for (int it = 0; it < LIGHT_ROUNDS; it++) {
            const bool pl = act && k != NONE;
            const u32 ck = pl ? S.cnt[k] : 0u;       // issued before the match (independent)
            const u32 pm = __match_any_sync(FULLMASK, pl ? k : (0x40000000u | lane));
            const bool ov = pl && (u32)__popc(pm & lanemask_lt()) >= ck;
            if (!__any_sync(FULLMASK, ov)) { pm_fin = pm; have_pm = true; break; }
            if (ov) k = first_ge(S, sw, k + 1, NC);
        }
        const u32 kpre = k;
        u32 peers = 0, rank = 0, flag = F_OK, myf = 0, mynk = NONE, mye = 0;
        u64 mys = 0;
        for (u32 round = 0;; round++) {
            n_rounds++;
            if (round > (u32)NC + 2) {
                if (lane == 0 && stats) stats[2] = 2;
                goto engine_end;
            }
            const bool part = act && k != NONE;
            peers = (round == 0 && have_pm) ? pm_fin : __match_any_sync(FULLMASK, part ? k : (0x40000000u | lane));
            rank = __popc(peers & lanemask_lt());
            const u32 leader = __ffs(peers) - 1;
            // Two parallel patterns cover almost every group; mixed groups fall back to the
            // leader's sequential replay below.
            //  (A) one block per request: request of rank q takes cached member q, valid when
            //      no request but the last leaves its block in the class;
            //  (B) one block for all: member 0 serves every request (head carve), valid when
            //      the remainder before each request is still in the class.
            const u32 npeer = __popc(peers);
            const u32 nh = part ? S.hn[k] : 0, nc = part ? S.cnt[k] : 0;
            const u32 hb = part ? S.hb[k] : 0;
            const u32 hbk = part ? hbase(k) : 0u, hmk = part ? hmask(k) : 0u;
            const u32 slotA = hbk + ((hb + rank) & hmk), slot0 = hbk + hb;
            const bool hasA = part && rank < nh;
            u32 fA = 0, nkA = NONE;
            u64 sA = 0;
            u32 eA = 0;
            if (hasA) {
                const uint4 mA = S.hc[slotA];
                fA = mA.x & ~HEAPBIT;
                sA = mA.y;
                eA = mA.z;
                const u64 zA = (u64)eA + 1 - sA - ri;
                nkA = zA ? cls_insert(zA, L) : NONE;
            }
            const bool okA = (__ballot_sync(FULLMASK, hasA && nkA == k && rank + 1 < npeer) & peers) == 0;
            bool okB = false, seq = false;
            if (__all_sync(FULLMASK, !part || okA)) {
                // every group takes one member per request (the common case): no prefix, no replay
                if (part) {
                    if (hasA) { flag = F_OK; myf = fA; mys = sA; mynk = (nkA == k) ? SAME : nkA; mye = eA; }
                    else flag = (rank < nc) ? F_MISS : F_OVER;
                }
            } else {
                if (part) S.lor[leader * 32 + rank] = lane;   // lane of rank q in the group
                __syncwarp();
                // segmented exclusive prefix of r over the group (Hillis-Steele over ranks)
                u64 incl = part ? ri : 0;
                // only groups that fail pattern A need the prefix (skip the scan when none does)
                const u32 maxpeer = __reduce_max_sync(FULLMASK, (part && !okA) ? npeer : 0u);
                for (u32 st = 1; st < maxpeer; st <<= 1) {
                    const u32 src = (part && rank >= st) ? S.lor[leader * 32 + rank - st] : lane;
                    const u64 t = __shfl_sync(FULLMASK, incl, src);
                    if (part && rank >= st) incl += t;
                }
                const u64 P = incl - (part ? ri : 0);
                u64 s0 = 0, z0 = 0;
                u32 f0 = 0, e0 = 0;
                if (part && nh) {
                    const uint4 m0 = S.hc[slot0];
                    f0 = m0.x & ~HEAPBIT;
                    s0 = m0.y;
                    e0 = m0.z;
                    z0 = (u64)e0 + 1 - s0;
                }
                const bool covB = part && nh && (rank == 0 || (P < z0 && z0 - P >= cls_lo(k, L)));
                const u32 uncov = __ballot_sync(FULLMASK, part && !covB);   // every lane must vote
                okB = !okA && (uncov & peers) == 0;
                if (part && okA) {
                    if (hasA) { flag = F_OK; myf = fA; mys = sA; mynk = (nkA == k) ? SAME : nkA; mye = eA; }
                    else flag = (rank < nc) ? F_MISS : F_OVER;
                } else if (part && okB) {
                    flag = F_OK; myf = f0; mys = s0 + P; mye = e0;
                    const u64 z = z0 - P - ri;
                    const u32 nk = z ? cls_insert(z, L) : NONE;
                    mynk = (nk == k) ? SAME : nk;
                }
                seq = part && !okA && !okB;
                if (seq && rank == 0) {
                    // replay the group in time order (shared memory only)
                    n_qsteps += npeer;
                    u32 b = 0, curf = 0;
                    u64 cur_s = 0, cur_e = 0;
                    bool need = true;
                    u32 q = 0;
                    for (; q < npeer; q++) {
                        const u32 lq = S.lor[lane * 32 + q];
                        if (need) {
                            if (b >= nh) break;
                            const u32 sl = hbase(k) + ((hb + b) & hmask(k));
                            const uint4 mq = S.hc[sl];
                            curf = mq.x & ~HEAPBIT;
                            cur_s = mq.y;
                            cur_e = (u64)mq.z + 1;
                            need = false;
                        }
                        const u64 rq = S.ch_r[lq];
                        S.res_flag[lq] = F_OK;
                        S.res_f[lq] = curf;
                        S.res_s[lq] = cur_s;
                        S.res_e[lq] = (u32)(cur_e - 1);
                        cur_s += rq;
                        const u64 z = cur_e - cur_s;
                        const u32 nk = z ? cls_insert(z, L) : NONE;
                        if (nk == k) S.res_nk[lq] = SAME;
                        else { S.res_nk[lq] = nk; b++; need = true; }
                    }
                    const u32 fl = (b < nc) ? F_MISS : F_OVER;
                    for (; q < npeer; q++) S.res_flag[S.lor[lane * 32 + q]] = fl;
                }
                __syncwarp();
                if (seq) {
                    flag = S.res_flag[lane];
                    myf = S.res_f[lane];
                    mys = S.res_s[lane];
                    mynk = S.res_nk[lane];
                    mye = S.res_e[lane];
                }
                __syncwarp();
            }
            const bool over = part && flag == F_OVER;
#ifdef ENGINE_DEBUG
            if (n_iter < 8)
                printf("it %llu pos %llu round %u lane %u act %d k %u rank %u flag %u f %u s %llu nk %u okA %d okB %d seq %d\n",
                       n_iter, pos, round, lane, (int)act, k, rank, flag, myf, mys, mynk, (int)okA, (int)okB, (int)seq);
#endif
            if (!__any_sync(FULLMASK, over)) break;
            if (over) { k = first_ge(S, sw, k + 1, NC); flag = F_OK; n_retarget++; }
        }
        if (act && k != NONE) { S.res_f[lane] = myf; S.res_s[lane] = mys; S.res_e[lane] = mye; }
        __syncwarp();
        t_spec += ENG_CLK() - t0;
        t0 = ENG_CLK();
        // ---- dirty requests: remainders dropped earlier in the chunk, cache misses ----
        const bool part = act && k != NONE;
        // in-class order key: address (f) — or, for LIFO bins, "after any fresh remainder"
        const u64 key = part ? (((u64)k << 32) | (LIFO ? 1u : myf)) : ~0ull;
        bool bad = part && flag == F_MISS;
        const bool dropper = part && flag == F_OK && mynk != SAME && mynk != NONE;
        // The droppers are compacted into shared memory in time order, and every lane scans the list
        // with broadcast loads: the loads are independent, so the scan pipelines instead of walking
        // the dropper mask with a find-first-set and two shuffles per dropper.
        const u32 dm = __ballot_sync(FULLMASK, dropper);
        const u32 nd = __popc(dm);
        if (dropper) {
            const u32 q = __popc(dm & lanemask_lt());
            S.dkey[q] = (((u64)mynk) << 32) | (LIFO ? 0u : myf);
            S.dlane[q] = lane;
        }
        __syncwarp();
        u32 samecls = 0;                     // droppers whose remainder joins my remainder's class
        {
            const bool chk = act && !fail0;
            const u64 clo = ((u64)ci) << 32;         // a drop class >= ci  <=>  dkey >= clo
#pragma unroll 4
            for (u32 q = 0; q < nd; q++) {
                const u64 dk = S.dkey[q];
                const u32 dl = S.dlane[q];
                if (chk && lane > dl && dk >= clo && dk < key) bad = true;
                if (dropper && (u32)(dk >> 32) == mynk) samecls |= 1u << dl;
            }
        }
        if (__any_sync(FULLMASK, act && kpre != k0)) {     // pre-moved lanes: skipped classes
            u32 sm = __ballot_sync(FULLMASK, part && flag == F_OK && mynk == SAME);
            while (sm) {
                const u32 d = __ffs(sm) - 1;
                sm &= sm - 1;
                const u32 sk = __shfl_sync(FULLMASK, k, d);
                if (act && kpre != k0 && k0 <= sk && sk < kpre) bad = true;
            }
        }
        const u32 badm = __ballot_sync(FULLMASK, bad);
        const u32 commit = badm ? (u32)(__ffs(badm) - 1) : limit;
#ifdef ENGINE_DEBUG
        if (lane == 0 && n_iter < 8) printf("it %llu commit %u badm %x\n", n_iter, commit, badm);
#endif
        if (commit == 0) {               // cannot happen (lane 0 is never dirty); never hang
            if (lane == 0 && stats) stats[2] = 1;
            goto engine_end;
        }
        const bool cm = act && lane < commit;
        t_dirty += ENG_CLK() - t0;
        t0 = ENG_CLK();
        // ---- commit: results and piece starts ----
        const u32 later = (lane < 31) ? (peers & (0xFFFFFFFEu << lane)) : 0u;   // peers after this lane
        const u32 nxt = later ? (u32)(__ffs(later) - 1) : NONE;
        const bool last_on_block = mynk != SAME || nxt >= commit;
        if (cm) {
            if (!part) out_u[i] = (wmode && ri != 0) ? WILD : HEAP_NULL_U64;
            else {
                out_u[i] = mys;
                if (last_on_block) {
                    fs[myf] = mys + ri;
                    if (LIFO && mynk != NONE) lf.stamp[myf] = (u32)(t_alloc + i);   // pushed remainder
                }
            }
        }
        // ---- class updates by group leaders: blocks that left the class; head carve ----
        __syncwarp();
        t_store += ENG_CLK() - t0;
        const u32 leftm = __ballot_sync(FULLMASK, cm && part && mynk != SAME);
        const u32 staym = __ballot_sync(FULLMASK, cm && part && mynk == SAME && last_on_block);
        // arrival groups (the first committed dropper of each remainder class leads its group)
        const bool cdrop = cm && dropper;
        const u32 g = samecls & (commit >= 32 ? FULLMASK : ((1u << commit) - 1u));   // committed ones
        const u32 mygrp = (cdrop && (g & lanemask_lt()) == 0) ? g : 0u;
        const u32 ctag = (u32)n_iter;
        auto handoff = [&](u32 rkv) {
            S.rk[lane] = rkv;
            S.dg[lane] = mygrp;
            S.dnk[lane] = mynk;
            if (lane == 0) {
                S.ctag = ctag;
                S.g_need = wmode ? 1u : 0u;          // a helper gathers the next chunk's candidates
                S.g_commit = commit;
                S.g_limit = limit;
                S.g_scan = scan_end;
                S.g_mx = mx_chunk;
            }
            __syncwarp();
            bar_arrive_n(1, nthr);
        };
        if (two) {
            // the classes this warp updates are tagged first (warp 1 applies only the arrival groups
            // of untagged classes); with three warps the classes with arrivals too (a class that
            // lost members and has none is refilled by warp 1), and the hand-off waits for the pops
            if (cm && part && rank == 0 && ((leftm | staym) & peers)) S.etag[k] = ctag;
            if (three && mygrp) S.atag[mynk] = ctag;
            __syncwarp();
            if (!three) handoff(NONE);
        }
        bool rf = false;                         // this leader's class lost members: refill
        if (cm && part && rank == 0) {
            const u32 left = __popc(leftm & peers);
            const u32 st = staym & peers;        // the surviving head was carved: new start
            const u32 b = S.hb[k];
            if (st) {
                // the carved block is the head now; it is no longer its batch-start CSR entry
                // (new start; for LIFO bins also the newest push), so mark it overflow-origin:
                // evicted later, it goes to the overflow set / spill stack and its start is
                // re-read from fs, never from the stale CSR copy
                const u32 d = __ffs(st) - 1;
                const u32 sl = hbase(k) + ((b + left) & hmask(k));
                S.hc[sl].y = (u32)(S.res_s[d] + S.ch_r[d]);
                S.hc[sl].x |= HEAPBIT;
            }
            if (left) {                          // pop `left` members: advance the ring base
                S.hb[k] = (unsigned char)((b + left) & hmask(k));
                S.hn[k] = (unsigned char)(S.hn[k] - left);
                S.cnt[k] -= left;
                rf = true;
            }
        }
        bool rfw = rf;                           // refilled by this warp
        if (three) {
            rfw = rf && S.atag[k] == ctag;
            handoff((rf && !rfw) ? k : NONE);
        }
        if constexpr (LIFO) {
            if (rf) refill_lifo(S, lf, csr, fs, fe, k, n_delmin);
        } else {
            // the leaders' refills run converged: every CSR part, then every overflow part
            __syncwarp();
            const long long ta = ENG_CLK();
            const bool rf2 = rfw && refill_csr(S, csr, k);
            __syncwarp();
            const long long tb = ENG_CLK();
            if (rf2) refill_ovf(S, hp, fs, fe, k, n_delmin);
            __syncwarp();
            const long long tc = ENG_CLK();
            t_pop += ta - t0; t_rcsr += tb - ta; t_rovf += tc - tb;
            n_refill += rf2;                     // diagnostics: refills that needed members
        }
        if (rf && S.cnt[k] == 0) clear_bit(S, k);
        __syncwarp();
        t_cls += ENG_CLK() - t0;
        t0 = ENG_CLK();
        // ---- remainders join their new classes (grouped by class, time order) ----
        // (two-warp engine: only the groups of classes this warp updated; warp 1 does the rest)
        if (mygrp && (!two || S.etag[mynk] == ctag)) {
            u32 mm = g;
            while (mm) {
                const u32 d = __ffs(mm) - 1;
                mm &= mm - 1;
                const u32 s2 = (u32)(S.res_s[d] + S.ch_r[d]);
                if constexpr (LIFO) arrive_lifo(S, lf, mynk, S.res_f[d], s2, S.res_e[d]);
                else arrive(S, hp, mynk, S.res_f[d], s2, S.res_e[d]);
            }
        }
        __syncwarp();
        if (two) bar_sync_n(2, nthr);            // the helpers' arrivals, refills and gather are in
        t_arr += ENG_CLK() - t0;
        if (!wmode) {
            pos += commit;
        } else if (two) {                            // warp 1 has gathered the next candidates
            prefetched = true;
            pos = S.nx_n ? S.nx_i[0] : S.nx_scan;
        } else if (commit < limit) {                 // carry the uncommitted candidates over
            keep = limit - commit;
            u64 ci_ = 0, cr_ = 0;
            u32 cc_ = 0;
            if (lane < keep) { ci_ = S.ch_i[commit + lane]; cr_ = S.ch_r[commit + lane]; cc_ = S.ch_c[commit + lane]; }
            __syncwarp();
            if (lane < keep) { S.ch_i[lane] = ci_; S.ch_r[lane] = cr_; S.ch_c[lane] = cc_; }
            resume = scan_end;
            pos = __shfl_sync(FULLMASK, ci_, 0);
        } else {
            keep = 0;
            pos = scan_end;
        }
        __syncwarp();
    }
engine_end:
    if (two) {                                   // release warp 1 and wait for its counters
        if (lane == 0) S.eng_done = 1;
        __syncwarp();
        bar_arrive_n(1, nthr);
        bar_sync_n(3, nthr);
    }
    if (slot_map)
        for (int k = lane; k < NC; k += 32) slot_map[k] = S.slot[k];   // for k_bitheap_clear
    if (stats) {
        u64 t = n_retarget, q = n_qsteps, dl = n_delmin, vis = hp.visits, nr = n_refill, ins = hp.inserts;
        if (two && lane == 0) { vis += S.w1_visits; ins += S.w1_inserts; dl += S.w1_delmin; }
        u64 tmax = (u64)t_refill;
        for (int o = 16; o > 0; o >>= 1) {
            nr += __shfl_xor_sync(FULLMASK, nr, o);
            const u64 x = __shfl_xor_sync(FULLMASK, tmax, o);
            tmax = x > tmax ? x : tmax;
        }
        for (int o = 16; o > 0; o >>= 1) {
            vis += __shfl_xor_sync(FULLMASK, vis, o);
            t += __shfl_xor_sync(FULLMASK, t, o);
            q += __shfl_xor_sync(FULLMASK, q, o);
            dl += __shfl_xor_sync(FULLMASK, dl, o);
            ins += __shfl_xor_sync(FULLMASK, ins, o);
        }
        if (lane == 0) {
            stats[0] += n_iter; stats[1] += t; stats[3] += n_rounds; stats[4] += q;
            stats[5] += t_spec; stats[6] += t_dirty; stats[7] += t_cls; stats[8] += t_arr; stats[9] += dl; stats[10] += vis; stats[11] += t_store;
            stats[12] += nr; stats[13] += tmax; stats[15] += ins;
            stats[16] += t_pop; stats[17] += t_rcsr; stats[18] += t_rovf; stats[19] += t_gather;
        }
    }
}

// zero the overflow-bitmap words still holding members after the engine: every such member is
// a piece in its final class, so visiting each surviving piece clears them all
__global__ void k_bitheap_clear(const u64 *__restrict__ fs, const u64 *__restrict__ fe, const u64 *F_dev,
                                const u32 *__restrict__ slot_map, u32 *bm, u64 w0, u64 w1, u64 w2, int NC,
                                int L) {
    PDL_ENTRY();
    const u64 F = *F_dev;
    const u64 nslots = (u64)NC;
    u32 *l0 = bm, *l1 = bm + nslots * w0, *l2 = bm + nslots * (w0 + w1);
    for (u64 f = (u64)blockIdx.x * blockDim.x + threadIdx.x; f < F; f += (u64)gridDim.x * blockDim.x) {
        const u64 z = fe[f] - fs[f];
        if (!z) continue;
        const u32 s = slot_map[cls_insert(z, L)];
        if (s == NONE) continue;
        l0[s * w0 + (f >> 5)] = 0;
        l1[s * w1 + (f >> 10)] = 0;
        l2[s * w2 + (f >> 15)] = 0;
    }
}

// ---------------------------------------------------------------- wilderness split ----
// Let K0 be the highest class with a member at the start of the alloc phase.  If (a) K0 has exactly
// one member w, (b) w minus the units T of EVERY request of the batch is still in a class Kf above
// every other member's class, and (c) every valid request's search class is <= Kf, then during
// the phase (i) w's class stays above every other piece's (pieces only shrink), (ii) a request
// takes w iff no other piece has class >= its search class (lowest (class, address) key among
// classes >= c_i; w is the only candidate left and it fits by (c)), and (iii) taking w changes no
// other class.  So the engine runs without w: a request that finds no class is marked WILD, and
// the WILD requests take consecutive pieces of w's low end in request order — result = start(w) +
// exclusive prefix sum of their units (Alg. 1 carve, applied one by one).
__global__ void __launch_bounds__(32) k_wild_setup(const u32 *__restrict__ off, const u32 *__restrict__ csr_f,
                                                   const u64 *__restrict__ fs, const u64 *__restrict__ fe,
                                                   u64 n, const u64 *n_in, int NC, int L, int enable, DevCtr *C) {
    PDL_ENTRY();
    // T = C->wild_acc[0] (units of all requests), cmax = C->wild_acc[1] (k_alloc_prep)
    if (n_in) n = *n_in;
    const u32 lane = lane_id();
    int kmax = -1, kmax2 = -1;           // highest and second-highest class with members
    for (int k = lane; k < NC; k += 32)
        if (off[k + 1] > off[k]) { kmax2 = kmax; kmax = k; }
    for (int o = 16; o > 0; o >>= 1) {   // merge (top, second) pairs across lanes
        const int a = __shfl_xor_sync(FULLMASK, kmax, o), b = __shfl_xor_sync(FULLMASK, kmax2, o);
        if (a > kmax) { kmax2 = max(kmax, b); kmax = a; }
        else kmax2 = max(kmax2, a == kmax ? b : a);
    }
    if (lane == 0) {
        const u64 T = C->wild_acc[0], cmax = C->wild_acc[1];
        u32 K0 = NONE, fw = NONE;
        const int k = kmax;
        if (enable && k >= 0 && off[k + 1] - off[k] == 1) {
            const u32 f = csr_f[off[k]];
            const u64 z = fe[f] - fs[f];
            if (z > T) {
                const u32 Kf = cls_insert(z - T, L);
                if ((int)Kf > kmax2 && cmax <= Kf) { K0 = (u32)k; fw = f; }
            }
        }
        C->wild[0] = K0;
        C->wild[1] = fw;
        C->wild_n = (K0 != NONE) ? n : 0;
        C->wild_start = (K0 != NONE) ? fs[fw] : 0;
        if (K0 != NONE) C->eng[14]++;           // diagnostics: batches served with the split
    }
}

// units of each WILD request (0 otherwise), for the prefix sum
__global__ void k_wild_flags(const u64 *__restrict__ out_u, const u64 *__restrict__ R, const DevCtr *C,
                             u32 *__restrict__ flags) {
    PDL_ENTRY();
    const u64 n = C->wild_n;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        flags[i] = out_u[i] == WILD ? (u32)R[i] : 0u;
}

// WILD request i takes [start(w) + pre_i, + r_i); w keeps what is left
__global__ void k_wild_apply(u64 *__restrict__ out_u, const u32 *__restrict__ pre, const DevCtr *C,
                             u64 *__restrict__ fs) {
    PDL_ENTRY();
    const u64 n = C->wild_n;
    if (!n) return;
    const u64 w0 = C->wild_start;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        if (out_u[i] == WILD) out_u[i] = w0 + pre[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) fs[C->wild[1]] = w0 + C->wild_total;
}

// class-sorted records {f, start, end - 1, 0} for the CSR (one gather after the class sort)
__global__ void k_csr_data(const u32 *__restrict__ csr_f, const u64 *__restrict__ fs, const u64 *__restrict__ fe,
                           const u64 *F_dev, uint4 *__restrict__ r4) {
    PDL_ENTRY();
    const u64 F = *F_dev;
    for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < F; p += (u64)gridDim.x * blockDim.x) {
        const u32 f = csr_f[p];
        r4[p] = make_uint4(f, (u32)fs[f], (u32)(fe[f] - 1), 0u);
    }
}

}  // namespace tlsfw
