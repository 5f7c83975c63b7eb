// engine_seq.cuh — sequential exact engine for SEGFIT / TLSF allocation batches, with every
// global-memory access moved off the critical chain onto helper warps.  ABLATION (HEAP_ENGINE=seq):
// exact (the whole GPU parity suite passes with it) but slower than the warp-chunk engine
// (engine_tlsf.cuh): measured on B200, config 5 batches 1-3, 850-900 cycles per request against
// ~400 — one thread runs ~120 mostly dependent instructions per request at 4-6 cycles each (ALU and
// branch latency, no ILP), while the chunk engine amortises its fixed cost over ~19 committed
// requests per 32-lane chunk.  See DESIGN.md §12.
//
// Semantics (identical to engine_tlsf.cuh and the oracle): requests are served one by one in
// request order; request i takes, among the free pieces whose class is >= its search class c_i,
// the one with the smallest (class, address) key (Alg. 4 + the bitmap/ffs fallback
// PAPER.md:332-337,440; TLSF two-level lookup PAPER.md:449; address order in a class, reading
// C9) and carves r_i units off its low end (Alg. 1).  Pieces are indexed by
// f = the address rank of their batch-start free block (each batch-start block holds at most one
// piece during the phase, and only its low end moves), so address order is f order.
//
// One CTA of 16 warps.
//  * Lane 0 of warp 0 ("main") runs the request chain alone (no warp collectives on the chain).
//    Its state lives in shared memory: the two-level availability bitmap (second-level words
//    cw[], the first-level word in a register); per class k the head member hd[k] = {f, start,
//    end-1, member count} and a sorted ring of up to H next members.  Invariant: hd and the ring
//    are the class's smallest members; every other ("outside") member is above the ring's tail.
//  * Warp 1 ("loader") streams the requests (units, search class) into a shared-memory ring.
//  * The other warps except 4, 8, 12 are helpers (no helper shares the main warp's scheduler:
//    warp w runs on sub-partition w mod 4).  The outside members of class k — its untouched
//    batch-start CSR suffix plus an overflow set O_k (a three-level bitmap over f in global
//    memory) — belong to helper k mod NHELP, which serves two messages from main through a FIFO in
//    shared memory: INS(k, piece) — the piece joins O_k — and REQ(k, m) — deliver the m smallest
//    outside members into a delivery slot.  Main merges a delivery when its completion appears.
//    Members sent to O_k after a REQ may be smaller than the delivered ones, so main keeps only the
//    delivered members below the smallest such member and gives the rest back (INS).  Main waits
//    on a helper only when a class's head is consumed while its ring is empty.
#pragma once
#include "common.cuh"

namespace tlsfs {

constexpr int H = 8;              // ring depth per class (power of two)
constexpr int MAX_NC = 928;       // classes of 2^32 units at SL_LOG2 = 5 (fl <= 28)
constexpr int NWARP = 16;
constexpr int NHELP = 11;         // warps 2, 3, 5, 6, 7, 9, 10, 11, 13, 14, 15
constexpr int QD = 64;            // message FIFO depth per helper (power of two)
constexpr int NSLOT = 64;         // delivery slots (at most one outstanding REQ per class)
constexpr int CQ = 128;           // completion FIFO depth (>= NSLOT, power of two)
constexpr int RB = 2048;          // request ring (power of two, multiple of 32)
#ifndef SEQ_TIMING
#define SEQ_TIMING 0
#endif
#ifndef SEQ_REQ_AT
#define SEQ_REQ_AT 4
#endif
constexpr u32 REQ_AT = SEQ_REQ_AT;  // post a refill when the ring holds fewer members
constexpr u32 NONE = 0xFFFFFFFFu;
constexpr u32 NOSLOT = 0xFFu;
constexpr u32 M_INS = 1, M_REQ = 2, M_STOP = 3;
constexpr u64 WILD = 0xFFFFFFFFFFFFFFFEull;   // result marker: served by the wilderness (k_wild_apply)

struct Smem {
    uint4 hd[MAX_NC];                 // head member {f, start, end-1, member count}
    uint4 rg[MAX_NC * H];             // ring entries {f, start, end-1, -} sorted by f
    u32 meta[MAX_NC];                 // hn | hb << 8 | outstanding slot << 16
    u32 insmin[MAX_NC];               // smallest f sent to O_k since the outstanding REQ
    u32 cw[32];                       // second-level availability words (first level: register)
    // helper-owned class state
    u32 ptr[MAX_NC], endp[MAX_NC], root[MAX_NC], slot[MAX_NC];
    u32 nslot;
    // main -> helper FIFOs
    uint4 q[NHELP][QD];
    u32 qhead[NHELP];                 // messages consumed (helper-written)
    u32 qt[NHELP], qhc[NHELP];        // main: tail, cached head
    // deliveries
    uint4 dl[NSLOT][H];
    u32 dn[NSLOT], dk[NSLOT];
    u32 fstk[NSLOT];
    u32 fsp;
    u32 ctail;                        // completion tail (helpers, atomicAdd)
    u32 cq[CQ];                       // completion entries: slot | lap << 16
    // request ring (loader -> main)
    u32 rr[RB], rc[RB];               // units (larger than 2^32 - 1: stored as 0 = fails), class
    u32 rfill;                        // requests staged, low 32 bits (loader-written)
    u32 rcons;                        // requests consumed, low 32 bits (main-written)
    u32 abort_;                       // main gave up (watchdog): helpers leave
};

__device__ __forceinline__ u32 sh_addr(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void st_vol_v4(uint4 *p, u32 x, u32 y, u32 z, u32 w) {
    asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sh_addr(p)), "r"(x), "r"(y), "r"(z),
                 "r"(w)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_vol_v4(const uint4 *p) {
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(sh_addr(p))
                 : "memory");
    return v;
}
__device__ __forceinline__ u32 ld_vol(const u32 *p) {
    u32 v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(sh_addr(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_vol(u32 *p, u32 v) {
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(sh_addr(p)), "r"(v) : "memory");
}

struct Csr {
    const u32 *f;   // class-sorted f
    const u32 *s;   // class-sorted batch-start start
    const u32 *e;   // class-sorted end - 1
};

// ------------------------------------------------------------------ helper side ----
// O_k: a three-level bitmap over f in global memory (a bit per piece, a bit per nonempty word, a
// bit per nonempty second-level word), one slot per class that ever needs one; the helper that
// owns class k is the only warp touching its slot.  root[k] is the exact minimum (NONE = empty).
struct Ovf {
    u32 *l0, *l1, *l2;
    u64 w0, w1, w2;
    u64 *pse;               // (end-1) << 32 | start of every piece in some O_k (helper-owned)
};

template <class SM>
__device__ __forceinline__ u32 ovf_slot(SM &S, u32 k) {
    u32 s = S.slot[k];
    if (s == NONE) {
        if (lane_id() == 0) s = atomicAdd(&S.nslot, 1u);
        s = __shfl_sync(FULLMASK, s, 0);
        if (lane_id() == 0) S.slot[k] = s;
        __syncwarp();
    }
    return s;
}

// warp-uniform: f joins O_k
template <class SM>
__device__ void ovf_insert(SM &S, const Ovf &O, u32 k, u32 f, u32 s, u32 e1) {
    const u64 sl = ovf_slot(S, k);
    u32 *a0 = O.l0 + sl * O.w0, *a1 = O.l1 + sl * O.w1, *a2 = O.l2 + sl * O.w2;
    if (lane_id() == 0) {
        O.pse[f] = ((u64)e1 << 32) | s;
        const u32 w = f >> 5;
        const u32 o0 = a0[w];
        a0[w] = o0 | (1u << (f & 31));
        if (!o0) {
            const u32 o1 = a1[w >> 5];
            a1[w >> 5] = o1 | (1u << (w & 31));
            if (!o1) a2[w >> 10] |= 1u << ((w >> 5) & 31);
        }
        if (f < S.root[k]) S.root[k] = f;
    }
    __syncwarp();
}

// warp-uniform: remove O_k's minimum h; returns the new minimum (NONE if empty).  Every set bit is
// above h (h is the minimum), so the search only looks upward.
template <class SM>
__device__ u32 ovf_extract(SM &S, const Ovf &O, u32 k, u32 h, bool &broken) {
    const u64 sl = S.slot[k];
    u32 *a0 = O.l0 + sl * O.w0, *a1 = O.l1 + sl * O.w1, *a2 = O.l2 + sl * O.w2;
    const u32 lane = lane_id();
    const u32 w = h >> 5;
    __syncwarp();                      // earlier lane-0 writes are visible to every lane
    u32 rest = a0[w] & ~(1u << (h & 31));
    if (lane == 0) a0[w] = rest;
    if (rest) return (w << 5) + __ffs(rest) - 1;
    const u32 v = w >> 5;
    rest = a1[v] & ~(1u << (w & 31));
    if (lane == 0) a1[v] = rest;
    u32 ww;
    if (rest) ww = (v << 5) + __ffs(rest) - 1;
    else {
        const u32 x = v >> 5;
        rest = a2[x] & ~(1u << (v & 31));
        if (lane == 0) a2[x] = rest;
        u32 vv = NONE;
        if (rest) vv = (x << 5) + __ffs(rest) - 1;
        else {
            for (u64 j0 = x + 1; j0 < O.w2; j0 += 32) {      // 32 words per step
                const u64 j = j0 + lane;
                const u32 t = j < O.w2 ? a2[j] : 0u;
                const u32 b = __ballot_sync(FULLMASK, t != 0);
                if (b) {
                    const u32 src = __ffs(b) - 1;
                    const u32 tv = __shfl_sync(FULLMASK, t, src);
                    vv = (u32)((j0 + src) << 5) + __ffs(tv) - 1;
                    break;
                }
            }
            if (vv == NONE) return NONE;
        }
        const u32 t1 = a1[vv];
        if (!t1) { broken = true; return NONE; }
        ww = (vv << 5) + __ffs(t1) - 1;
    }
    const u32 t0 = a0[ww];
    if (!t0) { broken = true; return NONE; }
    return (ww << 5) + __ffs(t0) - 1;
}

// A helper warp: serves INS / REQ messages from its FIFO in order until STOP (the caller's shared
// memory type SM provides the FIFOs, delivery slots, completion ring and the helper-owned class
// state ptr / endp / root / slot).  At STOP it publishes its classes' overflow slots (slot_map).
template <class SM, int NH>
__device__ void helper_loop(SM &S, u32 hid, const Csr &csr, const Ovf O, int NC, u32 *slot_map, u64 *stats) {
    const u32 lane = lane_id();
    bool broken = false;
    u64 nmsg = 0;
    for (u32 head = 0;; head++) {
        const u32 want = ((head / QD) + 1) & 0xFFFFFu;
        uint4 m;
        bool quit = false;
        for (;;) {
            m = ld_vol_v4(&S.q[hid][head & (QD - 1)]);
            if ((m.x >> 12) == want) break;
            if (ld_vol(&S.abort_)) { quit = true; break; }
            __nanosleep(100);
        }
        if (quit) break;
        if (lane == 0) st_vol(&S.qhead[hid], head + 1);
        const u32 type = (m.x >> 10) & 3, k = m.x & 0x3FF;
        if (type == M_STOP) {
            // every message for this helper's classes is done: publish their overflow slots
            if (slot_map)
                for (u32 k = hid + lane * NH; k < (u32)NC; k += 32 * NH) slot_map[k] = S.slot[k];
            break;
        }
        nmsg++;
        if (type == M_INS) {
            ovf_insert(S, O, k, m.y, m.z, m.w);
        } else {   // M_REQ: the m.y smallest of the CSR suffix and O_k into slot m.z
            const u32 want_n = m.y, slot = m.z;
            const u32 p = S.ptr[k], e = S.endp[k];
            u32 rt = S.root[k];
            const u32 mc = min(want_n, e - p);
            u32 cf = NONE, cs_ = 0, ce_ = 0;
            if (lane < mc) { cf = csr.f[p + lane]; cs_ = csr.s[p + lane]; ce_ = csr.e[p + lane]; }
            u32 got = 0, cp = 0;
            u32 of = 0, os = 0, oe = 0;
            while (got < want_n) {
                const u32 fc = __shfl_sync(FULLMASK, cf, cp & 31);
                const u32 sc = __shfl_sync(FULLMASK, cs_, cp & 31);
                const u32 ec = __shfl_sync(FULLMASK, ce_, cp & 31);
                const bool have_c = cp < mc;
                if (rt != NONE && (!have_c || rt < fc)) {
                    const u64 v = O.pse[rt];
                    if (lane == got) { of = rt; os = (u32)v; oe = (u32)(v >> 32); }
                    rt = ovf_extract(S, O, k, rt, broken);
                } else if (have_c) {
                    if (lane == got) { of = fc; os = sc; oe = ec; }
                    cp++;
                } else break;
                got++;
            }
            if (lane < got) S.dl[slot][lane] = make_uint4(of, os, oe, 0);
            if (lane == 0) { S.ptr[k] = p + cp; S.root[k] = rt; S.dn[slot] = got; }
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                const u32 pos = atomicAdd(&S.ctail, 1u);
                st_vol(&S.cq[pos & (CQ - 1)], slot | ((((pos / CQ) + 1) & 0xFFFFu) << 16));
            }
            __syncwarp();
        }
    }
    if (stats && lane == 0) {
        atomicAdd(&stats[10], nmsg);
        if (broken) stats[2] = 4;
    }
}

// ------------------------------------------------------------------ main side ----
// Everything below runs on one thread: plain shared-memory loads and stores, no warp collectives.
struct Main {
    Smem &S;
    u32 sw;            // first-level availability word
    int Mx;            // highest nonempty class (-1: none)
    u32 chead;         // completions consumed
    int NC, L;
    u64 n_wait = 0, n_req = 0, n_ins = 0, n_merge = 0, n_give = 0, n_arr = 0, n_pop = 0;
    long long t_wait = 0;
    bool broken = false;

    __device__ __forceinline__ u32 first_ge(u32 c) const {
        const u32 w = c >> 5;
        const u32 m = S.cw[w] & (0xFFFFFFFFu << (c & 31));
        if (m) return (w << 5) + __ffs(m) - 1;
        const u32 sm = (w >= 31) ? 0u : (sw & (0xFFFFFFFFu << (w + 1)));
        if (!sm) return NONE;
        const u32 w2 = __ffs(sm) - 1;
        return (w2 << 5) + __ffs(S.cw[w2]) - 1;
    }
    __device__ __forceinline__ void set_bit(u32 k) {
        const u32 w = k >> 5;
        S.cw[w] |= 1u << (k & 31);
        sw |= 1u << w;
        if ((int)k > Mx) Mx = (int)k;   // a remainder can land above a class that just emptied
    }
    __device__ __forceinline__ void clear_bit(u32 k) {
        const u32 w = k >> 5;
        const u32 v = S.cw[w] & ~(1u << (k & 31));
        S.cw[w] = v;
        if (!v) sw &= ~(1u << w);
        if ((int)k == Mx) {
            if (!sw) Mx = -1;
            else {
                const u32 ww = 31 - __clz(sw);
                const u32 cv = (ww == w) ? v : S.cw[ww];
                Mx = (int)(ww * 32 + 31 - __clz(cv));
            }
        }
    }

    __device__ __forceinline__ void post(u32 h, u32 type, u32 k, u32 y, u32 z, u32 w) {
        const u32 t = S.qt[h];
        if (t - S.qhc[h] >= (u32)QD) {
            u32 hh;
            long long spins = 0;
            while (t - (hh = ld_vol(&S.qhead[h])) >= (u32)QD) {
                if (++spins > (1ll << 26)) { broken = true; return; }
            }
            S.qhc[h] = hh;
        }
        const u32 lap = ((t / QD) + 1) & 0xFFFFFu;
        st_vol_v4(&S.q[h][t & (QD - 1)], k | (type << 10) | (lap << 12), y, z, w);
        S.qt[h] = t + 1;
    }
    // a member leaves the cached view of class k for O_k
    __device__ __forceinline__ void send_ins(u32 k, u32 meta, u32 f, u32 s, u32 e1) {
        n_ins++;
        post(k % NHELP, M_INS, k, f, s, e1);
        if ((meta >> 16) != NOSLOT && f < S.insmin[k]) S.insmin[k] = f;
    }
    // request the m smallest outside members of class k (false: no free slot)
    __device__ __forceinline__ bool post_req(u32 k) {
        const u32 sp = S.fsp;
        if (sp == 0) return false;
        const u32 slot = S.fstk[sp - 1];
        const u32 meta = S.meta[k];
        const u32 m = (u32)H - (meta & 0xFF);
        S.fsp = sp - 1;
        S.dk[slot] = k;
        S.insmin[k] = NONE;
        S.meta[k] = (meta & 0xFFFFu) | (slot << 16);
        n_req++;
        post(k % NHELP, M_REQ, k, m, slot, 0);
        return true;
    }
    // consume one completion if present; returns whether one was merged
    __device__ __forceinline__ bool poll() {
        const u32 v = ld_vol(&S.cq[chead & (CQ - 1)]);
        if ((v >> 16) != (((chead / CQ) + 1) & 0xFFFFu)) return false;
        chead++;
        merge(v & 0xFFFFu);
        return true;
    }
    __device__ __forceinline__ void merge(u32 slot) {
        n_merge++;
        const u32 k = S.dk[slot];
        const u32 nd = ld_vol(&S.dn[slot]);
        const u32 lim = S.insmin[k];
        const u32 meta = S.meta[k];
        const u32 n = meta & 0xFF, b = (meta >> 8) & 0xFF;
        u32 t = 0;
        for (; t < nd && n + t < (u32)H; t++) {
            const uint4 y = ld_vol_v4(&S.dl[slot][t]);
            if (y.x >= lim) break;
            S.rg[k * H + ((b + n + t) & (H - 1))] = y;
        }
        S.meta[k] = (n + t) | (b << 8) | (NOSLOT << 16);
        S.fstk[S.fsp] = slot;
        S.fsp = S.fsp + 1;
        // members beyond the ring's room or above a member sent to O_k after the REQ go back
        for (; t < nd; t++) {
            n_give++;
            const uint4 y = ld_vol_v4(&S.dl[slot][t]);
            post(k % NHELP, M_INS, k, y.x, y.y, y.z);
        }
    }
    // every remaining member of class k is outside: wait for the helper's delivery
    __device__ __forceinline__ u32 wait_ring(u32 k) {
        const long long t0 = clock64();
        n_wait++;
        long long spins = 0;
        u32 meta;
        while (((meta = S.meta[k]) & 0xFF) == 0) {
            if ((meta >> 16) == NOSLOT) {
                if (!post_req(k)) poll();
            } else if (!poll()) {
                if (++spins > (1ll << 26)) { broken = true; return meta; }
            }
        }
        t_wait += clock64() - t0;
        return meta;
    }
    // class k's head was consumed (carved to nothing or moved to another class)
    __device__ __forceinline__ void pop(u32 k, u32 cnt_before) {
        n_pop++;
        const u32 c = cnt_before - 1;
        if (c == 0) {
            S.hd[k].w = 0;
            clear_bit(k);
            return;
        }
        u32 meta = S.meta[k];
        if ((meta & 0xFF) == 0) {
            meta = wait_ring(k);
            if (broken) return;
        }
        const u32 n = meta & 0xFF, b = (meta >> 8) & 0xFF;
        uint4 e = S.rg[k * H + b];
        e.w = c;
        S.hd[k] = e;
        const u32 slot = meta >> 16;
        S.meta[k] = (n - 1) | (((b + 1) & (H - 1)) << 8) | (slot << 16);
        // outside after the pop = c - 1 - (n - 1)
        if (n - 1 < REQ_AT && slot == NOSLOT && c > n) post_req(k);
    }
    // a remainder piece f = [s, e1 + 1) joins class j
    __device__ __forceinline__ void arrive(u32 j, u32 f, u32 s, u32 e1) {
        n_arr++;
        const uint4 h = S.hd[j];
        const u32 meta = S.meta[j];
        const u32 c0 = h.w;
        if (c0 == 0) {
            S.hd[j] = make_uint4(f, s, e1, 1);
            set_bit(j);
            return;
        }
        u32 n = meta & 0xFF;
        const u32 b = (meta >> 8) & 0xFF;
        const u32 outside = c0 - 1 - n;
        uint4 *ring = &S.rg[j * H];
        if (f < h.x) {
            // the new piece is the head; the old head goes to the ring's front
            const u32 nb = (b - 1) & (H - 1);
            if (n == (u32)H) {           // the tail sits where the new front goes
                const uint4 t = ring[nb];
                send_ins(j, meta, t.x, t.y, t.z);
                n = H - 1;
            }
            ring[nb] = make_uint4(h.x, h.y, h.z, 0);
            S.hd[j] = make_uint4(f, s, e1, c0 + 1);
            S.meta[j] = (n + 1) | (nb << 8) | (meta & 0xFFFF0000u);
            return;
        }
        S.hd[j].w = c0 + 1;
        // the ring's entries (independent loads, issued together)
        uint4 x[H];
#pragma unroll
        for (int i = 0; i < H; i++) x[i] = ring[(b + i) & (H - 1)];
        u32 tail = 0;
#pragma unroll
        for (int i = 0; i < H; i++) if ((u32)i + 1 == n) tail = x[i].x;
        if (n == 0 || f > tail) {
            if (outside == 0 && n < (u32)H) {            // every member is cached: append
                ring[(b + n) & (H - 1)] = make_uint4(f, s, e1, 0);
                S.meta[j] = (n + 1) | (meta & 0xFFFFFF00u);
            } else {
                send_ins(j, meta, f, s, e1);
                if (n == 0 && (meta >> 16) == NOSLOT) post_req(j);
            }
            return;
        }
        // f lies inside the ring: sorted insertion (evicting the tail if the ring is full)
        if (n == (u32)H) {
            send_ins(j, meta, x[H - 1].x, x[H - 1].y, x[H - 1].z);
            n = H - 1;
        }
        u32 pos = 0;
#pragma unroll
        for (int i = 0; i < H; i++) pos += ((u32)i < n && x[i].x < f) ? 1u : 0u;
#pragma unroll
        for (int i = H - 2; i >= 0; i--)
            if ((u32)i >= pos && (u32)i < n) ring[(b + i + 1) & (H - 1)] = x[i];
        ring[(b + pos) & (H - 1)] = make_uint4(f, s, e1, 0);
        S.meta[j] = (n + 1) | (b << 8) | (S.meta[j] & 0xFFFF0000u);
    }
};

__global__ void __launch_bounds__(NWARP * 32, 1)
k_seq_engine(Csr csr, const u32 *__restrict__ off, u64 *__restrict__ fs, const u64 *__restrict__ R,
             const u32 *__restrict__ C, u64 n, u64 *__restrict__ out_u, u32 *bm, u64 w0, u64 w1, u64 w2,
             u64 *pse, u32 *slot_map, int NC, int L, u64 *stats, const u64 *n_in, const u32 *wild) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    if (n_in) n = *n_in;   // request count on the device (a hybrid heap's TLSF share)
    // wilderness split (engine_tlsf.cuh k_wild_setup): class Kw's single member is left out
    const u32 Kw = wild ? wild[0] : NONE;
    const bool wmode = Kw != NONE;
    const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // ---- init: class heads and rings from the CSR, FIFOs ----
    for (u32 k = tid; k < (u32)MAX_NC; k += blockDim.x) {
        u32 b = 0, e = 0;
        if ((int)k < NC) { b = off[k]; e = off[k + 1]; }
        if (k == Kw) b = e;
        const u32 cnt = e - b;
        const u32 hn = cnt > 0 ? min(cnt - 1, (u32)H) : 0u;
        if (cnt) S.hd[k] = make_uint4(csr.f[b], csr.s[b], csr.e[b], cnt);
        else S.hd[k] = make_uint4(0, 0, 0, 0);
        S.meta[k] = hn | (NOSLOT << 16);
        S.insmin[k] = NONE;
        S.ptr[k] = b + (cnt ? 1 + hn : 0);
        S.endp[k] = e;
        S.root[k] = NONE;
        S.slot[k] = NONE;
    }
    for (u32 x = tid; x < (u32)NC * H; x += blockDim.x) {
        const u32 k = x / H, j = x % H;
        u32 b = off[k], e = off[k + 1];
        if (k == Kw) b = e;
        if (b + 1 + j < e) S.rg[x] = make_uint4(csr.f[b + 1 + j], csr.s[b + 1 + j], csr.e[b + 1 + j], 0);
    }
    for (u32 x = tid; x < (u32)(NHELP * QD); x += blockDim.x) S.q[x / QD][x % QD] = make_uint4(0, 0, 0, 0);
    for (u32 x = tid; x < (u32)CQ; x += blockDim.x) S.cq[x] = 0;
    if (tid < (u32)NHELP) { S.qhead[tid] = 0; S.qt[tid] = 0; S.qhc[tid] = 0; }
    if (tid < (u32)NSLOT) S.fstk[tid] = tid;
    if (tid == 0) { S.fsp = NSLOT; S.ctail = 0; S.nslot = 0; S.abort_ = 0; S.rfill = 0; S.rcons = 0; }
    __syncthreads();
    if (warp == 0) {
        u32 swl = 0;
        for (int w = 0; w < 32; w++) {
            const int k = w * 32 + lane;
            const u32 bb = __ballot_sync(FULLMASK, k < NC && S.hd[k].w > 0);
            if (lane == 0) S.cw[w] = bb;
            if (bb) swl |= 1u << w;
        }
        __syncwarp();
        if (lane != 0) return;           // the chain runs on one thread; the other lanes leave
        {
            Main M{S, swl, -1, 0u, NC, L};
            if (swl) {
                const u32 ww = 31 - __clz(swl);
                M.Mx = (int)(ww * 32 + 31 - __clz(S.cw[ww]));
            }
            const long long t_begin = clock64();
            u64 avail = 0;                    // requests the loader has staged
            long long tt[6] = {0, 0, 0, 0, 0, 0};
#if SEQ_TIMING
#define SQT(j) { const long long _t = clock64(); tt[j] += _t - t_last; t_last = _t; }
            long long t_last = clock64();
#else
#define SQT(j)
#endif
            for (u64 i = 0; i < n && !M.broken; i++) {
                if (i == avail) {
                    long long spins = 0;
                    u32 fl;
                    while ((fl = ld_vol(&S.rfill)) == (u32)i)
                        if (++spins > (1ll << 28)) { M.broken = true; break; }
                    if (M.broken) break;
                    avail = i + (u32)(fl - (u32)i);
                    st_vol(&S.rcons, (u32)i);
                } else if ((i & 255) == 0) {
                    st_vol(&S.rcons, (u32)i);
                }
                SQT(0)
                const u32 r = S.rr[i & (RB - 1)], c = S.rc[i & (RB - 1)];
                u64 v;
                if (r == 0 || c >= (u32)NC) v = HEAP_NULL_U64;
                else if ((int)c > M.Mx) v = wmode ? WILD : HEAP_NULL_U64;   // the highest class only falls
                else {
                    const u32 k = M.first_ge(c);
                    if (k == NONE) v = wmode ? WILD : HEAP_NULL_U64;
                    else {
                        const uint4 h = S.hd[k];
                        v = h.y;
                        const u64 s2 = (u64)h.y + r;
                        fs[h.x] = s2;
                        const u64 z = (u64)h.z + 1 - s2;
                        const u32 nk = z ? cls_insert(z, L) : NONE;
                        SQT(1)
                        if (nk == k) S.hd[k].y = (u32)s2;
                        else {
                            M.pop(k, h.w);
                            SQT(2)
                            if (nk != NONE) M.arrive(nk, h.x, (u32)s2, h.z);
                            SQT(3)
                        }
                    }
                }
                out_u[i] = v;
                SQT(4)
                M.poll();
                SQT(5)
            }
#undef SQT
            st_vol(&S.rcons, (u32)n);
            // stop the helpers (after every message already posted)
            for (u32 hh = 0; hh < (u32)NHELP && !M.broken; hh++) M.post(hh, M_STOP, 0, 0, 0, 0);
            if (M.broken) st_vol(&S.abort_, 1u);
            if (stats) {
                stats[0] += M.n_pop; stats[1] += M.n_arr; stats[3] += M.n_req; stats[4] += M.n_ins;
                stats[5] += clock64() - t_begin; stats[6] += M.t_wait; stats[7] += M.n_wait; stats[8] += M.n_merge;
                stats[9] += M.n_give;
                stats[11] += tt[0]; stats[12] += tt[1]; stats[13] += tt[2]; stats[15] += tt[3];   // [14]: k_wild_setup
                if (M.broken) stats[2] = 5;
            }
        }
    } else if (warp == 1) {
        // ---- loader: requests into the ring, LB per round (LB / 32 independent loads per lane), at
        //      most RB - LB ahead of main ----
        constexpr int LB = 512;
        for (u64 base = 0; base < n; base += LB) {
            long long spins = 0;
            bool quit = false;
            while ((u32)(base + LB) - ld_vol(&S.rcons) > (u32)(RB - LB)) {
                if (ld_vol(&S.abort_) || ++spins > (1ll << 28)) { quit = true; break; }
                __nanosleep(32);
            }
            if (quit) break;
            u64 rv[LB / 32];
            u32 cv[LB / 32];
#pragma unroll
            for (int j = 0; j < LB / 32; j++) {
                const u64 i = base + j * 32 + lane;
                rv[j] = i < n ? R[i] : 0ull;
                cv[j] = i < n ? C[i] : 0u;
            }
#pragma unroll
            for (int j = 0; j < LB / 32; j++) {
                const u64 i = base + j * 32 + lane;
                S.rr[i & (RB - 1)] = rv[j] > 0xFFFFFFFFull ? 0u : (u32)rv[j];   // > 2^32 - 1 units never fit
                S.rc[i & (RB - 1)] = cv[j];
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                st_vol(&S.rfill, (u32)(base + LB < n ? base + LB : n));
            }
            __syncwarp();
        }
    } else if ((warp & 3) != 0) {
        helper_loop<Smem, NHELP>(S, warp - 2 - (warp >> 2), csr, Ovf{bm, bm + (u64)NC * w0, bm + (u64)NC * (w0 + w1), w0, w1, w2, pse},
                    NC, slot_map, stats);   // warps 2,3,5,6,7,9,10,11,13,14,15 -> helpers 0..10
    }
    // (no final barrier: main's lanes 1..31 left early; each helper published its slot_map entries)
}

}  // namespace tlsfs
