// engine_tlsf_h.cuh — the warp-chunk TLSF / SEGFIT engine of engine_tlsf.cuh with its global-memory
// work moved onto helper warps (engine_seq.cuh's helper protocol).
//
// Semantics and the chunk algorithm (speculation, light pre-rounds, patterns A/B and the replay,
// dirty check, commit of the clean prefix) are those of tlsfw::k_engine<false>; only the class
// state's slow half changes.  Per class, warp 0 keeps the sorted head cache of up to H smallest
// members in shared memory (as before); every other member ("outside": the untouched batch-start
// CSR suffix plus the overflow set O_k, a three-level bitmap over f in global memory) belongs to
// helper warp k mod NHELP:
//   * a cache that falls below REFILL_AT members while members remain outside posts REQ(k, m); the
//     helper delivers the m smallest outside members into a delivery slot, and warp 0 appends them
//     (keeping only those below any member sent outside since the REQ) at the top of a chunk;
//   * a remainder that does not belong in the cache, or a member evicted from a full cache, is
//     posted as INS(k, piece).
// So the engine warp never waits on global memory except when a chunk's first request finds its
// class's cache empty (it then waits for that class's delivery).  Warps 4, 8, 12 idle so that no
// helper shares warp 0's scheduler (warp w runs on sub-partition w mod 4).
// ABLATION (HEAP_ENGINE=helpers): exact (the GPU parity suite passes) but not faster.  Measured on
// B200, config 5 batch 5 (tools/seq_probe.py): class updates 2.6k -> 1.3k cycles per chunk, but the
// messaging (lane-parallel FIFO posts, delivery merges at the top of every chunk) costs ~1.6k and the
// arrivals phase +0.35k, and an asynchronous refill delivers fewer members per request (112k REQs
// against 48k synchronous refills per batch): 193.5 ms against 174.9 ms for engine_tlsf.cuh.  The
// global accesses it removes are mostly L1/L2 hits, about as cheap as the shared-memory handshake.
#pragma once
#include "common.cuh"
#include "engine_tlsf.cuh"
#include "engine_seq.cuh"

namespace tlsfh {

using tlsfw::H;
using tlsfw::MAX_NC;
using tlsfw::RB;
using tlsfw::NONE;
using tlsfw::SAME;
using tlsfw::F_OK;
using tlsfw::F_OVER;
using tlsfw::F_MISS;
using tlsfw::NIL64;
using tlsfw::WILD;
using tlsfs::QD;
using tlsfs::NSLOT;
using tlsfs::CQ;
using tlsfs::NOSLOT;
using tlsfs::M_INS;
using tlsfs::M_REQ;
using tlsfs::M_STOP;
using tlsfs::ld_vol;
using tlsfs::ld_vol_v4;
using tlsfs::st_vol;
using tlsfs::st_vol_v4;

constexpr int NWARP = 16;
constexpr int NHELP = 12;        // warps 1, 2, 3, 5, 6, 7, 9, 10, 11, 13, 14, 15
constexpr int REFILL_AT = tlsfw::REFILL_AT;
constexpr int NINS = 96;         // INS messages one chunk can produce (<= 32 arrivals + 32 evictions)
static_assert(H == 8, "delivery slots hold H = 8 members");

struct Smem {
    tlsfw::Smem E;                   // the engine warp's state (head caches, bitmaps, staging)
    // helper-owned class state (tlsfs::helper_loop)
    u32 ptr[MAX_NC], endp[MAX_NC], root[MAX_NC], slot[MAX_NC];
    u32 nslot;
    // warp 0 -> helper FIFOs, delivery slots, completion ring (tlsfs protocol)
    uint4 q[NHELP][QD];
    u32 qhead[NHELP];
    u32 qt[NHELP], qhc[NHELP];
    uint4 dl[NSLOT][H];
    u32 dn[NSLOT], dk[NSLOT];
    u32 fstk[NSLOT];
    u32 fsp;
    u32 ctail;
    u32 cq[CQ];
    u32 abort_;
    u32 rq[MAX_NC];                  // outstanding delivery slot of class k (NOSLOT: none)
    u32 insmin[MAX_NC];              // smallest f sent outside since that REQ
    uint4 ins[NINS];                 // this chunk's INS messages {k, f, start, end-1}
    u32 nins;
};

// ---- warp-uniform messaging (every lane calls with the same arguments; lane 0 writes) ----
__device__ __forceinline__ bool post(Smem &S, u32 h, u32 type, u32 k, u32 y, u32 z, u32 w) {
    const u32 t = S.qt[h];
    if (t - S.qhc[h] >= (u32)QD) {
        u32 hh;
        long long spins = 0;
        while (t - (hh = ld_vol(&S.qhead[h])) >= (u32)QD)
            if (++spins > (1ll << 26)) return false;
        if (lane_id() == 0) S.qhc[h] = hh;
    }
    const u32 lap = ((t / QD) + 1) & 0xFFFFFu;
    if (lane_id() == 0) {
        st_vol_v4(&S.q[h][t & (QD - 1)], k | (type << 10) | (lap << 12), y, z, w);
        S.qt[h] = t + 1;
    }
    __syncwarp();
    return true;
}

// lane-parallel: every lane with `valid` posts one message {k | type, y, z, w} to helper k % NHELP;
// lanes sharing a helper take consecutive FIFO positions in lane order (per-class message order is
// the caller's lane order)
__device__ __forceinline__ bool post_lanes(Smem &S, bool valid, u32 type, u32 k, u32 y, u32 z, u32 w) {
    const u32 lane = lane_id();
    const u32 h = valid ? k % NHELP : 0x40000000u | lane;
    const u32 peers = __match_any_sync(FULLMASK, h);
    const u32 rank = __popc(peers & lanemask_lt()), cnt = __popc(peers);
    bool ok = true;
    if (valid) {
        const u32 t = S.qt[h];
        if (t + cnt - S.qhc[h] > (u32)QD) {
            u32 hh;
            long long spins = 0;
            while (t + cnt - (hh = ld_vol(&S.qhead[h])) > (u32)QD)
                if (++spins > (1ll << 26)) { ok = false; break; }
            if (rank == 0) S.qhc[h] = hh;
        }
        const u32 pos = t + rank;
        const u32 lap = ((pos / QD) + 1) & 0xFFFFFu;
        st_vol_v4(&S.q[h][pos & (QD - 1)], k | (type << 10) | (lap << 12), y, z, w);
        __syncwarp(peers);
        if (rank == 0) S.qt[h] = t + cnt;
    }
    __syncwarp();
    return __all_sync(FULLMASK, ok);
}

// request the smallest outside members of class k into a free slot (false: none free)
__device__ __forceinline__ bool post_req(Smem &S, u32 k, bool &broken) {
    const u32 sp = S.fsp;
    if (sp == 0) return false;
    const u32 slot = S.fstk[sp - 1];
    const u32 m = (u32)H - S.E.hn[k];
    if (lane_id() == 0) {
        S.fsp = sp - 1;
        S.dk[slot] = k;
        S.rq[k] = slot;
        S.insmin[k] = NONE;
    }
    __syncwarp();
    if (!post(S, k % NHELP, M_REQ, k, m, slot, 0)) broken = true;
    return true;
}

// append a delivery to its class's cache (members below any member sent outside since the REQ and
// within the cache's room); the rest goes back outside
__device__ void merge(Smem &S, u32 slot, bool &broken) {
    const u32 lane = lane_id();
    const u32 k = S.dk[slot];
    const u32 nd = ld_vol(&S.dn[slot]);
    const u32 lim = S.insmin[k];
    const u32 n = S.E.hn[k], b = S.E.hb[k];
    uint4 y = make_uint4(NONE, 0, 0, 0);
    if (lane < nd) y = ld_vol_v4(&S.dl[slot][lane]);
    u32 take = __popc(__ballot_sync(FULLMASK, lane < nd && y.x < lim));
    if (take > (u32)H - n) take = (u32)H - n;
    if (lane < take) {
        const u32 ix = k * H + ((b + n + lane) & (H - 1));
        S.E.hf[ix] = y.x; S.E.hs[ix] = y.y; S.E.he[ix] = y.z;
    }
    if (lane == 0) {
        S.E.hn[k] = (unsigned char)(n + take);
        S.rq[k] = NOSLOT;
        S.fstk[S.fsp] = slot;
        S.fsp = S.fsp + 1;
    }
    __syncwarp();
    for (u32 t = take; t < nd; t++) {
        const u32 gf = __shfl_sync(FULLMASK, y.x, t), gs = __shfl_sync(FULLMASK, y.y, t),
                  ge = __shfl_sync(FULLMASK, y.z, t);
        if (!post(S, k % NHELP, M_INS, k, gf, gs, ge)) broken = true;
    }
}

// merge every completed delivery, one completion per lane (their classes differ: one outstanding
// REQ per class); members given back are queued in S.ins.  Returns how many were merged.
__device__ __forceinline__ u32 poll_all(Smem &S, u32 &chead, bool &broken) {
    const u32 lane = lane_id();
    const u32 p = chead + lane;
    const u32 v = ld_vol(&S.cq[p & (CQ - 1)]);
    const bool ready = (v >> 16) == (((p / CQ) + 1) & 0xFFFFu);
    const u32 rm = __ballot_sync(FULLMASK, ready);
    const u32 got = (~rm) ? (u32)(__ffs(~rm) - 1) : 32u;      // a prefix of the ring
    if (!got) return 0;
    const bool mine = lane < got;
    if (mine) {
        const u32 slot = v & 0xFFFFu;
        const u32 k = S.dk[slot];
        const u32 nd = ld_vol(&S.dn[slot]);
        const u32 lim = S.insmin[k];
        const u32 n = S.E.hn[k], b = S.E.hb[k];
        u32 t = 0;
        for (; t < nd && n + t < (u32)H; t++) {
            const uint4 y = ld_vol_v4(&S.dl[slot][t]);
            if (y.x >= lim) break;
            const u32 ix = k * H + ((b + n + t) & (H - 1));
            S.E.hf[ix] = y.x; S.E.hs[ix] = y.y; S.E.he[ix] = y.z;
        }
        S.E.hn[k] = (unsigned char)(n + t);
        S.rq[k] = NOSLOT;
        for (; t < nd; t++) {      // beyond the room, or above a member sent outside since the REQ
            const uint4 y = ld_vol_v4(&S.dl[slot][t]);
            const u32 q = atomicAdd(&S.nins, 1u);
            S.ins[q] = make_uint4(k, y.x, y.y, y.z);
        }
        S.fstk[S.fsp + lane] = slot;
    }
    __syncwarp();
    if (lane == 0) S.fsp = S.fsp + got;
    chead += got;
    __syncwarp();
    return got;
}

// post the queued INS messages (S.ins, 32 per round) and note members sent outside while a REQ is
// outstanding (insmin)
__device__ __forceinline__ u32 flush_ins(Smem &S, bool &broken) {
    const u32 lane = lane_id();
    const u32 ni = S.nins;
    for (u32 x0 = 0; x0 < ni; x0 += 32) {
        const bool v = x0 + lane < ni;
        uint4 m = make_uint4(0, 0, 0, 0);
        if (v) m = S.ins[x0 + lane];
        if (!post_lanes(S, v, M_INS, m.x, m.y, m.z, m.w)) broken = true;
        if (v && S.rq[m.x] != NOSLOT) atomicMin(&S.insmin[m.x], m.y);
    }
    __syncwarp();
    if (lane == 0) S.nins = 0;
    __syncwarp();
    return ni;
}

// a remainder piece f = [s, e1 + 1) joins class k (one lane per class; INS messages are queued in
// S.ins and posted by the whole warp after the phase)
__device__ void arrive_h(Smem &S, u32 k, u32 f, u32 s, u32 e1) {
    tlsfw::Smem &E = S.E;
    const u32 before = E.cnt[k]++;
    if (before == 0) tlsfw::set_bit(E, k);
    u32 n = E.hn[k];
    u32 *hf = &E.hf[k * H], *hs = &E.hs[k * H], *he = &E.he[k * H];
    const u32 b = E.hb[k];
#define RI(j) ((b + (j)) & (H - 1))
    // the cache must stay "the n smallest members": f enters it if it is below the cache's tail,
    // or if every member is cached (nothing outside could be smaller)
    if ((n > 0 && f < hf[RI(n - 1)]) || (n < (u32)H && before == n)) {
        u32 j;
        if (n == (u32)H) {      // evict the largest cached member: it goes outside
            const u32 p = atomicAdd(&S.nins, 1u);
            S.ins[p] = make_uint4(k, hf[RI(H - 1)], hs[RI(H - 1)], he[RI(H - 1)]);
            j = H - 1;
        } else {
            j = n;
            E.hn[k] = (unsigned char)(n + 1);
        }
        while (j > 0 && hf[RI(j - 1)] > f) {
            hf[RI(j)] = hf[RI(j - 1)]; hs[RI(j)] = hs[RI(j - 1)]; he[RI(j)] = he[RI(j - 1)];
            j--;
        }
        hf[RI(j)] = f; hs[RI(j)] = s; he[RI(j)] = e1;
    } else {
        const u32 p = atomicAdd(&S.nins, 1u);
        S.ins[p] = make_uint4(k, f, s, e1);
    }
#undef RI
}

__global__ void __launch_bounds__(NWARP * 32, 1)
k_engine_h(tlsfw::Csr csr, const u32 *__restrict__ off, u64 *__restrict__ fs, const u64 *__restrict__ R,
           const u32 *__restrict__ C, u64 n, u64 *__restrict__ out_u, u32 *bm, u64 w0, u64 w1, u64 w2, u64 *pse,
           u32 *slot_map, int NC, int L, u64 *stats, const u64 *n_in, const u32 *wild) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    tlsfw::Smem &E = S.E;
    if (n_in) n = *n_in;   // request count on the device (a hybrid heap's TLSF share)
    const u32 Kw = wild ? wild[0] : NONE;
    const bool wmode = Kw != NONE;
    const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // ---- init (whole CTA): caches = each class's H smallest batch-start members; the rest of the
    //      CSR range is outside (helper-owned) ----
    for (u32 k = tid; k < (u32)MAX_NC; k += blockDim.x) {
        u32 b = 0, e = 0;
        if ((int)k < NC) { b = off[k]; e = off[k + 1]; }
        if (k == Kw) b = e;     // the wilderness is not a member of the class state
        const u32 cnt = e - b, hn = min(cnt, (u32)H);
        E.cnt[k] = cnt;
        E.hn[k] = (unsigned char)hn;
        E.hb[k] = 0;
        S.ptr[k] = b + hn;
        S.endp[k] = e;
        S.root[k] = NONE;
        S.slot[k] = NONE;
        S.rq[k] = NOSLOT;
        S.insmin[k] = NONE;
    }
    for (u32 x = tid; x < (u32)NC * H; x += blockDim.x) {
        const u32 k = x / H, j = x % H;
        u32 b = off[k], e = off[k + 1];
        if (k == Kw) b = e;
        if (b + j < e) { E.hf[x] = csr.f[b + j]; E.hs[x] = csr.s[b + j]; E.he[x] = csr.e[b + j]; }
    }
    for (u32 x = tid; x < (u32)(NHELP * QD); x += blockDim.x) S.q[x / QD][x % QD] = make_uint4(0, 0, 0, 0);
    for (u32 x = tid; x < (u32)CQ; x += blockDim.x) S.cq[x] = 0;
    if (tid < (u32)NHELP) { S.qhead[tid] = 0; S.qt[tid] = 0; S.qhc[tid] = 0; }
    if (tid < (u32)NSLOT) S.fstk[tid] = tid;
    if (tid == 0) { S.fsp = NSLOT; S.ctail = 0; S.nslot = 0; S.abort_ = 0; S.nins = 0; }
    __syncthreads();
    if (warp != 0) {
        if ((warp & 3) != 0)
            tlsfs::helper_loop<Smem, NHELP>(S, warp - 1 - (warp >> 2), tlsfs::Csr{csr.f, csr.s, csr.e},
                                            tlsfs::Ovf{bm, bm + (u64)NC * w0, bm + (u64)NC * (w0 + w1), w0, w1, w2, pse},
                                            NC, slot_map, stats);
        return;
    }
    // ---------------------------------------------------------------- engine warp ----
    {
        u32 swl = 0;
        for (int w = 0; w < 32; w++) {
            int k = w * 32 + lane;
            u32 b = __ballot_sync(FULLMASK, k < NC && E.cnt[k] > 0);
            if (lane == 0) E.cw[w] = b;
            if (b) swl |= 1u << w;
        }
        if (lane == 0) E.sw = swl;
    }
    __syncwarp();
    bool broken = false;
    u32 chead = 0;
    u64 rb_base = 0, rb_end = 0;
    u32 keep = 0;
    u64 resume = 0;
    u64 n_iter = 0, n_retarget = 0, n_rounds = 0, n_qsteps = 0, n_wait = 0, n_req = 0, n_ins = 0;
    long long t_spec = 0, t_dirty = 0, t_cls = 0, t_arr = 0, t_store = 0, t_wait = 0, t0;
    u64 pos = 0;
    while (pos < n) {
        n_iter++;
        if (broken || n_iter > 4 * n + 64) {
            if (lane == 0 && stats) stats[2] = broken ? 4 : 3;
            break;
        }
        if (poll_all(S, chead, broken) && S.nins) flush_ins(S, broken);
        const u32 sw = E.sw;
        u64 i = NIL64, ri = 0, scan_end = 0;
        u32 ci = NONE, limit = 0;
        bool act = false;
        if (!wmode) {
            if (pos + 32 > rb_end) {
                rb_base = pos;
                rb_end = pos + RB < n ? pos + RB : n;
                for (u64 j = lane; j < rb_end - rb_base; j += 32) {
                    E.rbuf[j] = R[rb_base + j];
                    E.cbuf[j] = C[rb_base + j];
                }
                __syncwarp();
            }
            i = pos + lane;
            act = i < n;
            ri = act ? E.rbuf[i - rb_base] : 0;
            ci = act ? E.cbuf[i - rb_base] : NONE;
            limit = (n - pos) < 32 ? (u32)(n - pos) : 32u;
        } else {
            int Mx = -1;
            if (sw) {
                const u32 w = 31 - __clz(sw);
                Mx = (int)(w * 32 + 31 - __clz(E.cw[w]));
            }
            u32 ncand = keep;
            u64 sc = keep ? resume : pos;
            while (ncand < 32 && sc < n) {
                if (sc < rb_base || sc + 32 > rb_end) {
                    __syncwarp();
                    rb_base = sc;
                    rb_end = sc + RB < n ? sc + RB : n;
                    for (u64 j = lane; j < rb_end - rb_base; j += 32) {
                        E.rbuf[j] = R[rb_base + j];
                        E.cbuf[j] = C[rb_base + j];
                    }
                    __syncwarp();
                }
                const u64 j = sc + lane;
                const bool v = j < n;
                const u64 rj = v ? E.rbuf[j - rb_base] : 0;
                const u32 cj = v ? E.cbuf[j - rb_base] : NONE;
                const bool cand = v && rj != 0 && (int)cj <= Mx;
                const u32 cmask = __ballot_sync(FULLMASK, cand);
                const u32 nc = __popc(cmask);
                const u32 take = min(nc, 32u - ncand);
                const u32 rk = __popc(cmask & lanemask_lt());
                if (cand && rk < take) { E.ch_i[ncand + rk] = j; E.ch_r[ncand + rk] = rj; E.ch_c[ncand + rk] = cj; }
                u64 nsc = sc + 32 < n ? sc + 32 : n;
                const u32 firstout = __ballot_sync(FULLMASK, cand && rk == take);
                if (firstout) nsc = sc + __ffs(firstout) - 1;
                if (v && !cand && j < nsc) out_u[j] = rj != 0 ? WILD : HEAP_NULL_U64;
                ncand += take;
                sc = nsc;
            }
            __syncwarp();
            if (ncand == 0) { pos = sc; continue; }
            act = lane < ncand;
            if (act) { i = E.ch_i[lane]; ri = E.ch_r[lane]; ci = E.ch_c[lane]; }
            limit = ncand;
            scan_end = sc;
        }
        __syncwarp();
        E.ch_r[lane] = ri;
        __syncwarp();
        t0 = ENG_CLK();
        const bool fail0 = act && (ri == 0 || ci >= (u32)NC);
        u32 k = (act && !fail0) ? tlsfw::first_ge(E, sw, ci, NC) : NONE;
        // light pre-rounds (count model), as in tlsfw::k_engine
        const u32 k0 = k;
        u32 pm_fin = 0;
        bool have_pm = false;
#pragma unroll 1
        for (int it = 0; it < LIGHT_ROUNDS; it++) {
            const bool pl = act && k != NONE;
            const u32 ck = pl ? E.cnt[k] : 0u;
            const u32 pm = __match_any_sync(FULLMASK, pl ? k : (0x40000000u | lane));
            const bool ov = pl && (u32)__popc(pm & lanemask_lt()) >= ck;
            if (!__any_sync(FULLMASK, ov)) { pm_fin = pm; have_pm = true; break; }
            if (ov) k = tlsfw::first_ge(E, sw, k + 1, NC);
        }
        const u32 kpre = k;
        u32 peers = 0, rank = 0, flag = F_OK, myf = 0, mynk = NONE, mye = 0;
        u64 mys = 0;
        for (u32 round = 0;; round++) {
            n_rounds++;
            if (round > (u32)NC + 2) {
                if (lane == 0 && stats) stats[2] = 2;
                broken = true;
                break;
            }
            const bool part = act && k != NONE;
            peers = (round == 0 && have_pm) ? pm_fin : __match_any_sync(FULLMASK, part ? k : (0x40000000u | lane));
            rank = __popc(peers & lanemask_lt());
            const u32 leader = __ffs(peers) - 1;
            const u32 npeer = __popc(peers);
            const u32 nh = part ? E.hn[k] : 0, nc = part ? E.cnt[k] : 0;
            const u32 hb = part ? E.hb[k] : 0;
            const u32 slotA = k * H + ((hb + rank) & (H - 1)), slot0 = k * H + hb;
            const bool hasA = part && rank < nh;
            u32 fA = 0, nkA = NONE;
            u64 sA = 0;
            if (hasA) {
                fA = E.hf[slotA];
                sA = E.hs[slotA];
                const u64 zA = (u64)E.he[slotA] + 1 - sA - ri;
                nkA = zA ? cls_insert(zA, L) : NONE;
            }
            const bool okA = (__ballot_sync(FULLMASK, hasA && nkA == k && rank + 1 < npeer) & peers) == 0;
            bool okB = false, seq = false;
            if (__all_sync(FULLMASK, !part || okA)) {
                if (part) {
                    if (hasA) { flag = F_OK; myf = fA; mys = sA; mynk = (nkA == k) ? SAME : nkA; mye = E.he[slotA]; }
                    else flag = (rank < nc) ? F_MISS : F_OVER;
                }
            } else {
                if (part) E.lor[leader * 32 + rank] = lane;
                __syncwarp();
                u64 incl = part ? ri : 0;
                const u32 maxpeer = __reduce_max_sync(FULLMASK, (part && !okA) ? npeer : 0u);
                for (u32 st = 1; st < maxpeer; st <<= 1) {
                    const u32 src = (part && rank >= st) ? E.lor[leader * 32 + rank - st] : lane;
                    const u64 t = __shfl_sync(FULLMASK, incl, src);
                    if (part && rank >= st) incl += t;
                }
                const u64 P = incl - (part ? ri : 0);
                u64 s0 = 0, z0 = 0;
                u32 f0 = 0;
                if (part && nh) {
                    f0 = E.hf[slot0];
                    s0 = E.hs[slot0];
                    z0 = (u64)E.he[slot0] + 1 - s0;
                }
                const bool covB = part && nh && (rank == 0 || (P < z0 && z0 - P >= cls_lo(k, L)));
                const u32 uncov = __ballot_sync(FULLMASK, part && !covB);
                okB = !okA && (uncov & peers) == 0;
                if (part && okA) {
                    if (hasA) { flag = F_OK; myf = fA; mys = sA; mynk = (nkA == k) ? SAME : nkA; mye = E.he[slotA]; }
                    else flag = (rank < nc) ? F_MISS : F_OVER;
                } else if (part && okB) {
                    flag = F_OK; myf = f0; mys = s0 + P; mye = E.he[slot0];
                    const u64 z = z0 - P - ri;
                    const u32 nk = z ? cls_insert(z, L) : NONE;
                    mynk = (nk == k) ? SAME : nk;
                }
                seq = part && !okA && !okB;
                if (seq && rank == 0) {
                    n_qsteps += npeer;
                    u32 b = 0, curf = 0;
                    u64 cur_s = 0, cur_e = 0;
                    bool need = true;
                    u32 q = 0;
                    for (; q < npeer; q++) {
                        const u32 lq = E.lor[lane * 32 + q];
                        if (need) {
                            if (b >= nh) break;
                            const u32 sl = k * H + ((hb + b) & (H - 1));
                            curf = E.hf[sl];
                            cur_s = E.hs[sl];
                            cur_e = (u64)E.he[sl] + 1;
                            need = false;
                        }
                        const u64 rq = E.ch_r[lq];
                        E.res_flag[lq] = F_OK;
                        E.res_f[lq] = curf;
                        E.res_s[lq] = cur_s;
                        E.res_e[lq] = (u32)(cur_e - 1);
                        cur_s += rq;
                        const u64 z = cur_e - cur_s;
                        const u32 nk = z ? cls_insert(z, L) : NONE;
                        if (nk == k) E.res_nk[lq] = SAME;
                        else { E.res_nk[lq] = nk; b++; need = true; }
                    }
                    const u32 fl = (b < nc) ? F_MISS : F_OVER;
                    for (; q < npeer; q++) E.res_flag[E.lor[lane * 32 + q]] = fl;
                }
                __syncwarp();
                if (seq) {
                    flag = E.res_flag[lane];
                    myf = E.res_f[lane];
                    mys = E.res_s[lane];
                    mynk = E.res_nk[lane];
                    mye = E.res_e[lane];
                }
                __syncwarp();
            }
            const bool over = part && flag == F_OVER;
            if (!__any_sync(FULLMASK, over)) break;
            if (over) { k = tlsfw::first_ge(E, sw, k + 1, NC); flag = F_OK; n_retarget++; }
        }
        if (broken) break;
        if (act && k != NONE) { E.res_f[lane] = myf; E.res_s[lane] = mys; E.res_e[lane] = mye; }
        __syncwarp();
        t_spec += ENG_CLK() - t0;
        t0 = ENG_CLK();
        // ---- dirty requests: remainders dropped earlier in the chunk, cache misses ----
        const bool part = act && k != NONE;
        const u64 key = part ? (((u64)k << 32) | myf) : ~0ull;
        bool bad = part && flag == F_MISS;
        const bool dropper = part && flag == F_OK && mynk != SAME && mynk != NONE;
        u32 dm = __ballot_sync(FULLMASK, dropper);
        u32 samecls = 0;
        while (dm) {
            const u32 d = __ffs(dm) - 1;
            dm &= dm - 1;
            const u32 dk = __shfl_sync(FULLMASK, mynk, d);
            const u32 dfb = __shfl_sync(FULLMASK, myf, d);
            if (act && !fail0 && lane > d && ci <= dk && ((((u64)dk) << 32) | dfb) < key) bad = true;
            if (dropper && dk == mynk) samecls |= 1u << d;
        }
        if (__any_sync(FULLMASK, act && kpre != k0)) {
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
        t_dirty += ENG_CLK() - t0;
        if (commit == 0) {
            // the chunk's first request found its class's cache empty while members remain outside:
            // wait for that class's delivery, then retry the same candidates
            const u32 kw = __shfl_sync(FULLMASK, k, 0);
            if (kw == NONE || E.hn[kw] != 0) { broken = true; break; }   // impossible: never hang
            const long long tw = ENG_CLK();
            n_wait++;
            long long spins = 0;
            while (E.hn[kw] == 0 && !broken) {
                if (S.rq[kw] == NOSLOT) {
                    if (post_req(S, kw, broken)) n_req++;
                    else if (poll_all(S, chead, broken)) flush_ins(S, broken);
                } else if (poll_all(S, chead, broken)) {
                    if (S.nins) flush_ins(S, broken);
                } else if (++spins > (1ll << 26)) broken = true;
            }
            t_wait += ENG_CLK() - tw;
            if (wmode) { keep = limit; resume = scan_end; }
            __syncwarp();
            continue;
        }
        t0 = ENG_CLK();
        const bool cm = act && lane < commit;
        // ---- commit: results and piece starts ----
        const u32 later = (lane < 31) ? (peers & (0xFFFFFFFEu << lane)) : 0u;
        const u32 nxt = later ? (u32)(__ffs(later) - 1) : NONE;
        const bool last_on_block = mynk != SAME || nxt >= commit;
        if (cm) {
            if (!part) out_u[i] = (wmode && ri != 0) ? WILD : HEAP_NULL_U64;
            else {
                out_u[i] = mys;
                if (last_on_block) fs[myf] = mys + ri;
            }
        }
        // ---- class updates by group leaders: blocks that left the class; head carve ----
        __syncwarp();
        t_store += ENG_CLK() - t0;
        const u32 leftm = __ballot_sync(FULLMASK, cm && part && mynk != SAME);
        const u32 staym = __ballot_sync(FULLMASK, cm && part && mynk == SAME && last_on_block);
        bool want_req = false;
        if (cm && part && rank == 0) {
            const u32 left = __popc(leftm & peers);
            const u32 st = staym & peers;
            const u32 b = E.hb[k];
            if (st) {   // the carved block is the head now, with its new start
                const u32 d = __ffs(st) - 1;
                const u32 sl = k * H + ((b + left) & (H - 1));
                E.hs[sl] = (u32)(E.res_s[d] + E.ch_r[d]);
            }
            if (left) {
                E.hb[k] = (unsigned char)((b + left) & (H - 1));
                E.hn[k] = (unsigned char)(E.hn[k] - left);
                E.cnt[k] -= left;
                if (E.cnt[k] == 0) tlsfw::clear_bit(E, k);
                // refill asynchronously: the helper owning k delivers more members
                want_req = E.hn[k] < (u32)REFILL_AT && E.cnt[k] > E.hn[k] && S.rq[k] == NOSLOT;
            }
        }
        __syncwarp();
        {
            // one REQ per leader that wants one (distinct classes), slots from the free stack
            const u32 rm = __ballot_sync(FULLMASK, want_req);
            if (rm) {
                const u32 avail = S.fsp;
                const u32 rk = __popc(rm & lanemask_lt());
                const bool go = want_req && rk < avail;
                u32 slot = 0, m = 0;
                if (go) {
                    slot = S.fstk[avail - 1 - rk];
                    m = (u32)H - E.hn[k];
                    S.dk[slot] = k;
                    S.rq[k] = slot;
                    S.insmin[k] = NONE;
                }
                const u32 ng = __popc(__ballot_sync(FULLMASK, go));
                __syncwarp();
                if (lane == 0) S.fsp = avail - ng;
                if (!post_lanes(S, go, M_REQ, k, m, slot, 0)) broken = true;
                n_req += ng;
            }
        }
        t_cls += ENG_CLK() - t0;
        t0 = ENG_CLK();
        // ---- remainders join their new classes (grouped by class, time order) ----
        const bool cdrop = cm && dropper;
        const u32 g = samecls & (commit >= 32 ? FULLMASK : ((1u << commit) - 1u));
        if (cdrop && (g & lanemask_lt()) == 0) {
            u32 mm = g;
            while (mm) {
                const u32 d = __ffs(mm) - 1;
                mm &= mm - 1;
                const u32 s2 = (u32)(E.res_s[d] + E.ch_r[d]);
                arrive_h(S, mynk, E.res_f[d], s2, E.res_e[d]);
            }
        }
        __syncwarp();
        n_ins += flush_ins(S, broken);
        t_arr += ENG_CLK() - t0;
        if (!wmode) {
            pos += commit;
        } else if (commit < limit) {
            keep = limit - commit;
            u64 ci_ = 0, cr_ = 0;
            u32 cc_ = 0;
            if (lane < keep) { ci_ = E.ch_i[commit + lane]; cr_ = E.ch_r[commit + lane]; cc_ = E.ch_c[commit + lane]; }
            __syncwarp();
            if (lane < keep) { E.ch_i[lane] = ci_; E.ch_r[lane] = cr_; E.ch_c[lane] = cc_; }
            resume = scan_end;
            pos = __shfl_sync(FULLMASK, ci_, 0);
        } else {
            keep = 0;
            pos = scan_end;
        }
        __syncwarp();
    }
    // stop the helpers (after every message already posted); on a broken run let them leave
    for (u32 hh = 0; hh < (u32)NHELP && !broken; hh++)
        if (!post(S, hh, M_STOP, 0, 0, 0, 0)) broken = true;
    if (broken && lane == 0) st_vol(&S.abort_, 1u);
    if (stats) {
        if (lane == 0) {
            stats[0] += n_iter; stats[1] += n_retarget; stats[3] += n_rounds; stats[4] += n_qsteps;
            stats[5] += t_spec; stats[6] += t_dirty; stats[7] += t_cls; stats[8] += t_arr; stats[9] += n_req;
            stats[11] += t_store; stats[12] += n_wait; stats[13] += t_wait; stats[15] += n_ins;
            if (broken && !stats[2]) stats[2] = 6;
        }
    }
}

}  // namespace tlsfh
