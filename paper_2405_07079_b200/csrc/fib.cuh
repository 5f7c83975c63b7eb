// fib.cuh — Fibonacci buddies on sm_100a; reading C30.
//
// Classes S_0 = 1, S_1 = 2, S_k = S_{k-1} + S_{k-2} units; a class-k block splits into its low
// part of class k-1 and its high part of class R(k) = k-2 (class 1: 1 + 1, R(1) = 0).  The arena
// is the greedy (Zeckendorf) sum of Fibonacci roots, largest first.  Every block is a node of one
// root's split tree and a node is identified by (start, class); its parent and sibling follow from
// a walk down from its root (at most K+1 steps, the geometry lives in shared memory).
//
// State: per class the free node starts, sorted, back to back (the same CSR as binary buddies,
// ctr->bud_off / bud_cnt), so the free-batch classification, address sort and block table are
// shared with HEAP_BUDDY.
//
// Free (k_free_levels, one CTA): merges only go upward, so classes are settled bottom-up.  Step m
// forms the class-m parents: a free node (a, m-1) whose parent is (a, m) pairs with its free
// sibling (a + S_{m-1}, R(m)) (binary search in that class's list); both leave their lists and a
// joins class m.  A class-c list is complete once step c has merged the resident, freed and
// promoted nodes, and final after steps c+1 and c+2 (its possible parents) — the result is the
// set of maximal free tree nodes, the same set the oracle's one-by-one merge reaches.
//
// Alloc (k_alloc_engine, one warp): a split of class t for a class-j request leaves free high
// parts of classes t-2 ... j-1, i.e. also BELOW j, so the level-parallel scheme of binary buddies
// (lemma L6: leftovers stay at the demand's level) does not carry over.  The engine serves the
// requests one by one in request order, with every decision in shared memory: a 64-bit nonempty
// mask (smallest nonempty class >= j by one ffs), per class a 32-entry cache of its batch-start
// list (one coalesced warp load per 32 pops) and a sorted array of this batch's leftovers (binary
// search + warp-parallel shift).  k_alloc_rebuild then merges each class's unconsumed batch-start
// suffix with its leftovers (merge path, one CTA per class).
#pragma once
#include "common.cuh"
#include "buddy.cuh"

namespace fib {

constexpr int MAXC = 48;          // classes: S_45 < 2^32 <= S_46 ... (K <= 45)
constexpr int HC = 32;            // batch-start head cache per class (engine)
constexpr int LC = 1024;          // leftover capacity per class per alloc batch (engine)
constexpr u64 NONE64 = 0xFFFFFFFFFFFFFFFFull;

struct Geom {
    u64 S[MAXC];
    u64 rs[MAXC];      // root starts (increasing)
    u32 rk[MAXC];      // root classes (decreasing)
    u32 nroots, K;
};

// host: sizes and roots for A_u units
inline void make_geom(u64 A_u, Geom *g) {
    memset(g, 0, sizeof(Geom));
    int n = 0;
    g->S[n++] = 1;
    if (A_u >= 2) g->S[n++] = 2;
    while (n >= 2 && n < MAXC && g->S[n - 1] + g->S[n - 2] <= A_u) { g->S[n] = g->S[n - 1] + g->S[n - 2]; n++; }
    g->K = (u32)(n - 1);
    u64 s = 0, rem = A_u;
    while (rem) {
        int t = (int)g->K;
        while (g->S[t] > rem) t--;
        g->rs[g->nroots] = s;
        g->rk[g->nroots] = (u32)t;
        g->nroots++;
        s += g->S[t];
        rem -= g->S[t];
    }
}

__device__ __forceinline__ u32 rcls(u32 t) { return t >= 2 ? t - 2 : 0; }

// parent (start, class) of node (a, k); returns false for a root
__device__ __forceinline__ bool parent_of(const Geom &g, u64 a, u32 k, u64 *ps, u32 *pk) {
    u32 r = 0;
    while (r + 1 < g.nroots && g.rs[r + 1] <= a) r++;
    u64 s = g.rs[r];
    u32 t = g.rk[r];
    bool has = false;
    for (int guard = 0; guard < MAXC + 2 && !(s == a && t == k); guard++) {
        if (t == 0) return false;        // not a node (cannot happen for heap blocks)
        *ps = s; *pk = t; has = true;
        const u64 mid = s + g.S[t - 1];
        if (a < mid) t = t - 1;
        else { s = mid; t = rcls(t); }
    }
    return has;
}

// smallest class holding r units (g.K + 1 if none)
__device__ __forceinline__ u32 class_of_req(const Geom &g, u64 r) {
    u32 lo = 0, hi = g.K + 1;
    while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (g.S[mid] < r) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// freed (start, end) -> key = class of its size (sizes are exact class sizes), payload = index
__global__ void k_free_classes(const u64 *__restrict__ vs, const u64 *__restrict__ ve, const u64 *nv_dev,
                               const Geom *__restrict__ gp, u32 *__restrict__ key, u32 *__restrict__ val) {
    __shared__ Geom g;
    if (threadIdx.x == 0) g = *gp;
    __syncthreads();
    const u64 nv = *nv_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (u64)gridDim.x * blockDim.x) {
        key[i] = class_of_req(g, ve[i] - vs[i]);
        val[i] = (u32)i;
    }
}

__device__ __forceinline__ u64 bsearch_idx(const u64 *a, u64 n, u64 key) {
    u64 lo = 0, hi = n;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return (lo < n && a[lo] == key) ? lo : NONE64;
}

// ------------------------------------------------------------------ free phase ----
constexpr int NT = 1024;

__global__ void __launch_bounds__(NT) k_free_levels(const u64 *__restrict__ old_list, u64 *__restrict__ new_list,
                                                    const u64 *__restrict__ fr, const u32 *__restrict__ fr_off,
                                                    u64 *bufL, u32 *rem, u64 *promo, u64 *tmp,
                                                    const Geom *__restrict__ gp, DevCtr *ctr) {
    __shared__ Geom g;
    __shared__ u32 sm[33];
    __shared__ u64 ooff[MAXC + 1], loff[MAXC + 1], lcnt[MAXC + 1];
    __shared__ u32 foff[MAXC + 1];
    if (threadIdx.x == 0) g = *gp;
    __syncthreads();
    const u32 K = g.K;
    if (threadIdx.x <= K + 1) {
        ooff[threadIdx.x] = ctr->bud_off[threadIdx.x];
        foff[threadIdx.x] = fr_off[threadIdx.x];
    }
    __syncthreads();
    for (u32 m = 0; m <= K; m++) {
        if (threadIdx.x == 0) loff[m] = (m == 0) ? 0 : loff[m - 1] + lcnt[m - 1];   // lists packed as formed
        __syncthreads();
        // (a) parents of class m: left children (a, m-1) whose free sibling (a + S_{m-1}, R(m)) is listed
        u64 np = 0;
        if (m >= 1) {
            const u64 *Lm1 = bufL + loff[m - 1];
            const u64 nm1 = lcnt[m - 1];
            const u32 rc = rcls(m);
            const u64 *Lr = bufL + loff[rc];
            const u64 nr = lcnt[rc];
            for (u64 sb = 0; sb < nm1; sb += 32ull * NT) {      // super-rounds of <= 32 elements per thread
                const u64 nn = min(nm1 - sb, 32ull * NT);
                const u64 per = (nn + NT - 1) / NT, b0 = sb + (u64)threadIdx.x * per;
                u32 mk = 0;
                for (u64 q = 0; q < per && b0 + q < sb + nn; q++) {
                    const u64 i = b0 + q;
                    if (rem[loff[m - 1] + i]) continue;
                    const u64 a = Lm1[i];
                    u64 ps = 0;
                    u32 pk = 0;
                    if (!parent_of(g, a, m - 1, &ps, &pk) || pk != m || ps != a) continue;
                    const u64 jj = bsearch_idx(Lr, nr, a + g.S[m - 1]);
                    if (jj == NONE64 || rem[loff[rc] + jj]) continue;
                    mk |= 1u << q;
                }
                __syncthreads();          // every test read its flags before any pair is marked
                u32 tot;
                u32 pos = block_excl_scan<NT>(__popc(mk), sm, &tot);
                for (u64 q = 0; q < per; q++) {
                    if (!((mk >> q) & 1)) continue;
                    const u64 i = b0 + q;
                    const u64 a = Lm1[i];
                    rem[loff[m - 1] + i] = 1;
                    rem[loff[rc] + bsearch_idx(Lr, nr, a + g.S[m - 1])] = 1;
                    promo[np + pos++] = a;
                }
                np += tot;
                __syncthreads();
            }
        }
        // (b) class m's list: resident + freed + promoted, merged by address
        const u64 n_old = ooff[m + 1] - ooff[m], n_fr = foff[m + 1] - foff[m];
        u64 *Lm = bufL + loff[m];
        buddy::cta_merge_u64(old_list + ooff[m], n_old, fr + foff[m], n_fr, tmp);
        __syncthreads();
        buddy::cta_merge_u64(tmp, n_old + n_fr, promo, np, Lm);
        const u64 n = n_old + n_fr + np;
        for (u64 i = threadIdx.x; i < n; i += NT) rem[loff[m] + i] = 0;
        if (threadIdx.x == 0) lcnt[m] = n;
        __syncthreads();
    }
    // survivors, class by class, into the new CSR
    u64 out = 0;
    for (u32 c = 0; c <= K; c++) {
        const u64 base = loff[c];
        const u64 ns = buddy::cta_compact(lcnt[c], [&](u64 i) { return rem[base + i] == 0; },
                                          [&](u64 i, u64 p) { new_list[out + p] = bufL[base + i]; }, sm);
        if (threadIdx.x == 0) { ctr->bud_off[c] = out; ctr->bud_cnt[c] = ns; }
        out += ns;
        __syncthreads();
    }
    if (threadIdx.x == 0) { ctr->bud_off[K + 1] = out; ctr->bud_total = out; }
}

// ------------------------------------------------------------------ alloc phase ----
struct EngSmem {
    Geom g;
    u64 ptr[MAXC], end[MAXC];          // unconsumed part of the batch-start list beyond the cache
    u32 hh[MAXC], hn[MAXC];            // head cache window [hh, hn)
    u32 lh[MAXC], lt[MAXC];            // leftover window [lh, lt)
    u64 mask;
    u32 hc[MAXC * HC];
    u32 lo[1];                         // (K+1) * LC leftovers follow (dynamic)
};
inline size_t eng_smem(u32 K) { return sizeof(EngSmem) + (size_t)(K + 1) * LC * 4; }

__device__ __forceinline__ void eng_refill(EngSmem &S, const u64 *__restrict__ old_list, u32 t) {
    const u32 lane = lane_id();
    const u64 p = S.ptr[t], e = S.end[t];
    const u32 m = (u32)min((u64)HC, e - p);
    if (lane < m) S.hc[t * HC + lane] = (u32)old_list[p + lane];
    __syncwarp();
    if (lane == 0) { S.hh[t] = 0; S.hn[t] = m; S.ptr[t] = p + m; }
    __syncwarp();
}

// sorted insertion of leftover x into class c (whole warp)
__device__ __forceinline__ void eng_insert(EngSmem &S, u32 c, u32 x, DevCtr *ctr) {
    const u32 lane = lane_id();
    u32 *L = S.lo + (u64)c * LC;
    u32 h = S.lh[c], t = S.lt[c];
    if (t == (u32)LC) {
        if (h == 0) {                            // capacity: flag it (sticky), drop the leftover
            if (lane == 0) atomicOr(&ctr->error_flags, (u64)ERR_CAP_FREE);
            return;
        }
        for (u32 k = 0; k < t - h; k += 32) {    // move the window down to 0 (ascending chunks)
            const u32 i = k + lane;
            const u32 v = (i < t - h) ? L[h + i] : 0;
            __syncwarp();
            if (i < t - h) L[i] = v;
            __syncwarp();
        }
        t -= h;
        h = 0;
    }
    u32 a = h, b = t;                            // first element >= x
    while (a < b) {
        const u32 mid = (a + b) >> 1;
        if (L[mid] < x) a = mid + 1; else b = mid;
    }
    for (int top = (int)t - 1; top >= (int)a; top -= 32) {   // shift [a, t) up by one, top chunk first
        const int i = top - (int)lane;
        const u32 v = (i >= (int)a) ? L[i] : 0;
        __syncwarp();
        if (i >= (int)a) L[i + 1] = v;
        __syncwarp();
    }
    if (lane == 0) {
        L[a] = x;
        S.lh[c] = h;
        S.lt[c] = t + 1;
        S.mask |= 1ull << c;
    }
    __syncwarp();
}

// outputs: out_u[i] (units or FAIL), r[i] = S_j (units; 0 on failure); per class the first
// unconsumed batch-start index (fo), the leftovers (lo_g, lcnt) and the new list offsets (noff)
__global__ void __launch_bounds__(32, 1) k_alloc_engine(const u64 *__restrict__ sizes, u64 n, const u64 *n_in,
                                                        int alog2, const u64 *__restrict__ old_list,
                                                        const Geom *__restrict__ gp, DevCtr *ctr,
                                                        u64 *__restrict__ out_u, u64 *__restrict__ r_out,
                                                        u64 *__restrict__ fo, u64 *__restrict__ lo_g,
                                                        u64 *__restrict__ lcnt, u64 *__restrict__ noff) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    EngSmem &S = *reinterpret_cast<EngSmem *>(smem_raw);
    if (n_in) n = *n_in;
    const u32 lane = lane_id();
    if (lane == 0) S.g = *gp;
    __syncwarp();
    const u32 K = S.g.K;
    for (u32 t = lane; t <= K; t += 32) {
        S.ptr[t] = ctr->bud_off[t];
        S.end[t] = ctr->bud_off[t + 1];
        S.hh[t] = 0; S.hn[t] = 0; S.lh[t] = 0; S.lt[t] = 0;
    }
    __syncwarp();
    u64 mk = 0;
    for (u32 t = 0; t <= K; t++) if (S.end[t] > S.ptr[t]) mk |= 1ull << t;
    if (lane == 0) S.mask = mk;
    __syncwarp();
    const u64 amask = (1ull << alog2) - 1;
    for (u64 base = 0; base < n; base += 32) {
        const u64 my = base + lane;
        const u64 mys = my < n ? sizes[my] : 0;
        u64 res = buddy::FAIL, rz = 0;
        const u32 cnt = (u32)min((u64)32, n - base);
        for (u32 q = 0; q < cnt; q++) {
            const u64 s = __shfl_sync(FULLMASK, mys, q);
            const u64 r = (s >> alog2) + ((s & amask) != 0);
            const u32 j = (s == 0) ? K + 1 : class_of_req(S.g, r);
            u64 a = NONE64;
            const u64 m = (j <= K) ? (S.mask & (~0ull << j)) : 0;
            if (m) {
                const u32 t = (u32)(__ffsll((long long)m) - 1);
                const u32 hh = S.hh[t], hn = S.hn[t];
                if (hh == hn && S.ptr[t] < S.end[t]) eng_refill(S, old_list, t);
                const u32 hh2 = S.hh[t], hn2 = S.hn[t];
                const u64 hb = (hh2 < hn2) ? (u64)S.hc[t * HC + hh2] : NONE64;
                const u32 lh = S.lh[t], lt = S.lt[t];
                const u64 lb = (lh < lt) ? (u64)S.lo[(u64)t * LC + lh] : NONE64;
                __syncwarp();
                if (hb < lb) {
                    a = hb;
                    if (lane == 0) S.hh[t] = hh2 + 1;
                } else {
                    a = lb;
                    if (lane == 0) S.lh[t] = lh + 1;
                }
                __syncwarp();
                if (lane == 0 && S.hh[t] == S.hn[t] && S.ptr[t] == S.end[t] && S.lh[t] == S.lt[t])
                    S.mask &= ~(1ull << t);
                __syncwarp();
                for (u32 u = t; u > j; u--) eng_insert(S, rcls(u), (u32)(a + S.g.S[u - 1]), ctr);
            }
            if (lane == q) {
                res = a;
                rz = (a == NONE64) ? 0 : S.g.S[j];
            }
        }
        if (my < n) { out_u[my] = (res == NONE64) ? buddy::FAIL : res; r_out[my] = rz; }
    }
    __syncwarp();
    // leftovers to global, new offsets
    for (u32 t = 0; t <= K; t++) {
        const u32 lh = S.lh[t], lt = S.lt[t];
        for (u32 k = lane; k < lt - lh; k += 32) lo_g[(u64)t * LC + k] = S.lo[(u64)t * LC + lh + k];
    }
    if (lane == 0) {
        u64 o = 0;
        for (u32 t = 0; t <= K; t++) {
            const u64 first = S.ptr[t] - (S.hn[t] - S.hh[t]);   // cached but unpopped entries stay in the list
            fo[t] = first;
            lcnt[t] = S.lt[t] - S.lh[t];
            noff[t] = o;
            o += (S.end[t] - first) + lcnt[t];
        }
        noff[K + 1] = o;
    }
}

// one CTA per class: merge the unconsumed batch-start suffix with the leftovers
__global__ void __launch_bounds__(NT) k_alloc_rebuild(const u64 *__restrict__ old_list, u64 *__restrict__ new_list,
                                                      const Geom *__restrict__ gp, const DevCtr *ctr,
                                                      const u64 *__restrict__ fo, const u64 *__restrict__ lo_g,
                                                      const u64 *__restrict__ lcnt, const u64 *__restrict__ noff) {
    const u32 t = blockIdx.x;
    if (t > gp->K) return;
    const u64 first = fo[t], end = ctr->bud_off[t + 1];
    buddy::cta_merge_u64(old_list + first, end - first, lo_g + (u64)t * LC, lcnt[t], new_list + noff[t]);
}

__global__ void k_alloc_commit(DevCtr *ctr, const Geom *__restrict__ gp, const u64 *__restrict__ noff) {
    const u32 K = gp->K;
    for (u32 t = 0; t <= K; t++) {
        ctr->bud_off[t] = noff[t];
        ctr->bud_cnt[t] = noff[t + 1] - noff[t];
    }
    ctr->bud_off[K + 1] = noff[K + 1];
    ctr->bud_total = noff[K + 1];
}

// initial lists: one root per class at most (Zeckendorf roots have distinct classes)
__global__ void k_init_lists(DevCtr *ctr, u64 *list, const Geom *__restrict__ gp) {
    const u32 K = gp->K;
    u64 o = 0;
    for (u32 t = 0; t <= K; t++) {
        ctr->bud_off[t] = o;
        u64 c = 0;
        for (u32 r = 0; r < gp->nroots; r++)
            if (gp->rk[r] == t) { list[o + c] = gp->rs[r]; c++; }
        ctr->bud_cnt[t] = c;
        o += c;
    }
    ctr->bud_off[K + 1] = o;
    ctr->bud_total = o;
}

}  // namespace fib
