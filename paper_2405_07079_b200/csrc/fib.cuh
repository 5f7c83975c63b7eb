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

static_assert(sizeof(((DevCtr *)0)->bud_off) / sizeof(u64) >= MAXC, "DevCtr::bud_off must hold K + 2 class offsets");
static_assert(sizeof(((DevCtr *)0)->bud_cnt) / sizeof(u64) >= MAXC - 1, "DevCtr::bud_cnt must hold K + 1 counts");

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
    PDL_ENTRY();
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
    PDL_ENTRY();
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
// Engine state: class c is owned by lane c & 31 (c < 32: "half" 0, c >= 32: half 1), which keeps
// in registers its batch-start window (next list index, end), its head-cache window, its leftover
// window and the two candidate heads (batch-start head hb, leftover head lb).  A request reads the
// two heads of its class with two shuffles; only the owner updates; the nonempty mask is uniform.
// Shared memory holds the head caches and the sorted leftover arrays.
struct EngSmem {
    u64 S[MAXC];
    u32 hc[MAXC * HC];
    u32 lo[1];                         // (K+1) * LC leftovers follow (dynamic)
};
inline size_t eng_smem(u32 K) { return sizeof(EngSmem) + (size_t)(K + 1) * LC * 4; }

struct Cls {                           // one class's state, held by its owner lane
    u64 ptr, end;                      // batch-start list: next index to cache, end
    u32 hh, hn;                        // cache window [hh, hn) in S.hc
    u32 lh, lt;                        // leftover window [lh, lt) in S.lo
    u64 hb, lb;                        // current heads (NONE64 if none)
};

// C0 / C1 are two named register sets (classes lane, lane + 32); hf is warp-uniform, so these
// selections compile to selects / uniform branches, never to local memory
#define CSEL(f) (hf ? C1.f : C0.f)
#define CWITH(hf_, body) do { if (hf_) { Cls &x = C1; body; } else { Cls &x = C0; body; } } while (0)

// outputs: out_u[i] (units or FAIL), r[i] = S_j (units; 0 on failure); per class the first
// unconsumed batch-start index (fo), the leftovers (lo_g, lcnt) and the new list offsets (noff)
__global__ void __launch_bounds__(32, 1) k_alloc_engine(const u64 *__restrict__ sizes, u64 n, const u64 *n_in,
                                                        int alog2, const u64 *__restrict__ old_list,
                                                        const Geom *__restrict__ gp, DevCtr *ctr,
                                                        u64 *__restrict__ out_u, u64 *__restrict__ r_out,
                                                        u64 *__restrict__ fo, u64 *__restrict__ lo_g,
                                                        u64 *__restrict__ lcnt, u64 *__restrict__ noff) {
    PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    EngSmem &S = *reinterpret_cast<EngSmem *>(smem_raw);
    if (n_in) n = *n_in;
    const u32 lane = lane_id();
    const u32 K = gp->K;
    for (u32 t = lane; t < (u32)MAXC; t += 32) S.S[t] = (t <= K) ? gp->S[t] : NONE64;
    // owner state of classes lane and lane + 32; initial caches (one coalesced load per class)
    Cls C0, C1;
#pragma unroll
    for (int hf = 0; hf < 2; hf++) {
        const u32 c = lane + 32 * hf;
        CWITH(hf, {
            x.ptr = x.end = 0; x.hh = x.hn = x.lh = x.lt = 0; x.hb = x.lb = NONE64;
            if (c <= K) { x.ptr = ctr->bud_off[c]; x.end = ctr->bud_off[c + 1]; }
        });
    }
    for (u32 t = 0; t <= K; t++) {
        const u32 hf = t >> 5;
        const u64 p0 = __shfl_sync(FULLMASK, CSEL(ptr), t & 31), e0 = __shfl_sync(FULLMASK, CSEL(end), t & 31);
        const u32 m = (u32)min((u64)HC, e0 - p0);
        if (lane < m) S.hc[t * HC + lane] = (u32)old_list[p0 + lane];
    }
    __syncwarp();
    u64 mask = 0;
#pragma unroll
    for (int hf = 0; hf < 2; hf++) {
        const u32 c = lane + 32 * hf;
        CWITH(hf, {
            if (c <= K) {
                const u32 m = (u32)min((u64)HC, x.end - x.ptr);
                x.hn = m;
                x.ptr += m;
                x.hb = m ? (u64)S.hc[c * HC] : NONE64;
            }
        });
        const u32 bal = __ballot_sync(FULLMASK, CSEL(hb) != NONE64);
        mask |= (u64)bal << (32 * hf);
    }
    const u64 amask = (1ull << alog2) - 1;
    u64 n_ins = 0, n_shift = 0, n_ref = 0;
    long long cyc_ins = 0;
    const long long cyc0 = clock64();
    for (u64 base = 0; base < n; base += 32) {
        const u64 my = base + lane;
        const u64 mys = my < n ? sizes[my] : 0;
        u64 res = NONE64, rz = 0;
        const u32 cnt = (u32)min((u64)32, n - base);
        // every lane classes its own request first (smallest class holding r = the number of
        // class sizes below r, a binary search over the ascending S), then the requests are
        // served one by one
        u32 myj = K + 1;
        {
            const u64 myr = (mys >> alog2) + ((mys & amask) != 0);
            if (mys != 0) {
                u32 lo = 0, hi = K + 1;                  // first t with S[t] >= myr
                while (lo < hi) {
                    const u32 mid = (lo + hi) >> 1;
                    if (S.S[mid] < myr) lo = mid + 1; else hi = mid;
                }
                myj = lo;
            }
        }
        for (u32 q = 0; q < cnt; q++) {
            const u32 j = __shfl_sync(FULLMASK, myj, q);
            const u64 m = (j <= K) ? (mask & (~0ull << j)) : 0;
            u64 a = NONE64;
            if (m) {
                const u32 t = (u32)(__ffsll((long long)m) - 1), ow = t & 31, hf = t >> 5;
                {
                    const u64 hb0 = CSEL(hb), lb0 = CSEL(lb);  // the owner's two heads: one shuffle of the smaller
                    a = __shfl_sync(FULLMASK, hb0 < lb0 ? hb0 : lb0, ow);
                }
                int fl = 0;                                       // bit 0: refill needed, bit 1: nonempty
                if (lane == ow) {                                 // pop, next head
                    CWITH(hf, {
                        if (x.hb < x.lb) {
                            x.hh++;
                            if (x.hh < x.hn) x.hb = S.hc[t * HC + x.hh];
                            else { x.hb = NONE64; fl = x.ptr < x.end; }
                        } else {
                            x.lh++;
                            x.lb = (x.lh < x.lt) ? (u64)S.lo[(u64)t * LC + x.lh] : NONE64;
                        }
                        fl |= (x.hb != NONE64 || x.lb != NONE64) ? 2 : 0;
                    });
                }
                fl = __shfl_sync(FULLMASK, fl, ow);               // (a refill leaves the class nonempty)
                if (fl & 1) {                                     // refill the cache (whole warp)
                    const u64 p0 = __shfl_sync(FULLMASK, CSEL(ptr), ow), e0 = __shfl_sync(FULLMASK, CSEL(end), ow);
                    const u32 mm = (u32)min((u64)HC, e0 - p0);
                    if (lane < mm) S.hc[t * HC + lane] = (u32)old_list[p0 + lane];
                    __syncwarp();
                    if (lane == ow) CWITH(hf, { x.hh = 0; x.hn = mm; x.ptr = p0 + mm; x.hb = S.hc[t * HC]; });
                    n_ref++;
                }
                if (!fl) mask &= ~(1ull << t);
                // split keeping the low part: the high parts (a + S_{u-1}, R(u)) stay free
                const long long c0 = clock64();
                for (u32 u = t; u > j; u--) {
                    const u32 c = rcls(u), oc = c & 31, hc2 = c >> 5;
                    const u32 xv = (u32)(a + S.S[u - 1]);
                    u32 h = __shfl_sync(FULLMASK, hc2 ? C1.lh : C0.lh, oc), tt = __shfl_sync(FULLMASK, hc2 ? C1.lt : C0.lt, oc);
                    u32 *L = S.lo + (u64)c * LC;
                    n_ins++;
                    if (tt == (u32)LC) {
                        if (h == 0) {                            // capacity: flag (sticky), drop
                            if (lane == 0) atomicOr(&ctr->error_flags, (u64)ERR_CAP_FREE);
                            continue;
                        }
                        for (u32 k = 0; k < tt - h; k += 32) {   // move the window down to 0
                            const u32 i = k + lane;
                            const u32 v = (i < tt - h) ? L[h + i] : 0;
                            __syncwarp();
                            if (i < tt - h) L[i] = v;
                            __syncwarp();
                        }
                        tt -= h;
                        h = 0;
                    }
                    // insertion point: the tail (common), else a 32-way warp search
                    u32 lo2 = h, hi2 = tt;
                    if (tt == h || L[tt - 1] < xv) lo2 = tt;
                    while (hi2 - lo2 > 1 && lo2 < tt) {
                        const u32 seg = (hi2 - lo2 + 31) / 32;
                        const u32 i = lo2 + lane * seg;
                        const u32 k = __popc(__ballot_sync(FULLMASK, i < hi2 && L[i] < xv));
                        if (k == 0) { hi2 = lo2; break; }
                        lo2 = lo2 + (k - 1) * seg + 1;
                        hi2 = min(hi2, lo2 - 1 + seg);
                        if (seg == 1) { hi2 = lo2; break; }
                    }
                    if (lo2 < hi2 && L[lo2] < xv) lo2++;
                    n_shift += tt - lo2;
                    for (int top = (int)tt - 1; top >= (int)lo2; top -= 32) {   // shift [lo2, tt) up by one
                        const int i = top - (int)lane;
                        const u32 v = (i >= (int)lo2) ? L[i] : 0;
                        __syncwarp();
                        if (i >= (int)lo2) L[i + 1] = v;
                        __syncwarp();
                    }
                    if (lane == 0) L[lo2] = xv;
                    __syncwarp();
                    if (lane == oc) CWITH(hc2, { x.lh = h; x.lt = tt + 1; x.lb = L[h]; });
                    mask |= 1ull << c;
                }
                cyc_ins += clock64() - c0;
            }
            if (lane == q) {
                res = a;
                rz = (a == NONE64) ? 0 : S.S[j];
            }
        }
        if (my < n) { out_u[my] = (res == NONE64) ? buddy::FAIL : res; r_out[my] = rz; }
    }
    __syncwarp();
    if (lane == 0) {                 // diagnostics (heap_debug_counters)
        ctr->eng[0] += clock64() - cyc0; ctr->eng[1] += cyc_ins; ctr->eng[3] += n_ins;
        ctr->eng[4] += n_shift; ctr->eng[6] += n_ref;
    }
    // leftovers to global; per class first unconsumed list index, leftover count, new offsets
    for (u32 t = 0; t <= K; t++) {
        const u32 hf = t >> 5;
        const u32 lh = __shfl_sync(FULLMASK, CSEL(lh), t & 31), lt = __shfl_sync(FULLMASK, CSEL(lt), t & 31);
        for (u32 k = lane; k < lt - lh; k += 32) lo_g[(u64)t * LC + k] = S.lo[(u64)t * LC + lh + k];
    }
    u64 o = 0;
    for (u32 t = 0; t <= K; t++) {
        const u32 hf = t >> 5;
        const u64 f = __shfl_sync(FULLMASK, CSEL(ptr) - (CSEL(hn) - CSEL(hh)), t & 31);   // unpopped cache entries stay
        const u64 c = __shfl_sync(FULLMASK, (u64)(CSEL(lt) - CSEL(lh)), t & 31);
        const u64 e = __shfl_sync(FULLMASK, CSEL(end), t & 31);
        if (lane == 0) { fo[t] = f; lcnt[t] = c; noff[t] = o; }
        o += (e - f) + c;
    }
    if (lane == 0) noff[K + 1] = o;
}

// one CTA per class: merge the unconsumed batch-start suffix with the leftovers
__global__ void __launch_bounds__(NT) k_alloc_rebuild(const u64 *__restrict__ old_list, u64 *__restrict__ new_list,
                                                      const Geom *__restrict__ gp, const DevCtr *ctr,
                                                      const u64 *__restrict__ fo, const u64 *__restrict__ lo_g,
                                                      const u64 *__restrict__ lcnt, const u64 *__restrict__ noff) {
    PDL_ENTRY();
    const u32 t = blockIdx.x;
    if (t > gp->K) return;
    const u64 first = fo[t], end = ctr->bud_off[t + 1];
    buddy::cta_merge_u64(old_list + first, end - first, lo_g + (u64)t * LC, lcnt[t], new_list + noff[t]);
}

__global__ void k_alloc_commit(DevCtr *ctr, const Geom *__restrict__ gp, const u64 *__restrict__ noff) {
    PDL_ENTRY();
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
    PDL_ENTRY();
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
