// heap.cu — libheap: the C ABI (include/heap.h) over the sm_100a kernels.
//
// Host side: argument checks, workspace carving, and the kernel sequence of each batch.
// Nothing here synchronises with the device except heap_stats / heap_export.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <algorithm>
#include <vector>
#include "../../include/heap.h"
#include <nccl.h>
#include "common.cuh"
#include "prims.cuh"
#include "micro.cuh"
#include "table.cuh"
#include "buddy.cuh"
#include "fits.cuh"
#include "engine_tlsf.cuh"
#include "pool.cuh"
#include "dbuddy.cuh"
#include "partial.cuh"
#include "fib.cuh"

namespace {

inline u64 align_up(u64 x, u64 a) { return (x + a - 1) / a * a; }
inline int ilog2(u64 x) { int r = -1; while (x) { x >>= 1; r++; } return r; }
inline u64 next_pow2(u64 x) { u64 p = 1; while (p < x) p <<= 1; return p; }

// host mirror of the class mapping, used only to size the class range (NC)
inline u64 h_cls_insert(u64 u, int L) {
    if (u < (1ull << L)) return u;
    int m = ilog2(u);
    return ((u64)(m - L + 1) << L) + ((u >> (m - L)) - (1ull << L));
}

struct Layout {
    u64 A_u, cap_f, cap_m, tcap, sort_cap, scan_cap, hist_cap, ff_tree, bud_cap, dpool, bpool;
    int nlev, K, NC, L, FB;
    // offsets
    u64 o_ctr, o_stats, o_tbl, o_fs0, o_fs1, o_fe0, o_fe1, o_kA, o_kB, o_vA, o_vB, o_flags, o_pos,
        o_hist, o_tsum, o_vs, o_ve, o_vsc, o_vec, o_ms, o_me, o_r, o_c, o_out, o_off, o_child,
        o_sib, o_cs, o_bm, o_slot, bm_w0, bm_w1, bm_w2, bm_bytes, o_tree, o_lvl, o_bk0, o_bk1, o_dtm, o_dsrc, o_baddr, o_daddr, o_btm, o_bsrc, o_bufA, o_bufB,
        o_promo, o_bq0, o_bq1, o_fr, o_froff, o_reqoff, o_ft0, o_ft1, o_vt, o_mt, o_lnext, total;
    // HEAP_HYBRID: pool geometry and arrays, then the TLSF heap's own workspace at o_sub
    pool::Geom geo;
    u64 o_pctr, o_bits, o_sbcnt, o_sbpre, o_tsz, o_tout, o_toff, o_tidx, o_coff, o_sstats, o_sub, sub_total;
    u64 o_gin, o_gout;   // graph path: staging of the request / result words
    // HEAP_DOUBLE_BUDDY: the 3-unit heap's geometry and the split / merge buffers
    u64 dbl_A, dbl_n3, o_dctr, o_ca, o_cb, o_ia, o_ib, o_ra, o_rb, o_sstats2, o_sub2, sub2_total;
    // HEAP_FIB_BUDDY: geometry, leftovers, level lists (fib.cuh)
    fib::Geom fg;
    u64 o_fgeom, o_flo, o_fbufL, o_frem, o_fscr;
    // HEAP_PARTIAL_FREE: live-start bitmap (partial.cuh)
    bool partial;
    partial::Lbm lbm;
    u64 o_lbm, lbm_words;
};

bool make_layout(u64 arena, u64 align, int policy, u64 max_live, u64 max_batch, Layout *Lo) {
    if (align == 0 || (align & (align - 1)) || arena == 0 || arena % align) return false;
    const bool partial_free = (policy & HEAP_PARTIAL_FREE) != 0;
    policy &= ~HEAP_PARTIAL_FREE;
    if (policy < HEAP_FIRST_FIT || policy > HEAP_FIB_BUDDY) return false;
    // partial frees need address coalescing (C29)
    if (partial_free && policy != HEAP_FIRST_FIT && policy != HEAP_BEST_FIT && policy != HEAP_SEGFIT &&
        policy != HEAP_TLSF && policy != HEAP_NEXT_FIT)
        return false;
    if (max_live == 0 || max_batch == 0 || max_batch >= (1ull << 31) || max_live >= (1ull << 30)) return false;
    Layout &L = *Lo;
    memset(&L, 0, sizeof(L));
    L.partial = partial_free;
    L.A_u = arena / align;
    if (L.A_u > (1ull << 32)) return false;
    if (policy == HEAP_DOUBLE_BUDDY) {
        // reading C28 (dbuddy.cuh): the 3-unit heap gets floor(arena / 6 align) units at the top
        L.dbl_n3 = arena / (6 * align);
        L.dbl_A = arena - 3 * align * L.dbl_n3;
        Layout la, lb;
        if (!make_layout(L.dbl_A, align, HEAP_BUDDY, max_live, max_batch, &la)) return false;
        if (L.dbl_n3 && !make_layout(L.dbl_n3, 1, HEAP_BUDDY, max_live, max_batch, &lb)) return false;
        u64 o = 0;
        auto take = [&](u64 bytes) { u64 r = o; o = align_up(o + bytes, 256); return r; };
        L.o_ctr = take(sizeof(DevCtr));
        L.o_stats = take(sizeof(heap_stats_t));
        L.o_dctr = take(sizeof(dbl::Ctr));
        L.o_flags = take(max_batch * 4 + 4);
        L.o_pos = take(max_batch * 4 + 4);
        L.o_kA = take(max_batch * 4 + 4);
        L.o_kB = take(max_batch * 4 + 4);
        L.o_tsum = take((prims::ntiles_of(max_batch) + 16) * 4);
        L.o_tsz = take(max_batch * 8);
        L.o_toff = take(max_batch * 8);
        L.o_ca = take(max_batch * 8);
        L.o_cb = take(max_batch * 8);
        L.o_ia = take(max_batch * 4);
        L.o_ib = take(max_batch * 4);
        L.o_ra = take(max_batch * 8);
        L.o_rb = take(max_batch * 8);
        L.o_sstats = take(sizeof(heap_stats_t));
        L.o_sstats2 = take(sizeof(heap_stats_t));
        L.o_gin = take(max_batch * 8);
        L.o_gout = take(max_batch * 8);
        L.o_sub = take(la.total);
        L.sub_total = la.total;
        if (L.dbl_n3) { L.o_sub2 = take(lb.total); L.sub2_total = lb.total; }
        L.total = o;
        return true;
    }
    if (policy == HEAP_HYBRID) {
        // reading C26 (pool.cuh): pools of align*2^j <= 4096 B objects share the first half of the
        // arena, each a whole number of pages; the TLSF heap covers the rest
        pool::Geom &G = L.geo;
        G.alog2 = ilog2(align);
        for (u64 o = align; o <= pool::PAGE; o <<= 1) G.J++;
        G.S = G.J ? arena / (2 * (u64)G.J) / pool::PAGE * pool::PAGE : 0;
        G.pool_end = (u64)G.J * G.S;
        u64 wb = 0;
        for (int j = 0; j < G.J; j++) {
            G.wbase[j] = wb;
            G.nslots[j] = G.S >> (G.alog2 + j);
            wb += align_up((G.nslots[j] + 31) / 32, 32);
        }
        G.wbase[G.J] = wb;
        G.nwords = wb;
        G.nsb = wb / 32;
        if (G.nslots[0] >= (1ull << 32)) return false;          // u32 slot ranks
        Layout sub;
        if (!make_layout(arena - G.pool_end, align, HEAP_TLSF, max_live, max_batch, &sub)) return false;
        const u64 scan_cap = std::max(std::max(max_batch, G.nwords), (u64)256 * prims::ntiles_of(max_batch) + 16);
        u64 o = 0;
        auto take = [&](u64 bytes) { u64 r = o; o = align_up(o + bytes, 256); return r; };
        L.o_ctr = take(sizeof(DevCtr));
        L.o_stats = take(sizeof(heap_stats_t));
        L.o_pctr = take(sizeof(pool::Ctr));
        L.o_bits = take(G.nwords * 4 + 4);
        L.o_sbcnt = take(G.nsb * 4 + 4);
        L.o_sbpre = take(G.nsb * 4 + 4);
        L.o_kA = take(max_batch * 4);
        L.o_kB = take(max_batch * 4);
        L.o_vA = take(max_batch * 4);
        L.o_vB = take(max_batch * 4);
        L.o_flags = take(scan_cap * 4);
        L.o_pos = take(scan_cap * 4);
        L.o_hist = take((256 * prims::ntiles_of(max_batch) + 512) * 4);
        L.o_tsum = take((prims::ntiles_of(scan_cap) + 16) * 4);
        L.o_tsz = take(max_batch * 8);
        L.o_tout = take(max_batch * 8);
        L.o_toff = take(max_batch * 8);
        L.o_tidx = take(max_batch * 4);
        L.o_coff = take((pool::MAXJ + 2) * 4);
        L.o_sstats = take(sizeof(heap_stats_t));
        L.o_gin = take(max_batch * 8);
        L.o_gout = take(max_batch * 8);
        L.o_sub = take(sub.total);
        L.sub_total = sub.total;
        L.total = o;
        return true;
    }
    L.K = ilog2(L.A_u);
    const bool fibp = policy == HEAP_FIB_BUDDY;
    if (fibp) {                               // Fibonacci classes (reading C30)
        fib::make_geom(L.A_u, &L.fg);
        L.K = (int)L.fg.K;
    }
    L.L = (policy == HEAP_TLSF) ? 5 : 0;
    L.NC = (int)h_cls_insert(L.A_u, L.L) + 1;
    L.cap_f = max_live + 1;
    if (policy == HEAP_BUDDY || fibp) L.cap_f = (max_live + 1) * 2 * (u64)(L.K + 1);
    L.cap_m = L.cap_f + max_batch;
    L.tcap = next_pow2(2 * max_live);
    if (L.tcap < 1024) L.tcap = 1024;
    L.sort_cap = std::max(std::max(max_batch, L.cap_f), max_live) + 16;
    L.hist_cap = 256 * prims::ntiles_of(L.sort_cap) + 512;   // u64 lookback words of the onesweep tiles
    L.scan_cap = std::max(std::max(L.cap_m, L.sort_cap), L.hist_cap);
    L.scan_cap = std::max(L.scan_cap, L.tcap);
    L.FB = ilog2(L.cap_f) + 1;
    // first-fit tree levels
    u64 n = L.cap_f;
    L.nlev = 1;
    L.ff_tree = n;
    while (n > 32) { n = (n + 31) / 32; L.ff_tree += n; L.nlev++; }
    L.bud_cap = L.cap_f + max_batch;
    L.dpool = 2 * max_batch + 256;
    L.bpool = max_batch + 256;
    u64 o = 0;
    auto take = [&](u64 bytes) { u64 r = o; o = align_up(o + bytes, 256); return r; };
    L.o_ctr = take(sizeof(DevCtr));
    L.o_stats = take(sizeof(heap_stats_t));
    L.o_tbl = take(L.tcap * 8);
    L.o_fs0 = take(L.cap_f * 8);
    L.o_fs1 = take(L.cap_f * 8);
    if (policy != HEAP_BUDDY && !fibp) { L.o_fe0 = take(L.cap_f * 8); L.o_fe1 = take(L.cap_f * 8); }
    L.o_kA = take(L.sort_cap * 4);
    L.o_kB = take(L.sort_cap * 4);
    L.o_vA = take(L.sort_cap * 4);
    L.o_vB = take(L.sort_cap * 4);
    L.o_flags = take(L.scan_cap * 4);
    L.o_pos = take(L.scan_cap * 4);
    L.o_hist = take(L.hist_cap * 4);
    L.o_tsum = take((prims::ntiles_of(L.scan_cap) + 16) * 4);
    L.o_vs = take(max_batch * 8);
    L.o_ve = take(max_batch * 8);
    L.o_vsc = take(max_batch * 8);
    L.o_vec = take(max_batch * 8);
    L.o_ms = take(std::max(L.cap_m, max_live + 16) * 8);
    L.o_me = take(std::max(L.cap_m, max_live + 16) * 8);
    L.o_r = take(max_batch * 8);
    L.o_c = take(max_batch * 4);
    L.o_out = take(max_batch * 8);
    L.o_gin = take(max_batch * 8);
    L.o_gout = take(max_batch * 8);
    L.o_off = take((fits::MAX_NC + 8) * 4);
    if (policy == HEAP_TLSF || policy == HEAP_SEGFIT) {
        L.o_cs = take(L.cap_f * 16);          // CSR records {f, start, end - 1, 0} (engine_tlsf.cuh)
        // overflow bitmaps: one three-level slot per class (engine_tlsf.cuh)
        L.bm_w0 = (L.cap_f + 31) / 32;
        L.bm_w1 = (L.bm_w0 + 31) / 32;
        L.bm_w2 = (L.bm_w1 + 31) / 32;
        L.bm_bytes = (u64)L.NC * (L.bm_w0 + L.bm_w1 + L.bm_w2) * 4;
        L.o_bm = take(L.bm_bytes);
        L.o_slot = take(tlsfw::MAX_NC * 4);
    }
    if (policy == HEAP_SEGFIT_LIFO) {
        L.o_cs = take(L.cap_f * 16);
        L.o_ft0 = take(L.cap_f * 4);          // push stamps of the free pieces (double buffer)
        L.o_ft1 = take(L.cap_f * 4);
        L.o_vt = take(max_batch * 4);         // stamps of this batch's frees
        L.o_mt = take(L.cap_m * 4);           // stamps of the merged array
        L.o_lnext = take(L.cap_f * 4);        // spill-stack links
        L.o_bk0 = take(L.cap_f * 8);          // (class, stamp) sort keys
        L.o_bk1 = take(L.cap_f * 8);
    }
    if (policy == HEAP_FIRST_FIT || policy == HEAP_NEXT_FIT) {
        L.o_tree = take(L.ff_tree * 8);
        L.o_lvl = take(fits::FF_MAX_LEVELS * 8);
    }
    if (policy == HEAP_BEST_FIT) {
        L.o_bk0 = take(L.cap_f * 8);
        L.o_bk1 = take(L.cap_f * 8);
    }
    if (L.partial) {
        L.lbm_words = partial::lbm_layout(L.A_u, &L.lbm);
        L.o_lbm = take(L.lbm_words * 4);
    }
    if (fibp) {
        L.o_fgeom = take(sizeof(fib::Geom));
        L.o_flo = take((u64)(L.K + 1) * fib::LC * 8);
        L.o_fbufL = take(2 * L.bud_cap * 8);  // every level list: <= 2 x (resident + freed) nodes
        L.o_frem = take(2 * L.bud_cap * 4);
        L.o_fscr = take(4 * (fib::MAXC + 2) * 8);
    }
    if (policy == HEAP_BUDDY || fibp) {
        L.o_dtm = take(L.dpool * 4);
        L.o_dsrc = take(L.dpool * 4);
        L.o_baddr = take(L.bpool * 8);
        L.o_daddr = take(L.dpool * 8);
        L.o_btm = take(L.bpool * 4);
        L.o_bsrc = take(L.bpool * 4);
        L.o_bufA = take(L.bud_cap * 8);
        L.o_bufB = take(L.bud_cap * 8);
        L.o_promo = take(L.bud_cap * 8);
        if (policy == HEAP_BUDDY) { L.o_bq0 = take(L.cap_f * 8); L.o_bq1 = take(L.cap_f * 8); }
        L.o_fr = take(max_batch * 8);
        L.o_froff = take(64 * 4);
        L.o_reqoff = take(64 * 4);
    }
    L.total = o;
    return true;
}

template <typename T> T *at(void *ws, u64 off) { return reinterpret_cast<T *>(static_cast<char *>(ws) + off); }

}  // namespace

struct heap {
    u64 arena, align, max_live, max_batch;
    int policy, alog2, sms, G;
    int wild_split;          // TLSF/SEGFIT wilderness split (engine_tlsf.cuh); env HEAP_WILD_SPLIT=0 disables
    int bf_flat;             // BEST_FIT: the flat one-array engine instead of the blocked one (env HEAP_BF_FLAT=1)
    int micro;               // small heap: each batch is one single-CTA launch (micro.cuh); env HEAP_MICRO=0 disables
    const u64 *hidx = nullptr;   // heap_free_batch_handles on a micro heap: the handle indices (else null)
    u64 hlen = 0;
    int pdl;                 // programmatic dependent launches (env HEAP_PDL=0 disables)
    int eng_warps;           // TLSF/SEGFIT engine: 2 = arrivals on a second warp (default), 1 = one warp (HEAP_ENGINE_WARPS=1)
    int bud_levels;          // BUDDY free phase: the level-by-level kernel instead of the parallel form (env HEAP_BUDDY_LEVELS=1)
    Layout L;
    void *ws;
    size_t ws_bytes;
    int cur;
    u64 launches;
    DevCtr *ctr;
    heap_stats_t *dstats;
    u64 *tbl, *fs[2], *fe[2];
    u64 *bq[2] = {nullptr, nullptr};   // BUDDY: the free set in address order (start << 6 | order)
    u32 *kA, *kB, *vA, *vB, *flags, *pos, *hist, *tsum;
    u64 *vs, *ve, *vsc, *vec, *ms, *me, *r, *out;
    u32 *c, *off, *child, *sib, *bm, *slot;
    uint4 *cs;
    u32 *ft[2], *vt, *mt, *lnext;             // SEGFIT_LIFO stamps and spill links
    u64 *tree, *lvl;
    u64 *bk[2];
    u32 *dtm, *dsrc, *btm, *bsrc, *froff, *reqoff;
    u64 *baddr, *daddr, *bufA, *bufB, *promo, *fr;
    fib::Geom *fgeom;                         // HEAP_FIB_BUDDY
    u64 *flo, *fbufL, *fscr;
    u32 *frem;
    // HEAP_HYBRID
    heap *sub;                                // HYBRID: the TLSF heap on [pool_end, arena); DOUBLE: the binary heap
    heap *sub2;                               // DOUBLE_BUDDY: the 3-unit heap (NULL if it has no units)
    dbl::Ctr *dctr;
    u64 *ca, *cb, *ra, *rb;
    u32 *ia, *ib;
    heap_stats_t *sstats2;
    pool::Ctr *pctr;
    u32 *bits, *sbcnt, *sbpre, *tidx, *coff;
    u64 *tsz, *tout, *toff;
    heap_stats_t *sstats;
    // graph path: one instantiated graph per (op, ping-pong state); see graph_batch()
    struct GSlot {
        cudaGraphExec_t exec = nullptr;
        cudaGraph_t graph = nullptr;          // kept alive: the exec's node handles refer to it
        cudaGraphNode_t set_n = nullptr, cin = nullptr, cout = nullptr;
        int cur_after = 0, subcur_after = 0, sub2cur_after = 0;
        u64 nlaunch = 0;
    };
    int graphs;
    cudaStream_t cap;
    GSlot gs[2][2][2];
    u64 *gin, *gout;
    // tracing
    u64 prof_mask;
    int tag;                                  // tag of the launches being issued
    struct Rec { int tag; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
};

namespace {
cudaEvent_t prof_event(heap *h) {
    if (!h->pool.empty()) { cudaEvent_t e = h->pool.back(); h->pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

// programmatic dependent launch (common.cuh PDL_ENTRY): the launch attribute lets this kernel be
// scheduled while the previous one drains; the kernel itself waits for its completion
template <typename... P, typename... A>
static void launch_pdl(void (*kern)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

#define LAUNCH(h, kern, grid, block, smem, stream, ...)                                   \
    do {                                                                                  \
        bool _p = ((h)->prof_mask >> (h)->tag) & 1;                                       \
        heap::Rec _r{(h)->tag, nullptr, nullptr};                                         \
        if (_p) { _r.a = prof_event(h); _r.b = prof_event(h); cudaEventRecord(_r.a, (cudaStream_t)(stream)); } \
        if ((h)->pdl) launch_pdl((kern), (grid), (block), (smem), (cudaStream_t)(stream), __VA_ARGS__); \
        else kern<<<(grid), (block), (smem), (cudaStream_t)(stream)>>>(__VA_ARGS__);        \
        if (_p) { cudaEventRecord(_r.b, (cudaStream_t)(stream)); (h)->recs.push_back(_r); } \
        (h)->launches++;                                                                  \
    } while (0)
#define TAG(h, t) ((h)->tag = (t))

namespace {

__global__ void k_init(DevCtr *ctr, u64 *tbl, u64 tcap, u64 *fs, u64 *fe, u64 A_u, int buddy, int K) {
    PDL_ENTRY();
    const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x, nth = (u64)gridDim.x * blockDim.x;
    for (u64 i = tid; i < tcap; i += nth) tbl[i] = table::EMPTY;
    if (tid == 0) {
        memset(ctr, 0, sizeof(DevCtr));
        if (buddy == 2) {
            // HEAP_FIB_BUDDY: the root lists are written by fib::k_init_lists
        } else if (!buddy) {
            fs[0] = 0;      // the heap itself is the one free block (Alg. 6)
            fe[0] = A_u;
            ctr->F = 1;
            ctr->lifo_clock = 1;
        } else {
            // greedy decomposition into maximal aligned power-of-two blocks (C13):
            // one block per set bit of A_u, largest first
            u64 s = 0, o = 0;
            for (int t = 0; t <= K + 1; t++) ctr->bud_off[t] = 0;
            u64 addr[40];
            for (int t = K; t >= 0; t--) {
                addr[t] = s;
                if ((A_u >> t) & 1) s += 1ull << t;
            }
            for (int t = 0; t <= K; t++) {
                ctr->bud_off[t] = o;
                u64 c = (A_u >> t) & 1;
                ctr->bud_cnt[t] = c;
                if (c) fs[o++] = addr[t];
            }
            ctr->bud_off[K + 1] = o;
            ctr->bud_total = o;
            // the same roots in address order (largest first) for the parallel free phase (fe = bq)
            u64 q = 0;
            for (int t = K; t >= 0; t--)
                if ((A_u >> t) & 1) fe[q++] = (addr[t] << buddy::QSH) | (u64)t;
            ctr->bud_qn = q;
        }
    }
}

// radix sort of *n_dev keys (ping-pong); returns the buffer index (0 = a, 1 = b) holding the result
template <typename K, bool HV>
int radix_sort(heap *h, K *ka, K *kb, u32 *va, u32 *vb, const u64 *n_dev, int bits, cudaStream_t s,
               bool hist_done = false) {
    // onesweep (prims.cuh): one histogram launch for every pass (none when the keys' producer
    // counted them: hist_done), then one launch per pass
    const int passes = (bits + 7) / 8;
    u64 *flags = reinterpret_cast<u64 *>(h->hist);
    if (!hist_done) LAUNCH(h, prims::k_os_hist<K>, h->sms, prims::OS_NT, 0, s, ka, n_dev, passes, h->ctr);
    K *kin = ka, *kout = kb;
    u32 *vin = va, *vout = vb;
    for (int p = 0; p < passes; p++) {
        LAUNCH(h, (prims::k_os_scatter<K, HV>), h->G, prims::OS_NT, (prims::os_smem<K, HV>()), s, kin, vin, kout,
               vout, n_dev, p, flags, h->ctr);
        K *tk = kin; kin = kout; kout = tk;
        u32 *tv = vin; vin = vout; vout = tv;
    }
    return passes & 1;
}

// exclusive scan of u32 in[*n_dev] into out, grand total into *total (single pass, prims.cuh)
void scan(heap *h, const u32 *in, u32 *out, const u64 *n_dev, u64 *total, cudaStream_t s) {
    LAUNCH(h, prims::k_scan_1p, h->G, prims::OS_NT, 0, s, in, out, n_dev, total, reinterpret_cast<u64 *>(h->tsum),
           h->ctr);
}

__global__ void k_set_F(DevCtr *ctr) {
    PDL_ENTRY();
    ctr->F = ctr->tmp[1];
    if (ctr->eng[2]) ctr->error_flags |= ERR_ENGINE;   // engine watchdog fired: results invalid
}

// ---- table rebuild (tombstone purge), each kernel a no-op unless the flag is set ----
// k_rb_collect decides (every CTA reads the same tbl_used; block 0 records the flag for the other
// two kernels) and counts the live slots into tmp[5] (zero between rebuilds); k_rb_clear moves the
// count to rb_n and re-zeroes tmp[5]; k_rb_insert re-inserts rb_n slots.
__global__ void k_rb_collect(DevCtr *ctr, const u64 *tbl, u64 tcap, u64 *scratch, u64 thresh) {
    PDL_ENTRY();
    const bool rb = ctr->tbl_used > thresh;
    if (blockIdx.x == 0 && threadIdx.x == 0) ctr->tmp[4] = rb ? 1 : 0;
    if (!rb) return;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < tcap; i += (u64)gridDim.x * blockDim.x) {
        u64 v = tbl[i];
        if (table::is_live(v)) scratch[atomicAdd(&ctr->tmp[5], 1ull)] = v;
    }
}
__global__ void k_rb_clear(DevCtr *ctr, u64 *tbl, u64 tcap) {
    PDL_ENTRY();
    if (!ctr->tmp[4]) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) { ctr->rb_n = ctr->tmp[5]; ctr->tmp[5] = 0; }
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < tcap; i += (u64)gridDim.x * blockDim.x)
        tbl[i] = table::EMPTY;
}
__global__ void k_rb_insert(DevCtr *ctr, u64 *tbl, u64 tmask, u64 max_lines, const u64 *scratch) {
    PDL_ENTRY();
    if (!ctr->tmp[4]) return;
    const u64 n = ctr->rb_n;
    const u32 g = lane_id() / table::TILE_LANES;
    const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((u64)gridDim.x * blockDim.x) >> 5;
    for (u64 base = gw * table::KPW; base < n; base += nw * table::KPW) {
        u64 i = base + g;
        bool in = i < n;
        u64 v = in ? scratch[i] : 0;
        int rc = table::insert(tbl, tmask, in ? table::slot_key(v) : 0, in ? table::slot_size(v) : 1, in, max_lines);
        if (rc == 2) atomicOr(&ctr->error_flags, (u64)ERR_TABLE_FULL);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) { ctr->tbl_used = n; ctr->tbl_tombs = 0; }
}

void maybe_rebuild(heap *h, cudaStream_t s) {
    u64 thresh = h->L.tcap / 4 * 3;
    TAG(h, HEAP_TAG_REBUILD);
    LAUNCH(h, k_rb_collect, h->G, 256, 0, s, h->ctr, h->tbl, h->L.tcap, h->ms, thresh);
    LAUNCH(h, k_rb_clear, h->G, 256, 0, s, h->ctr, h->tbl, h->L.tcap);
    LAUNCH(h, k_rb_insert, h->G, 256, 0, s, h->ctr, h->tbl, h->L.tcap - 1, h->L.tcap / table::LINE, h->ms);
}

// ---- statistics ----
__global__ void __launch_bounds__(1024) k_stats(const DevCtr *ctr, const u64 *fs, const u64 *fe, int buddy, int K,
                                                u64 arena, u64 align, int alog2, u64 meta, heap_stats_t *out,
                                                const u64 *fibS) {
    PDL_ENTRY();
    __shared__ u64 sm[33];
    u64 nfree, fu = 0, big = 0;
    if (!buddy) {
        nfree = ctr->F;
        for (u64 i = threadIdx.x; i < nfree; i += blockDim.x) {
            u64 z = fe[i] - fs[i];
            fu += z;
            big = z > big ? z : big;
        }
        fu = block_sum64<1024>(fu, sm);
        big = warp_max64(big);
        __shared__ u64 bm;
        if (threadIdx.x == 0) bm = 0;
        __syncthreads();
        if (lane_id() == 0) atomicMax(&bm, big);
        __syncthreads();
        big = bm;
    } else {
        nfree = 0;
        for (int t = 0; t <= K; t++) {
            const u64 z = fibS ? fibS[t] : (1ull << t);   // Fibonacci or power-of-two class size
            nfree += ctr->bud_cnt[t];
            fu += ctr->bud_cnt[t] * z;
            if (ctr->bud_cnt[t]) big = z;
        }
    }
    if (threadIdx.x == 0) {
        out->arena_bytes = arena;
        out->align = align;
        out->live_bytes = ctr->live_units << alog2;
        out->free_bytes = fu << alog2;
        out->n_live = ctr->n_live;
        out->n_free = nfree;
        out->largest_free = big << alog2;
        out->high_water_end = ctr->high_water_units << alog2;
        out->allocs_ok = ctr->allocs_ok;
        out->allocs_failed = ctr->allocs_failed;
        out->frees_ok = ctr->frees_ok;
        out->frees_invalid = ctr->frees_invalid;
        out->frees_double = ctr->frees_double;
        out->frees_null = ctr->frees_null;
        out->metadata_bytes = meta;
        out->error_flags = ctr->error_flags;
    }
}

// ---- export ----
__global__ void k_export_free(const u64 *fs, const u64 *fe, const u64 *F_dev, int alog2, u64 *pairs, u64 cap) {
    PDL_ENTRY();
    const u64 F = *F_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < F && i < cap; i += (u64)gridDim.x * blockDim.x) {
        pairs[2 * i] = fs[i] << alog2;
        pairs[2 * i + 1] = (fe[i] - fs[i]) << alog2;
    }
}
__global__ void k_bud_keys(const u64 *list, const DevCtr *ctr, int K, u32 *key, u32 *val) {
    PDL_ENTRY();
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < ctr->bud_total; i += (u64)gridDim.x * blockDim.x) {
        int t = 0;
        while (t < K && ctr->bud_off[t + 1] <= i) t++;
        key[i] = (u32)list[i];
        val[i] = (u32)t;
    }
}
__global__ void k_export_pairs_u32(const u32 *key, const u32 *val, const u64 *n_dev, int alog2, int val_is_order,
                                   u64 *pairs, u64 cap, const u64 *fibS = nullptr) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n && i < cap; i += (u64)gridDim.x * blockDim.x) {
        pairs[2 * i] = (u64)key[i] << alog2;
        u64 z = val_is_order ? (fibS ? fibS[val[i]] : (1ull << val[i])) : ((u64)val[i] + 1);
        pairs[2 * i + 1] = z << alog2;
    }
}
__global__ void k_tbl_flags(const u64 *tbl, u64 tcap, u32 *flags) {
    PDL_ENTRY();
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < tcap; i += (u64)gridDim.x * blockDim.x)
        flags[i] = table::is_live(tbl[i]) ? 1u : 0u;
}
__global__ void k_tbl_compact(const u64 *tbl, u64 tcap, const u32 *flags, const u32 *pos, u32 *key, u32 *val,
                              u64 cap) {
    PDL_ENTRY();
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < tcap; i += (u64)gridDim.x * blockDim.x)
        if (flags[i] && pos[i] < cap) {
            u64 v = tbl[i];
            key[pos[i]] = (u32)table::slot_key(v);
            val[pos[i]] = (u32)(v & 0xFFFFFFFFull);
        }
}
__global__ void k_set_u64(u64 *p, u64 v) {
    PDL_ENTRY(); *p = v; }
__global__ void k_clamp(const u64 *in, u64 *out, u64 cap) {
    PDL_ENTRY(); *out = *in < cap ? *in : cap; }

}  // namespace

extern "C" {

size_t heap_workspace_bytes(uint64_t arena_bytes, uint64_t align, int policy, uint64_t max_live_blocks,
                            uint64_t max_batch) {
    Layout L;
    if (!make_layout(arena_bytes, align, policy, max_live_blocks, max_batch, &L)) return 0;
    return (size_t)L.total;
}

int heap_create(uint64_t arena_bytes, uint64_t align, int policy, uint64_t max_live_blocks, uint64_t max_batch,
                void *d_workspace, size_t workspace_bytes, heap_stream_t s, heap_t **h_out) {
    if (!h_out) return HEAP_EINVAL;
    *h_out = nullptr;
    Layout L;
    if (!make_layout(arena_bytes, align, policy, max_live_blocks, max_batch, &L)) return HEAP_EINVAL;
    if (!d_workspace || ((uintptr_t)d_workspace & 255)) return HEAP_EINVAL;
    if (workspace_bytes < L.total) return HEAP_ENOMEM;
    heap *h = new (std::nothrow) heap();
    if (!h) return HEAP_ENOMEM;
    policy &= ~HEAP_PARTIAL_FREE;            // the flag lives in L.partial
    h->arena = arena_bytes; h->align = align; h->policy = policy;
    h->max_live = max_live_blocks; h->max_batch = max_batch;
    h->alog2 = ilog2(align);
    {
        const char *ws = getenv("HEAP_WILD_SPLIT");
        h->wild_split = (ws && ws[0] == '0') ? 0 : 1;
        const char *bf = getenv("HEAP_BF_FLAT");
        h->bf_flat = (bf && bf[0] >= '1' && bf[0] <= '3') ? bf[0] - '0' : 0;
        const char *ew = getenv("HEAP_ENGINE_WARPS");
        h->eng_warps = (ew && (ew[0] == '1' || ew[0] == '3')) ? ew[0] - '0' : 2;
        const char *pd = getenv("HEAP_PDL");
        h->pdl = (pd && pd[0] == '0') ? 0 : 1;
        const char *bl = getenv("HEAP_BUDDY_LEVELS");
        h->bud_levels = (bl && bl[0] == '1') ? 1 : 0;
        const char *mi = getenv("HEAP_MICRO");
        const bool fitp = policy == HEAP_FIRST_FIT || policy == HEAP_NEXT_FIT || policy == HEAP_BEST_FIT ||
                          policy == HEAP_SEGFIT || policy == HEAP_TLSF;
        h->micro = (fitp && !L.partial && max_live_blocks + 1 <= micro::MICRO_F && L.A_u <= 0xFFFFFFFFull &&
                    max_batch <= micro::MICRO_N && !(mi && mi[0] == '0')) ? 1 : 0;
    }
    h->L = L;
    h->ws = d_workspace; h->ws_bytes = workspace_bytes;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    h->sms = sms;
    h->G = sms * 4;
    if (const char *gg = getenv("HEAP_GRID")) { const int g = atoi(gg); if (g > 0) h->G = g; }   // dev knob: grid of the grid-stride kernels
    if (cudaFuncSetAttribute(tlsfw::k_engine<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(tlsfw::Smem)) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    if (cudaFuncSetAttribute(tlsfw::k_engine<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(tlsfw::Smem)) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    if (cudaFuncSetAttribute(prims::k_os_scatter<u32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)prims::os_smem<u32, false>()) != cudaSuccess ||
        cudaFuncSetAttribute(prims::k_os_scatter<u32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)prims::os_smem<u32, true>()) != cudaSuccess ||
        cudaFuncSetAttribute(prims::k_os_scatter<u64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)prims::os_smem<u64, false>()) != cudaSuccess ||
        cudaFuncSetAttribute(prims::k_os_scatter<u64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)prims::os_smem<u64, true>()) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    if (cudaFuncSetAttribute(micro::k_micro_free, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)micro::FREE_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(micro::k_micro_alloc<micro::P_FF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)micro::ALLOC_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(micro::k_micro_alloc<micro::P_NF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)micro::ALLOC_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(micro::k_micro_alloc<micro::P_BF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)micro::ALLOC_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(micro::k_micro_alloc<micro::P_CLS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)micro::ALLOC_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(micro::k_micro_step<micro::P_FF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)micro::STEP_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(micro::k_micro_step<micro::P_NF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)micro::STEP_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(micro::k_micro_step<micro::P_BF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)micro::STEP_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(micro::k_micro_step<micro::P_CLS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)micro::STEP_SMEM) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    if (cudaFuncSetAttribute(fits::k_bf_engine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(fits::BfSmem)) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    if (cudaFuncSetAttribute(fits::k_bf_cls_engine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)fits::BF_ENGINE_SMEM) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    if (cudaFuncSetAttribute(fits::k_bf_spec_engine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)fits::BF_ENGINE_SMEM2) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    if (cudaFuncSetAttribute(buddy::k_free_levels, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)buddy::FREE_SMEM) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    if (cudaFuncSetAttribute(buddy::k_alloc_levels, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)buddy::ALLOC_SMEM) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    void *w = d_workspace;
    if (policy == HEAP_DOUBLE_BUDDY) {
        cudaStream_t st = (cudaStream_t)s;
        h->ctr = at<DevCtr>(w, L.o_ctr);
        h->dstats = at<heap_stats_t>(w, L.o_stats);
        h->dctr = at<dbl::Ctr>(w, L.o_dctr);
        h->flags = at<u32>(w, L.o_flags); h->pos = at<u32>(w, L.o_pos);
        h->kA = at<u32>(w, L.o_kA); h->kB = at<u32>(w, L.o_kB); h->tsum = at<u32>(w, L.o_tsum);
        h->tsz = at<u64>(w, L.o_tsz); h->toff = at<u64>(w, L.o_toff);
        h->ca = at<u64>(w, L.o_ca); h->cb = at<u64>(w, L.o_cb); h->ia = at<u32>(w, L.o_ia); h->ib = at<u32>(w, L.o_ib);
        h->ra = at<u64>(w, L.o_ra); h->rb = at<u64>(w, L.o_rb);
        h->sstats = at<heap_stats_t>(w, L.o_sstats); h->sstats2 = at<heap_stats_t>(w, L.o_sstats2);
        h->gin = at<u64>(w, L.o_gin); h->gout = at<u64>(w, L.o_gout);
        h->graphs = 1;
        h->cur = 0; h->launches = 0; h->prof_mask = 0; h->tag = HEAP_TAG_MISC;
        if (cudaMemsetAsync(h->ctr, 0, sizeof(DevCtr), st) != cudaSuccess ||
            cudaMemsetAsync(h->dctr, 0, sizeof(dbl::Ctr), st) != cudaSuccess ||
            cudaMemsetAsync(h->tsum, 0, (prims::ntiles_of(max_batch) + 16) * 4, st) != cudaSuccess) { delete h; return HEAP_ECUDA; }
        int rc = heap_create(L.dbl_A, align, HEAP_BUDDY, max_live_blocks, max_batch, at<char>(w, L.o_sub), L.sub_total,
                             s, &h->sub);
        if (rc == HEAP_OK && L.dbl_n3)
            rc = heap_create(L.dbl_n3, 1, HEAP_BUDDY, max_live_blocks, max_batch, at<char>(w, L.o_sub2), L.sub2_total, s,
                             &h->sub2);
        if (rc != HEAP_OK) { if (h->sub) heap_destroy(h->sub); delete h; return rc; }
        *h_out = h;
        return HEAP_OK;
    }
    if (policy == HEAP_HYBRID) {
        cudaStream_t st = (cudaStream_t)s;
        h->ctr = at<DevCtr>(w, L.o_ctr);
        h->dstats = at<heap_stats_t>(w, L.o_stats);
        h->pctr = at<pool::Ctr>(w, L.o_pctr);
        h->bits = at<u32>(w, L.o_bits); h->sbcnt = at<u32>(w, L.o_sbcnt); h->sbpre = at<u32>(w, L.o_sbpre);
        h->kA = at<u32>(w, L.o_kA); h->kB = at<u32>(w, L.o_kB); h->vA = at<u32>(w, L.o_vA); h->vB = at<u32>(w, L.o_vB);
        h->flags = at<u32>(w, L.o_flags); h->pos = at<u32>(w, L.o_pos); h->hist = at<u32>(w, L.o_hist);
        h->tsum = at<u32>(w, L.o_tsum);
        h->tsz = at<u64>(w, L.o_tsz); h->tout = at<u64>(w, L.o_tout); h->toff = at<u64>(w, L.o_toff);
        h->tidx = at<u32>(w, L.o_tidx); h->coff = at<u32>(w, L.o_coff); h->sstats = at<heap_stats_t>(w, L.o_sstats);
        h->gin = at<u64>(w, L.o_gin); h->gout = at<u64>(w, L.o_gout);
        h->graphs = 1;
        h->cur = 0; h->launches = 0; h->prof_mask = 0; h->tag = HEAP_TAG_MISC;
        if (cudaMemsetAsync(h->ctr, 0, sizeof(DevCtr), st) != cudaSuccess ||
            cudaMemsetAsync(h->pctr, 0, sizeof(pool::Ctr), st) != cudaSuccess ||
            cudaMemsetAsync(h->hist, 0, L.o_tsum - L.o_hist, st) != cudaSuccess ||
            cudaMemsetAsync(h->tsum, 0, L.o_tsz - L.o_tsum, st) != cudaSuccess) { delete h; return HEAP_ECUDA; }
        LAUNCH(h, pool::k_init, h->G, 256, 0, st, L.geo, h->bits, h->sbcnt, h->pctr);
        int rc = heap_create(arena_bytes - L.geo.pool_end, align, HEAP_TLSF, max_live_blocks, max_batch,
                             at<char>(w, L.o_sub), L.sub_total, s, &h->sub);
        if (rc != HEAP_OK) { delete h; return rc; }
        if (cudaGetLastError() != cudaSuccess) { heap_destroy(h->sub); delete h; return HEAP_ECUDA; }
        *h_out = h;
        return HEAP_OK;
    }
    h->ctr = at<DevCtr>(w, L.o_ctr);
    h->dstats = at<heap_stats_t>(w, L.o_stats);
    h->tbl = at<u64>(w, L.o_tbl);
    h->fs[0] = at<u64>(w, L.o_fs0); h->fs[1] = at<u64>(w, L.o_fs1);
    h->fe[0] = L.o_fe0 ? at<u64>(w, L.o_fe0) : nullptr; h->fe[1] = L.o_fe1 ? at<u64>(w, L.o_fe1) : nullptr;
    h->kA = at<u32>(w, L.o_kA); h->kB = at<u32>(w, L.o_kB); h->vA = at<u32>(w, L.o_vA); h->vB = at<u32>(w, L.o_vB);
    h->flags = at<u32>(w, L.o_flags); h->pos = at<u32>(w, L.o_pos); h->hist = at<u32>(w, L.o_hist);
    h->tsum = at<u32>(w, L.o_tsum);
    h->vs = at<u64>(w, L.o_vs); h->ve = at<u64>(w, L.o_ve); h->vsc = at<u64>(w, L.o_vsc); h->vec = at<u64>(w, L.o_vec);
    h->ms = at<u64>(w, L.o_ms); h->me = at<u64>(w, L.o_me);
    h->r = at<u64>(w, L.o_r); h->c = at<u32>(w, L.o_c); h->out = at<u64>(w, L.o_out);
    h->off = at<u32>(w, L.o_off);
    h->gin = at<u64>(w, L.o_gin); h->gout = at<u64>(w, L.o_gout);
    h->graphs = 1;
    h->cs = L.o_cs ? at<uint4>(w, L.o_cs) : nullptr;
    h->bm = L.o_bm ? at<u32>(w, L.o_bm) : nullptr; h->slot = L.o_slot ? at<u32>(w, L.o_slot) : nullptr;
    if (h->bm && cudaMemsetAsync(h->bm, 0, L.bm_bytes, (cudaStream_t)s) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    // lookback words of the single-pass sort / scan: never-published (epoch tags start above 0)
    if (cudaMemsetAsync(h->hist, 0, L.hist_cap * 4, (cudaStream_t)s) != cudaSuccess ||
        cudaMemsetAsync(h->tsum, 0, (prims::ntiles_of(L.scan_cap) + 16) * 4, (cudaStream_t)s) != cudaSuccess) {
        delete h;
        return HEAP_ECUDA;
    }
    h->tree = L.o_tree ? at<u64>(w, L.o_tree) : nullptr; h->lvl = L.o_lvl ? at<u64>(w, L.o_lvl) : nullptr;
    h->bk[0] = L.o_bk0 ? at<u64>(w, L.o_bk0) : nullptr; h->bk[1] = L.o_bk1 ? at<u64>(w, L.o_bk1) : nullptr;
    if (policy == HEAP_SEGFIT_LIFO) {
        h->ft[0] = at<u32>(w, L.o_ft0); h->ft[1] = at<u32>(w, L.o_ft1);
        h->vt = at<u32>(w, L.o_vt); h->mt = at<u32>(w, L.o_mt); h->lnext = at<u32>(w, L.o_lnext);
        // the initial whole-heap block was pushed at time 0; pushes of batches start at 1
        if (cudaMemsetAsync(h->ft[0], 0, 4, (cudaStream_t)s) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    }
    if (policy == HEAP_FIB_BUDDY) {
        h->fgeom = at<fib::Geom>(w, L.o_fgeom);
        h->flo = at<u64>(w, L.o_flo); h->fbufL = at<u64>(w, L.o_fbufL); h->frem = at<u32>(w, L.o_frem);
        h->fscr = at<u64>(w, L.o_fscr);
        if (cudaMemcpyAsync(h->fgeom, &L.fg, sizeof(fib::Geom), cudaMemcpyHostToDevice, (cudaStream_t)s) != cudaSuccess ||
            // the limit is per function and process-wide: always the largest any heap needs
            // (K <= MAXC - 3 = 45), so a small heap never lowers it under a live larger one
            cudaFuncSetAttribute(fib::k_alloc_engine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)fib::eng_smem(fib::MAXC - 3)) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    }
    if (policy == HEAP_BUDDY || policy == HEAP_FIB_BUDDY) {
        h->dtm = at<u32>(w, L.o_dtm); h->dsrc = at<u32>(w, L.o_dsrc); h->baddr = at<u64>(w, L.o_baddr); h->daddr = at<u64>(w, L.o_daddr);
        h->btm = at<u32>(w, L.o_btm); h->bsrc = at<u32>(w, L.o_bsrc);
        h->bufA = at<u64>(w, L.o_bufA); h->bufB = at<u64>(w, L.o_bufB); h->promo = at<u64>(w, L.o_promo);
        if (L.o_bq0) { h->bq[0] = at<u64>(w, L.o_bq0); h->bq[1] = at<u64>(w, L.o_bq1); }
        h->fr = at<u64>(w, L.o_fr); h->froff = at<u32>(w, L.o_froff); h->reqoff = at<u32>(w, L.o_reqoff);
    }
    if (L.partial) {
        h->L.lbm.w = at<u32>(w, L.o_lbm);      // all free: no live starts
        if (cudaMemsetAsync(h->L.lbm.w, 0, L.lbm_words * 4, (cudaStream_t)s) != cudaSuccess) { delete h; return HEAP_ECUDA; }
    }
    h->cur = 0;
    h->launches = 0;
    h->prof_mask = 0;
    h->tag = HEAP_TAG_MISC;
    cudaStream_t st = (cudaStream_t)s;
    LAUNCH(h, k_init, h->G, 256, 0, st, h->ctr, h->tbl, L.tcap, h->fs[0], policy == HEAP_BUDDY ? h->bq[0] : h->fe[0],
           L.A_u, policy == HEAP_BUDDY ? 1 : (policy == HEAP_FIB_BUDDY ? 2 : 0), L.K);
    if (policy == HEAP_FIB_BUDDY) LAUNCH(h, fib::k_init_lists, 1, 1, 0, st, h->ctr, h->fs[0], h->fgeom);
    if (policy == HEAP_FIRST_FIT || policy == HEAP_NEXT_FIT) {
        u64 offs[fits::FF_MAX_LEVELS] = {0};
        u64 n = L.cap_f, o = 0;
        for (int l = 0; l < L.nlev && l < fits::FF_MAX_LEVELS; l++) { offs[l] = o; o += n; n = (n + 31) / 32; }
        for (int l = 0; l < fits::FF_MAX_LEVELS; l++) LAUNCH(h, k_set_u64, 1, 1, 0, st, h->lvl + l, offs[l]);
    }
    if (cudaGetLastError() != cudaSuccess) { delete h; return HEAP_ECUDA; }
    *h_out = h;
    return HEAP_OK;
}

int heap_destroy(heap_t *h) {
    if (!h) return HEAP_EINVAL;
    if (h->sub) heap_destroy(h->sub);
    if (h->sub2) heap_destroy(h->sub2);
    for (auto &a : h->gs)
        for (auto &b : a)
            for (auto &g : b) {
                if (g.exec) cudaGraphExecDestroy(g.exec);
                if (g.graph) cudaGraphDestroy(g.graph);
            }
    if (h->cap) cudaStreamDestroy(h->cap);
    for (auto &r : h->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : h->pool) cudaEventDestroy(e);
    delete h;
    return HEAP_OK;
}

uint64_t heap_launch_count(const heap_t *h) {
    return h ? h->launches + (h->sub ? h->sub->launches : 0) + (h->sub2 ? h->sub2->launches : 0) : 0;
}

}  // extern "C"

// The batch sequences.  `n` bounds the request count; when `n_in` is given the actual count is
// read from device memory by the first kernel (a hybrid heap hands its TLSF heap the requests
// its pools did not take without a host round trip).
static int free_impl(heap *h, const uint64_t *d_offsets, uint64_t n, const u64 *n_in, cudaStream_t s) {
    const Layout &L = h->L;
    const int cur = h->cur, nxt = cur ^ 1;
    const bool fibp = h->policy == HEAP_FIB_BUDDY;
    const bool bud = h->policy == HEAP_BUDDY || fibp;
    DevCtr *C = h->ctr;
    u64 *n_dev = &C->tmp[0];
    if (h->micro) {          // small heap: the whole free batch in one single-CTA launch (micro.cuh)
        TAG(h, HEAP_TAG_MICRO);
        LAUNCH(h, micro::k_micro_free, 1, micro::MT, micro::FREE_SMEM, s, (const u64 *)d_offsets, n, n_in, h->alog2,
               L.A_u, h->fs[cur], h->fe[cur], h->fs[nxt], h->fe[nxt], h->tbl, L.tcap - 1, L.tcap / table::LINE,
               L.cap_f, C, h->hidx, h->hlen);
        h->cur = nxt;
        if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
        return HEAP_OK;
    }
    // 1. classify (null / unaligned / out of range) and compact the candidate keys
    TAG(h, HEAP_TAG_CLASSIFY);
    const int kbits = ilog2(L.A_u - 1 > 0 ? L.A_u - 1 : 1) + 1;   // address-sort key width (4 passes at most)
    LAUNCH(h, fits::k_free_classify, h->G, prims::NT, 0, s, (const u64 *)d_offsets, n, n_in, h->alog2, L.A_u, h->kA,
           h->flags, n_dev, C, (kbits + 7) / 8);
    TAG(h, HEAP_TAG_SCAN);
    scan(h, h->flags, h->pos, n_dev, &C->nk, s);
    TAG(h, HEAP_TAG_COMPACT);
    LAUNCH(h, fits::k_compact<u32>, h->G, 256, 0, s, h->kA, h->flags, h->pos, n_dev, h->kB);
    // 2. sort the keys (address order; duplicates become adjacent)
    TAG(h, HEAP_TAG_SORT);   // (digits counted by k_free_classify)
    int rb = radix_sort<u32, false>(h, h->kB, h->kA, nullptr, nullptr, &C->nk, kbits, s, true);
    u32 *keys = rb ? h->kA : h->kB;
    // 3. block-table lookup + delete; classify double / invalid
    TAG(h, HEAP_TAG_LOOKUP);
    if (L.partial) {
        // containing-block resolution through the live-start bitmap, then the winners' table
        // updates (tombstone or shrink) — partial.cuh, reading C29
        LAUNCH(h, partial::k_resolve, h->G, 256, 0, s, keys, &C->nk, h->tbl, L.tcap - 1, L.tcap / table::LINE,
               L.lbm, h->fs[cur], &C->F, h->vA, h->vB, h->vs, C);
        LAUNCH(h, partial::k_apply, h->G, 256, 0, s, keys, &C->nk, h->vA, h->vB, h->vs, h->tbl, L.tcap - 1,
               L.tcap / table::LINE, L.lbm, h->flags, h->vs, h->ve, C);
    } else {
        LAUNCH(h, fits::k_free_lookup, h->G, 256, 0, s, keys, &C->nk, h->tbl, L.tcap - 1, L.tcap / table::LINE,
               bud ? nullptr : h->fs[cur], bud ? nullptr : &C->F, bud ? h->fs[cur] : nullptr, L.K,
               h->flags, h->vs, h->ve, C);
    }
    TAG(h, HEAP_TAG_SCAN);
    scan(h, h->flags, h->pos, &C->nk, &C->nv, s);
    TAG(h, HEAP_TAG_COMPACT);
    LAUNCH(h, fits::k_compact2<u64>, h->G, 256, 0, s, h->vs, h->ve, h->flags, h->pos, &C->nk, h->vsc, h->vec);
    if (!bud) {
        // 4. merge path with the free array, 5. coalesce maximal runs
        const bool lifo = h->policy == HEAP_SEGFIT_LIFO;
        TAG(h, HEAP_TAG_MERGE);
        if (lifo)   // the valid frees are pushed in ascending address order: stamps clock + rank
            LAUNCH(h, fits::k_free_stamps, h->G, 256, 0, s, &C->nv, C, h->vt);
        LAUNCH(h, prims::k_merge, h->G, prims::NT, 0, s, h->fs[cur], h->fe[cur], &C->F, h->vsc, h->vec, &C->nv,
               h->ms, h->me, &C->M, lifo ? h->ft[cur] : nullptr, lifo ? h->vt : nullptr, lifo ? h->mt : nullptr);
        TAG(h, HEAP_TAG_COALESCE);
        LAUNCH(h, fits::k_coal_flags, h->G, 256, 0, s, h->ms, h->me, &C->M, h->flags);
        scan(h, h->flags, h->pos, &C->M, &C->F, s);
        LAUNCH(h, fits::k_coal_write, h->G, 256, 0, s, h->ms, h->me, &C->M, h->flags, h->pos, h->fs[nxt],
               h->fe[nxt], L.cap_f, C);
        if (lifo) {   // a coalesced run is pushed by its last free: the run's largest stamp
            LAUNCH(h, fits::k_coal_stamp_head, h->G, 256, 0, s, h->mt, &C->M, h->flags, h->pos, h->ft[nxt], L.cap_f);
            LAUNCH(h, fits::k_coal_stamp, h->G, 256, 0, s, h->mt, &C->M, h->flags, h->pos, h->ft[nxt], L.cap_f);
            LAUNCH(h, fits::k_clock_add, 1, 1, 0, s, C, &C->nv, 0ull);
        }
    } else {
        // 4b. group freed blocks by order, 5b. level-by-level buddy merge
        TAG(h, HEAP_TAG_BUDDY_FREE);
        if (!fibp && !h->bud_levels) {
            // parallel form (buddy.cuh): old blocks in address order, merged with the freed ones,
            // coalesced into maximal runs, each run's greedy decomposition grouped by order
            // the free set is kept in address order too (bq, maintained by both phases)
            LAUNCH(h, buddy::k_bud_merge, h->G, 256, 0, s, h->bq[cur], C, h->vsc, h->vec, &C->nv, h->ms, h->me, &C->M);
            LAUNCH(h, fits::k_coal_flags, h->G, 256, 0, s, h->ms, h->me, &C->M, h->flags);
            scan(h, h->flags, h->pos, &C->M, &C->tmp[2], s);
            LAUNCH(h, fits::k_coal_write, h->G, 256, 0, s, h->ms, h->me, &C->M, h->flags, h->pos, h->bufA, h->bufB,
                   L.bud_cap, C);
            LAUNCH(h, buddy::k_bud_count, h->G, 256, 0, s, h->bufA, h->bufB, &C->tmp[2], h->flags);
            scan(h, h->flags, h->pos, &C->tmp[2], &C->tmp[3], s);
            LAUNCH(h, buddy::k_bud_write, h->G, prims::OS_NT, 0, s, h->bufA, h->bufB, &C->tmp[2], h->pos, h->promo, h->kA,
                   h->vA, h->bq[nxt], L.cap_f, C);
            const int r2 = radix_sort<u32, true>(h, h->kA, h->kB, h->vA, h->vB, &C->tmp[3], 8, s, true);
            LAUNCH(h, buddy::k_bud_lists, h->G, 256, 0, s, r2 ? h->vB : h->vA, &C->tmp[3], h->promo, h->fs[nxt], L.K, C);
            h->cur = nxt;
            if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
            return HEAP_OK;
        }
        if (fibp) LAUNCH(h, fib::k_free_classes, h->G, 256, 0, s, h->vsc, h->vec, &C->nv, h->fgeom, h->kA, h->vA);
        else LAUNCH(h, buddy::k_free_orders, h->G, 256, 0, s, h->vsc, h->vec, &C->nv, h->kA, h->vA);
        int r2 = radix_sort<u32, true>(h, h->kA, h->kB, h->vA, h->vB, &C->nv, 8, s);
        u32 *ok = r2 ? h->kB : h->kA, *ov = r2 ? h->vB : h->vA;
        LAUNCH(h, fits::k_cls_off, h->G, 256, 0, s, ok, &C->nv, L.K + 1, h->froff);
        LAUNCH(h, buddy::k_gather_u64, h->G, 256, 0, s, h->vsc, ov, &C->nv, h->fr);
        if (fibp)
            LAUNCH(h, fib::k_free_levels, 1, fib::NT, 0, s, h->fs[cur], h->fs[nxt], h->fr, h->froff, h->fbufL, h->frem,
                   h->promo, h->bufA, h->fgeom, C);
        else
            LAUNCH(h, buddy::k_free_levels, 1, buddy::NT, buddy::FREE_SMEM, s, h->fs[cur], h->fs[nxt], h->fr, h->froff,
                   h->bufA, h->bufB, h->promo, L.K, C);
    }
    h->cur = nxt;
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    return HEAP_OK;
}

static int alloc_impl(heap *h, const uint64_t *d_sizes, uint64_t *d_out, uint64_t n, const u64 *n_in, cudaStream_t s) {
    const Layout &L = h->L;
    const int cur = h->cur, nxt = cur ^ 1;
    DevCtr *C = h->ctr;
    if (h->policy == HEAP_FIB_BUDDY) {
        // one warp serves the requests in order (fib.cuh), then each class's list is rebuilt
        TAG(h, HEAP_TAG_BUDDY_ALLOC);
        u64 *fo = h->fscr, *lcnt = h->fscr + (fib::MAXC + 2), *noff = h->fscr + 2 * (fib::MAXC + 2);
        LAUNCH(h, fib::k_alloc_engine, 1, 32, fib::eng_smem(L.fg.K), s, (const u64 *)d_sizes, n, n_in, h->alog2,
               h->fs[cur], h->fgeom, C, h->out, h->r, fo, h->flo, lcnt, noff);
        LAUNCH(h, fib::k_alloc_rebuild, L.K + 1, fib::NT, 0, s, h->fs[cur], h->fs[nxt], h->fgeom, C, fo, h->flo, lcnt,
               noff);
        LAUNCH(h, fib::k_alloc_commit, 1, 1, 0, s, C, h->fgeom, noff);
        TAG(h, HEAP_TAG_FINISH);
        LAUNCH(h, fits::k_alloc_finish, h->G, 256, 0, s, h->r, h->out, n, n_in, h->alog2, (u64 *)d_out,
               h->tbl, L.tcap - 1, L.tcap / table::LINE, C, h->max_live, (const u32 *)nullptr);
        h->cur = nxt;
        maybe_rebuild(h, s);
        if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
        return HEAP_OK;
    }
    if (h->policy == HEAP_BUDDY) {
        TAG(h, HEAP_TAG_BUDDY_ALLOC);
        LAUNCH(h, buddy::k_alloc_orders, h->G, prims::OS_NT, 0, s, (const u64 *)d_sizes, n, n_in, h->alog2, L.A_u, L.K,
               h->kA, h->vA, &C->tmp[0], C);
        radix_sort<u32, true>(h, h->kA, h->kB, h->vA, h->vB, &C->tmp[0], 8, s, true);   // 1 pass: result in kB/vB
        LAUNCH(h, buddy::k_alloc_levels, 1, buddy::NT, buddy::ALLOC_SMEM, s, h->vB, (const u32 *)nullptr, h->fs[cur], h->fs[nxt], h->dtm,
               h->dsrc, h->daddr, h->baddr, h->btm, h->bsrc, h->out, L.K, C);
        LAUNCH(h, buddy::k_bud_scatter, h->G, 256, 0, s, h->dsrc, h->daddr, C, h->out, h->fs[cur], h->fs[nxt], L.K);
        if (!h->bud_levels) {   // the address-ordered free set: survivors compacted, leftovers inserted
            LAUNCH(h, buddy::k_bud_qflags, h->G, 256, 0, s, h->bq[cur], C, h->flags);
            scan(h, h->flags, h->pos, &C->bud_qn, &C->tmp[2], s);
            LAUNCH(h, buddy::k_bud_qwrite, h->G, 256, 0, s, h->bq[cur], h->flags, h->pos, &C->tmp[2], L.K,
                   h->bq[nxt], C);
        }
        TAG(h, HEAP_TAG_FINISH);   // (units 2^order read from the order keys: no k_alloc_r pass)
        LAUNCH(h, fits::k_alloc_finish, h->G, 256, 0, s, h->r, h->out, n, n_in, h->alog2, (u64 *)d_out,
               h->tbl, L.tcap - 1, L.tcap / table::LINE, C, h->max_live, (const u32 *)h->kA);
        h->cur = nxt;
        maybe_rebuild(h, s);
        if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
        return HEAP_OK;
    }
    if (h->micro) {          // small heap: the whole alloc batch in one single-CTA launch (micro.cuh)
        TAG(h, HEAP_TAG_MICRO);
#define MICRO_ALLOC(P)                                                                                          \
    LAUNCH(h, micro::k_micro_alloc<P>, 1, micro::MT, micro::ALLOC_SMEM, s, (const u64 *)d_sizes, n, n_in, h->alog2, \
           L.A_u, L.L, h->fs[cur], h->fe[cur], h->fs[nxt], h->fe[nxt], (u64 *)d_out, h->tbl, L.tcap - 1,             \
           L.tcap / table::LINE, L.tcap, h->ms, C, h->max_live)
        switch (h->policy) {
            case HEAP_FIRST_FIT: MICRO_ALLOC(micro::P_FF); break;
            case HEAP_NEXT_FIT: MICRO_ALLOC(micro::P_NF); break;
            case HEAP_BEST_FIT: MICRO_ALLOC(micro::P_BF); break;
            default: MICRO_ALLOC(micro::P_CLS); break;
        }
#undef MICRO_ALLOC
        h->cur = nxt;
        if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
        return HEAP_OK;
    }
    const bool lifo = (h->policy == HEAP_SEGFIT_LIFO);
    const bool cls = (h->policy == HEAP_TLSF || h->policy == HEAP_SEGFIT || lifo);
    TAG(h, HEAP_TAG_ALLOC_PREP);
    const bool wild = cls && !lifo;          // the wilderness split needs the batch's totals
    if (wild) LAUNCH(h, fits::k_zero2, 1, 1, 0, s, C->wild_acc);
    LAUNCH(h, fits::k_alloc_prep, h->G, 256, 0, s, (const u64 *)d_sizes, n, n_in, h->alog2, L.A_u, L.L, cls ? 1 : 0, h->r, h->c,
           wild ? C->wild_acc : (u64 *)nullptr);
    if (lifo) {
        // class-major, newest-push-first CSR (the bins as the paper's stacks), then the engine
        TAG(h, HEAP_TAG_INDEX);
        LAUNCH(h, fits::k_lifo_keys, h->G, 256, 0, s, h->fs[cur], h->fe[cur], h->ft[cur], &C->F, h->bk[0], h->vA);
        int rb = radix_sort<u64, true>(h, h->bk[0], h->bk[1], h->vA, h->vB, &C->F, 32 + ilog2((u64)L.NC) + 1, s);
        u64 *sk = h->bk[rb];
        u32 *sv = rb ? h->vB : h->vA;
        LAUNCH(h, fits::k_u64_hi, h->G, 256, 0, s, sk, &C->F, h->kA);
        LAUNCH(h, fits::k_cls_off, h->G, 256, 0, s, h->kA, &C->F, L.NC, h->off);
        LAUNCH(h, tlsfw::k_csr_data, h->G, 256, 0, s, sv, h->fs[cur], h->fe[cur], &C->F, h->cs);
        TAG(h, HEAP_TAG_ENGINE);
        tlsfw::Csr csr{h->cs};
        tlsfw::Lifo lf{h->lnext, h->ft[cur], &C->lifo_clock};
        LAUNCH(h, tlsfw::k_engine<true>, 1, 32, sizeof(tlsfw::Smem), s, csr, h->off, h->fs[cur], h->fe[cur], h->r,
               h->c, n, h->out, nullptr, 0ull, 0ull, 0ull, h->slot, L.NC, L.L, C->eng, lf, n_in, (const u32 *)nullptr);
        TAG(h, HEAP_TAG_INDEX);
        LAUNCH(h, fits::k_clock_add, 1, 1, 0, s, C, n_in, (u64)n);
    } else if (cls) {
        TAG(h, HEAP_TAG_INDEX);
        const int cbits = ilog2((u64)L.NC) + 1;
        LAUNCH(h, fits::k_cls_keys, h->G, 256, 0, s, h->fs[cur], h->fe[cur], &C->F, L.L, h->kA, h->vA, C,
               (cbits + 7) / 8);
        int rb = radix_sort<u32, true>(h, h->kA, h->kB, h->vA, h->vB, &C->F, cbits, s, true);
        u32 *sk = rb ? h->kB : h->kA, *sv = rb ? h->vB : h->vA;
        LAUNCH(h, fits::k_cls_off, h->G, 256, 0, s, sk, &C->F, L.NC, h->off);
        LAUNCH(h, tlsfw::k_csr_data, h->G, 256, 0, s, sv, h->fs[cur], h->fe[cur], &C->F, h->cs);
        LAUNCH(h, tlsfw::k_wild_setup, 1, 32, 0, s, h->off, sv, h->fs[cur], h->fe[cur], n, n_in, L.NC, L.L,
               h->wild_split, C);
        TAG(h, HEAP_TAG_ENGINE);
        {
            tlsfw::Csr csr{h->cs};
            LAUNCH(h, tlsfw::k_engine<false>, 1, h->eng_warps * 32, sizeof(tlsfw::Smem), s, csr, h->off, h->fs[cur], h->fe[cur], h->r,
                   h->c, n, h->out, h->bm, L.bm_w0, L.bm_w1, L.bm_w2, h->slot, L.NC, L.L, C->eng, tlsfw::Lifo{}, n_in,
                   (const u32 *)C->wild);
        }
        TAG(h, HEAP_TAG_FINISH);
        LAUNCH(h, tlsfw::k_wild_flags, h->G, 256, 0, s, h->out, h->r, C, h->flags);
        scan(h, h->flags, h->pos, &C->wild_n, &C->wild_total, s);
        LAUNCH(h, tlsfw::k_wild_apply, h->G, 256, 0, s, h->out, h->pos, C, h->fs[cur]);
        TAG(h, HEAP_TAG_INDEX);
        LAUNCH(h, tlsfw::k_bitheap_clear, h->G, 256, 0, s, h->fs[cur], h->fe[cur], &C->F, h->slot, h->bm,
               L.bm_w0, L.bm_w1, L.bm_w2, L.NC, L.L);
    } else if (h->policy == HEAP_FIRST_FIT || h->policy == HEAP_NEXT_FIT) {
        u64 offs[fits::FF_MAX_LEVELS] = {0};
        u64 m = L.cap_f, o = 0;
        for (int l = 0; l < L.nlev; l++) { offs[l] = o; o += m; m = (m + 31) / 32; }
        TAG(h, HEAP_TAG_INDEX);
        LAUNCH(h, fits::k_ff_leaves, h->G, 256, 0, s, h->fs[cur], h->fe[cur], &C->F, h->tree);
        for (int l = 1; l < L.nlev; l++)
            LAUNCH(h, fits::k_ff_level, h->G, 256, 0, s, h->tree + offs[l - 1], h->tree + offs[l], &C->F, l);
        TAG(h, HEAP_TAG_ENGINE);
        LAUNCH(h, fits::k_ff_engine, 1, 32, 0, s, h->tree, h->lvl, L.nlev, h->fs[cur], &C->F, h->r, n, n_in, h->out,
               h->policy == HEAP_NEXT_FIT ? &C->rover : (u64 *)nullptr);
    } else {   // BEST_FIT
        TAG(h, HEAP_TAG_INDEX);
        int bits = 33 + L.FB;
        LAUNCH(h, fits::k_bf_keys, h->G, 256, 0, s, h->fs[cur], h->fe[cur], &C->F, L.FB, h->bk[0], C, (bits + 7) / 8);
        int rb = radix_sort<u64, false>(h, h->bk[0], h->bk[1], nullptr, nullptr, &C->F, bits, s, true);
        u64 *keys = h->bk[rb];
        TAG(h, HEAP_TAG_ENGINE);
        if (h->bf_flat) {      // ablation (HEAP_BF_FLAT=1): the one-array engine
            size_t smem = L.cap_f * 8;
            if (smem <= 200 * 1024) {
                cudaFuncSetAttribute(fits::k_bf_engine_flat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                LAUNCH(h, fits::k_bf_engine_flat<true>, 1, 32, smem, s, keys, &C->F, L.FB, h->fs[cur], h->r, n, n_in, h->out);
            } else {
                LAUNCH(h, fits::k_bf_engine_flat<false>, 1, 32, 0, s, keys, &C->F, L.FB, h->fs[cur], h->r, n, n_in, h->out);
            }
        } else if (h->bf_flat == 2) {   // ablation (HEAP_BF_FLAT=2): the blocked engine without the class index
            LAUNCH(h, fits::k_bf_engine, 1, 32, sizeof(fits::BfSmem), s, keys, &C->F, L.FB, h->fs[cur], h->r, n, n_in,
                   h->out);
        } else if (h->bf_flat == 3) {   // ablation (HEAP_BF_FLAT=3): one request at a time on the class index
            LAUNCH(h, fits::k_bf_cls_engine, 1, 32, fits::BF_ENGINE_SMEM, s, keys, &C->F, L.FB, h->fs[cur], h->r, n,
                   n_in, h->out, L.A_u <= 0xFFFFFFFFull ? 1 : 0, C->eng);
        } else {
            LAUNCH(h, fits::k_bf_spec_engine, 1, 32, fits::BF_ENGINE_SMEM2, s, keys, &C->F, L.FB, h->fs[cur], h->r, n,
                   n_in, h->out, L.A_u <= 0xFFFFFFFFull ? 1 : 0, C->eng);
        }
    }
    // compact the surviving pieces into the other buffer (address order is kept)
    TAG(h, HEAP_TAG_COMPACT);
    LAUNCH(h, fits::k_piece_flags, h->G, 256, 0, s, h->fs[cur], h->fe[cur], &C->F, h->flags);
    scan(h, h->flags, h->pos, &C->F, &C->tmp[1], s);
    LAUNCH(h, fits::k_compact<u64>, h->G, 256, 0, s, h->fs[cur], h->flags, h->pos, &C->F, h->fs[nxt]);
    LAUNCH(h, fits::k_compact<u64>, h->G, 256, 0, s, h->fe[cur], h->flags, h->pos, &C->F, h->fe[nxt]);
    if (lifo) LAUNCH(h, fits::k_compact<u32>, h->G, 256, 0, s, h->ft[cur], h->flags, h->pos, &C->F, h->ft[nxt]);
    LAUNCH(h, k_set_F, 1, 1, 0, s, C);
    TAG(h, HEAP_TAG_FINISH);
    LAUNCH(h, fits::k_alloc_finish, h->G, 256, 0, s, h->r, h->out, n, n_in, h->alog2, (u64 *)d_out, h->tbl, L.tcap - 1,
           L.tcap / table::LINE, C, h->max_live, (const u32 *)nullptr);
    if (L.partial) LAUNCH(h, partial::k_set_bits, h->G, 256, 0, s, h->out, n, n_in, L.lbm);
    h->cur = nxt;
    maybe_rebuild(h, s);
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    return HEAP_OK;
}

static int hybrid_free(heap *h, const uint64_t *d_offsets, uint64_t n, const u64 *n_in, cudaStream_t s);
static int hybrid_alloc(heap *h, const uint64_t *d_sizes, uint64_t *d_out, uint64_t n, const u64 *n_in, cudaStream_t s);

// ---- HEAP_DOUBLE_BUDDY (dbuddy.cuh): split a batch between the two buddy heaps ----
static int double_free(heap *h, const uint64_t *d_offsets, uint64_t n, const u64 *n_in, cudaStream_t s) {
    dbl::Ctr *D = h->dctr;
    const int has3 = h->sub2 != nullptr;
    TAG(h, HEAP_TAG_CLASSIFY);
    LAUNCH(h, dbl::k_free_split, h->G, 256, 0, s, (const u64 *)d_offsets, n, n_in, h->L.dbl_A, 3 * h->align, has3,
           h->flags, h->kA, h->tsz, h->toff, D);
    TAG(h, HEAP_TAG_SCAN);
    scan(h, h->flags, h->pos, &D->nreq, &D->nA, s);
    scan(h, h->kA, h->kB, &D->nreq, &D->nB, s);
    TAG(h, HEAP_TAG_COMPACT);
    LAUNCH(h, dbl::k_compact_idx, h->G, 256, 0, s, h->tsz, h->flags, h->pos, &D->nreq, h->ca, (u32 *)nullptr);
    LAUNCH(h, dbl::k_compact_idx, h->G, 256, 0, s, h->toff, h->kA, h->kB, &D->nreq, h->cb, (u32 *)nullptr);
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    int rc = free_impl(h->sub, (const uint64_t *)h->ca, n, &D->nA, s);
    if (rc == HEAP_OK && has3) rc = free_impl(h->sub2, (const uint64_t *)h->cb, n, &D->nB, s);
    return rc;
}

static int double_alloc(heap *h, const uint64_t *d_sizes, uint64_t *d_out, uint64_t n, const u64 *n_in, cudaStream_t s) {
    dbl::Ctr *D = h->dctr;
    const int has3 = h->sub2 != nullptr;
    TAG(h, HEAP_TAG_ALLOC_PREP);
    LAUNCH(h, dbl::k_alloc_split, h->G, 256, 0, s, (const u64 *)d_sizes, n, n_in, h->alog2, h->arena / h->align, has3,
           h->flags, h->kA, h->tsz, h->toff, D);
    TAG(h, HEAP_TAG_SCAN);
    scan(h, h->flags, h->pos, &D->nreq, &D->nA, s);
    scan(h, h->kA, h->kB, &D->nreq, &D->nB, s);
    TAG(h, HEAP_TAG_COMPACT);
    LAUNCH(h, dbl::k_compact_idx, h->G, 256, 0, s, h->tsz, h->flags, h->pos, &D->nreq, h->ca, h->ia);
    LAUNCH(h, dbl::k_compact_idx, h->G, 256, 0, s, h->toff, h->kA, h->kB, &D->nreq, h->cb, h->ib);
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    int rc = alloc_impl(h->sub, (const uint64_t *)h->ca, (uint64_t *)h->ra, n, &D->nA, s);
    if (rc == HEAP_OK && has3) rc = alloc_impl(h->sub2, (const uint64_t *)h->cb, (uint64_t *)h->rb, n, &D->nB, s);
    if (rc != HEAP_OK) return rc;
    TAG(h, HEAP_TAG_FINISH);
    LAUNCH(h, dbl::k_scatter, h->G, 256, 0, s, h->ra, h->ia, &D->nA, 0ull, 1ull, (u64 *)d_out);
    if (has3) LAUNCH(h, dbl::k_scatter, h->G, 256, 0, s, h->rb, h->ib, &D->nB, h->L.dbl_A, 3 * h->align, (u64 *)d_out);
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    return HEAP_OK;
}

static int batch_free(heap *h, const uint64_t *in, uint64_t n, const u64 *n_in, cudaStream_t s) {
    if (h->policy == HEAP_DOUBLE_BUDDY) return double_free(h, in, n, n_in, s);
    return h->policy == HEAP_HYBRID ? hybrid_free(h, in, n, n_in, s) : free_impl(h, in, n, n_in, s);
}
static int batch_alloc(heap *h, const uint64_t *in, uint64_t *out, uint64_t n, const u64 *n_in, cudaStream_t s) {
    if (h->policy == HEAP_DOUBLE_BUDDY) return double_alloc(h, in, out, n, n_in, s);
    return h->policy == HEAP_HYBRID ? hybrid_alloc(h, in, out, n, n_in, s) : alloc_impl(h, in, out, n, n_in, s);
}

// ---- CUDA-graph path ----
// A batch is ~30-90 small launches whose host-side arguments depend only on the policy, the
// capacities and the ping-pong state (every count is read from device memory), so one graph per
// (op, ping-pong state) serves every n: its first node writes n to the device, a memcpy node
// stages the caller's request words into the workspace, the captured batch runs on the staging
// buffers with a device-side count, and (alloc) a memcpy node copies the results out.  Each call
// only patches those three nodes and launches the graph: one launch instead of dozens.
__global__ void k_set_req_n(DevCtr *ctr, u64 n) {
    PDL_ENTRY(); ctr->req_n = n; }

#define GRAPH_TRY(x)                                                                       \
    do {                                                                                   \
        cudaError_t _e = (x);                                                              \
        if (_e != cudaSuccess) {                                                           \
            if (getenv("HEAP_DEBUG")) fprintf(stderr, "libheap graph: %s: %s\n", #x, cudaGetErrorString(_e)); \
            return HEAP_ECUDA;                                                             \
        }                                                                                  \
    } while (0)

static bool use_graph(heap *h, cudaStream_t s) {
    if (!h->graphs || h->prof_mask || (h->sub && h->sub->prof_mask) || (h->sub2 && h->sub2->prof_mask)) return false;
    // a single-launch (micro) batch is already one launch: the graph's count-setting kernel and
    // staging copies would only add nodes (measured: config 1, 4 of the 7 nodes per batch)
    if (h->micro && !getenv("HEAP_MICRO_GRAPH")) return false;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone) return false;
    return true;
}

static int graph_batch(heap *h, int op, const uint64_t *in, uint64_t *out, uint64_t n, cudaStream_t s) {
    heap *sub = h->sub;
    const int sc = sub ? sub->cur : 0;
    heap::GSlot &g = h->gs[op][h->cur][sc];
    DevCtr *ctr = h->ctr;
    void *kargs[2] = {(void *)&ctr, (void *)&n};
    cudaKernelNodeParams kp = {};
    kp.func = (void *)k_set_req_n;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = kargs;
    if (!g.exec) {
        if (!h->cap) CUDA_TRY(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
        const int cur0 = h->cur;
        heap *sub2 = h->sub2;
        const int sc2 = sub2 ? sub2->cur : 0;
        const u64 l0 = h->launches, ls0 = sub ? sub->launches : 0, ls2 = sub2 ? sub2->launches : 0;
        cudaGraph_t body = nullptr;
        CUDA_TRY(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
        const uint64_t *gin = (const uint64_t *)h->gin;
        int rc = op == 0 ? batch_free(h, gin, h->max_batch, &ctr->req_n, h->cap)
                         : batch_alloc(h, gin, (uint64_t *)h->gout, h->max_batch, &ctr->req_n, h->cap);
        cudaError_t e = cudaStreamEndCapture(h->cap, &body);
        g.cur_after = h->cur;
        g.subcur_after = sub ? sub->cur : 0;
        g.sub2cur_after = sub2 ? sub2->cur : 0;
        g.nlaunch = (h->launches - l0) + (sub ? sub->launches - ls0 : 0) + (sub2 ? sub2->launches - ls2 : 0) + 1;
        h->cur = cur0;                                 // nothing ran yet: restore the host state
        h->launches = l0;
        if (sub) { sub->cur = sc; sub->launches = ls0; }
        if (sub2) { sub2->cur = sc2; sub2->launches = ls2; }
        if (rc != HEAP_OK || e != cudaSuccess) {
            if (getenv("HEAP_DEBUG")) fprintf(stderr, "libheap graph: capture rc %d: %s\n", rc, cudaGetErrorString(e));
            if (body) cudaGraphDestroy(body);
            cudaGetLastError();
            return rc ? rc : HEAP_ECUDA;
        }
        cudaGraph_t G = nullptr;
        cudaGraphNode_t child = nullptr;
        GRAPH_TRY(cudaGraphCreate(&G, 0));
        GRAPH_TRY(cudaGraphAddKernelNode(&g.set_n, G, nullptr, 0, &kp));
        GRAPH_TRY(cudaGraphAddMemcpyNode1D(&g.cin, G, &g.set_n, 1, h->gin, in, n * 8, cudaMemcpyDefault));
        GRAPH_TRY(cudaGraphAddChildGraphNode(&child, G, &g.cin, 1, body));
        if (op == 1) GRAPH_TRY(cudaGraphAddMemcpyNode1D(&g.cout, G, &child, 1, out, h->gout, n * 8, cudaMemcpyDefault));
        cudaGraphExec_t ex = nullptr;
        GRAPH_TRY(cudaGraphInstantiate(&ex, G, 0));
        g.exec = ex;
        g.graph = G;
        cudaGraphDestroy(body);
    } else {
        GRAPH_TRY(cudaGraphExecKernelNodeSetParams(g.exec, g.set_n, &kp));
        GRAPH_TRY(cudaGraphExecMemcpyNodeSetParams1D(g.exec, g.cin, h->gin, in, n * 8, cudaMemcpyDefault));
        if (op == 1) GRAPH_TRY(cudaGraphExecMemcpyNodeSetParams1D(g.exec, g.cout, out, h->gout, n * 8, cudaMemcpyDefault));
    }
    GRAPH_TRY(cudaGraphLaunch(g.exec, s));
    h->cur = g.cur_after;
    if (sub) sub->cur = g.subcur_after;
    if (h->sub2) h->sub2->cur = g.sub2cur_after;
    h->launches += g.nlaunch;
    return HEAP_OK;
}

// ---- HEAP_HYBRID (pool.cuh): pools in front of the TLSF heap `sub` ----
static int hybrid_free(heap *h, const uint64_t *d_offsets, uint64_t n, const u64 *n_in, cudaStream_t s) {
    const pool::Geom &G = h->L.geo;
    pool::Ctr *P = h->pctr;
    TAG(h, HEAP_TAG_CLASSIFY);
    LAUNCH(h, pool::k_free, h->G, 256, 0, s, (const u64 *)d_offsets, n, n_in, G, h->bits, h->sbcnt, P, h->flags, h->toff);
    TAG(h, HEAP_TAG_SCAN);
    scan(h, h->flags, h->pos, &P->nreq, &P->n_tl, s);
    TAG(h, HEAP_TAG_COMPACT);
    LAUNCH(h, fits::k_compact<u64>, h->G, 256, 0, s, h->toff, h->flags, h->pos, &P->nreq, h->tsz);
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    return free_impl(h->sub, (const uint64_t *)h->tsz, n, &P->n_tl, s);
}

static int hybrid_alloc(heap *h, const uint64_t *d_sizes, uint64_t *d_out, uint64_t n, const u64 *n_in, cudaStream_t s) {
    const pool::Geom &G = h->L.geo;
    pool::Ctr *P = h->pctr;
    // 1. pool class per request, stable counting sort by class (request order within a class)
    TAG(h, HEAP_TAG_ALLOC_PREP);
    LAUNCH(h, pool::k_keys, h->G, 256, 0, s, (const u64 *)d_sizes, n, n_in, G, h->kA, h->vA, P);
    TAG(h, HEAP_TAG_SORT);
    int rb = radix_sort<u32, true>(h, h->kA, h->kB, h->vA, h->vB, &P->nreq, 4, s);
    u32 *sk = rb ? h->kB : h->kA, *sv = rb ? h->vB : h->vA;
    TAG(h, HEAP_TAG_INDEX);
    LAUNCH(h, fits::k_cls_off, h->G, 256, 0, s, sk, &P->nreq, G.J + 1, h->coff);
    LAUNCH(h, pool::k_take, 1, 1, 0, s, h->coff, G, P);
    // 2. ranks of the free slots: scan of the superblock free counts, then one warp per superblock
    scan(h, h->sbcnt, h->sbpre, &P->nsb, &P->scan_total, s);
    TAG(h, HEAP_TAG_ENGINE);
    LAUNCH(h, pool::k_select, h->G, 256, 0, s, G, h->bits, h->sbcnt, h->sbpre, h->coff, sv, P, (u64 *)d_out);
    // 3. everything else, in request order, through the TLSF heap
    TAG(h, HEAP_TAG_COMPACT);
    LAUNCH(h, pool::k_tl_flags, h->G, 256, 0, s, sk, sv, h->coff, &P->nreq, G, P, h->flags);
    scan(h, h->flags, h->pos, &P->nreq, &P->n_tl, s);
    LAUNCH(h, pool::k_tl_compact, h->G, 256, 0, s, (const u64 *)d_sizes, h->flags, h->pos, &P->nreq, h->tsz, h->tidx);
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    int rc = alloc_impl(h->sub, (const uint64_t *)h->tsz, (uint64_t *)h->tout, n, &P->n_tl, s);
    if (rc != HEAP_OK) return rc;
    TAG(h, HEAP_TAG_FINISH);
    LAUNCH(h, pool::k_tl_scatter, h->G, 256, 0, s, h->tout, h->tidx, &P->n_tl, G.pool_end, (u64 *)d_out);
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    return HEAP_OK;
}

// offsets by handle: d_table[d_idx[i]] (an index >= table_len frees nothing).  A single-launch
// (micro) heap reads them inside its free kernel; other heaps gather them into the graph staging
// buffer of the alloc side (unused during a free batch) and run the plain free batch on it.
__global__ void k_gather_handles(const u64 *__restrict__ table, u64 tlen, const u64 *__restrict__ idx, u64 n,
                                 u64 *__restrict__ out) {
    PDL_ENTRY();
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 x = idx[i];
        out[i] = x < tlen ? table[x] : HEAP_NULL_U64;
    }
}

extern "C" {

int heap_free_batch(heap_t *h, const uint64_t *d_offsets, uint64_t n, heap_stream_t sp) {
    if (!h || n > h->max_batch || (n && !d_offsets)) return HEAP_EINVAL;
    if (n == 0) return HEAP_OK;
    if (use_graph(h, (cudaStream_t)sp)) return graph_batch(h, 0, d_offsets, nullptr, n, (cudaStream_t)sp);
    return batch_free(h, d_offsets, n, nullptr, (cudaStream_t)sp);
}

int heap_free_batch_handles(heap_t *h, const uint64_t *d_table, uint64_t table_len, const uint64_t *d_idx,
                            uint64_t n, heap_stream_t sp) {
    if (!h || n > h->max_batch || (n && (!d_table || !d_idx))) return HEAP_EINVAL;
    if (n == 0) return HEAP_OK;
    cudaStream_t s = (cudaStream_t)sp;
    if (h->micro) {
        h->hidx = (const u64 *)d_idx;
        h->hlen = table_len;
        const int rc = batch_free(h, d_table, n, nullptr, s);
        h->hidx = nullptr;
        h->hlen = 0;
        return rc;
    }
    LAUNCH(h, k_gather_handles, h->G, 256, 0, s, (const u64 *)d_table, (u64)table_len, (const u64 *)d_idx, (u64)n,
           (u64 *)h->gout);
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    return heap_free_batch(h, (const uint64_t *)h->gout, n, sp);
}

int heap_step(heap_t *h, const uint64_t *d_offsets, const uint64_t *d_idx, uint64_t table_len, uint64_t nf,
              const uint64_t *d_sizes, uint64_t *d_out, uint64_t na, heap_stream_t sp) {
    if (!h || nf > h->max_batch || na > h->max_batch || (nf && !d_offsets) || (na && (!d_sizes || !d_out)))
        return HEAP_EINVAL;
    if (h->micro && (nf || na)) {          // one launch: the free batch, then the alloc batch
        const Layout &L = h->L;
        const int cur = h->cur, nxt = cur ^ 1;
        DevCtr *C = h->ctr;
        cudaStream_t s = (cudaStream_t)sp;
        TAG(h, HEAP_TAG_MICRO);
#define MICRO_STEP(P)                                                                                            \
    LAUNCH(h, micro::k_micro_step<P>, 1, micro::MT, micro::STEP_SMEM, s, (const u64 *)d_offsets, (u64)nf,          \
           (const u64 *)d_idx, (u64)(d_idx ? table_len : 0), (const u64 *)d_sizes, (u64)na, (u64 *)d_out, h->alog2, \
           L.A_u, L.L, h->fs[cur], h->fe[cur], h->fs[nxt], h->fe[nxt], h->tbl, L.tcap - 1, L.tcap / table::LINE,   \
           L.tcap, L.cap_f, h->ms, C, h->max_live)
        switch (h->policy) {
            case HEAP_FIRST_FIT: MICRO_STEP(micro::P_FF); break;
            case HEAP_NEXT_FIT: MICRO_STEP(micro::P_NF); break;
            case HEAP_BEST_FIT: MICRO_STEP(micro::P_BF); break;
            default: MICRO_STEP(micro::P_CLS); break;
        }
#undef MICRO_STEP
        h->cur = cur ^ (nf ? 1 : 0) ^ (na ? 1 : 0);
        if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
        return HEAP_OK;
    }
    int rc = HEAP_OK;
    if (nf) rc = d_idx ? heap_free_batch_handles(h, d_offsets, table_len, d_idx, nf, sp)
                       : heap_free_batch(h, d_offsets, nf, sp);
    if (rc != HEAP_OK) return rc;
    return na ? heap_alloc_batch(h, d_sizes, d_out, na, sp) : HEAP_OK;
}

int heap_alloc_batch(heap_t *h, const uint64_t *d_sizes, uint64_t *d_out, uint64_t n, heap_stream_t sp) {
    if (!h || n > h->max_batch || (n && (!d_sizes || !d_out))) return HEAP_EINVAL;
    if (n == 0) return HEAP_OK;
    if (use_graph(h, (cudaStream_t)sp)) return graph_batch(h, 1, d_sizes, d_out, n, (cudaStream_t)sp);
    return batch_alloc(h, d_sizes, d_out, n, nullptr, (cudaStream_t)sp);
}

int heap_set_graphs(heap_t *h, int enable) {
    if (!h) return HEAP_EINVAL;
    h->graphs = enable ? 1 : 0;
    return HEAP_OK;
}

static u64 meta_bytes(const heap *h) { return (u64)h->L.total; }

int heap_stats_async(heap_t *h, heap_stats_t *d_out, heap_stream_t sp) {
    if (!h || !d_out) return HEAP_EINVAL;
    cudaStream_t s = (cudaStream_t)sp;
    TAG(h, HEAP_TAG_MISC);
    if (h->policy == HEAP_DOUBLE_BUDDY) {
        int rc = heap_stats_async(h->sub, h->sstats, sp);
        if (rc == HEAP_OK && h->sub2) rc = heap_stats_async(h->sub2, h->sstats2, sp);
        if (rc != HEAP_OK) return rc;
        LAUNCH(h, dbl::k_stats, 1, 1, 0, s, h->sstats, h->sstats2, h->sub2 ? 1 : 0, h->dctr, h->arena, h->align,
               h->L.dbl_A, meta_bytes(h), d_out);
        if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
        return HEAP_OK;
    }
    if (h->policy == HEAP_HYBRID) {
        int rc = heap_stats_async(h->sub, h->sstats, sp);
        if (rc != HEAP_OK) return rc;
        CUDA_TRY(cudaMemsetAsync(&h->pctr->runs, 0, 2 * sizeof(u64), s));
        LAUNCH(h, pool::k_marks, h->G, 256, 0, s, h->L.geo, h->bits, (u32 *)nullptr, (u32 *)nullptr, h->pctr);
        LAUNCH(h, pool::k_stats, 1, 1, 0, s, h->sstats, h->pctr, h->L.geo, h->arena, h->align, meta_bytes(h), d_out);
        if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
        return HEAP_OK;
    }
    LAUNCH(h, k_stats, 1, 1024, 0, s, h->ctr, h->fs[h->cur], h->fe[h->cur],
           (h->policy == HEAP_BUDDY || h->policy == HEAP_FIB_BUDDY) ? 1 : 0, h->L.K,
           h->arena, h->align, h->alog2, meta_bytes(h), d_out,
           h->policy == HEAP_FIB_BUDDY ? (const u64 *)h->fgeom : (const u64 *)nullptr);
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    return HEAP_OK;
}

int heap_stats(heap_t *h, heap_stats_t *h_out, heap_stream_t sp) {
    if (!h || !h_out) return HEAP_EINVAL;
    int rc = heap_stats_async(h, h->dstats, sp);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)sp;
    CUDA_TRY(cudaMemcpyAsync(h_out, h->dstats, sizeof(heap_stats_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (h_out->error_flags) return HEAP_ECAPACITY;
    return HEAP_OK;
}

int heap_export(heap_t *h, uint64_t *d_free_pairs, uint64_t cap_free, uint64_t *d_live_pairs, uint64_t cap_live,
                uint64_t *h_counts, heap_stream_t sp) {
    if (!h || !h_counts) return HEAP_EINVAL;
    cudaStream_t s = (cudaStream_t)sp;
    TAG(h, HEAP_TAG_MISC);
    if (h->policy == HEAP_DOUBLE_BUDDY) {
        // the binary heap's blocks (below A_bytes), then the 3-unit heap's converted to bytes
        uint64_t ca[2] = {0, 0}, cb[2] = {0, 0};
        int rc = heap_export(h->sub, d_free_pairs, cap_free, d_live_pairs, cap_live, ca, sp);
        if (rc != HEAP_OK) return rc;
        if (h->sub2) {
            uint64_t *fp2 = (d_free_pairs && cap_free > ca[0]) ? d_free_pairs + 2 * ca[0] : nullptr;
            uint64_t *lp2 = (d_live_pairs && cap_live > ca[1]) ? d_live_pairs + 2 * ca[1] : nullptr;
            const u64 cf2 = fp2 ? cap_free - ca[0] : 0, cl2 = lp2 ? cap_live - ca[1] : 0;
            rc = heap_export(h->sub2, fp2, cf2, lp2, cl2, cb, sp);
            if (rc != HEAP_OK) return rc;
            if (fp2) LAUNCH(h, dbl::k_pairs_to_bytes, h->G, 256, 0, s, (u64 *)fp2, std::min<u64>(cb[0], cf2), h->L.dbl_A, 3 * h->align);
            if (lp2) LAUNCH(h, dbl::k_pairs_to_bytes, h->G, 256, 0, s, (u64 *)lp2, std::min<u64>(cb[1], cl2), h->L.dbl_A, 3 * h->align);
            CUDA_TRY(cudaStreamSynchronize(s));
        }
        if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
        h_counts[0] = ca[0] + cb[0];
        h_counts[1] = ca[1] + cb[1];
        return HEAP_OK;
    }
    if (h->policy == HEAP_HYBRID) {
        // pool runs / live objects first (below pool_end, address order), then the TLSF heap's
        const pool::Geom &G = h->L.geo;
        pool::Ctr *P = h->pctr;
        CUDA_TRY(cudaMemsetAsync(&P->runs, 0, 2 * sizeof(u64), s));
        LAUNCH(h, pool::k_marks, h->G, 256, 0, s, G, h->bits, h->flags, h->pos, P);
        scan(h, h->flags, h->flags, &P->nwords, &P->scan_total, s);
        scan(h, h->pos, h->pos, &P->nwords, &P->scan_total, s);
        u64 pc[2] = {0, 0};
        CUDA_TRY(cudaMemcpyAsync(pc, &P->runs, 2 * sizeof(u64), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        const u64 R = pc[0], LV = pc[1];
        if ((d_free_pairs && cap_free) || (d_live_pairs && cap_live)) {
            LAUNCH(h, pool::k_emit, h->G, 256, 0, s, G, h->bits, h->flags, h->pos, (u64 *)d_free_pairs,
                   d_free_pairs ? cap_free : 0, (u64 *)d_live_pairs, d_live_pairs ? cap_live : 0);
            if (d_free_pairs && cap_free)
                LAUNCH(h, pool::k_end_to_size, h->G, 256, 0, s, (u64 *)d_free_pairs, std::min<u64>(R, cap_free));
        }
        uint64_t *fp2 = (d_free_pairs && cap_free > R) ? d_free_pairs + 2 * R : nullptr;
        uint64_t *lp2 = (d_live_pairs && cap_live > LV) ? d_live_pairs + 2 * LV : nullptr;
        const u64 cf2 = fp2 ? cap_free - R : 0, cl2 = lp2 ? cap_live - LV : 0;
        uint64_t sc[2] = {0, 0};
        int rc = heap_export(h->sub, fp2, cf2, lp2, cl2, sc, sp);
        if (rc != HEAP_OK) return rc;
        if (fp2) LAUNCH(h, pool::k_shift_pairs, h->G, 256, 0, s, (u64 *)fp2, std::min((u64)sc[0], cf2), G.pool_end);
        if (lp2) LAUNCH(h, pool::k_shift_pairs, h->G, 256, 0, s, (u64 *)lp2, std::min((u64)sc[1], cl2), G.pool_end);
        CUDA_TRY(cudaStreamSynchronize(s));
        if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
        h_counts[0] = R + sc[0];
        h_counts[1] = LV + sc[1];
        return HEAP_OK;
    }
    const Layout &L = h->L;
    DevCtr *C = h->ctr;
    int alog = h->alog2;
    u64 counts[2] = {0, 0};
    // free blocks
    if (h->policy != HEAP_BUDDY && h->policy != HEAP_FIB_BUDDY) {
        if (d_free_pairs && cap_free)
            LAUNCH(h, k_export_free, h->G, 256, 0, s, h->fs[h->cur], h->fe[h->cur], &C->F, alog, (u64 *)d_free_pairs, cap_free);
        CUDA_TRY(cudaMemcpyAsync(&counts[0], &C->F, 8, cudaMemcpyDeviceToHost, s));
    } else {
        LAUNCH(h, k_bud_keys, h->G, 256, 0, s, h->fs[h->cur], C, L.K, h->kA, h->vA);
        int rb = radix_sort<u32, true>(h, h->kA, h->kB, h->vA, h->vB, &C->bud_total, 32, s);
        u32 *k = rb ? h->kB : h->kA, *v = rb ? h->vB : h->vA;
        if (d_free_pairs && cap_free)
            LAUNCH(h, k_export_pairs_u32, h->G, 256, 0, s, k, v, &C->bud_total, alog, 1, (u64 *)d_free_pairs, cap_free,
                   h->policy == HEAP_FIB_BUDDY ? (const u64 *)h->fgeom : (const u64 *)nullptr);
        CUDA_TRY(cudaMemcpyAsync(&counts[0], &C->bud_total, 8, cudaMemcpyDeviceToHost, s));
    }
    // live blocks: collect table slots, sort by key
    LAUNCH(h, k_set_u64, 1, 1, 0, s, &C->tmp[6], L.tcap);
    LAUNCH(h, k_tbl_flags, h->G, 256, 0, s, h->tbl, L.tcap, h->flags);
    scan(h, h->flags, h->pos, &C->tmp[6], &C->tmp[7], s);
    LAUNCH(h, k_tbl_compact, h->G, 256, 0, s, h->tbl, L.tcap, h->flags, h->pos, h->kA, h->vA, L.sort_cap);
    LAUNCH(h, k_clamp, 1, 1, 0, s, &C->tmp[7], &C->tmp[3], L.sort_cap);
    int rb = radix_sort<u32, true>(h, h->kA, h->kB, h->vA, h->vB, &C->tmp[3], 32, s);
    u32 *k = rb ? h->kB : h->kA, *v = rb ? h->vB : h->vA;
    if (d_live_pairs && cap_live)
        LAUNCH(h, k_export_pairs_u32, h->G, 256, 0, s, k, v, &C->tmp[3], alog, 0, (u64 *)d_live_pairs, cap_live,
               (const u64 *)nullptr);
    CUDA_TRY(cudaMemcpyAsync(&counts[1], &C->tmp[7], 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (cudaGetLastError() != cudaSuccess) return HEAP_ECUDA;
    h_counts[0] = counts[0];
    h_counts[1] = counts[1];
    return HEAP_OK;
}

int heap_debug_counters(heap_t *h, uint64_t *h_out, int n, heap_stream_t sp) {
    if (!h || !h_out || n < 0 || n > 32) return HEAP_EINVAL;
    cudaStream_t s = (cudaStream_t)sp;
    CUDA_TRY(cudaMemcpyAsync(h_out, (h->sub ? h->sub : h)->ctr->eng, n * sizeof(u64), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return HEAP_OK;
}

int heap_profile_enable(heap_t *h, uint64_t tag_mask) {
    if (!h) return HEAP_EINVAL;
    h->prof_mask = tag_mask;
    if (h->sub) h->sub->prof_mask = tag_mask;
    if (h->sub2) h->sub2->prof_mask = tag_mask;
    return HEAP_OK;
}

int heap_profile_read(heap_t *h, double *h_ms, uint64_t *h_launches) {
    if (!h) return HEAP_EINVAL;
    for (auto &r : h->recs) {
        if (cudaEventSynchronize(r.b) != cudaSuccess) return HEAP_ECUDA;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        if (h_ms) h_ms[r.tag] += ms;
        if (h_launches) h_launches[r.tag] += 1;
        h->pool.push_back(r.a);
        h->pool.push_back(r.b);
    }
    h->recs.clear();
    if (h->sub2) { int rc = heap_profile_read(h->sub2, h_ms, h_launches); if (rc) return rc; }
    if (h->sub) return heap_profile_read(h->sub, h_ms, h_launches);
    return HEAP_OK;
}

const char *heap_tag_name(int tag) {
    static const char *names[HEAP_NTAGS] = {"classify", "scan", "sort", "table_lookup", "compact", "merge",
                                            "coalesce", "alloc_prep", "index_build", "engine", "finish",
                                            "table_rebuild", "buddy_free_levels", "buddy_alloc_levels",
                                            "misc", "micro"};
    return (tag >= 0 && tag < HEAP_NTAGS) ? names[tag] : "?";
}

int heap_stats_allgather(heap_t *h, ncclComm_t comm, heap_stats_t *d_all, heap_stream_t sp) {
    if (!h || !comm || !d_all) return HEAP_EINVAL;
    // this rank's record goes to the heap's own 128-byte stats slot in the workspace, then every
    // rank's record to d_all[rank] (the only inter-GPU bytes of the path)
    int rc = heap_stats_async(h, h->dstats, sp);
    if (rc != HEAP_OK) return rc;
    if (ncclAllGather(h->dstats, d_all, sizeof(heap_stats_t) / sizeof(uint64_t), ncclUint64, comm,
                      (cudaStream_t)sp) != ncclSuccess)
        return HEAP_ENCCL;
    return HEAP_OK;
}

int heap_nccl_unique_id(uint8_t *h_id) {
    if (!h_id) return HEAP_EINVAL;
    ncclUniqueId id;
    static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
    if (ncclGetUniqueId(&id) != ncclSuccess) return HEAP_ENCCL;
    memcpy(h_id, id.internal, sizeof(id.internal));
    return HEAP_OK;
}

int heap_nccl_comm_init(ncclComm_t *h_comm, int nranks, const uint8_t *h_id, int rank) {
    if (!h_comm || !h_id || nranks < 1 || rank < 0 || rank >= nranks) return HEAP_EINVAL;
    ncclUniqueId id;
    memcpy(id.internal, h_id, sizeof(id.internal));
    return ncclCommInitRank(h_comm, nranks, id, rank) == ncclSuccess ? HEAP_OK : HEAP_ENCCL;
}

int heap_nccl_comm_init_all(ncclComm_t *h_comms, int ndev, const int *h_devs) {
    if (!h_comms || ndev < 1) return HEAP_EINVAL;
    return ncclCommInitAll(h_comms, ndev, h_devs) == ncclSuccess ? HEAP_OK : HEAP_ENCCL;
}

int heap_nccl_comm_destroy(ncclComm_t comm) {
    if (!comm) return HEAP_EINVAL;
    return ncclCommDestroy(comm) == ncclSuccess ? HEAP_OK : HEAP_ENCCL;
}

const char *heap_strerror(int code) {
    switch (code) {
    case HEAP_ENCCL: return "NCCL error";
    case HEAP_OK: return "ok";
    case HEAP_EINVAL: return "invalid argument";
    case HEAP_ENOMEM: return "workspace too small / out of host memory";
    case HEAP_ECAPACITY: return "metadata capacity exceeded in a batch";
    case HEAP_ECUDA: return "CUDA error";
    default: return "unknown error";
    }
}

}  // extern "C"
