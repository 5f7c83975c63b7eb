/*
 * oracle_l.cpp — Oracle-L: the plain, slow, single-threaded CPU reference for the
 * batched device heap.  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2405_07079_b200/) never links or calls it, and this file shares
 * no code, header, table or constant with the CUDA path.
 *
 * What it computes (arXiv 2405.07079, "Host-Based Allocators for Device Memory"):
 *   - the allocator never reads the memory it manages, so all metadata is out of band
 *     (PAPER.md:39,55,61): here `live` plays the block table keyed by address
 *     (§3.3) and `freeb` the address-sorted free list (§3.1 HAL role,
 *     PAPER.md:166-168); the heap starts as one free block (Alg. 6 :617-618).
 *   - alloc splits the chosen free block from its low end (Alg. 1).
 *   - free coalesces with the free neighbour ending at the block and/or the one starting
 *     right after it (Alg. 2; Alg. 5).
 *   - policies (the candidate key; lowest key wins, readings C2-C13):
 *       FIRST_FIT  first block with size >= r, by address
 *       BEST_FIT   min (size, start) over size >= r               (Alg. 3 :298-317)
 *       SEGFIT     TLSF mapping with SL_LOG2 = 0: search bin = ceil(log2 r), block bin =
 *                  floor(log2 size) (+1 shift), address order within a bin
 *                                                                 (Alg. 4 :332-351, :440)
 *       TLSF       SL_LOG2 = 5 two-level classes, min (cls, start) with cls >= search class
 *
 *       BUDDY      binary buddy: smallest nonempty order >= k, lowest address, split keeping
 *                  the low half, merge with a free buddy a XOR 2^k
 *       SEGFIT_LIFO the paper's segregated fit verbatim: power-of-two bins used as stacks —
 *                  alloc pops the head (newest push) of the first nonempty bin >= ceil(log2 r),
 *                  every free / remainder is pushed at the head of its bin (Alg. 4/5)
 *       NEXT_FIT   first fit resumed at a rover ("each traversal of the free list
 *                  resumes from the last position"): the first block with start >= rover and
 *                  size >= r, else (wrap) the first from the lowest address; after a carve the
 *                  rover is the end of the allocation (reading C27)
 *       DOUBLE_BUDDY double buddies ("two heaps with staggered class sizes, e.g.
 *                  2, 4, 8, ... and 3, 6, 12, ..."): a binary buddy heap of align-sized units on
 *                  [0, A_bytes) and one of 3*align-sized units on [A_bytes, arena); a request
 *                  goes to the heap whose class is smaller (no fallback; reading C28)
 *       FIB_BUDDY  Fibonacci buddies ("every Fibonacci number is the sum of two other
 *                  Fibonacci numbers, blocks can be split recursively"): classes S_0 = 1, S_1 = 2,
 *                  S_k = S_{k-1} + S_{k-2} units; a class-k block splits into its low part of class
 *                  k-1 and its high part of class k-2 (class 1: two class-0 halves); the arena is
 *                  the greedy (Zeckendorf) sum of Fibonacci roots, largest first.  An alloc takes the
 *                  smallest nonempty class >= the request's, lowest address, and splits keeping the
 *                  low part ("the first is split further", :116); a free merges a block with its
 *                  tree sibling while the sibling is free (reading C30)
 *       HYBRID     §5.3's hybrid: requests below a page (0 < s < 4096 B) go
 *                  to object pools managed by bitmasks (§3.2) — pool j holds
 *                  objects of align*2^j bytes, an allocation takes the pool's lowest free slot
 *                  (first fit over the bitmask), a full pool falls back to the segregated-fit
 *                  heap — and everything else to a TLSF heap on the rest of the arena
 *                  (layout: DESIGN.md reading C26)
 *   - batch driver (canonical order, BASELINE.json north_star): a free batch classifies every
 *     offset against the batch-start state, then frees the valid ones in ascending address
 *     order; an alloc batch serves requests in request order, HEAP_NULL on failure.
 *   - partial (tail) deallocation, policy flag PARTIAL (0x100) on FIRST_FIT, BEST_FIT, SEGFIT,
 *     TLSF and NEXT_FIT: "freeing the last 2kB of a 10kB block ... the in-use block will be shrunk"
 *     (Alg. 2 :205-212 `search(used_list, addr)` then `it.size = addr - it.addr`):
 *     an offset inside a live block frees from that offset to the block's end.  Per live block
 *     of the batch-start state, the lowest offset of the batch inside it frees (the whole block
 *     if it is the start); every other offset inside it is a double free (C29).
 * Everything is in units of `align` (reading C14).  Sizes of s bytes become
 * r = ceil(s / align) units; s = 0 or r > A_u fails (C17).
 */
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <vector>
#include <algorithm>
#include <utility>
#include <tuple>

namespace {

const uint64_t HEAP_NULL = ~0ull;
enum { FIRST_FIT = 1, BEST_FIT = 2, SEGFIT = 3, TLSF = 4, BUDDY = 5, SEGFIT_LIFO = 6, HYBRID = 7, NEXT_FIT = 8,
       DOUBLE_BUDDY = 9, FIB_BUDDY = 10 };
const int PARTIAL = 0x100;    /* policy flag: partial (tail) deallocation */
const uint64_t PAGE = 4096;   /* "allocations smaller than a page (<4kB)" */

/* floor(log2 u) for u >= 1, written as a plain loop */
int floor_log2(uint64_t u) {
    int m = -1;
    while (u) { u >>= 1; m++; }
    return m;
}

/* TLSF class of a free block of u units (insert mapping; Masmano's TLSF as read in
 * DESIGN.md C10).  Classes below 2^L units are exact; above, first level fl = m - L + 1
 * with m = floor(log2 u), second level = the next L bits below the leading one. */
uint64_t insert_class(uint64_t u, int L) {
    if (u < (1ull << L)) return u;                       /* fl = 0, sl = u */
    int m = floor_log2(u);
    uint64_t fl = (uint64_t)(m - L + 1);
    uint64_t sl = (u >> (m - L)) - (1ull << L);
    return fl * (1ull << L) + sl;
}
/* search class: round the request up to the next class boundary so that every block of
 * that class or above fits (Alg. 4 "1 << ceil(log2(size))", generalised) */
uint64_t search_class(uint64_t u, int L) {
    if (u < (1ull << L)) return insert_class(u, L);
    int m = floor_log2(u);
    return insert_class(u + (1ull << (m - L)) - 1, L);
}

struct Counters {
    uint64_t allocs_ok = 0, allocs_failed = 0, frees_ok = 0, frees_invalid = 0,
             frees_double = 0, frees_null = 0, high_water_end = 0;
};

struct Heap {
    int policy;
    bool partial = false;                 /* PARTIAL flag: an interior offset frees the block's tail */
    int L;
    uint64_t align, A_u, arena_bytes;
    std::map<uint64_t, uint64_t> live;    /* start -> size (units): the block table */
    std::map<uint64_t, uint64_t> freeb;   /* start -> size (units): free list, address order */
    std::set<std::pair<uint64_t, uint64_t>> cls_index;   /* (class, start): SEGFIT/TLSF bins */
    /* SEGFIT_LIFO bins: (class, ~push stamp, start) — the head of a bin is its newest push */
    std::set<std::tuple<uint64_t, uint64_t, uint64_t>> lifo_index;
    std::map<uint64_t, uint64_t> stamp_of;                 /* start -> push stamp */
    uint64_t clock = 0;
    uint64_t rover = 0;                                   /* NEXT_FIT: where the next scan starts */
    std::vector<std::set<uint64_t>> bfree;                /* BUDDY / FIB_BUDDY: free starts per class */
    std::vector<uint64_t> FS;                             /* FIB_BUDDY: class sizes S_k (units) */
    std::vector<std::pair<uint64_t, int>> roots;          /* FIB_BUDDY: (start, class) of the roots */
    int K = 0;                                            /* BUDDY: max order */
    Counters c;
    /* HYBRID: J pools of S bytes each at [j*S, (j+1)*S), then the TLSF heap `sub` on
     * [pool_end, arena).  A pool's bitmask is kept as "every slot >= fresh[j] is free" plus the
     * set of free slots below fresh[j]; its lowest free slot is min(freed.begin(), fresh). */
    int J = 0;
    uint64_t S = 0, pool_end = 0;
    std::vector<uint64_t> fresh, nslots;
    std::vector<std::set<uint64_t>> freed;
    uint64_t pool_live_n = 0, pool_live_b = 0;
    Heap *sub = nullptr;
    /* DOUBLE_BUDDY: heap `sub` (units of align on [0, A_bytes)) and `sub3` (units of 3*align on
     * [A_bytes, arena)); sub3 is a plain buddy heap whose "bytes" are those 3*align units */
    Heap *sub3 = nullptr;
    uint64_t A_bytes = 0, N3 = 0;
    ~Heap() { delete sub; delete sub3; }

    bool slot_free(int j, uint64_t t) const { return t >= fresh[j] || freed[j].count(t); }
    /* lowest free slot of pool j, or HEAP_NULL when the pool is full */
    uint64_t pool_lowest_free(int j) const {
        if (!freed[j].empty()) return *freed[j].begin();
        return fresh[j] < nslots[j] ? fresh[j] : HEAP_NULL;
    }
    void pool_take(int j, uint64_t t) {
        if (t == fresh[j]) fresh[j]++;
        else freed[j].erase(t);
    }

    /* ---- free-list edits (keep the class index in step) ---- */
    void free_insert(uint64_t s, uint64_t z) {
        freeb[s] = z;
        if (policy == SEGFIT || policy == TLSF) cls_index.insert({insert_class(z, L), s});
        if (policy == SEGFIT_LIFO) {
            /* "Place new block at head of free list in its size class" (Alg. 4 :350-355,
             * Alg. 5 :427-433): a push gets the next tick of a logical clock; the bin's head
             * is its most recent push. */
            uint64_t st = clock++;
            stamp_of[s] = st;
            lifo_index.insert({insert_class(z, 0), ~st, s});
        }
    }
    void free_erase(uint64_t s) {
        auto it = freeb.find(s);
        if (policy == SEGFIT || policy == TLSF) cls_index.erase({insert_class(it->second, L), s});
        if (policy == SEGFIT_LIFO) {
            lifo_index.erase({insert_class(it->second, 0), ~stamp_of[s], s});   /* unlink (remove()) */
            stamp_of.erase(s);
        }
        freeb.erase(it);
    }

    bool is_free_start(uint64_t u) const {
        if (policy == BUDDY || policy == FIB_BUDDY) {
            for (const auto &st : bfree) if (st.count(u)) return true;
            return false;
        }
        return freeb.count(u) != 0;
    }

    /* ---- Alg. 2 / Alg. 5: deallocate a live block with 3-way coalescing ---- */
    void free_block(uint64_t o) {
        uint64_t size = live[o];
        live.erase(o);
        if (policy == BUDDY) { buddy_free(o, size); return; }
        if (policy == FIB_BUDDY) { fib_free(o, size); return; }
        free_range(o, o + size);
    }
    /* partial deallocation (Alg. 2 :205-212): the live block at a keeps [a, o), [o, end) is freed */
    void free_tail(uint64_t a, uint64_t o) {
        uint64_t end = a + live[a];
        live[a] = o - a;                        /* it.size = addr - it.addr */
        free_range(o, end);
    }
    /* insert [o, end) into the free list, merging with the free neighbours on both sides */
    void free_range(uint64_t o, uint64_t end) {
        uint64_t start = o;
        /* left: the free block whose end is o */
        auto it = freeb.lower_bound(o);
        if (it != freeb.begin()) {
            auto left = std::prev(it);
            if (left->first + left->second == o) { start = left->first; free_erase(left->first); }
        }
        /* right: the free block starting at end */
        auto right = freeb.find(end);
        if (right != freeb.end()) { end = right->first + right->second; free_erase(right->first); }
        free_insert(start, end - start);
    }
    /* the live block containing unit u (search(used_list, addr), Alg. 2 :205), or HEAP_NULL */
    uint64_t containing_live(uint64_t u) const {
        auto it = live.upper_bound(u);
        if (it == live.begin()) return HEAP_NULL;
        --it;
        return (u < it->first + it->second) ? it->first : HEAP_NULL;
    }

    /* buddy merge: while the buddy a XOR 2^k is a free block of order k, merge */
    void buddy_free(uint64_t o, uint64_t size) {
        int k = floor_log2(size);
        while (k < K) {
            uint64_t b = o ^ (1ull << k);
            auto it = bfree[k].find(b);
            if (it == bfree[k].end()) break;
            bfree[k].erase(it);
            o = std::min(o, b);
            k++;
        }
        bfree[k].insert(o);
    }

    /* ---- Fibonacci buddies (reading C30) ---- */
    int fib_class_of_size(uint64_t z) const {              /* exact class of a block size */
        for (int k = 0; k < (int)FS.size(); k++) if (FS[k] == z) return k;
        return -1;
    }
    static int fib_left(int t) { return t - 1; }           /* low child's class */
    static int fib_right(int t) { return t >= 2 ? t - 2 : 0; }   /* high child's class (class 1: 1 + 1) */
    /* walk from the root holding a down to the node (a, k); returns false if (a, k) is a root,
     * else the sibling (q, qk) and the parent (p, pk) */
    bool fib_family(uint64_t a, int k, uint64_t *q, int *qk, uint64_t *p, int *pk) const {
        for (const auto &r : roots) {
            if (a < r.first || a >= r.first + FS[r.second]) continue;
            uint64_t s = r.first;
            int t = r.second;
            bool has_parent = false;
            while (!(s == a && t == k)) {
                uint64_t mid = s + FS[fib_left(t)];
                *p = s; *pk = t; has_parent = true;
                if (a < mid) { *q = mid; *qk = fib_right(t); t = fib_left(t); }
                else { *q = s; *qk = fib_left(t); s = mid; t = fib_right(t); }
            }
            return has_parent;
        }
        return false;
    }
    /* free: while the tree sibling is a free block, remove it and move up to the parent */
    void fib_free(uint64_t a, uint64_t size) {
        int k = fib_class_of_size(size);
        for (;;) {
            uint64_t q = 0, p = 0;
            int qk = 0, pk = 0;
            if (!fib_family(a, k, &q, &qk, &p, &pk) || !bfree[qk].count(q)) break;
            bfree[qk].erase(q);
            a = p;
            k = pk;
        }
        bfree[k].insert(a);
    }

    /* ---- Alg. 1: allocate r units from the chosen free block (low-end split) ---- */
    uint64_t take(uint64_t s, uint64_t r) {
        uint64_t z = freeb[s];
        free_erase(s);
        if (z > r) free_insert(s + r, z - r);   /* free_it.address += size; free_it.size -= size */
        live[s] = r;                            /* record the rounded request (Alg. 4 :348) */
        return s;
    }

    uint64_t alloc_units(uint64_t r) {
        if (policy == FIRST_FIT) {
            for (const auto &kv : freeb)
                if (kv.second >= r) return take(kv.first, r);
            return HEAP_NULL;
        }
        if (policy == NEXT_FIT) {
            /* scan from the rover to the end of the list, then from the start up to the rover */
            auto at = freeb.lower_bound(rover);
            for (auto it = at; it != freeb.end(); ++it)
                if (it->second >= r) { rover = it->first + r; return take(it->first, r); }
            for (auto it = freeb.begin(); it != at; ++it)
                if (it->second >= r) { rover = it->first + r; return take(it->first, r); }
            return HEAP_NULL;
        }
        if (policy == BEST_FIT) {
            /* Alg. 3: scan the whole free list, keep the smallest fitting block; exact match
             * ends the scan.  Ties go to the lowest address (reading C3). */
            bool found = false; uint64_t bs = 0, bz = 0;
            for (const auto &kv : freeb) {
                if (kv.second < r) continue;
                if (!found || kv.second < bz) { found = true; bs = kv.first; bz = kv.second; }
                if (kv.second == r) break;
            }
            return found ? take(bs, r) : HEAP_NULL;
        }
        if (policy == SEGFIT || policy == TLSF) {
            /* Alg. 4 + availability bitmap/ffs fallback: the first
             * nonempty bin at or above the search class, its lowest-address block (C9). */
            uint64_t c = search_class(r, L);
            auto it = cls_index.lower_bound({c, 0});
            if (it == cls_index.end()) return HEAP_NULL;
            return take(it->second, r);
        }
        if (policy == SEGFIT_LIFO) {
            /* Alg. 4 as written: bin = ceil(log2 size) (+1 shift), the first nonempty bin at or
             * above it (availability bitmap + ffs), pop its HEAD (the block pushed
             * last, "it = ht[free_lists[order]]", :336-337), split from the low end and push the
             * remainder at the head of its bin (:342-356). */
            uint64_t c = search_class(r, 0);
            auto it = lifo_index.lower_bound({c, 0, 0});
            if (it == lifo_index.end()) return HEAP_NULL;
            return take(std::get<2>(*it), r);
        }
        if (policy == FIB_BUDDY) {
            /* r is already a class size S_j: the smallest nonempty class >= j, lowest address;
             * split keeping the low part, the high parts stay free */
            int j = fib_class_of_size(r);
            int t = j;
            while (t <= K && bfree[t].empty()) t++;
            if (t > K) return HEAP_NULL;
            uint64_t a = *bfree[t].begin();
            bfree[t].erase(bfree[t].begin());
            for (int u = t; u > j; u--) bfree[fib_right(u)].insert(a + FS[fib_left(u)]);
            live[a] = r;
            return a;
        }
        /* BUDDY: r is already a power of two */
        int k = floor_log2(r);
        int j = k;
        while (j <= K && bfree[j].empty()) j++;
        if (j > K) return HEAP_NULL;
        uint64_t a = *bfree[j].begin();
        bfree[j].erase(bfree[j].begin());
        for (int t = j - 1; t >= k; t--) bfree[t].insert(a + (1ull << t));  /* split, keep low half */
        live[a] = r;
        return a;
    }
};

}  // namespace

extern "C" {

void *oracle_create(uint64_t arena_bytes, uint64_t align, int policy) {
    if (align == 0 || (align & (align - 1)) || arena_bytes == 0 || arena_bytes % align) return nullptr;
    const bool partial = (policy & PARTIAL) != 0;
    policy &= ~PARTIAL;
    if (policy < FIRST_FIT || policy > FIB_BUDDY) return nullptr;
    /* partial frees need address coalescing: not for buddies or the object pools */
    if (partial && (policy == BUDDY || policy == HYBRID || policy == DOUBLE_BUDDY || policy == SEGFIT_LIFO ||
                    policy == FIB_BUDDY))
        return nullptr;
    if (policy == DOUBLE_BUDDY) {
        /* reading C28: the 3-unit heap gets floor(arena / (6 align)) units at the top of the
         * arena, the binary heap everything below (at least half) */
        Heap *h = new Heap();
        h->policy = DOUBLE_BUDDY;
        h->align = align;
        h->arena_bytes = arena_bytes;
        h->A_u = arena_bytes / align;
        h->N3 = arena_bytes / (6 * align);
        h->A_bytes = arena_bytes - 3 * align * h->N3;
        h->sub = (Heap *)oracle_create(h->A_bytes, align, BUDDY);
        h->sub3 = h->N3 ? (Heap *)oracle_create(h->N3, 1, BUDDY) : nullptr;
        return h;
    }
    if (policy == HYBRID) {
        /* reading C26: pool classes align*2^j <= PAGE; the first half of the arena is split
         * evenly between the pools, each share rounded down to a whole number of pages */
        Heap *h = new Heap();
        h->policy = HYBRID;
        h->align = align;
        h->arena_bytes = arena_bytes;
        h->A_u = arena_bytes / align;
        for (uint64_t o = align; o <= PAGE; o <<= 1) h->J++;
        if (h->J) h->S = arena_bytes / (2 * (uint64_t)h->J) / PAGE * PAGE;
        h->pool_end = (uint64_t)h->J * h->S;
        for (int j = 0; j < h->J; j++) {
            h->nslots.push_back(h->S / (align << j));
            h->fresh.push_back(0);
            h->freed.emplace_back();
        }
        h->sub = (Heap *)oracle_create(arena_bytes - h->pool_end, align, TLSF);
        return h;
    }
    Heap *h = new Heap();
    h->policy = policy;
    h->partial = partial;
    h->L = (policy == TLSF) ? 5 : 0;
    h->align = align;
    h->arena_bytes = arena_bytes;
    h->A_u = arena_bytes / align;
    if (policy == FIB_BUDDY) {
        /* S_0 = 1, S_1 = 2, S_k = S_{k-1} + S_{k-2} up to the arena; roots: the greedy
         * (Zeckendorf) decomposition of A_u, largest first, at increasing addresses */
        h->FS.push_back(1);
        if (h->A_u >= 2) h->FS.push_back(2);
        while (h->FS.size() >= 2 && h->FS[h->FS.size() - 1] + h->FS[h->FS.size() - 2] <= h->A_u)
            h->FS.push_back(h->FS[h->FS.size() - 1] + h->FS[h->FS.size() - 2]);
        h->K = (int)h->FS.size() - 1;
        h->bfree.assign(h->K + 1, std::set<uint64_t>());
        uint64_t s = 0, rem = h->A_u;
        while (rem) {
            int t = h->K;
            while (h->FS[t] > rem) t--;
            h->roots.push_back({s, t});
            h->bfree[t].insert(s);
            s += h->FS[t];
            rem -= h->FS[t];
        }
        return h;
    }
    if (policy == BUDDY) {
        h->K = floor_log2(h->A_u);
        h->bfree.assign(h->K + 1, std::set<uint64_t>());
        /* greedy decomposition of [0, A_u) into maximal aligned power-of-two blocks (C13) */
        uint64_t s = 0;
        while (s < h->A_u) {
            int t = h->K;
            while (t > 0 && ((s & ((1ull << t) - 1)) || s + (1ull << t) > h->A_u)) t--;
            h->bfree[t].insert(s);
            s += 1ull << t;
        }
    } else {
        h->free_insert(0, h->A_u);   /* "at least one entry: the heap itself" */
    }
    return h;
}

void oracle_destroy(void *p) { delete (Heap *)p; }

/* frees: classify every copy against the batch-start state, then free the valid live starts
 * in ascending address order.  Classification (reading C16):
 *   HEAP_NULL -> null; unaligned / out of range / neither live nor free start -> invalid;
 *   live start -> first copy frees, other copies double; start of a free block -> double. */
void oracle_free_batch(void *p, const uint64_t *offsets, uint64_t n);

/* HYBRID frees: the same per-copy classification; a pool offset must be a slot start of its
 * pool (a multiple of the object size inside the pool's share) — an allocated slot frees
 * (its bit returns to one), a free slot is a double free; every offset at or
 * above pool_end is the TLSF heap's, relative to pool_end. */
static void hybrid_free_batch(Heap *h, const uint64_t *offsets, uint64_t n) {
    std::vector<uint64_t> v(offsets, offsets + n);
    std::sort(v.begin(), v.end());
    std::vector<uint64_t> sub_offs;
    for (uint64_t i = 0; i < n; i++) {
        uint64_t o = v[i];
        bool dup = (i > 0 && v[i - 1] == o);
        if (o == HEAP_NULL) { h->c.frees_null++; continue; }
        if (o >= h->pool_end) { sub_offs.push_back(o - h->pool_end); continue; }
        int j = (int)(o / h->S);
        uint64_t rel = o % h->S, oj = h->align << j;
        if (rel % oj) { h->c.frees_invalid++; continue; }
        uint64_t t = rel / oj;
        if (h->slot_free(j, t) || dup) { h->c.frees_double++; continue; }
        h->c.frees_ok++;
        h->freed[j].insert(t);
        h->pool_live_n--;
        h->pool_live_b -= oj;
    }
    oracle_free_batch(h->sub, sub_offs.data(), sub_offs.size());
}

/* DOUBLE_BUDDY frees: an offset below A_bytes is the binary heap's; above, it must be a whole
 * number of 3*align units past A_bytes and is the 3-unit heap's unit index (else invalid) */
static void double_free_batch(Heap *h, const uint64_t *offsets, uint64_t n) {
    std::vector<uint64_t> a, b;
    const uint64_t u3 = 3 * h->align;
    for (uint64_t i = 0; i < n; i++) {
        uint64_t o = offsets[i];
        if (o == HEAP_NULL) { h->c.frees_null++; continue; }
        if (o < h->A_bytes) { a.push_back(o); continue; }
        if ((o - h->A_bytes) % u3 || !h->sub3) { h->c.frees_invalid++; continue; }
        b.push_back((o - h->A_bytes) / u3);
    }
    oracle_free_batch(h->sub, a.data(), a.size());
    if (h->sub3) oracle_free_batch(h->sub3, b.data(), b.size());
}

void oracle_free_batch(void *p, const uint64_t *offsets, uint64_t n) {
    Heap *h = (Heap *)p;
    if (h->policy == HYBRID) { hybrid_free_batch(h, offsets, n); return; }
    if (h->policy == DOUBLE_BUDDY) { double_free_batch(h, offsets, n); return; }
    std::vector<uint64_t> v(offsets, offsets + n);
    std::sort(v.begin(), v.end());
    std::set<uint64_t> claimed;                          /* live blocks already freed from */
    std::vector<std::pair<uint64_t, uint64_t>> to_free;  /* (block start, freed from) */
    for (uint64_t i = 0; i < n; i++) {
        uint64_t o = v[i];
        if (o == HEAP_NULL) { h->c.frees_null++; continue; }
        if (o % h->align || o / h->align >= h->A_u) { h->c.frees_invalid++; continue; }
        uint64_t u = o / h->align;
        uint64_t a = HEAP_NULL;
        if (h->live.count(u)) a = u;
        else if (h->is_free_start(u)) { h->c.frees_double++; continue; }
        else if (h->partial) a = h->containing_live(u);
        if (a == HEAP_NULL) { h->c.frees_invalid++; continue; }
        if (claimed.count(a)) { h->c.frees_double++; continue; }   /* a copy, or a higher offset */
        claimed.insert(a);
        h->c.frees_ok++;
        to_free.push_back({a, u});
    }
    for (auto &f : to_free) {                       /* ascending address order */
        if (f.first == f.second) h->free_block(f.first);
        else h->free_tail(f.first, f.second);
    }
}

void oracle_alloc_batch(void *p, const uint64_t *sizes, uint64_t n, uint64_t *out) {
    Heap *h = (Heap *)p;
    if (h->policy == DOUBLE_BUDDY) {
        /* r units -> binary class 2^ceil(log2 r) or 3-unit class 3 * 2^ceil(log2 ceil(r/3)),
         * whichever is smaller (they are never equal); that heap alone serves it (C28) */
        for (uint64_t i = 0; i < n; i++) {
            uint64_t s = sizes[i];
            uint64_t r = s / h->align + (s % h->align != 0);
            uint64_t p2 = 1, q = (r + 2) / 3, p3 = 1;
            while (p2 < r) p2 <<= 1;
            while (p3 < q) p3 <<= 1;
            uint64_t o = HEAP_NULL;
            if (s != 0 && r <= h->A_u && h->sub3 && 3 * p3 < p2) {
                uint64_t t = q, u = HEAP_NULL;
                oracle_alloc_batch(h->sub3, &t, 1, &u);
                o = (u == HEAP_NULL) ? HEAP_NULL : h->A_bytes + u * 3 * h->align;
            } else {
                oracle_alloc_batch(h->sub, &s, 1, &o);
            }
            out[i] = o;
        }
        return;
    }
    if (h->policy == HYBRID) {
        /* request order; a sub-page request takes the lowest free slot of the smallest pool whose
         * objects hold it, else (pool full, or s >= PAGE, or s = 0) the TLSF heap serves it */
        for (uint64_t i = 0; i < n; i++) {
            uint64_t s = sizes[i];
            if (s > 0 && s < PAGE && h->J > 0) {
                int j = 0;
                while ((h->align << j) < s) j++;
                uint64_t t = h->pool_lowest_free(j);
                if (t != HEAP_NULL) {
                    uint64_t oj = h->align << j;
                    h->pool_take(j, t);
                    out[i] = (uint64_t)j * h->S + t * oj;
                    h->pool_live_n++;
                    h->pool_live_b += oj;
                    h->c.allocs_ok++;
                    h->c.high_water_end = std::max(h->c.high_water_end, out[i] + oj);
                    continue;
                }
            }
            uint64_t o = HEAP_NULL;
            oracle_alloc_batch(h->sub, &s, 1, &o);
            out[i] = (o == HEAP_NULL) ? HEAP_NULL : o + h->pool_end;
        }
        return;
    }
    for (uint64_t i = 0; i < n; i++) {
        uint64_t s = sizes[i];
        uint64_t r = s / h->align + (s % h->align != 0);     /* ceil(s / align) */
        uint64_t u = HEAP_NULL;
        if (s != 0 && r <= h->A_u) {
            if (h->policy == FIB_BUDDY) {
                uint64_t z = HEAP_NULL;                          /* the smallest class holding r */
                for (uint64_t x : h->FS) if (x >= r) { z = x; break; }
                if (z != HEAP_NULL) u = h->alloc_units(z);
                if (u != HEAP_NULL) r = z;
            } else if (h->policy == BUDDY) {
                uint64_t p2 = 1;
                while (p2 < r) p2 <<= 1;                        /* round up to a power of two */
                if (p2 <= h->A_u) u = h->alloc_units(p2);
                if (u != HEAP_NULL) r = p2;
            } else {
                u = h->alloc_units(r);
            }
        }
        if (u == HEAP_NULL) { out[i] = HEAP_NULL; h->c.allocs_failed++; }
        else {
            out[i] = u * h->align;
            h->c.allocs_ok++;
            h->c.high_water_end = std::max(h->c.high_water_end, (u + r) * h->align);
        }
    }
}

/* stats in the heap_stats_t field order (include/heap.h): 16 x u64, bytes */
/* maximal runs of free slots of pool j as (first slot, count) — "coalescence is implicit" in a
 * bitmask; runs never cross a pool boundary */
static std::vector<std::pair<uint64_t, uint64_t>> pool_runs(const Heap *h, int j) {
    std::vector<std::pair<uint64_t, uint64_t>> runs;
    uint64_t t = 0, N = h->nslots[j];
    while (t < N) {
        if (!h->slot_free(j, t)) { t++; continue; }
        uint64_t a = t;
        while (t < N && h->slot_free(j, t)) t++;
        runs.push_back({a, t - a});
    }
    return runs;
}

void oracle_stats(void *p, uint64_t *o) {
    Heap *h = (Heap *)p;
    if (h->policy == DOUBLE_BUDDY) {
        uint64_t a[16], b[16] = {0};
        oracle_stats(h->sub, a);
        if (h->sub3) oracle_stats(h->sub3, b);
        const uint64_t u3 = 3 * h->align;
        uint64_t live = a[2] + b[2] * u3;
        uint64_t hw = std::max(a[7], b[7] ? h->A_bytes + b[7] * u3 : 0);
        uint64_t vals[16] = {h->arena_bytes, h->align, live, h->arena_bytes - live, a[4] + b[4], a[5] + b[5],
                             std::max(a[6], b[6] * u3), hw, a[8] + b[8], a[9] + b[9], a[10] + b[10],
                             a[11] + b[11] + h->c.frees_invalid, a[12] + b[12], a[13] + b[13] + h->c.frees_null, 0, 0};
        memcpy(o, vals, sizeof(vals));
        return;
    }
    if (h->policy == HYBRID) {
        /* pools + TLSF heap; largest_free is the TLSF heap's (reading C26); counters add up */
        uint64_t sv[16];
        oracle_stats(h->sub, sv);
        uint64_t runs = 0;
        for (int j = 0; j < h->J; j++) runs += pool_runs(h, j).size();
        uint64_t live_b = h->pool_live_b + sv[2];
        uint64_t hw = std::max(h->c.high_water_end, sv[7] ? sv[7] + h->pool_end : 0);
        uint64_t vals[16] = {h->arena_bytes, h->align, live_b, h->arena_bytes - live_b, h->pool_live_n + sv[4],
                             runs + sv[5], sv[6], hw, h->c.allocs_ok + sv[8], h->c.allocs_failed + sv[9],
                             h->c.frees_ok + sv[10], h->c.frees_invalid + sv[11], h->c.frees_double + sv[12],
                             h->c.frees_null + sv[13], 0, 0};
        memcpy(o, vals, sizeof(vals));
        return;
    }
    uint64_t live_b = 0, free_b = 0, nfree = 0, largest = 0;
    for (const auto &kv : h->live) live_b += kv.second;
    if (h->policy == BUDDY || h->policy == FIB_BUDDY) {
        for (int k = 0; k <= h->K; k++) {
            uint64_t z = (h->policy == BUDDY) ? (1ull << k) : h->FS[k];
            nfree += h->bfree[k].size();
            free_b += (uint64_t)h->bfree[k].size() * z;
            if (!h->bfree[k].empty()) largest = std::max<uint64_t>(largest, z);
        }
    } else {
        for (const auto &kv : h->freeb) { free_b += kv.second; nfree++; largest = std::max(largest, kv.second); }
    }
    uint64_t a = h->align;
    uint64_t vals[16] = {h->arena_bytes, a, live_b * a, free_b * a, (uint64_t)h->live.size(), nfree,
                         largest * a, h->c.high_water_end, h->c.allocs_ok, h->c.allocs_failed,
                         h->c.frees_ok, h->c.frees_invalid, h->c.frees_double, h->c.frees_null, 0, 0};
    memcpy(o, vals, sizeof(vals));
}

/* export: free (start,size) pairs in address order and live (start,size) pairs, bytes.
 * counts[0] = #free, counts[1] = #live; pairs written only up to the capacities. */
void oracle_export(void *p, uint64_t *free_pairs, uint64_t cap_free, uint64_t *live_pairs,
                   uint64_t cap_live, uint64_t *counts) {
    Heap *h = (Heap *)p;
    if (h->policy == DOUBLE_BUDDY) {
        /* the binary heap's blocks (below A_bytes), then the 3-unit heap's, in bytes */
        std::vector<uint64_t> fp, lp;
        const uint64_t u3 = 3 * h->align;
        for (int part = 0; part < 2; part++) {
            Heap *x = part ? h->sub3 : h->sub;
            if (!x) continue;
            uint64_t sc[2];
            oracle_export(x, nullptr, 0, nullptr, 0, sc);
            std::vector<uint64_t> sf(2 * sc[0] + 2), sl(2 * sc[1] + 2);
            oracle_export(x, sf.data(), sc[0], sl.data(), sc[1], sc);
            const uint64_t base = part ? h->A_bytes : 0, mul = part ? u3 : 1;
            for (uint64_t k = 0; k < sc[0]; k++) { fp.push_back(base + sf[2 * k] * mul); fp.push_back(sf[2 * k + 1] * mul); }
            for (uint64_t k = 0; k < sc[1]; k++) { lp.push_back(base + sl[2 * k] * mul); lp.push_back(sl[2 * k + 1] * mul); }
        }
        counts[0] = fp.size() / 2;
        counts[1] = lp.size() / 2;
        for (uint64_t k = 0; k < counts[0] && k < cap_free; k++) { free_pairs[2 * k] = fp[2 * k]; free_pairs[2 * k + 1] = fp[2 * k + 1]; }
        for (uint64_t k = 0; k < counts[1] && k < cap_live; k++) { live_pairs[2 * k] = lp[2 * k]; live_pairs[2 * k + 1] = lp[2 * k + 1]; }
        return;
    }
    if (h->policy == HYBRID) {
        /* pool runs / objects first (they lie below pool_end), then the TLSF heap's, shifted */
        std::vector<uint64_t> fp, lp;
        for (int j = 0; j < h->J; j++) {
            uint64_t oj = h->align << j, base = (uint64_t)j * h->S;
            for (auto &r : pool_runs(h, j)) { fp.push_back(base + r.first * oj); fp.push_back(r.second * oj); }
            for (uint64_t t = 0; t < h->fresh[j]; t++)
                if (!h->freed[j].count(t)) { lp.push_back(base + t * oj); lp.push_back(oj); }
        }
        uint64_t sc[2];
        oracle_export(h->sub, nullptr, 0, nullptr, 0, sc);
        std::vector<uint64_t> sf(2 * sc[0] + 2), sl(2 * sc[1] + 2);
        oracle_export(h->sub, sf.data(), sc[0], sl.data(), sc[1], sc);
        for (uint64_t k = 0; k < sc[0]; k++) { fp.push_back(sf[2 * k] + h->pool_end); fp.push_back(sf[2 * k + 1]); }
        for (uint64_t k = 0; k < sc[1]; k++) { lp.push_back(sl[2 * k] + h->pool_end); lp.push_back(sl[2 * k + 1]); }
        counts[0] = fp.size() / 2;
        counts[1] = lp.size() / 2;
        for (uint64_t k = 0; k < counts[0] && k < cap_free; k++) { free_pairs[2 * k] = fp[2 * k]; free_pairs[2 * k + 1] = fp[2 * k + 1]; }
        for (uint64_t k = 0; k < counts[1] && k < cap_live; k++) { live_pairs[2 * k] = lp[2 * k]; live_pairs[2 * k + 1] = lp[2 * k + 1]; }
        return;
    }
    uint64_t a = h->align, i = 0;
    if (h->policy == BUDDY || h->policy == FIB_BUDDY) {
        std::map<uint64_t, uint64_t> all;
        for (int k = 0; k <= h->K; k++)
            for (uint64_t s : h->bfree[k]) all[s] = (h->policy == BUDDY) ? (1ull << k) : h->FS[k];
        for (const auto &kv : all) { if (i < cap_free) { free_pairs[2 * i] = kv.first * a; free_pairs[2 * i + 1] = kv.second * a; } i++; }
    } else {
        for (const auto &kv : h->freeb) { if (i < cap_free) { free_pairs[2 * i] = kv.first * a; free_pairs[2 * i + 1] = kv.second * a; } i++; }
    }
    counts[0] = i;
    i = 0;
    for (const auto &kv : h->live) { if (i < cap_live) { live_pairs[2 * i] = kv.first * a; live_pairs[2 * i + 1] = kv.second * a; } i++; }
    counts[1] = i;
}

/* the TLSF mapping, exported so tests can pin it against the paper's log2 formulas */
uint64_t oracle_insert_class(uint64_t u, int L) { return insert_class(u, L); }
uint64_t oracle_search_class(uint64_t u, int L) { return search_class(u, L); }

}  // extern "C"
