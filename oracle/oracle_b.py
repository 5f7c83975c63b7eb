"""Oracle-B — brute-force allocator over a unit bitmap.  TEST INFRASTRUCTURE ONLY.

Structurally different from Oracle-L: it keeps no free list at all.  The state is
one bit per unit of the arena (set = free), as in the paper's bitmask allocator
(§3.2), plus the live map (start -> size) that a free needs.
Free blocks are DERIVED on every call:

* fits / SEGFIT / TLSF: the maximal runs of free units (coalescing is implicit in
  the bitmap);
* BUDDY: the maximal aligned free power-of-two blocks inside the root blocks of the
  arena's greedy decomposition (binary buddies).

An alloc enumerates every derived block and applies the policy key of DESIGN.md
§5 directly (lowest key wins), then clears the bits it hands out.  The class
mapping is written here from its *defining property* (search class = the smallest
class whose lower bound is >= the request) rather than Oracle-L's formula, so the
two oracles pin each other.  O(arena units) per op: tiny heaps and config 1 only.
"""
from __future__ import annotations

import numpy as np

HEAP_NULL = (1 << 64) - 1
FIRST_FIT, BEST_FIT, SEGFIT, TLSF, BUDDY = 1, 2, 3, 4, 5
NEXT_FIT = 8
PARTIAL = 0x100     # policy flag: partial (tail) deallocation (Alg. 2 :205-212)


def cls_of(u: int, L: int) -> int:
    """Class of a block of u units: exact below 2^L, else (fl, sl) from the top L+1 bits."""
    if u < (1 << L):
        return u
    m = u.bit_length() - 1
    return (m - L + 1) * (1 << L) + ((u >> (m - L)) - (1 << L))


def cls_lo(c: int, L: int) -> int:
    """Smallest block size (units) of class c."""
    fl, sl = divmod(c, 1 << L)
    return sl if fl == 0 else ((1 << L) + sl) << (fl - 1)


def search_cls(u: int, L: int) -> int:
    """Smallest class all of whose blocks hold u units: min{c : lo(c) >= u}."""
    c = cls_of(u, L)
    while cls_lo(c, L) < u:
        c += 1
    return c


class OracleB:
    def __init__(self, arena_bytes: int, align: int, policy: int):
        assert align > 0 and align & (align - 1) == 0 and arena_bytes % align == 0
        self.partial = bool(policy & PARTIAL)
        policy &= ~PARTIAL
        assert not (self.partial and policy == BUDDY)
        self.align, self.policy = align, policy
        self.A = arena_bytes // align
        self.bits = np.ones(self.A, dtype=bool)
        self.live: dict[int, int] = {}
        # owner[u] = start of the live block holding unit u, -1 if u is free (a per-unit map
        # instead of Oracle-L's ordered search, so a partial free is located differently)
        self.owner = np.full(self.A, -1, dtype=np.int64)
        self.L = 5 if policy == TLSF else 0
        self.roots = []
        if policy == BUDDY:
            s, K = 0, self.A.bit_length() - 1
            while s < self.A:
                t = K
                while t > 0 and (s % (1 << t) or s + (1 << t) > self.A):
                    t -= 1
                self.roots.append((s, t))
                s += 1 << t
        self._counts = dict(allocs_ok=0, allocs_failed=0, frees_ok=0, frees_invalid=0,
                           frees_double=0, frees_null=0)
        self.rover = 0       # NEXT_FIT (reading C27): only allocations move it
        self.hw = 0          # max over successful allocations of its end (units)

    @property
    def counts(self):
        """Outcome counters, plus the two size statistics of heap_stats_t derived here from the
        bitmap: the largest derived free block and the high-water end (the largest end of any
        allocation so far, the 'provisioned' extent of PAPER.md:518's fragmentation measure)."""
        c = dict(self._counts)
        c["largest_free"] = max((z for _, z in self.blocks()), default=0) * self.align
        c["high_water_end"] = self.hw * self.align
        return c

    # ---- derived free blocks ----
    def runs(self):
        b = self.bits.astype(np.int8)
        d = np.diff(np.concatenate(([0], b, [0])))
        starts = np.flatnonzero(d == 1)
        ends = np.flatnonzero(d == -1)
        return [(int(s), int(e - s)) for s, e in zip(starts, ends)]

    def buddy_blocks(self):
        out = []

        def rec(s, t):
            if self.bits[s:s + (1 << t)].all():
                out.append((s, 1 << t))
            elif t > 0:
                rec(s, t - 1)
                rec(s + (1 << (t - 1)), t - 1)
        for s, t in self.roots:
            rec(s, t)
        return out

    def blocks(self):
        return self.buddy_blocks() if self.policy == BUDDY else self.runs()

    # ---- ops ----
    def alloc_units(self, r: int):
        blocks = self.blocks()
        if self.policy == FIRST_FIT:
            cand = [(s, s, z) for s, z in blocks if z >= r]
        elif self.policy == NEXT_FIT:
            # key (wrapped, start): blocks at or after the rover first, then from address 0
            cand = [((s < self.rover, s), s, z) for s, z in blocks if z >= r]
        elif self.policy == BEST_FIT:
            cand = [((z, s), s, z) for s, z in blocks if z >= r]
        elif self.policy in (SEGFIT, TLSF):
            c = search_cls(r, self.L)
            cand = [((cls_of(z, self.L), s), s, z) for s, z in blocks if cls_of(z, self.L) >= c]
        else:
            cand = [((z, s), s, z) for s, z in blocks if z >= r]   # (order, start), z = 2^order
        if not cand:
            return None
        _, s, _ = min(cand)
        self.bits[s:s + r] = False
        self.owner[s:s + r] = s
        self.live[s] = r
        self.rover = s + r
        self.hw = max(self.hw, s + r)
        return s

    def alloc_batch(self, sizes):
        out = np.empty(len(sizes), dtype=np.uint64)
        for i, sz in enumerate(int(x) for x in sizes):
            r = -(-sz // self.align)
            u = None
            if sz != 0 and r <= self.A:
                if self.policy == BUDDY:
                    p = 1
                    while p < r:
                        p <<= 1
                    r = p
                    u = self.alloc_units(r) if r <= self.A else None
                else:
                    u = self.alloc_units(r)
            if u is None:
                out[i] = HEAP_NULL
                self._counts["allocs_failed"] += 1
            else:
                out[i] = u * self.align
                self._counts["allocs_ok"] += 1
        return out

    def free_batch(self, offsets):
        free_starts = {s for s, _ in self.blocks()}
        seen = set()
        to_free = []
        for o in sorted(int(x) for x in offsets):
            if o == HEAP_NULL:
                self._counts["frees_null"] += 1
            elif o % self.align or o // self.align >= self.A:
                self._counts["frees_invalid"] += 1
            else:
                u = o // self.align
                a = int(self.owner[u])
                if u in free_starts:
                    self._counts["frees_double"] += 1
                elif a < 0 or (a != u and not self.partial):
                    self._counts["frees_invalid"] += 1
                elif a in seen:            # a copy, or a second offset inside one live block
                    self._counts["frees_double"] += 1
                else:
                    seen.add(a)
                    self._counts["frees_ok"] += 1
                    to_free.append((a, u))
        for a, u in to_free:
            end = a + self.live[a]
            if u == a:
                del self.live[a]
            else:
                self.live[a] = u - a      # the in-use block is shrunk
            self.bits[u:end] = True
            self.owner[u:end] = -1

    def export(self):
        fp = np.array([(s * self.align, z * self.align) for s, z in self.blocks()],
                      dtype=np.uint64).reshape(-1, 2)
        lp = np.array(sorted((s * self.align, z * self.align) for s, z in self.live.items()),
                      dtype=np.uint64).reshape(-1, 2)
        return fp, lp


class OracleBLifo:
    """Brute-force twin of Oracle-L's SEGFIT_LIFO (the paper's Alg. 4/5 with stack bins).

    Free blocks are a flat Python list of [start, size, stamp]; every decision is a linear
    scan: alloc takes the minimum (bin, -stamp) over blocks whose bin >= ceil-bin of the
    request (Alg. 4 pops the head of the first nonempty bin, :332-337, :440); a free removes
    the free neighbours ending at / starting right after the block and pushes the merged block
    (Alg. 5 :374-436).  Every push takes the next tick of a logical clock."""

    def __init__(self, arena_bytes: int, align: int, policy: int = 6):
        assert policy == 6
        self.align, self.A = align, arena_bytes // align
        self.free = [[0, self.A, 0]]
        self.clock = 1
        self.live: dict[int, int] = {}
        self.counts = dict(allocs_ok=0, allocs_failed=0, frees_ok=0, frees_invalid=0,
                           frees_double=0, frees_null=0)

    @staticmethod
    def _bin(size):            # floor(log2 size) + 1 (our class numbering, SL_LOG2 = 0)
        return size.bit_length()

    @staticmethod
    def _req_bin(r):           # ceil(log2 r) + 1
        return (r - 1).bit_length() + 1

    def _push(self, s, z):
        self.free.append([s, z, self.clock])
        self.clock += 1

    def alloc_units(self, r):
        c = self._req_bin(r)
        cand = [(self._bin(z), -st, i) for i, (s, z, st) in enumerate(self.free) if self._bin(z) >= c]
        if not cand:
            return None
        _, _, i = min(cand)
        s, z, _ = self.free.pop(i)
        if z > r:
            self._push(s + r, z - r)
        self.live[s] = r
        return s

    def alloc_batch(self, sizes):
        out = np.empty(len(sizes), dtype=np.uint64)
        for i, sz in enumerate(int(x) for x in sizes):
            r = -(-sz // self.align)
            u = self.alloc_units(r) if sz != 0 and r <= self.A else None
            if u is None:
                out[i] = HEAP_NULL
                self.counts["allocs_failed"] += 1
            else:
                out[i] = u * self.align
                self.counts["allocs_ok"] += 1
        return out

    def free_batch(self, offsets):
        free_starts = {s for s, _, _ in self.free}
        seen, to_free = set(), []
        for o in sorted(int(x) for x in offsets):
            if o == HEAP_NULL:
                self.counts["frees_null"] += 1
            elif o % self.align or o // self.align >= self.A:
                self.counts["frees_invalid"] += 1
            else:
                u = o // self.align
                if u in self.live:
                    if u in seen:
                        self.counts["frees_double"] += 1
                    else:
                        seen.add(u)
                        self.counts["frees_ok"] += 1
                        to_free.append(u)
                elif u in free_starts:
                    self.counts["frees_double"] += 1
                else:
                    self.counts["frees_invalid"] += 1
        for u in to_free:
            z = self.live.pop(u)
            s, e = u, u + z
            for blk in list(self.free):
                if blk[0] + blk[1] == u:
                    s = blk[0]
                    self.free.remove(blk)
                elif blk[0] == u + z:
                    e = blk[0] + blk[1]
                    self.free.remove(blk)
            self._push(s, e - s)

    def export(self):
        fp = np.array(sorted((s * self.align, z * self.align) for s, z, _ in self.free),
                      dtype=np.uint64).reshape(-1, 2)
        lp = np.array(sorted((s * self.align, z * self.align) for s, z in self.live.items()),
                      dtype=np.uint64).reshape(-1, 2)
        return fp, lp


class OracleBHybrid:
    """Brute-force twin of Oracle-L's HYBRID (§5.3).

    The pools are kept literally as the paper's bitmasks (§3.2): one numpy
    boolean per object, True = free; an allocation takes the first True (np.flatnonzero) and a
    free sets it back.  Requests the pools do not take go to an OracleB TLSF heap (unit bitmap,
    blocks derived on every call) covering [pool_end, arena).  The layout is recomputed here from
    the words of DESIGN.md reading C26, not from Oracle-L's code."""

    PAGE = 4096

    def __init__(self, arena_bytes: int, align: int, policy: int = 7):
        assert policy == 7
        self.align, self.arena = align, arena_bytes
        self.obj = [align << j for j in range(64) if (align << j) <= self.PAGE]
        share = arena_bytes // (2 * len(self.obj)) if self.obj else 0
        self.S = share - share % self.PAGE
        self.pool_end = len(self.obj) * self.S
        self.pools = [np.ones(self.S // o, dtype=bool) for o in self.obj]
        self.sub = OracleB(arena_bytes - self.pool_end, align, TLSF)
        self.own = dict(allocs_ok=0, frees_ok=0, frees_invalid=0, frees_double=0, frees_null=0)
        self.pool_hw = 0

    @property
    def counts(self):
        c = dict(self.sub.counts)
        for k, v in self.own.items():
            c[k] = c.get(k, 0) + v
        # largest_free is the TLSF heap's (reading C26); the high-water end spans pools and heap
        sub_hw = c["high_water_end"]
        c["high_water_end"] = max(self.pool_hw, sub_hw + self.pool_end if sub_hw else 0)
        return c

    @property
    def live(self):        # for the exhaustive enumerations: every live start (bytes)
        return [int(o) for o, _ in self.export()[1]]

    def alloc_batch(self, sizes):
        out = np.empty(len(sizes), dtype=np.uint64)
        for i, s in enumerate(int(x) for x in sizes):
            fits = [j for j, o in enumerate(self.obj) if o >= s]
            if 0 < s < self.PAGE and fits:
                j = fits[0]
                free = np.flatnonzero(self.pools[j])
                if len(free):
                    t = int(free[0])
                    self.pools[j][t] = False
                    out[i] = j * self.S + t * self.obj[j]
                    self.own["allocs_ok"] += 1
                    self.pool_hw = max(self.pool_hw, int(out[i]) + self.obj[j])
                    continue
            o = int(self.sub.alloc_batch(np.array([s], dtype=np.uint64))[0])
            out[i] = HEAP_NULL if o == HEAP_NULL else o + self.pool_end
        return out

    def free_batch(self, offsets):
        sub, seen, to_free = [], set(), []
        for o in sorted(int(x) for x in offsets):
            if o == HEAP_NULL:
                self.own["frees_null"] += 1
            elif o >= self.pool_end:
                sub.append(o - self.pool_end)
            else:
                j = o // self.S
                rel = o - j * self.S
                if rel % self.obj[j]:
                    self.own["frees_invalid"] += 1
                    continue
                t = rel // self.obj[j]
                if self.pools[j][t] or (j, t) in seen:
                    self.own["frees_double"] += 1
                else:
                    seen.add((j, t))
                    to_free.append((j, t))
                    self.own["frees_ok"] += 1
        for j, t in to_free:
            self.pools[j][t] = True
        self.sub.free_batch(np.array(sub, dtype=np.uint64))

    def export(self):
        fp, lp = [], []
        for j, (o, bits) in enumerate(zip(self.obj, self.pools)):
            base = j * self.S
            t = 0
            while t < len(bits):
                if not bits[t]:
                    lp.append((base + t * o, o))
                    t += 1
                    continue
                a = t
                while t < len(bits) and bits[t]:
                    t += 1
                fp.append((base + a * o, (t - a) * o))
        sf, sl = self.sub.export()
        fp += [(int(s) + self.pool_end, int(z)) for s, z in sf]
        lp += [(int(s) + self.pool_end, int(z)) for s, z in sl]
        return (np.array(fp, dtype=np.uint64).reshape(-1, 2), np.array(lp, dtype=np.uint64).reshape(-1, 2))


class OracleBDouble:
    """Brute-force twin of Oracle-L's DOUBLE_BUDDY (reading C28): two OracleB
    binary-buddy heaps (unit bitmaps, blocks derived on every call), the second counting in
    units of 3*align.  The class choice is written from its definition: the smallest block of
    either family {2^k} / {3 * 2^k} (units) that holds the request."""

    def __init__(self, arena_bytes: int, align: int, policy: int = 9):
        assert policy == 9
        self.align, self.arena = align, arena_bytes
        self.N3 = arena_bytes // (6 * align)
        self.A_bytes = arena_bytes - 3 * align * self.N3
        self.a = OracleB(self.A_bytes, align, BUDDY)
        self.b = OracleB(self.N3, 1, BUDDY) if self.N3 else None
        self.own = dict(frees_null=0, frees_invalid=0)

    @property
    def counts(self):
        c = dict(self.a.counts)
        if self.b:
            for k, v in self.b.counts.items():
                c[k] += v
        for k, v in self.own.items():
            c[k] += v
        del c["largest_free"], c["high_water_end"]   # per-heap statistics: not additive
        return c

    @property
    def live(self):
        return [int(o) for o, _ in self.export()[1]]

    def alloc_batch(self, sizes):
        out = np.empty(len(sizes), dtype=np.uint64)
        for i, s in enumerate(int(x) for x in sizes):
            r = -(-s // self.align)
            two = next(1 << k for k in range(80) if (1 << k) >= r)
            three = next(3 << k for k in range(80) if (3 << k) >= r)
            if s and r <= self.arena // self.align and self.b and three < two:
                u = int(self.b.alloc_batch(np.array([three // 3], dtype=np.uint64))[0])
                out[i] = HEAP_NULL if u == HEAP_NULL else self.A_bytes + u * 3 * self.align
            else:
                out[i] = self.a.alloc_batch(np.array([s], dtype=np.uint64))[0]
        return out

    def free_batch(self, offsets):
        fa, fb = [], []
        for o in (int(x) for x in offsets):
            if o == HEAP_NULL:
                self.own["frees_null"] += 1
            elif o < self.A_bytes:
                fa.append(o)
            elif self.b is None or (o - self.A_bytes) % (3 * self.align):
                self.own["frees_invalid"] += 1
            else:
                fb.append((o - self.A_bytes) // (3 * self.align))
        self.a.free_batch(np.array(fa, dtype=np.uint64))
        if self.b:
            self.b.free_batch(np.array(fb, dtype=np.uint64))

    def export(self):
        fa, la = self.a.export()
        fp, lp = [tuple(map(int, x)) for x in fa], [tuple(map(int, x)) for x in la]
        if self.b:
            fb, lb = self.b.export()
            m = 3 * self.align
            fp += [(self.A_bytes + int(s) * m, int(z) * m) for s, z in fb]
            lp += [(self.A_bytes + int(s) * m, int(z) * m) for s, z in lb]
        return (np.array(fp, dtype=np.uint64).reshape(-1, 2), np.array(lp, dtype=np.uint64).reshape(-1, 2))


class OracleBFib:
    """Brute-force twin of Oracle-L's FIB_BUDDY (Fibonacci buddies; reading C30).

    No free lists at all: a unit bitmap plus the live map.  The arena is cut greedily into
    Fibonacci roots (largest first); a block of size F splits into its low part of the previous
    Fibonacci size and its high part of the one before (2 = 1 + 1).  The free blocks are DERIVED
    on every call as the maximal fully-free nodes of those split trees, so merging is implicit.
    An alloc takes the smallest free node holding the request (ties: lowest address) and uses the
    node of the request's size at its start (descending through low parts); a free sets bits."""

    def __init__(self, arena_bytes: int, align: int, policy: int = 10):
        assert policy == 10
        self.align, self.A = align, arena_bytes // align
        fib = [1]
        if self.A >= 2:
            fib.append(2)
        while len(fib) >= 2 and fib[-1] + fib[-2] <= self.A:
            fib.append(fib[-1] + fib[-2])
        self.fib = fib
        self.roots, s, rem = [], 0, self.A
        while rem:
            z = max(x for x in fib if x <= rem)
            self.roots.append((s, z))
            s, rem = s + z, rem - z
        self.bits = np.ones(self.A, dtype=bool)
        self.live: dict[int, int] = {}
        self.counts = dict(allocs_ok=0, allocs_failed=0, frees_ok=0, frees_invalid=0,
                           frees_double=0, frees_null=0)

    def _children(self, s, z):
        i = self.fib.index(z)
        lo = self.fib[i - 1] if i >= 1 else None
        if lo is None:
            return []
        hi = z - lo                      # 2 = 1 + 1, otherwise the Fibonacci number before lo
        return [(s, lo), (s + lo, hi)]

    def blocks(self):
        out = []

        def rec(s, z):
            if self.bits[s:s + z].all():
                out.append((s, z))
            else:
                for c in self._children(s, z):
                    rec(*c)
        for r in self.roots:
            rec(*r)
        return sorted(out)

    def alloc_batch(self, sizes):
        out = np.empty(len(sizes), dtype=np.uint64)
        for i, sz in enumerate(int(x) for x in sizes):
            r = -(-sz // self.align)
            fits = [x for x in self.fib if x >= r]
            cand = [(z, s) for s, z in self.blocks() if fits and z >= fits[0]] if sz else []
            if not cand:
                out[i] = HEAP_NULL
                self.counts["allocs_failed"] += 1
                continue
            _, s = min(cand)
            self.bits[s:s + fits[0]] = False
            self.live[s] = fits[0]
            out[i] = s * self.align
            self.counts["allocs_ok"] += 1
        return out

    def free_batch(self, offsets):
        free_starts = {s for s, _ in self.blocks()}
        seen, to_free = set(), []
        for o in sorted(int(x) for x in offsets):
            if o == HEAP_NULL:
                self.counts["frees_null"] += 1
            elif o % self.align or o // self.align >= self.A:
                self.counts["frees_invalid"] += 1
            else:
                u = o // self.align
                if u in self.live and u not in seen:
                    seen.add(u)
                    self.counts["frees_ok"] += 1
                    to_free.append(u)
                elif u in self.live or u in free_starts:
                    self.counts["frees_double"] += 1
                else:
                    self.counts["frees_invalid"] += 1
        for u in to_free:
            self.bits[u:u + self.live.pop(u)] = True

    def export(self):
        fp = np.array([(s * self.align, z * self.align) for s, z in self.blocks()], dtype=np.uint64).reshape(-1, 2)
        lp = np.array(sorted((s * self.align, z * self.align) for s, z in self.live.items()),
                      dtype=np.uint64).reshape(-1, 2)
        return fp, lp
