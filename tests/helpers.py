"""Shared test helpers: trace replay, invariant checker, golden-file parser.

Nothing here implements allocator arithmetic; the invariants are the paper's
properties checked on exported state.
"""
from __future__ import annotations

import os

import numpy as np

HEAP_NULL = (1 << 64) - 1
POLICY = {"FIRST": 1, "BEST": 2, "SEGFIT": 3, "TLSF": 4, "BUDDY": 5, "LIFO": 6, "HYBRID": 7, "NEXT": 8, "DOUBLE": 9, "FIB": 10}
PARTIAL = 0x100      # policy flag: partial (tail) deallocation (include/heap.h HEAP_PARTIAL_FREE)
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class IdMap:
    """id -> offset map of a trace (HEAP_NULL for failed or not-yet-made allocs)."""

    def __init__(self, n: int):
        self.a = np.full(max(n, 1), HEAP_NULL, dtype=np.uint64)

    def ensure(self, n):
        if n > self.a.size:
            b = np.full(max(n, 2 * self.a.size), HEAP_NULL, dtype=np.uint64)
            b[: self.a.size] = self.a
            self.a = b

    def offsets(self, ids: np.ndarray) -> np.ndarray:
        return self.a[ids.astype(np.int64)] if ids.size else np.zeros(0, dtype=np.uint64)

    def record(self, first: int, out: np.ndarray):
        self.ensure(first + out.size)
        self.a[first:first + out.size] = out


def replay(heap, trace, idmap: IdMap | None = None, on_batch=None, max_batches=None):
    """Drive ``heap`` (free_batch / alloc_batch) with a tracegen.Trace."""
    idmap = idmap or IdMap(1 << 16)
    for bi, (fids, sizes, first) in enumerate(trace):
        if max_batches is not None and bi >= max_batches:
            break
        offs = idmap.offsets(fids)
        heap.free_batch(offs)
        out = heap.alloc_batch(sizes)
        idmap.record(first, np.asarray(out, dtype=np.uint64))
        if on_batch is not None:
            on_batch(bi, offs, sizes, out)
    return idmap


def replay_partial(heaps, cfg, seed: int, p_tail=0.5, p_extra=0.15, p_wild=0.05, on_batch=None):
    """Drive ``heaps`` in lockstep with a tracegen trace whose frees are partly turned into
    partial (tail) frees (policy flag PARTIAL).  Every input comes from the trace,
    a seeded numpy generator and heaps[0] (the oracle) — never from the heap under test:
    for a freed id of u units at offset o, with probability p_tail the offset becomes
    o + d*align, d uniform in [1, u) (the id keeps its d-unit head, which the trace then never
    frees: a leak, as a caller that shrinks a block and forgets it); extra offsets are added
    inside the same block (a second offset: a double free) or anywhere in the arena (start,
    interior or free memory).  Returns the per-batch outputs of heaps[0]."""
    rng = np.random.default_rng(seed)
    align, A_u = cfg.align, cfg.arena_bytes // cfg.align
    idmap = IdMap(1 << 12)
    units = {}
    for bi, (fids, sizes, first) in enumerate(__import__("tracegen").Trace(cfg)):
        offs = [int(x) for x in idmap.offsets(fids)]
        extra = []
        for j, fid in enumerate(int(x) for x in fids):
            o = offs[j]
            if o == HEAP_NULL:
                continue
            z = units.get(fid, 1)
            x = rng.random()
            if x < p_tail and z > 1:
                d = 1 + int(rng.integers(z - 1))
                offs[j] = o + d * align
                if rng.random() < p_extra:
                    extra.append(o + int(rng.integers(d, z)) * align)
            elif x < p_tail + p_extra:
                extra.append(o + int(rng.integers(z)) * align)
            if rng.random() < p_wild:
                extra.append(int(rng.integers(A_u)) * align)
        batch = np.array(offs + extra, dtype=np.uint64)
        outs = []
        for h in heaps:
            h.free_batch(batch)
            outs.append(np.asarray(h.alloc_batch(sizes), dtype=np.uint64))
        for k, sz in enumerate(int(x) for x in sizes):
            units[first + k] = -(-sz // align)
        idmap.record(first, outs[0])
        if on_batch is not None:
            on_batch(bi, batch, sizes, outs)


def hybrid_layout(arena: int, align: int):
    """(share S, pool_end, object sizes) of a HYBRID heap, reading C26."""
    obj = [align << j for j in range(64) if (align << j) <= 4096]
    share = arena // (2 * len(obj)) if obj else 0
    S = share - share % 4096
    return S, len(obj) * S, obj


def double_layout(arena: int, align: int):
    """(A_bytes, N3) of a DOUBLE_BUDDY heap, reading C28."""
    n3 = arena // (6 * align)
    return arena - 3 * align * n3, n3


def check_double_invariants(free_pairs, live_pairs, arena: int, align: int):
    """DOUBLE_BUDDY: each heap separately satisfies the buddy invariants in its own units."""
    A_bytes, n3 = double_layout(arena, align)
    fp = np.asarray(free_pairs, dtype=np.uint64).reshape(-1, 2)
    lp = np.asarray(live_pairs, dtype=np.uint64).reshape(-1, 2)
    lo_f, lo_l = fp[fp[:, 0] < A_bytes], lp[lp[:, 0] < A_bytes]
    check_invariants(lo_f, lo_l, A_bytes, align, True)
    if n3:
        m = np.uint64(3 * align)
        hi_f, hi_l = fp[fp[:, 0] >= A_bytes], lp[lp[:, 0] >= A_bytes]
        assert np.all((hi_f[:, 0] - np.uint64(A_bytes)) % m == 0) and np.all(hi_f[:, 1] % m == 0)
        assert np.all((hi_l[:, 0] - np.uint64(A_bytes)) % m == 0) and np.all(hi_l[:, 1] % m == 0)
        to_u = lambda a: np.c_[(a[:, 0] - np.uint64(A_bytes)) // m, a[:, 1] // m]  # noqa: E731
        check_invariants(to_u(hi_f), to_u(hi_l), n3, 1, True)


def check_invariants(free_pairs, live_pairs, arena: int, align: int, buddy: bool, region_edges=()):
    """I1 no overlap, I2 tiling/conservation, I3 full coalescing, I4 alignment.
    ``region_edges``: addresses where two free blocks may touch (HYBRID pool boundaries: pools
    and the TLSF heap never coalesce with each other)."""
    fp = np.asarray(free_pairs, dtype=np.uint64).reshape(-1, 2)
    lp = np.asarray(live_pairs, dtype=np.uint64).reshape(-1, 2)
    allb = np.concatenate([np.c_[fp, np.zeros(len(fp), np.uint64)],
                           np.c_[lp, np.ones(len(lp), np.uint64)]])
    allb = allb[np.argsort(allb[:, 0], kind="stable")]
    # I4 alignment and positive sizes
    assert np.all(allb[:, 0] % align == 0) and np.all(allb[:, 1] % align == 0)
    assert np.all(allb[:, 1] > 0)
    # I1 + I2: sorted blocks tile [0, arena) exactly
    if len(allb):
        assert allb[0, 0] == 0
        ends = allb[:, 0] + allb[:, 1]
        assert np.all(ends[:-1] == allb[1:, 0]), "overlap or gap"
        assert ends[-1] == arena
    else:
        assert arena == 0
    assert int(fp[:, 1].sum()) + int(lp[:, 1].sum()) == arena
    # I3 coalescing
    if len(fp):
        fps = fp[np.argsort(fp[:, 0])]
        if not buddy:
            touch = fps[:-1, 0] + fps[:-1, 1] == fps[1:, 0]
            edges = np.array(sorted(region_edges), dtype=np.uint64)
            assert np.all(~touch | np.isin(fps[1:, 0], edges)), "adjacent free blocks"
        else:
            sz = fps[:, 1]
            assert np.all(sz & (sz - 1) == 0)
            assert np.all(fps[:, 0] % sz == 0), "buddy block not aligned to its size"
            s = set(map(tuple, fps.tolist()))
            for a, z in s:
                assert (a ^ z, z) not in s, "two free buddies not merged"


def parse_golden(name: str):
    cases = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            body, _, cite = line.partition("@")
            head, ops, expect = [x.strip() for x in body.split("|")]
            pol, arena, align = head.split()
            batches = []
            for b in ops.split("/"):
                fr = [int(t[1:]) for t in b.split() if t.startswith("f")]
                al = [int(t[1:]) for t in b.split() if t.startswith("a")]
                batches.append((fr, al))
            outs, _, frees = expect.partition("#")
            outs = [int(x) for x in outs.split()]
            frees = frees.strip()
            if frees == "*":
                fl = None
            else:
                fl = [tuple(int(v) for v in x.split(":")) for x in frees.split()]
            pol, _, flag = pol.partition("+")
            pid = POLICY[pol] | (PARTIAL if flag == "P" else 0)
            cases.append(dict(policy=pid, arena=int(arena), align=int(align),
                              batches=batches, outs=outs, frees=fl, cite=cite.strip()))
    return cases


def fib_roots(arena: int, align: int):
    """(sizes, roots) of a FIB_BUDDY heap in units (reading C30): the Fibonacci sizes
    1, 2, 3, 5, ... up to the arena and its greedy (Zeckendorf) root decomposition."""
    A = arena // align
    fib = [1] + ([2] if A >= 2 else [])
    while len(fib) >= 2 and fib[-1] + fib[-2] <= A:
        fib.append(fib[-1] + fib[-2])
    roots, s, rem = [], 0, A
    while rem:
        z = max(x for x in fib if x <= rem)
        roots.append((s, z))
        s, rem = s + z, rem - z
    return fib, roots


def check_fib_invariants(free_pairs, live_pairs, arena: int, align: int):
    """FIB_BUDDY: tiling (I1/I2), every block is a node of a root's Fibonacci split tree, and no
    two free siblings coexist (I3: complete merging)."""
    fp = np.asarray(free_pairs, dtype=np.uint64).reshape(-1, 2)
    lp = np.asarray(live_pairs, dtype=np.uint64).reshape(-1, 2)
    check_invariants(np.zeros((0, 2), np.uint64), np.concatenate([fp, lp]), arena, align, True)
    fib, roots = fib_roots(arena, align)
    nodes = {}

    def rec(s, z, parent):
        nodes[(s, z)] = parent
        i = fib.index(z)
        if i >= 1:
            lo = fib[i - 1]
            rec(s, lo, (s, z))
            rec(s + lo, z - lo, (s, z))
    if arena // align <= 1 << 14:
        for r in roots:
            rec(*r, None)
        a = int(align)
        free = {(int(s) // a, int(z) // a) for s, z in fp}
        for blk in free | {(int(s) // a, int(z) // a) for s, z in lp}:
            assert blk in nodes, f"block {blk} is not a tree node"
        kids = {}
        for blk in free:
            if nodes[blk] is not None:
                kids.setdefault(nodes[blk], []).append(blk)
        assert all(len(v) < 2 for v in kids.values()), "two free siblings not merged"
