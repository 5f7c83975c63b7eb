"""Pins for the oracle (-m "not gpu").

The oracle is only trusted because these tests tie it to something other than
itself: the paper's formulas and worked examples (tests/golden/, each line cited),
closed forms (fresh-heap prefix sums, buddy addresses), the paper's invariants,
and a structurally different brute-force oracle (Oracle-B) including exhaustive
enumeration on tiny heaps.  A plausible slip in Oracle-L (wrong split end, missing
left/right merge, off-by-one class, wrong tie-break, LIFO instead of address order,
wrong buddy half) fails at least one of them.
"""
from __future__ import annotations

import itertools
import random

import numpy as np
import pytest

import tracegen as tg
from oracle import OracleL, insert_class, search_class
import copy

from oracle.oracle_b import OracleB, OracleBDouble, OracleBFib, OracleBHybrid, OracleBLifo, cls_lo, cls_of, search_cls
from tests.helpers import (HEAP_NULL, PARTIAL, IdMap, check_double_invariants, check_fib_invariants, check_invariants,
                           double_layout, fib_roots, hybrid_layout, parse_golden, replay, replay_partial)

FIT_POLICIES = [1, 2, 3, 4]
ALL_POLICIES = [1, 2, 3, 4, 5, 6, 8]


def run_case(H, case):
    h = H(case["arena"], case["align"], case["policy"])
    outs = []
    for fr, al in case["batches"]:
        h.free_batch(np.array(fr, dtype=np.uint64))
        outs = [int(x) for x in h.alloc_batch(np.array(al, dtype=np.uint64))]
    return h, outs


@pytest.mark.parametrize("case", parse_golden("spec_examples.txt"), ids=lambda c: c["cite"][:40])
def test_golden_examples(case):
    impls = [OracleL]
    if case["arena"] // case["align"] <= 1 << 16:
        impls.append(_twin(case["policy"]))
    for H in impls:
        h, outs = run_case(H, case)
        assert outs == case["outs"], (H.__name__, case["cite"])
        if case["frees"] is not None:
            fp, _ = h.export()
            assert [tuple(int(v) for v in p) for p in fp] == case["frees"], (H.__name__, case["cite"])


# ---------------- TLSF / segregated-fit class mapping ----------------

def test_segfit_mapping_is_paper_log2():
    """SL_LOG2 = 0: block bin = floor(log2 size), request bin = ceil(log2 size)
    (Alg. 4 PAPER.md:332 '1 << ceil(log2(size))', :351/:429 'floor(log2(...))');
    our class numbers carry a +1 shift (C7)."""
    for u in list(range(1, 1 << 14)) + [2**31 - 1, 2**31, 2**31 + 1, 2**32 - 1, 2**32]:
        fl = u.bit_length() - 1                  # floor(log2 u)
        cl = (u - 1).bit_length()                # ceil(log2 u)
        assert insert_class(u, 0) == fl + 1
        assert search_class(u, 0) == cl + 1


def test_mapping_spec_examples():
    """SPEC.md:416-418,425-427 (derived from Alg. 4): bins 3000->11, 4096->12; requests
    1000->10, 1024->10 (align 1, our classes shifted by +1); TLSF SLI=16: 2432 -> sl 3."""
    assert insert_class(3000, 0) - 1 == 11
    assert insert_class(4096, 0) - 1 == 12
    assert search_class(1000, 0) - 1 == 10
    assert search_class(1024, 0) - 1 == 10
    assert insert_class(2432, 4) % 16 == 3


@pytest.mark.parametrize("L", [0, 4, 5])
def test_mapping_defining_properties(L):
    """insert class brackets the size; search class is the smallest class whose every
    block fits (lo >= u) — Oracle-B's definition, checked against Oracle-L's formula."""
    us = list(range(1, 1 << 13)) + [random.Random(L).randrange(1, 1 << 32) for _ in range(3000)]
    for u in us:
        c = insert_class(u, L)
        assert c == cls_of(u, L)
        assert cls_lo(c, L) <= u < cls_lo(c + 1, L)
        s = search_class(u, L)
        assert s == search_cls(u, L)
        assert cls_lo(s, L) >= u and (s == 0 or cls_lo(s - 1, L) < u)


def test_tlsf_worked_values():
    """Worked values at align 16, SL_LOG2=5 (C10 table)."""
    L = 5
    def fs(c):
        return divmod(c, 32)
    assert fs(insert_class(16 // 16, L)) == (0, 1)
    assert fs(insert_class(496 // 16, L)) == (0, 31)
    assert fs(insert_class(512 // 16, L)) == (1, 0)
    assert fs(insert_class(-(-1000 // 16), L)) == (1, 31) and fs(search_class(63, L)) == (1, 31)
    assert fs(insert_class(1024 // 16, L)) == (2, 0) and cls_lo(insert_class(64, L), L) == 64
    assert fs(insert_class(-(-3000 // 16), L)) == (3, 15) and fs(search_class(188, L)) == (3, 15)
    assert fs(insert_class(-(-3010 // 16), L)) == (3, 15) and fs(search_class(189, L)) == (3, 16)
    assert cls_lo(search_class(189, L), L) == 192
    assert fs(insert_class((4 << 30) // 16, L)) == (24, 0)
    assert fs(insert_class((64 << 30) // 16, L)) == (28, 0)


def test_segfit_nearly_4x_bound():
    """a request served from its own (power-of-two) bin gets a block
    'nearly 4x larger' at worst, i.e. strictly below 4x."""
    worst = 0.0
    for u in range(1, 8193):
        c = search_class(u, 0)
        biggest = cls_lo(c + 1, 0) - 1
        assert biggest < 4 * u
        worst = max(worst, biggest / u)
    assert worst > 3.9


def test_tlsf_good_fit_failure():
    """I6: TLSF rounds the request up to its search class, so it can fail while a block
    >= r exists one class below (Masmano's good fit).  65 units: block class (2,0), search
    class (2,1) -> NULL; first fit takes it."""
    for H in (OracleL, OracleB):
        h = H(65, 1, tg.TLSF)
        assert int(h.alloc_batch([65])[0]) == HEAP_NULL
        h = H(65, 1, tg.FIRST_FIT)
        assert int(h.alloc_batch([65])[0]) == 0


# ---------------- closed forms ----------------

@pytest.mark.parametrize("policy", FIT_POLICIES)
def test_fresh_heap_prefix_sums(policy):
    """L3: with no frees every fit policy bump-allocates: out[i] = sum_{j<i} r_j * align
    (Alg. 1 split from the low end of the single free block)."""
    rng = np.random.default_rng(policy)
    align = 16
    sizes = rng.integers(1, 5000, size=400).astype(np.uint64)
    r = -(-sizes.astype(np.int64) // align)
    arena = int(r.sum() * align * 4)
    h = OracleL(arena, align, policy)
    out = h.alloc_batch(sizes).astype(np.int64)
    expect = np.concatenate([[0], np.cumsum(r)[:-1]]) * align
    assert np.array_equal(out, expect)


def test_buddy_closed_forms():
    """Buddy: a fresh heap serving only order-k requests returns
    i*2^k; non-increasing orders return prefix sums; buddy of a is a XOR 2^k."""
    A = 1 << 12
    for k in range(0, 6):
        h = OracleL(A, 1, tg.BUDDY)
        n = A >> k
        out = h.alloc_batch(np.full(n, 1 << k, dtype=np.uint64)).astype(np.int64)
        assert np.array_equal(out, np.arange(n) << k)
        assert int(h.alloc_batch([1])[0]) == HEAP_NULL
    rng = np.random.default_rng(7)
    ks = np.sort(rng.integers(0, 8, size=40))[::-1]
    h = OracleL(A, 1, tg.BUDDY)
    out = h.alloc_batch((1 << ks).astype(np.uint64)).astype(np.int64)
    assert np.array_equal(out, np.concatenate([[0], np.cumsum(1 << ks)[:-1]]))
    # freeing every block restores the single root block (merge with a XOR 2^k)
    h.free_batch(out.astype(np.uint64))
    fp, lp = h.export()
    assert fp.tolist() == [[0, A]] and len(lp) == 0


def test_free_all_restores_whole_heap():
    """'free-then-alloc of the full heap size succeeds when nothing else is live'
     — full coalescing, Alg. 2 / Alg. 5."""
    for policy in FIT_POLICIES:
        h = OracleL(1 << 16, 16, policy)
        t = tg.Trace(tg.custom(policy, 1 << 16, 16, 64, total_ops=2000, idx=91))
        im = replay(h, t)
        live = im.a[im.a != HEAP_NULL]
        h.free_batch(live)
        fp, lp = h.export()
        assert fp.tolist() == [[0, 1 << 16]] and len(lp) == 0
        assert int(h.alloc_batch([1 << 16])[0]) == (0 if policy != tg.TLSF else 0)


def test_free_classification():
    """Error taxonomy (C16): null, invalid (interior, unaligned,
    out of range, never allocated), double (free block start, or second copy)."""
    for H in (OracleL, OracleB):
        h = H(1024, 16, tg.FIRST_FIT)
        a = [int(x) for x in h.alloc_batch([16, 32, 16])]      # 0, 16, 48
        assert a == [0, 16, 48]
        h.free_batch(np.array([HEAP_NULL, 16, 16, 17, 32, 2048, 64, 0], dtype=np.uint64))
        c = h.stats() if H is OracleL else h.counts
        assert c["frees_null"] == 1 and c["frees_ok"] == 2 and c["frees_double"] == 2
        assert c["frees_invalid"] == 3
        fp, lp = h.export()
        assert [tuple(int(v) for v in p) for p in lp] == [(48, 16)]
        assert [tuple(int(v) for v in p) for p in fp] == [(0, 48), (64, 960)]


# ---------------- cross-oracle ----------------

def _run_both(policy, arena, align, batch, ops, sizes, rho, idx, size_kind=0):
    cfg = tg.custom(policy, arena, align, batch, rho=rho, total_ops=ops, sizes=sizes,
                    size_kind=size_kind, idx=idx)
    hl, hb = OracleL(arena, align, policy), _twin(policy)(arena, align, policy)
    im_l, im_b = IdMap(ops), IdMap(ops)
    for bi, (fids, sz, first) in enumerate(tg.Trace(cfg)):
        ol, ob = im_l.offsets(fids), im_b.offsets(fids)
        assert np.array_equal(ol, ob)
        hl.free_batch(ol)
        hb.free_batch(ob)
        xl, xb = hl.alloc_batch(sz), hb.alloc_batch(sz)
        assert np.array_equal(xl, xb), (policy, bi)
        im_l.record(first, xl)
        im_b.record(first, xb)
        fl, ll = hl.export()
        fb, lb = hb.export()
        assert np.array_equal(fl, fb) and np.array_equal(ll, lb), (policy, bi)
        if policy == 9:
            check_double_invariants(fl, ll, arena, align)
        elif policy == 10:
            check_fib_invariants(fl, ll, arena, align)
        else:
            check_invariants(fl, ll, arena, align, policy == tg.BUDDY, _edges(policy, arena, align))
    st = hl.stats()
    for k, v in hb.counts.items():
        assert st[k] == v, k


@pytest.mark.parametrize("policy", ALL_POLICIES)
@pytest.mark.parametrize("seed", range(4))
def test_oracle_l_equals_oracle_b(policy, seed):
    if policy == tg.BUDDY:
        _run_both(policy, 1 << 14, 16, 24, 1500, (0, 8), (1, 2), 80 + seed, size_kind=1)
    else:
        _run_both(policy, 1 << 14, 16, 24, 1500, (4, 10), (2, 5) if seed % 2 else (1, 2), 80 + seed)


def test_config1_oracle_l_equals_oracle_b():
    """Config 1 exactly (first fit, 1 MiB, 16 B, slot trace, 1000 ops)."""
    cfg = tg.CONFIGS[1]
    hl = OracleL(cfg.arena_bytes, cfg.align, cfg.policy)
    hb = OracleB(cfg.arena_bytes, cfg.align, cfg.policy)
    im_l, im_b = IdMap(1000), IdMap(1000)
    for fids, sz, first in tg.Trace(cfg):
        hl.free_batch(im_l.offsets(fids))
        hb.free_batch(im_b.offsets(fids))
        xl, xb = hl.alloc_batch(sz), hb.alloc_batch(sz)
        assert np.array_equal(xl, xb)
        im_l.record(first, xl)
        im_b.record(first, xb)
    fl, ll = hl.export()
    fb, lb = hb.export()
    assert np.array_equal(fl, fb) and np.array_equal(ll, lb)


@pytest.mark.parametrize("policy", ALL_POLICIES)
def test_exhaustive_tiny_heaps(policy):
    """Every op sequence of length <= 4 over an 8-unit heap (alloc 1..8 units, free any
    live block; one op per batch), Oracle-L == Oracle-B on every output and state."""
    A = 8

    def leaves(depth, seq, hb):
        yield seq
        if depth == 0:
            return
        for s in range(1, A + 1):
            hb2 = _clone_b(hb)
            hb2.alloc_batch([s])
            yield from leaves(depth - 1, seq + [("a", s)], hb2)
        for o in list(hb.live):
            hb2 = _clone_b(hb)
            hb2.free_batch([o])
            yield from leaves(depth - 1, seq + [("f", o)], hb2)

    n = 0
    for seq in leaves(4, [], _twin(policy)(A, 1, policy)):
        hl, hb = OracleL(A, 1, policy), _twin(policy)(A, 1, policy)
        for op, v in seq:
            if op == "a":
                assert int(hl.alloc_batch([v])[0]) == int(hb.alloc_batch([v])[0]), seq
            else:
                hl.free_batch([v])
                hb.free_batch([v])
        fl, ll = hl.export()
        fb, lb = hb.export()
        assert np.array_equal(fl, fb) and np.array_equal(ll, lb), seq
        st = hl.stats()
        assert all(st[k] == v for k, v in hb.counts.items()), seq   # incl. largest_free, high_water_end
        n += 1
    assert n > 1000


def _twin(policy):
    return {6: OracleBLifo, 7: OracleBHybrid, 9: OracleBDouble, 10: OracleBFib}.get(policy, OracleB)


def _edges(policy, arena, align):
    if policy != 7:
        return ()
    S, pool_end, obj = hybrid_layout(arena, align)
    return tuple(j * S for j in range(1, len(obj) + 1)) if S else ()


def _clone_b(h):
    if isinstance(h, OracleBLifo):
        c = OracleBLifo.__new__(OracleBLifo)
        c.__dict__.update(h.__dict__)
        c.free = [list(b) for b in h.free]
        c.live = dict(h.live)
        c.counts = dict(h.counts)
        return c
    c = OracleB.__new__(OracleB)
    c.__dict__.update(h.__dict__)
    c.bits = h.bits.copy()
    c.live = dict(h.live)
    c._counts = dict(h._counts)
    return c


@pytest.mark.parametrize("cfg_id", [2, 3, 4])
def test_invariants_on_scaled_configs(cfg_id):
    """I1-I4 after every batch of a scaled-down config trace, plus conservation of
    bytes in the stats (live + free = arena) and counters = per-request outcomes."""
    cfg = tg.CONFIGS[cfg_id]
    arena = cfg.arena_bytes >> 6 if cfg_id != 2 else cfg.arena_bytes >> 2
    batch = max(cfg.batch >> 6, 64)
    t = tg.Trace(tg.custom(cfg.policy, arena, cfg.align, batch, rho=(cfg.rho_num, cfg.rho_den),
                           total_ops=batch * 12, sizes=(cfg.a, cfg.b), size_kind=cfg.size_kind,
                           idx=cfg.idx))
    h = OracleL(arena, cfg.align, cfg.policy)
    tot = dict(ok=0, fail=0)

    def on_batch(bi, offs, sizes, out):
        fp, lp = h.export()
        check_invariants(fp, lp, arena, cfg.align, cfg.policy == tg.BUDDY)
        st = h.stats()
        assert st["live_bytes"] + st["free_bytes"] == arena
        assert st["n_live"] == len(lp) and st["n_free"] == len(fp)
        tot["ok"] += int(np.sum(out != HEAP_NULL))
        tot["fail"] += int(np.sum(out == HEAP_NULL))
        assert st["allocs_ok"] == tot["ok"] and st["allocs_failed"] == tot["fail"]
    replay(h, t, on_batch=on_batch)


def test_free_order_independence():
    """L1: the state after a free batch does not depend on the order of its frees
    (address-keyed selection), checked by freeing in random orders one by one."""
    for policy in ALL_POLICIES:
        arena = 1 << 12
        base = OracleL(arena, 1, policy)
        sizes = np.random.default_rng(policy).integers(1, 40, size=60).astype(np.uint64)
        out = base.alloc_batch(sizes)
        live = out[out != HEAP_NULL]
        pick = live[::2]
        ref = OracleL(arena, 1, policy)
        ref.alloc_batch(sizes)
        ref.free_batch(pick)
        want = ref.export()
        for perm_seed in range(3):
            h = OracleL(arena, 1, policy)
            h.alloc_batch(sizes)
            for o in np.random.default_rng(perm_seed).permutation(pick):
                h.free_batch([o])
            got = h.export()
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_lifo_differs_from_address_order_and_fragments_more():
    """The paper's segregated fit (LIFO bins) and our address-ordered reading (C9) diverge on
    the paper's own workload shape (malloc-large: 1 KiB-16 MiB), and TLSF
    fragments less than segregated fit ("A Two-Level Segregated Fit allocator would see
    improved fragmentation").  Fragmentation = 1 - live / high-water."""
    frag = {}
    outs = {}
    for pol in (6, 3, 4):
        cfg = tg.Config(95, "malloc-large", pol, 1 << 36, 1024, 1, 0, 1, 2, 5000, 0, 10, 24, n_slots=1000)
        h = OracleL(cfg.arena_bytes, cfg.align, pol)
        im, fr, allout = IdMap(6000), [], []
        for fids, sz, first in tg.Trace(cfg, batch=2):      # one step (free, alloc) per batch
            h.free_batch(im.offsets(fids))
            out = h.alloc_batch(sz)
            im.record(first, out)
            allout.append(out)
            st = h.stats()
            fr.append(1 - st["live_bytes"] / max(st["high_water_end"], 1))
        frag[pol] = float(np.mean(fr[len(fr) // 2:]))
        outs[pol] = np.concatenate(allout)
    assert not np.array_equal(outs[6], outs[3])
    assert frag[4] < frag[3] and frag[4] < frag[6]


# ---------------- HYBRID (§5.3 pools + TLSF; reading C26) ----------------

@pytest.mark.parametrize("seed", range(4))
def test_hybrid_oracle_l_equals_oracle_b(seed):
    """Sizes LU8[16 B, 16 KiB): most requests go to the pools, the rest (and pool overflow,
    forced by the small shares) to the TLSF heap; Oracle-L == the bitmask twin everywhere."""
    _run_both(7, 1 << 18, 16, 48, 3000, (4, 14), (2, 5) if seed % 2 else (1, 3), 90 + seed)


def test_hybrid_layout_and_classification():
    """The layout read from C26 (share = half the arena split over the pools, whole pages) and
    the free taxonomy on pool offsets: interior of an object -> invalid, free slot -> double,
    second copy -> double, TLSF-region rules unchanged."""
    S, pool_end, obj = hybrid_layout(1 << 20, 16)
    assert (S, pool_end, obj[0], obj[-1], len(obj)) == (57344, 516096, 16, 4096, 9)
    assert hybrid_layout(1 << 16, 16)[0] == 0               # too small for a page per pool
    for H in (OracleL, OracleBHybrid):
        h = H(1 << 20, 16, 7)
        a = [int(x) for x in h.alloc_batch([16, 16, 100, 5000])]
        assert a == [0, 16, 3 * S, pool_end]
        h.free_batch(np.array([HEAP_NULL, 8, 16, 16, 32, 3 * S + 64, 3 * S, pool_end + 16, 1 << 21,
                               pool_end], dtype=np.uint64))
        c = h.stats() if H is OracleL else h.counts
        assert (c["frees_null"], c["frees_ok"], c["frees_double"], c["frees_invalid"]) == (1, 3, 2, 4), H
        fp, lp = h.export()
        assert [tuple(int(v) for v in p) for p in lp] == [(0, 16)]
        assert int(h.alloc_batch([1])[0]) == 16              # lowest free slot again
    h = OracleL(1 << 16, 16, 7)                             # no pools: plain TLSF
    t = OracleL(1 << 16, 16, 4)
    sz = np.array([100, 16, 3000, 5], dtype=np.uint64)
    assert np.array_equal(h.alloc_batch(sz), t.alloc_batch(sz))


def test_hybrid_exhaustive_tiny():
    """Every sequence of <= 4 ops (alloc of 8 sizes spanning every pool, the pool/TLSF edge and
    OOM, or free of any live block) on a 24 KiB heap with 1 KiB alignment: pools of 4 x 1 KiB,
    2 x 2 KiB, 1 x 4 KiB and a 12 KiB TLSF heap.  Oracle-L == Oracle-B on every output/state."""
    arena, align = 24576, 1024
    sizes = [1, 1024, 1025, 2049, 4095, 4096, 5000, 12288]

    def leaves(depth, seq, hb):
        yield seq
        if depth == 0:
            return
        for s in sizes:
            hb2 = copy.deepcopy(hb)
            hb2.alloc_batch([s])
            yield from leaves(depth - 1, seq + [("a", s)], hb2)
        for o in hb.live:
            hb2 = copy.deepcopy(hb)
            hb2.free_batch([o])
            yield from leaves(depth - 1, seq + [("f", o)], hb2)

    n = 0
    for seq in leaves(4, [], OracleBHybrid(arena, align)):
        hl, hb = OracleL(arena, align, 7), OracleBHybrid(arena, align)
        for op, v in seq:
            if op == "a":
                assert int(hl.alloc_batch([v])[0]) == int(hb.alloc_batch([v])[0]), seq
            else:
                hl.free_batch([v])
                hb.free_batch([v])
        fl, ll = hl.export()
        fb, lb = hb.export()
        assert np.array_equal(fl, fb) and np.array_equal(ll, lb), seq
        st = hl.stats()
        assert st["n_free"] == len(fl) and st["n_live"] == len(ll)
        assert st["live_bytes"] + st["free_bytes"] == arena
        n += 1
    assert n > 4000


# ---------------- DOUBLE_BUDDY (two staggered buddy heaps; reading C28) ----------------

@pytest.mark.parametrize("seed", range(4))
def test_double_buddy_oracle_l_equals_oracle_b(seed):
    _run_both(9, 6 * 1024 * 16, 16, 24, 1200, (4, 12), (1, 2) if seed % 2 else (2, 5), 110 + seed)


def test_double_buddy_layout_classes_and_taxonomy():
    """Layout (the 3-unit heap gets floor(arena / 6 align) units at the top), the class choice
    (smaller of 2^a and 3 * 2^b units — never equal), frees at a non-multiple of 3*align past
    A_bytes are invalid, and both heaps merge buddies back."""
    assert double_layout(98304, 16) == (49152, 1024)
    assert double_layout(1000, 16) == (1000 - 48 * 10, 10)
    for r in range(1, 5000):
        two = 1 << (r - 1).bit_length()
        three = 3 * (1 << (-(-r // 3) - 1).bit_length())
        assert two != three and max(two, three) >= r and min(two, three) >= r
    for H in (OracleL, OracleBDouble):
        h = H(98304, 16, 9)
        a = [int(x) for x in h.alloc_batch([48, 16, 96])]
        assert a == [49152, 32768, 49248], H               # 96 B = 6 units -> 3-unit class 6
        h.free_batch(np.array([49152 + 16, 49152 + 48, 49152, 49152, HEAP_NULL, 32768], dtype=np.uint64))
        c = h.stats() if H is OracleL else h.counts
        assert (c["frees_ok"], c["frees_invalid"], c["frees_double"], c["frees_null"]) == (2, 1, 2, 1), (H, c)   # 49152+48 is a free 3-unit block start: double
        fp, lp = h.export()
        assert [tuple(int(v) for v in p) for p in lp] == [(49248, 96)]
        check_double_invariants(fp, lp, 98304, 16)


def test_double_buddy_exhaustive_tiny():
    """Every sequence of <= 4 ops on a 12-unit heap (align 1: 3-unit heap of 2 units = [6, 12),
    binary heap of 6 units = 4 @0 + 2 @4): allocs of 1..7 units, frees of any live block."""
    arena = 12

    def leaves(depth, seq, hb):
        yield seq
        if depth == 0:
            return
        for s in range(1, 8):
            hb2 = copy.deepcopy(hb)
            hb2.alloc_batch([s])
            yield from leaves(depth - 1, seq + [("a", s)], hb2)
        for o in hb.live:
            hb2 = copy.deepcopy(hb)
            hb2.free_batch([o])
            yield from leaves(depth - 1, seq + [("f", o)], hb2)

    n = 0
    for seq in leaves(4, [], OracleBDouble(arena, 1)):
        hl, hb = OracleL(arena, 1, 9), OracleBDouble(arena, 1)
        for op, v in seq:
            if op == "a":
                assert int(hl.alloc_batch([v])[0]) == int(hb.alloc_batch([v])[0]), seq
            else:
                hl.free_batch([v])
                hb.free_batch([v])
        fl, ll = hl.export()
        fb, lb = hb.export()
        assert np.array_equal(fl, fb) and np.array_equal(ll, lb), seq
        n += 1
    assert n > 2000


# ---------------- partial (tail) deallocation: policy flag PARTIAL ----------------

PARTIAL_POLICIES = [1, 2, 3, 4, 8]


def test_partial_free_classification():
    """Reading C29 on a hand-built state: an interior offset of a live block frees its tail;
    per live block the lowest offset of the batch wins, every other offset inside it (and a
    copy of the winner) is a double free; an interior offset of FREE memory stays invalid; on a
    heap without the flag an interior offset is invalid (C6)."""
    for H in (OracleL, OracleB):
        h = H(1024, 16, tg.FIRST_FIT | PARTIAL)
        assert [int(x) for x in h.alloc_batch([64, 64, 64])] == [0, 64, 128]     # free [192, 1024)
        h.free_batch(np.array([32, 48, 32, 64, 96, 512, 512 + 8, HEAP_NULL], dtype=np.uint64))
        c = h.stats() if H is OracleL else h.counts
        # 32 -> tail of block 0 (ok); 48, second 32 -> double; 64 -> whole block 1 (ok); 96 -> double;
        # 512 -> interior of the free block [192, 1024): invalid; 520 unaligned: invalid
        assert (c["frees_ok"], c["frees_double"], c["frees_invalid"], c["frees_null"]) == (2, 3, 2, 1), (H, c)
        fp, lp = h.export()
        assert [tuple(int(v) for v in p) for p in lp] == [(0, 32), (128, 64)]
        assert [tuple(int(v) for v in p) for p in fp] == [(32, 96), (192, 832)]
        g = H(1024, 16, tg.FIRST_FIT)
        g.alloc_batch([64])
        g.free_batch(np.array([32], dtype=np.uint64))
        c = g.stats() if H is OracleL else g.counts
        assert c["frees_invalid"] == 1 and c["frees_ok"] == 0


def test_partial_tail_then_start_equals_whole_free():
    """Freeing a block's tail and then its start (two batches) leaves the same state as freeing
    the whole block at once: conservation of the block's bytes across the split (I2)."""
    for policy in PARTIAL_POLICIES:
        a, b = OracleL(1 << 14, 16, policy | PARTIAL), OracleL(1 << 14, 16, policy)
        for h in (a, b):
            h.alloc_batch([1000, 3000, 200])
        a.free_batch(np.array([1008 + 1600], dtype=np.uint64))        # tail of the 3000-byte block
        a.free_batch(np.array([1008], dtype=np.uint64))               # then its start
        b.free_batch(np.array([1008], dtype=np.uint64))
        for x, y in zip(a.export(), b.export()):
            assert np.array_equal(x, y), policy


@pytest.mark.parametrize("policy", PARTIAL_POLICIES)
@pytest.mark.parametrize("seed", range(3))
def test_partial_oracle_l_equals_oracle_b(policy, seed):
    """Random traces with tail frees, second offsets and wild offsets: Oracle-L (ordered live-map
    search) == Oracle-B (per-unit owner map over a bitmap) on every output, state and counter;
    invariants I1-I4 after every batch."""
    arena, align = 1 << 14, 16
    cfg = tg.custom(policy, arena, align, 24, rho=(1, 2), total_ops=1200, sizes=(4, 10), idx=120 + seed)
    hl, hb = OracleL(arena, align, policy | PARTIAL), OracleB(arena, align, policy | PARTIAL)

    def check(bi, batch, sizes, outs):
        assert np.array_equal(outs[0], outs[1]), (policy, bi)
        fl, ll = hl.export()
        fb, lb = hb.export()
        assert np.array_equal(fl, fb) and np.array_equal(ll, lb), (policy, bi)
        check_invariants(fl, ll, arena, align, False)

    replay_partial([hl, hb], cfg, seed, on_batch=check)
    st = hl.stats()
    for k, v in hb.counts.items():
        assert st[k] == v, k
    assert st["frees_ok"] > 0 and st["frees_double"] > 0 and st["frees_invalid"] > 0


@pytest.mark.parametrize("policy", PARTIAL_POLICIES)
def test_partial_exhaustive_tiny_heaps(policy):
    """Every sequence of 3 single-op batches over an 8-unit heap: alloc 1..8 units or free ANY
    unit offset (live start, interior, free memory), Oracle-L == Oracle-B everywhere."""
    A, pol = 8, policy | PARTIAL
    n = 0
    for seq in itertools.product([("a", s) for s in range(1, A + 1)] + [("f", o) for o in range(A)], repeat=3):
        hl, hb = OracleL(A, 1, pol), OracleB(A, 1, pol)
        for op, v in seq:
            if op == "a":
                assert int(hl.alloc_batch([v])[0]) == int(hb.alloc_batch([v])[0]), seq
            else:
                hl.free_batch([v])
                hb.free_batch([v])
        fl, ll = hl.export()
        fb, lb = hb.export()
        assert np.array_equal(fl, fb) and np.array_equal(ll, lb), seq
        st = hl.stats()
        assert all(st[k] == v for k, v in hb.counts.items()), seq
        n += 1
    assert n == 16 ** 3


def test_partial_rejected_where_undefined():
    """The flag needs address coalescing: buddies, pools and LIFO bins reject it."""
    for policy in (tg.BUDDY, tg.HYBRID, tg.DOUBLE_BUDDY, tg.SEGFIT_LIFO, tg.FIB_BUDDY):
        with pytest.raises(ValueError):
            OracleL(1 << 14, 16, policy | PARTIAL)


# ---------------- Fibonacci buddies (reading C30) ----------------

def test_fib_roots_and_closed_forms():
    """Zeckendorf roots (every positive integer is a sum of non-consecutive Fibonacci numbers);
    a fresh Fibonacci-sized heap fed only 1-unit requests fills in address order (0, 1, 2, ...,
    the low part is always split further) — several roots fill smallest root first — and
    freeing everything restores the roots."""
    for A in (1, 2, 3, 4, 7, 8, 12, 20, 21, 100, 1000, 4181):
        fib, roots = fib_roots(A, 1)
        sizes = [z for _, z in roots]
        assert sum(sizes) == A and sizes == sorted(sizes, reverse=True)
        assert all(fib.index(a) - fib.index(b) >= 2 for a, b in zip(sizes, sizes[1:]))   # non-consecutive
        h = OracleL(A, 1, tg.FIB_BUDDY)
        assert [tuple(int(v) for v in p) for p in h.export()[0]] == roots
        out = h.alloc_batch([1] * A)
        if len(roots) == 1:              # one root: the low part is always split further
            assert [int(x) for x in out] == list(range(A)), A
        else:                            # smaller roots are used first, each in address order
            want = [u for s, z in sorted(roots, key=lambda r: r[1]) for u in range(s, s + z)]
            assert [int(x) for x in out] == want, A
        assert int(h.alloc_batch([1])[0]) == HEAP_NULL
        h.free_batch(out)
        assert [tuple(int(v) for v in p) for p in h.export()[0]] == roots


def test_fib_requests_round_up_to_fibonacci_sizes():
    """A request of r units takes a block of the smallest Fibonacci size >= r (live sizes), and
    the split leaves exactly the high parts of the descended classes free."""
    h = OracleL(89, 1, tg.FIB_BUDDY)
    out = [int(x) for x in h.alloc_batch([4, 6, 9, 1])]
    fp, lp = h.export()
    assert sorted(int(z) for _, z in lp) == [1, 5, 8, 13]
    # 89 -> 55|34 -> 34|21 -> 21|13 -> 13|8 -> 8|5 -> 5|3: the 5 at 0 leaves high parts 3@5, 5@8,
    # 8@13, 13@21, 21@34, 34@55; 6 units take 8@13, 9 units 13@21, 1 unit splits 3@5 -> 2|1 -> 1|1
    assert out == [0, 13, 21, 5]
    assert [tuple(int(v) for v in p) for p in fp] == [(6, 1), (7, 1), (8, 5), (34, 21), (55, 34)]


@pytest.mark.parametrize("seed", range(4))
def test_fib_buddy_oracle_l_equals_oracle_b(seed):
    _run_both(tg.FIB_BUDDY, 1 << 14, 16, 24, 1500, (4, 11), (2, 5) if seed % 2 else (1, 2), 90 + seed)


def test_fib_buddy_exhaustive_tiny():
    """Every sequence of <= 4 single-op batches over a 12-unit heap (roots 8 + 3 + 1): alloc 1..12
    units or free any live block; Oracle-L == Oracle-B (derived maximal free tree nodes)."""
    A = 12

    def leaves(depth, seq, hb):
        yield seq
        if depth == 0:
            return
        for s in range(1, A + 1):
            hb2 = copy.deepcopy(hb)
            hb2.alloc_batch([s])
            yield from leaves(depth - 1, seq + [("a", s)], hb2)
        for o in list(hb.live):
            hb2 = copy.deepcopy(hb)
            hb2.free_batch([o])
            yield from leaves(depth - 1, seq + [("f", o)], hb2)

    n = 0
    for seq in leaves(3, [], OracleBFib(A, 1)):
        hl, hb = OracleL(A, 1, tg.FIB_BUDDY), OracleBFib(A, 1)
        for op, v in seq:
            if op == "a":
                assert int(hl.alloc_batch([v])[0]) == int(hb.alloc_batch([v])[0]), seq
            else:
                hl.free_batch([v])
                hb.free_batch([v])
        fl, ll = hl.export()
        fb, lb = hb.export()
        assert np.array_equal(fl, fb) and np.array_equal(ll, lb), seq
        check_fib_invariants(fl, ll, A, 1)
        n += 1
    assert n > 1000


def test_buddy_roots_closed_form():
    """A buddy arena that is not a power of two starts as its binary digits, largest first at
    increasing addresses (the greedy decomposition of reading C13 into maximal aligned powers of
    two): A_u = sum 2^b_j (b_0 > b_1 > ...) gives free blocks
    (sum_{i<j} 2^b_i, 2^b_j).  Written from the binary expansion, not from either oracle's loop."""
    for A in list(range(1, 70)) + [96, 100, 1000, 4095, (1 << 20) + (1 << 7) + 3, (1 << 33) - 1]:
        bits = [b for b in range(A.bit_length() - 1, -1, -1) if A >> b & 1]
        want, s = [], 0
        for b in bits:
            want.append((s, 1 << b))
            s += 1 << b
        for H in ((OracleL, OracleB) if A < (1 << 21) else (OracleL,)):
            fp, lp = H(A, 1, tg.BUDDY).export()
            assert [tuple(int(v) for v in p) for p in fp] == want, (H.__name__, A)
            assert len(lp) == 0
        # the largest root is the largest free block; nothing allocated yet
        st = OracleL(A, 1, tg.BUDDY).stats()
        assert st["largest_free"] == 1 << bits[0] and st["high_water_end"] == 0 and st["n_free"] == len(bits)


def _greedy_runs(fp, A, align):
    """Maximal free runs of `fp` (byte pairs), each decomposed greedily: at x the largest 2^s units
    with x % 2^s == 0 and x + 2^s <= the run's end."""
    runs = []
    for s_, z in (tuple(int(v) for v in p) for p in fp):
        if runs and runs[-1][1] == s_:
            runs[-1][1] = s_ + z
        else:
            runs.append([s_, s_ + z])
    out = []
    for x, y in runs:
        x //= align
        y //= align
        while x < y:
            s_ = (x & -x).bit_length() - 1 if x else 63
            s_ = min(s_, (y - x).bit_length() - 1)
            out.append((x * align, (1 << s_) * align))
            x += 1 << s_
    return out


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_buddy_free_set_is_greedy_decomposition_of_runs(seed):
    """The lemma behind the GPU's parallel buddy free phase (buddy.cuh k_bud_*): after
    any sequence of batches the buddy free set (Oracle-L's one-by-one merges) equals
    the greedy decomposition of its maximal free runs into maximal aligned power-of-two blocks —
    including arenas that are not a power of two (the greedy never crosses a root boundary).
    Checked after every batch of random traces on several arena shapes."""
    rng = np.random.default_rng(seed)
    for A_u in (1 << 12, (1 << 12) + (1 << 9) + 7, 3000, 1 << 10):
        align = 16
        o = OracleL(A_u * align, align, tg.BUDDY)
        live = []
        for _ in range(40):
            nf = int(rng.integers(0, len(live) + 1)) if live else 0
            idx = rng.permutation(len(live))[:nf]
            frees = np.array([live[i] for i in idx], dtype=np.uint64)
            live = [v for i, v in enumerate(live) if i not in set(idx.tolist())]
            o.free_batch(frees)
            sizes = (1 << rng.integers(0, 8, size=int(rng.integers(1, 40)))) * align
            out = o.alloc_batch(sizes.astype(np.uint64))
            live += [int(v) for v in out if v != (1 << 64) - 1]
            fp, _ = o.export()
            got = [tuple(int(v) for v in p) for p in fp]
            assert got == _greedy_runs(fp, A_u, align), (A_u, seed)


def test_size_statistics_closed_forms():
    """largest_free and high_water_end (heap_stats_t) on hand-worked sequences, for both oracles:
    a fresh heap's largest block is the arena; after allocations of r_0, r_1, ... the high-water
    end is sum r_i (L3) and the largest free block the tail; a free below the top does not lower
    the high-water end (it is the provisioned extent of PAPER.md:518, not the live extent)."""
    for H in (OracleL, OracleB):
        for pol in (tg.FIRST_FIT, tg.BEST_FIT, tg.TLSF, tg.SEGFIT, tg.NEXT_FIT):
            h = H(1024, 16, pol)
            c = h.stats() if H is OracleL else h.counts
            assert (c["largest_free"], c["high_water_end"]) == (1024, 0)
            a = [int(x) for x in h.alloc_batch([100, 16, 300])]   # 112, 16, 304 bytes
            assert a == [0, 112, 128], (H, pol)
            c = h.stats() if H is OracleL else h.counts
            assert (c["largest_free"], c["high_water_end"]) == (1024 - 432, 432), (H, pol)
            h.free_batch(np.array([128], dtype=np.uint64))          # the top block: coalesces with the tail
            c = h.stats() if H is OracleL else h.counts
            assert (c["largest_free"], c["high_water_end"]) == (1024 - 128, 432), (H, pol)
            h.free_batch(np.array([0], dtype=np.uint64))
            c = h.stats() if H is OracleL else h.counts
            assert (c["largest_free"], c["high_water_end"]) == (1024 - 128, 432), (H, pol)
        h = H(1024, 16, tg.BUDDY)
        a = [int(x) for x in h.alloc_batch([16, 100])]                # orders 16 B and 128 B
        assert a == [0, 128]
        c = h.stats() if H is OracleL else h.counts
        assert (c["largest_free"], c["high_water_end"]) == (512, 256)
