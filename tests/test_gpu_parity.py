"""GPU parity: the CUDA path (through the C ABI) against Oracle-L, bit-exact.

Integer work throughout, so the bar is exact equality of every returned offset, the final
free-block set, the live set, and the counters (north_star).  Small cases compare every
batch; the BASELINE configs are run at full size where the oracle finishes in seconds to
minutes, and config 5 compares its first batches exactly plus invariants.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import tracegen as tg
from oracle import OracleL
from tests.helpers import HEAP_NULL, IdMap, check_invariants, hybrid_layout

pytestmark = pytest.mark.gpu

COUNTERS = ("live_bytes", "free_bytes", "n_live", "n_free", "largest_free", "high_water_end",
            "allocs_ok", "allocs_failed", "frees_ok", "frees_invalid", "frees_double", "frees_null")


class Gpu:
    """numpy-in / numpy-out adapter over the product binding (same interface as OracleL)."""

    def __init__(self, arena, align, policy, max_live, max_batch, graphs=True):
        from paper_2405_07079_b200 import Heap
        self.h = Heap(arena, align, policy, max_live, max_batch)
        self.h.set_graphs(graphs)

    def free_batch(self, offs):
        a = np.ascontiguousarray(np.asarray(offs, dtype=np.uint64))
        self.h.free_batch(torch.from_numpy(a.view(np.int64)).cuda())

    def alloc_batch(self, sizes):
        a = np.ascontiguousarray(np.asarray(sizes, dtype=np.uint64))
        out = self.h.alloc_batch(torch.from_numpy(a.view(np.int64)).cuda())
        return out.cpu().numpy().view(np.uint64).copy()

    def stats(self):
        return self.h.stats()

    def export(self):
        fp, lp = self.h.export()
        return fp.numpy().view(np.uint64), lp.numpy().view(np.uint64)


def compare_state(g, o, ctx=""):
    gs0 = g.stats()
    assert gs0["error_flags"] == 0, f"capacity error flags {gs0['error_flags']} {ctx}"
    gf, gl = g.export()
    of, ol = o.export()
    assert gf.shape == of.shape and np.array_equal(gf, of), f"free set differs {ctx}"
    assert gl.shape == ol.shape and np.array_equal(gl, ol), f"live set differs {ctx}"
    gs, os_ = g.stats(), o.stats()
    assert gs["rc"] == 0 and gs["error_flags"] == 0, gs
    for k in COUNTERS:
        assert gs[k] == os_[k], (k, gs[k], os_[k], ctx)


def run_parity(cfg, max_live, max_batch, total_ops=None, every_batch_state=False, max_batches=None,
               batch=None, graphs=True):
    t = tg.Trace(cfg, total_ops=total_ops, batch=batch)
    g = Gpu(cfg.arena_bytes, cfg.align, cfg.policy, max_live, max_batch, graphs)
    o = OracleL(cfg.arena_bytes, cfg.align, cfg.policy)
    im = IdMap(1 << 16)
    for bi, (fids, sizes, first) in enumerate(t):
        if max_batches is not None and bi >= max_batches:
            break
        offs = im.offsets(fids)
        g.free_batch(offs)
        o.free_batch(offs)
        go = g.alloc_batch(sizes)
        oo = o.alloc_batch(sizes)
        if not np.array_equal(go, oo):
            bad = np.flatnonzero(go != oo)
            raise AssertionError(f"{cfg.name} batch {bi}: {len(bad)} offsets differ, first at {bad[0]}: "
                                 f"gpu {go[bad[0]]} oracle {oo[bad[0]]}")
        im.record(first, go)
        if every_batch_state:
            compare_state(g, o, f"{cfg.name} batch {bi}")
    compare_state(g, o, cfg.name)
    return g, o


SMALL = [
    # (policy, arena, align, batch, ops, sizes, rho, size_kind)
    (tg.FIRST_FIT, 1 << 16, 16, 24, 1500, (4, 10), (1, 2), 0),
    (tg.BEST_FIT, 1 << 16, 16, 24, 1500, (4, 10), (1, 2), 0),
    (tg.SEGFIT, 1 << 16, 16, 24, 1500, (4, 10), (1, 2), 0),
    (tg.TLSF, 1 << 16, 16, 24, 1500, (4, 10), (1, 2), 0),
    (tg.BUDDY, 1 << 16, 16, 24, 1500, (0, 8), (1, 2), 1),
    (tg.FIRST_FIT, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5), 0),
    (tg.BEST_FIT, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5), 0),
    (tg.SEGFIT, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5), 0),
    (tg.TLSF, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5), 0),
    (tg.BUDDY, 1 << 24, 64, 3000, 40000, (6, 16), (1, 2), 1),
    (tg.TLSF, (1 << 22) + 48, 16, 5000, 60000, (4, 12), (1, 3), 0),     # non power-of-two arena
    (tg.SEGFIT_LIFO, 1 << 16, 16, 24, 1500, (4, 10), (1, 2), 0),        # the paper's stack bins
    (tg.SEGFIT_LIFO, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5), 0),
    (tg.SEGFIT_LIFO, 1 << 28, 16, 16384, 200000, (4, 12), (2, 5), 0),
    (tg.BUDDY, (1 << 20) + (1 << 14) + 256, 256, 700, 9000, (8, 18), (1, 2), 1),
    (tg.HYBRID, 1 << 18, 16, 48, 3000, (4, 14), (1, 3), 0),              # §5.3 pools + TLSF
    (tg.HYBRID, 1 << 22, 16, 3000, 40000, (4, 14), (2, 5), 0),
    (tg.HYBRID, 1 << 24, 64, 5000, 60000, (4, 13), (1, 2), 0),
    (tg.NEXT_FIT, 1 << 16, 16, 24, 1500, (4, 10), (1, 2), 0),           # first fit from a rover
    (tg.NEXT_FIT, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5), 0),
    (tg.NEXT_FIT, 1 << 28, 16, 4096, 120000, (4, 20), (1, 2), 0),       # config-2 shaped
    (tg.DOUBLE_BUDDY, 6 * 4096 * 16, 16, 24, 1500, (4, 12), (1, 2), 0),  # two staggered buddy heaps
    (tg.DOUBLE_BUDDY, (1 << 24) + 4096, 64, 3000, 40000, (6, 16), (2, 5), 0),
    (tg.DOUBLE_BUDDY, 1 << 30, 256, 20000, 200000, (8, 24), (1, 2), 0),
    (tg.FIB_BUDDY, 1 << 16, 16, 24, 1500, (4, 10), (1, 2), 0),          # Fibonacci buddies
    (tg.FIB_BUDDY, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5), 0),
    (tg.FIB_BUDDY, (1 << 30) + 12345 * 256, 256, 20000, 200000, (8, 24), (1, 2), 0),   # several roots
]


@pytest.mark.parametrize("case", SMALL, ids=lambda c: f"p{c[0]}-A{c[1]}-B{c[3]}")
def test_small_every_batch(case):
    pol, arena, align, batch, ops, sizes, rho, kind = case
    cfg = tg.custom(pol, arena, align, batch, rho=rho, total_ops=ops, sizes=sizes, size_kind=kind,
                    idx=60 + pol)
    run_parity(cfg, max_live=max(1 << 15, 8 * batch), max_batch=batch, every_batch_state=batch < 100)


WILD_CASES = [
    # (policy, arena, align, batch, ops, sizes, rho): TLSF / SEGFIT heaps whose top class holds one
    # large piece (the wilderness) for most batches, plus small arenas where it does not
    (tg.TLSF, 1 << 16, 16, 24, 1500, (4, 10), (1, 2)),
    (tg.TLSF, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5)),
    (tg.SEGFIT, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5)),
    (tg.TLSF, (1 << 30) + 4096, 16, 65536, 400000, (4, 12), (2, 5)),   # config-3 shaped batches
    (tg.TLSF, 1 << 20, 16, 2000, 30000, (4, 11), (2, 5)),              # wilderness runs out
]


@pytest.mark.parametrize("split", [True, False], ids=["split", "plain"])
@pytest.mark.parametrize("case", WILD_CASES, ids=lambda c: f"p{c[0]}-A{c[1]}-B{c[3]}")
def test_wild_split_both_paths(case, split, monkeypatch):
    """The TLSF/SEGFIT engine with and without the wilderness split (engine_tlsf.cuh
    k_wild_setup): both bit-exact with Oracle-L; with the split on, the large cases must
    actually have used it (diagnostic counter 14 = batches served with the split)."""
    monkeypatch.setenv("HEAP_WILD_SPLIT", "1" if split else "0")
    pol, arena, align, batch, ops, sizes, rho = case
    cfg = tg.custom(pol, arena, align, batch, rho=rho, total_ops=ops, sizes=sizes, idx=80 + pol)
    g, _ = run_parity(cfg, max_live=max(1 << 15, 8 * batch), max_batch=batch, every_batch_state=batch < 100)
    used = g.h.debug_counters()[14]
    if not split:
        assert used == 0
    elif arena >= 1 << 24:
        assert used > 0


@pytest.mark.parametrize("warps", ["1", "2"])
@pytest.mark.parametrize("case", WILD_CASES[1:4], ids=lambda c: f"p{c[0]}-A{c[1]}-B{c[3]}")
def test_engine_one_and_two_warps(case, warps, monkeypatch):
    """The TLSF/SEGFIT engine with its arrivals applied by a second warp concurrently with the class
    updates (default) and with one warp doing both (HEAP_ENGINE_WARPS=1): both bit-exact with
    Oracle-L, state compared after every batch."""
    monkeypatch.setenv("HEAP_ENGINE_WARPS", warps)
    pol, arena, align, batch, ops, sizes, rho = case
    cfg = tg.custom(pol, arena, align, batch, rho=rho, total_ops=ops, sizes=sizes, idx=85 + pol)
    run_parity(cfg, max_live=max(1 << 15, 8 * batch), max_batch=batch, every_batch_state=True)


BF_CASES = [
    # (arena, batch, ops, sizes, rho): blocked engine (chunk pool) and, for the 20000-request
    # batches, the flat global-memory fallback
    (1 << 16, 24, 1500, (4, 10), (1, 2)),
    (1 << 14, 64, 4000, (4, 10), (1, 3)),               # the heap fills: the key list empties and refills
    (1 << 24, 3000, 40000, (4, 14), (2, 5)),
    (256 << 20, 4096, 120000, (4, 20), (1, 2)),        # config-2 shaped
    (1 << 26, 20000, 200000, (4, 12), (1, 2)),        # fallback: too many requests for the pool
]


@pytest.mark.parametrize("engine", ["0", "3", "2", "1"], ids=["spec", "classes", "blocked", "flat"])
@pytest.mark.parametrize("case", BF_CASES, ids=lambda c: f"A{c[0]}-B{c[1]}")
def test_best_fit_engines(case, engine, monkeypatch):
    """BEST_FIT's speculative-chunk, class-indexed, blocked (chunked) and flat engines (fits.cuh
    k_bf_spec_engine, k_bf_cls_engine, k_bf_engine, bf_flat), each bit-exact with Oracle-L."""
    monkeypatch.setenv("HEAP_BF_FLAT", engine)
    arena, batch, ops, sizes, rho = case
    cfg = tg.custom(tg.BEST_FIT, arena, 16, batch, rho=rho, total_ops=ops, sizes=sizes, idx=90)
    run_parity(cfg, max_live=max(1 << 15, 8 * batch), max_batch=batch, every_batch_state=batch < 100)


def test_wild_split_guards(monkeypatch):
    """The split's three conditions (engine_tlsf.cuh k_wild_setup) each switched off by a batch
    built to violate it, and on for batches that satisfy them; zero-size and oversize requests
    in a split batch (written as failures by the candidate gather).  Every batch must match
    Oracle-L; diagnostic counter 14 counts the batches served with the split.  (The heaps are
    small enough for the single-launch path, which has no split: the general path is forced.)"""
    monkeypatch.setenv("HEAP_MICRO", "0")
    U = 16
    arena = 1 << 24                                    # 2^20 units
    for pol in (tg.TLSF, tg.SEGFIT):
        def step(g, o, frees, sizes, expect_split, ctx):
            before = g.h.debug_counters()[14]
            f = np.asarray(frees, dtype=np.uint64)
            g.free_batch(f)
            o.free_batch(f)
            a = np.asarray(sizes, dtype=np.uint64)
            go, oo = g.alloc_batch(a), o.alloc_batch(a)
            assert np.array_equal(go, oo), (pol, ctx, go, oo)
            compare_state(g, o, f"p{pol} {ctx}")
            assert (g.h.debug_counters()[14] - before == 1) == expect_split, (pol, ctx)
            return go

        g, o = Gpu(arena, U, pol, 1024, 64), OracleL(arena, U, pol)
        # the wilderness (one member) serves four blocks: on
        blk = step(g, o, [], [100000 * U, U, 100000 * U, U], True, "fill")
        # (b) two 100000-unit holes; requests large enough to pull the wilderness down to the
        # holes' class: off
        step(g, o, [blk[0], blk[2]], [250000 * U, 250000 * U, 250000 * U, 16], False, "b")
        # (a) the top class now holds the wilderness and both holes: off
        step(g, o, [], [16, 4096], False, "a")
        g2, o2 = Gpu(arena, U, pol, 1024, 64), OracleL(arena, U, pol)
        # (c) a request whose search class is above the wilderness's final class: off
        step(g2, o2, [], [600000 * U, 300000 * U], False, "c")
        # on, with zero-size and oversize requests among the candidates and the skipped ones
        step(g2, o2, [], [16, 0, 48, arena * 4, 4096, 0, 32] * 5, True, "on+invalid")


def test_config1_exact():
    cfg = tg.CONFIGS[1]
    run_parity(cfg, cfg.max_live, 1000, every_batch_state=True)


def test_config2_full():
    cfg = tg.CONFIGS[2]
    run_parity(cfg, cfg.max_live, cfg.batch)


def test_config3_full():
    cfg = tg.CONFIGS[3]
    run_parity(cfg, cfg.max_live, cfg.batch)


def test_config4_full():
    cfg = tg.CONFIGS[4]
    run_parity(cfg, cfg.max_live, cfg.batch)


def test_config5_first_batches():
    """Config 5 at full size (64 GiB arena = 2^32 units, 1M-request batches): the first
    batches exactly (the oracle computes them in seconds), state compared after each."""
    cfg = tg.CONFIGS[5]
    run_parity(cfg, cfg.max_live, cfg.batch, max_batches=3)


@pytest.mark.parametrize("micro", ["1", "0"], ids=["micro", "general"])
def test_edge_cases(micro, monkeypatch):
    """Empty batches, NULL / interior / unaligned / out-of-range / duplicate frees,
    zero and oversize requests, OOM in a tiny arena, the last unit of a 2^32-unit arena — on the
    single-launch small-heap path (micro.cuh) and on the general path."""
    monkeypatch.setenv("HEAP_MICRO", micro)
    for pol in (1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 1 | 0x100, 4 | 0x100):
        arena, align = 1 << 12, 16
        g = Gpu(arena, align, pol, 256, 64)
        o = OracleL(arena, align, pol)
        for h in (g, o):
            h.free_batch(np.zeros(0, np.uint64))
        sizes = np.array([16, 0, 5000, 64, 1, 100, 4096, 32], dtype=np.uint64)
        go, oo = g.alloc_batch(sizes), o.alloc_batch(sizes)
        assert np.array_equal(go, oo), pol
        live = oo[oo != HEAP_NULL]
        frees = np.array([HEAP_NULL, live[0], live[0], live[0] + 16, 3, arena * 2, live[-1], 7 * 16],
                         dtype=np.uint64)
        g.free_batch(frees)
        o.free_batch(frees)
        compare_state(g, o, f"edge p{pol}")
        # fill to OOM
        big = np.full(64, 200, dtype=np.uint64)
        assert np.array_equal(g.alloc_batch(big), o.alloc_batch(big))
        compare_state(g, o, f"edge-oom p{pol}")
    # 2^32-unit arena: allocate right up to the end
    g = Gpu(1 << 36, 16, tg.TLSF, 64, 64)
    o = OracleL(1 << 36, 16, tg.TLSF)
    sizes = np.array([(1 << 36) - 32, 16, 16, 16], dtype=np.uint64)
    assert np.array_equal(g.alloc_batch(sizes), o.alloc_batch(sizes))
    compare_state(g, o, "2^32 units")


@pytest.mark.parametrize("micro", ["1", "0"], ids=["micro", "general"])
def test_table_rebuild_under_churn(micro, monkeypatch):
    """Small live capacity with heavy churn forces tombstone purges of the block table (in the
    micro kernel's own purge, and in the general path's rebuild launches)."""
    monkeypatch.setenv("HEAP_MICRO", micro)
    cfg = tg.custom(tg.TLSF, 1 << 22, 16, 256, rho=(1, 2), total_ops=60000, sizes=(4, 10), idx=77)
    run_parity(cfg, max_live=600, max_batch=256)


MICRO_CASES = [
    # (arena, align, batch, ops, sizes, rho): heaps small enough for the single-launch path
    # (max_live 4096 -> at most 4097 free pieces), live blocks kept below the capacity
    (1 << 16, 16, 24, 1500, (4, 10), (1, 2)),
    (1 << 22, 16, 1000, 40000, (4, 14), (1, 2)),
    (1 << 20, 16, 500, 10000, (4, 12), (2, 5)),
    (1 << 18, 16, 3000, 30000, (4, 9), (1, 2)),          # the arena fills: failed requests
    ((1 << 22) + 48, 16, 700, 14000, (4, 13), (1, 2)),   # non power-of-two arena
    (1 << 21, 64, 256, 8000, (6, 12), (1, 2)),           # align 64
]


@pytest.mark.parametrize("micro", ["1", "0"], ids=["micro", "general"])
@pytest.mark.parametrize("pol", [tg.FIRST_FIT, tg.NEXT_FIT, tg.BEST_FIT, tg.SEGFIT, tg.TLSF],
                         ids=lambda p: tg.POLICY_NAME[p])
@pytest.mark.parametrize("case", MICRO_CASES, ids=lambda c: f"A{c[0]}-B{c[2]}")
def test_micro_and_general_paths(case, pol, micro, monkeypatch):
    """The small-heap path (micro.cuh: one single-CTA launch per free batch and per alloc batch,
    brute-force exact argmin engine) and the general path, each bit-exact with Oracle-L on every
    batch, state compared after every batch (the two interleave through the same state)."""
    monkeypatch.setenv("HEAP_MICRO", micro)
    arena, align, batch, ops, sizes, rho = case
    cfg = tg.custom(pol, arena, align, batch, rho=rho, total_ops=ops, sizes=sizes, idx=40 + pol)
    run_parity(cfg, max_live=4096, max_batch=batch, every_batch_state=True)


BUDDY_CASES = [
    # (policy, arena, align, batch, ops, sizes, rho)
    (tg.BUDDY, 1 << 16, 16, 24, 1500, (0, 8), (1, 2)),
    (tg.BUDDY, 1 << 24, 64, 3000, 40000, (6, 16), (1, 2)),
    (tg.BUDDY, (1 << 20) + (1 << 14) + 256, 256, 700, 9000, (8, 18), (1, 2)),   # several roots
    (tg.BUDDY, (1 << 30) + (1 << 23) + (1 << 12), 256, 8192, 120000, (8, 24), (1, 2)),
    (tg.DOUBLE_BUDDY, (1 << 24) + 4096, 64, 3000, 40000, (6, 16), (2, 5)),
]


@pytest.mark.parametrize("levels", ["0", "1"], ids=["parallel", "levels"])
@pytest.mark.parametrize("case", BUDDY_CASES, ids=lambda c: f"p{c[0]}-A{c[1]}-B{c[3]}")
def test_buddy_free_forms(case, levels, monkeypatch):
    """Binary-buddy free phase in its parallel form (runs of free space decomposed greedily into
    maximal aligned blocks, buddy.cuh k_bud_*) and in the level-by-level form (k_free_levels):
    both bit-exact with Oracle-L, state compared after every batch."""
    monkeypatch.setenv("HEAP_BUDDY_LEVELS", levels)
    pol, arena, align, batch, ops, sizes, rho = case
    kind = 1 if pol == tg.BUDDY else 0
    cfg = tg.custom(pol, arena, align, batch, rho=rho, total_ops=ops, sizes=sizes, size_kind=kind, idx=20 + pol)
    run_parity(cfg, max_live=max(1 << 15, 8 * batch), max_batch=batch, every_batch_state=True)


def test_invariants_config3_prefix():
    cfg = tg.CONFIGS[3]
    g, _ = run_parity(cfg, cfg.max_live, cfg.batch, max_batches=10)
    fp, lp = g.export()
    check_invariants(fp, lp, cfg.arena_bytes, cfg.align, False)


@pytest.mark.timeout(1800)
def test_config5_full_size_properties():
    """Config 5 at full size for 85 batches, every returned offset of every batch exactly against
    the oracle, in bench.py's launch configuration (batch graphs): the batches the driver's bench
    (``--warmup 5 --steps 20``) warms up on and times (0..24, state compared after batch 24) and on
    to a late window (80..84, the heap near 17M live blocks; the paper separates warm-up from
    steady state), final state compared, plus properties that hold at
    any size — I1-I4 on the exported state, conservation, counter consistency, and every returned
    offset of the last batch is a live block of the rounded request size, pairwise disjoint."""
    cfg = tg.CONFIGS[5]
    g = Gpu(cfg.arena_bytes, cfg.align, cfg.policy, cfg.max_live, cfg.batch)
    o = OracleL(cfg.arena_bytes, cfg.align, cfg.policy)
    nb = 85
    im = IdMap(cfg.batch * nb)
    nreq = 0
    last = None
    for bi, (fids, sizes, first) in enumerate(tg.Trace(cfg, total_ops=cfg.batch * nb)):
        offs = im.offsets(fids)
        g.free_batch(offs)
        go = g.alloc_batch(sizes)
        o.free_batch(offs)
        oo = o.alloc_batch(sizes)
        if not np.array_equal(go, oo):
            bad = np.flatnonzero(go != oo)
            raise AssertionError(f"config 5 batch {bi}: {len(bad)} offsets differ, first at {bad[0]}")
        im.record(first, go)
        nreq += len(sizes)
        last = (sizes, go)
        if bi == 24:
            compare_state(g, o, "config 5 after batch 24")
    compare_state(g, o, "config 5 after batch 84")
    st = g.stats()
    assert st["error_flags"] == 0 and st["rc"] == 0
    assert st["allocs_ok"] + st["allocs_failed"] == nreq
    assert st["live_bytes"] + st["free_bytes"] == cfg.arena_bytes
    fp, lp = g.export()
    assert len(lp) == st["n_live"] and len(fp) == st["n_free"]
    check_invariants(fp, lp, cfg.arena_bytes, cfg.align, False)
    sizes, out = last
    ok = out != HEAP_NULL
    starts = lp[:, 0]
    idx = np.searchsorted(starts, out[ok])
    assert np.all(starts[idx] == out[ok])
    r = -(-sizes[ok].astype(np.int64) // cfg.align) * cfg.align
    assert np.array_equal(lp[idx, 1].astype(np.int64), r)
    so = np.sort(out[ok])
    assert len(np.unique(so)) == len(so)


def test_hybrid_edges_and_full_pools():
    """HYBRID with real pools: pool-offset taxonomy (interior, free slot, duplicate copies),
    request sizes at the pool/TLSF edge (4095 / 4096 / 0), pools driven to exhaustion so
    requests fall back to the TLSF heap, then freed back."""
    arena, align = 1 << 20, 16
    S, pool_end, obj = hybrid_layout(arena, align)
    g = Gpu(arena, align, tg.HYBRID, 4096, 4096)
    o = OracleL(arena, align, tg.HYBRID)
    sizes = np.array([16, 0, 4095, 4096, 1, 100, 2048, 2049, 5000, 1 << 21], dtype=np.uint64)
    go, oo = g.alloc_batch(sizes), o.alloc_batch(sizes)
    assert np.array_equal(go, oo)
    frees = np.array([HEAP_NULL, oo[0], oo[0], oo[0] + 8, 3 * S + 64, 16 * 5, oo[3], pool_end + 16, arena * 3],
                     dtype=np.uint64)
    g.free_batch(frees)
    o.free_batch(frees)
    compare_state(g, o, "hybrid taxonomy")
    big = np.full(4000, 3000, dtype=np.uint64)          # pool 8 holds S/4096 = 14 objects
    assert np.array_equal(g.alloc_batch(big), o.alloc_batch(big))
    small = np.full(4096, 16, dtype=np.uint64)           # pool 0 holds 3584: the rest fall back
    gs, os_ = g.alloc_batch(small), o.alloc_batch(small)
    assert np.array_equal(gs, os_)
    compare_state(g, o, "hybrid full pools")
    g.free_batch(gs[::3].copy())
    o.free_batch(os_[::3].copy())
    assert np.array_equal(g.alloc_batch(small[:1000]), o.alloc_batch(small[:1000]))
    compare_state(g, o, "hybrid refill")
    fp, lp = g.export()
    check_invariants(fp, lp, arena, align, False, tuple(j * S for j in range(1, len(obj) + 1)))


def test_hybrid_config5_shape():
    """The config-5 trace (64 GiB, 1M-request batches, LU8[16 B, 4 KiB)) on a HYBRID heap: every
    request is below a page, so the pools serve it; three batches exact, counters compared."""
    cfg = tg.CONFIGS[5]
    g = Gpu(cfg.arena_bytes, cfg.align, tg.HYBRID, 1 << 16, cfg.batch)
    o = OracleL(cfg.arena_bytes, cfg.align, tg.HYBRID)
    im = IdMap(cfg.batch * 3)
    for bi, (fids, sizes, first) in enumerate(tg.Trace(cfg, total_ops=cfg.batch * 3)):
        offs = im.offsets(fids)
        g.free_batch(offs)
        o.free_batch(offs)
        go = g.alloc_batch(sizes)
        assert np.array_equal(go, o.alloc_batch(sizes)), bi
        im.record(first, go)
    gs, os_ = g.stats(), o.stats()
    assert gs["error_flags"] == 0
    for k in COUNTERS:
        assert gs[k] == os_[k], k


@pytest.mark.parametrize("pol", [tg.FIRST_FIT, tg.BEST_FIT, tg.TLSF, tg.BUDDY, tg.SEGFIT_LIFO, tg.HYBRID, tg.NEXT_FIT,
                                 tg.DOUBLE_BUDDY, tg.FIB_BUDDY, tg.TLSF | 0x100])
def test_direct_launch_path(pol):
    """The same batches with batch graphs disabled (direct launches, the path tracing uses), and
    a heap switching between the two paths mid-trace."""
    kind = 1 if pol == tg.BUDDY else 0
    sizes = (6, 16) if pol == tg.BUDDY else (4, 14)
    cfg = tg.custom(pol, 1 << 22, 16, 500, rho=(2, 5), total_ops=8000, sizes=sizes, size_kind=kind, idx=70 + pol)
    run_parity(cfg, max_live=1 << 15, max_batch=500, graphs=False)
    t = tg.Trace(cfg)
    g = Gpu(cfg.arena_bytes, cfg.align, pol, 1 << 15, 500)
    o = OracleL(cfg.arena_bytes, cfg.align, pol)
    im = IdMap(1 << 14)
    for bi, (fids, sz, first) in enumerate(t):
        g.h.set_graphs(bi % 3 != 1)
        offs = im.offsets(fids)
        g.free_batch(offs)
        o.free_batch(offs)
        go = g.alloc_batch(sz)
        assert np.array_equal(go, o.alloc_batch(sz)), bi
        im.record(first, go)
    compare_state(g, o, "mixed paths")


# ---------------- partial (tail) deallocation: HEAP_PARTIAL_FREE (reading C29) ----------------

PARTIAL_CASES = [
    # (policy, arena, align, batch, ops, sizes, rho)
    (tg.FIRST_FIT, 1 << 16, 16, 24, 1500, (4, 10), (1, 2)),
    (tg.BEST_FIT, 1 << 16, 16, 24, 1500, (4, 10), (1, 2)),
    (tg.SEGFIT, 1 << 16, 16, 24, 1500, (4, 10), (1, 2)),
    (tg.TLSF, 1 << 16, 16, 24, 1500, (4, 10), (1, 2)),
    (tg.NEXT_FIT, 1 << 16, 16, 24, 1500, (4, 10), (1, 2)),
    (tg.TLSF, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5)),
    (tg.FIRST_FIT, 1 << 24, 16, 3000, 40000, (4, 14), (2, 5)),
    (tg.BEST_FIT, 1 << 26, 16, 4096, 60000, (4, 20), (1, 2)),          # config-2 shaped sizes
    (tg.TLSF, (1 << 30) + 4096, 16, 65536, 400000, (4, 12), (2, 5)),   # config-3 shaped batches
]


@pytest.mark.parametrize("case", PARTIAL_CASES, ids=lambda c: f"p{c[0]}-A{c[1]}-B{c[3]}")
def test_partial_free_parity(case):
    """Traces whose frees are partly tail frees, second offsets inside a block and wild
    offsets (tests/helpers.replay_partial): every output, the final state and all counters
    equal Oracle-L; the state is compared after every batch on the small heaps."""
    from tests.helpers import PARTIAL, replay_partial
    pol, arena, align, batch, ops, sizes, rho = case
    cfg = tg.custom(pol, arena, align, batch, rho=rho, total_ops=ops, sizes=sizes, idx=140 + pol)
    o = OracleL(arena, align, pol | PARTIAL)
    g = Gpu(arena, align, pol | PARTIAL, max(1 << 15, 8 * batch), 3 * batch)

    def check(bi, offs, sizes, outs):
        if not np.array_equal(outs[0], outs[1]):
            bad = np.flatnonzero(outs[0] != outs[1])
            raise AssertionError(f"batch {bi}: {len(bad)} offsets differ, first at {bad[0]}")
        if batch < 100:
            compare_state(g, o, f"batch {bi}")

    replay_partial([o, g], cfg, 7 + pol, on_batch=check)
    compare_state(g, o, "end")
    st = o.stats()
    assert st["frees_ok"] > 0 and st["frees_double"] > 0 and st["frees_invalid"] > 0


def test_partial_free_edges():
    """The paper's 10 KiB example; several offsets inside one block (lowest wins, the rest are
    double); start + interior of one block (whole free); interior of free memory (invalid);
    empty and all-null batches; a predecessor search that climbs every bitmap level (a 2^31-unit
    block in a 2^32-unit arena, tail freed near its end); a tail free of the last unit."""
    from tests.helpers import PARTIAL
    cases = [
        (1 << 14, 16, [[10240]], [[8192]]),
        (1 << 16, 16, [[1024, 1024, 4096]], [[1040, 1024 + 512, 1024 + 2032, 1040]]),
        (1 << 16, 16, [[1024, 1024]], [[1024, 1024 + 16, 2048 + 512, 4096 + 32, 60000 * 16 // 16]]),
        (1 << 16, 16, [[1024]], [[], [(1 << 64) - 1] * 5, [16, 32, 48]]),
        (1 << 36, 16, [[1 << 35, 4096]], [[(1 << 35) - 16, (1 << 35) + 16]]),
        (1 << 16, 16, [[64, 64]], [[48, 112]]),
    ]
    for pol in (tg.FIRST_FIT, tg.TLSF):
        for arena, align, allocs, frees in cases:
            o = OracleL(arena, align, pol | PARTIAL)
            g = Gpu(arena, align, pol | PARTIAL, 1 << 12, 1 << 10)
            for a in allocs:
                assert np.array_equal(g.alloc_batch(a), o.alloc_batch(a))
            for f in frees:
                g.free_batch(f)
                o.free_batch(f)
                compare_state(g, o, f"{pol} {arena} {f}")
            # the heap keeps working after the tail frees
            assert np.array_equal(g.alloc_batch([16, 4096, 1 << 20]), o.alloc_batch([16, 4096, 1 << 20]))
            compare_state(g, o, f"{pol} {arena} after")


def test_fib_buddy_config4_shape_and_edges():
    """Config 4's trace (2^34-byte arena, 256 B units: roots 2^26 units = 39088169 + 24157817 +
    ... ; 64K-request batches of power-of-two sizes) on Fibonacci buddies, every batch exact; then
    a fresh Fibonacci-sized heap fed 1-unit requests fills in address order and frees back to its
    root; empty / all-null / double / invalid free batches."""
    c4 = tg.CONFIGS[4]
    cfg = tg.Config(c4.idx, "cfg4-as-fib", tg.FIB_BUDDY, c4.arena_bytes, c4.align, c4.model, c4.batch, c4.rho_num,
                    c4.rho_den, c4.batch * 12, c4.size_kind, c4.a, c4.b, max_live=c4.max_live)
    run_parity(cfg, c4.max_live, c4.batch)
    A = 4181
    g, o = Gpu(A * 16, 16, tg.FIB_BUDDY, 1 << 13, 1 << 13), OracleL(A * 16, 16, tg.FIB_BUDDY)
    out = g.alloc_batch([16] * A)
    assert np.array_equal(out, o.alloc_batch([16] * A))
    assert np.array_equal(out, np.arange(A, dtype=np.uint64) * 16)
    for batch in ([], [HEAP_NULL] * 3, [16, 16, 17, 1 << 40], out[::2], out[1::2]):
        g.free_batch(batch)
        o.free_batch(batch)
        compare_state(g, o, f"fib edge {len(batch)}")
    assert [tuple(int(v) for v in p) for p in g.export()[0]] == [(0, A * 16)]


def test_fib_buddy_arena_extremes():
    """Fibonacci buddies at the arena extremes: 1, 2, 3 and 7 units (one or a few tiny roots; K = 0
    for one unit) and 2^32 units (K = 45, the largest class table and engine shared memory), each
    filled, partly freed and refilled against Oracle-L."""
    for arena, align, sizes in ((16, 16, [16, 16]), (32, 16, [16, 16, 16]), (48, 16, [32, 16, 16]),
                                (112, 16, [16, 48, 32, 16, 16]),
                                (1 << 36, 16, [1 << 35, 16, 4096, 1 << 30, 3 << 20, 1 << 34, 16])):
        g, o = Gpu(arena, align, tg.FIB_BUDDY, 1 << 10, 1 << 10), OracleL(arena, align, tg.FIB_BUDDY)
        out = g.alloc_batch(sizes)
        assert np.array_equal(out, o.alloc_batch(sizes)), arena
        compare_state(g, o, f"fib {arena} filled")
        g.free_batch(out[::2])
        o.free_batch(out[::2])
        compare_state(g, o, f"fib {arena} half freed")
        assert np.array_equal(g.alloc_batch(sizes[::-1]), o.alloc_batch(sizes[::-1])), arena
        compare_state(g, o, f"fib {arena} refilled")


@pytest.mark.parametrize("pol", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 1 | 0x100, 4 | 0x100])
def test_arena_extremes_all_policies(pol):
    """Every policy at the arena extremes: 1 unit, 3 units and 2^32 units (the largest arena the
    32-bit unit keys allow): whole-arena, oversize, zero and minimum requests, free everything,
    allocate again — every output, the state and the counters against Oracle-L."""
    for arena in (16, 48, 1 << 36):
        g, o = Gpu(arena, 16, pol, 256, 64), OracleL(arena, 16, pol)
        sizes = np.array([16, arena, arena + 16, 0, 32, arena // 2, 16, 1 << 20], dtype=np.uint64)
        go, oo = g.alloc_batch(sizes), o.alloc_batch(sizes)
        assert np.array_equal(go, oo), (pol, arena)
        compare_state(g, o, f"p{pol} {arena} alloc")
        live = oo[oo != HEAP_NULL]
        g.free_batch(live)
        o.free_batch(live)
        compare_state(g, o, f"p{pol} {arena} free all")
        assert np.array_equal(g.alloc_batch(sizes[::-1].copy()), o.alloc_batch(sizes[::-1].copy())), (pol, arena)
        compare_state(g, o, f"p{pol} {arena} realloc")


@pytest.mark.parametrize("mode", ["handles", "step", "step_offsets"])
@pytest.mark.parametrize("micro", ["1", "0"], ids=["single_launch", "general"])
@pytest.mark.parametrize("policy", [tg.FIRST_FIT, tg.BEST_FIT, tg.TLSF, tg.BUDDY])
def test_free_batch_handles(policy, micro, mode, monkeypatch):
    """heap_free_batch_handles frees table[idx[i]] exactly as heap_free_batch frees the gathered
    offsets, and heap_step (free batch + alloc batch in one call: one kernel on a single-launch
    heap) equals the two calls: a handle table on the device (the alloc results written into it),
    frees by index, including indices past the table (no-op nulls), repeated and HEAP_NULL
    entries, batches without frees or allocs; every batch against Oracle-L."""
    from paper_2405_07079_b200 import Heap
    monkeypatch.setenv("HEAP_MICRO", micro)
    kind, sizes = (1, (4, 10)) if policy == tg.BUDDY else (0, (4, 12))
    cfg = tg.custom(policy, 1 << 20, 16, 128, total_ops=6000, sizes=sizes, size_kind=kind, idx=93)
    h = Heap(cfg.arena_bytes, cfg.align, policy, 1 << 12, 256)
    o = OracleL(cfg.arena_bytes, cfg.align, policy)
    table = torch.full((8192,), -1, dtype=torch.int64, device="cuda")
    rng = np.random.default_rng(7)
    for bi, (fids, sz, first) in enumerate(tg.Trace(cfg)):
        idx = fids.astype(np.int64)
        if bi % 3 == 2 and len(idx):          # an index past the table and a repeated handle
            idx = np.concatenate([idx, [table.numel() + 5, idx[0]]])
            rng.shuffle(idx)
        offs = np.where(idx < table.numel(), table.cpu().numpy()[np.minimum(idx, table.numel() - 1)], -1)
        if bi % 7 == 3:                       # a batch without allocs, then one without frees
            sz = sz[:0]
        if bi % 7 == 4:
            idx, offs = idx[:0], offs[:0]
        sd = torch.from_numpy(sz.view(np.int64)).cuda()
        dst = table[first:first + len(sz)]
        if mode == "handles":
            h.free_batch_handles(table, torch.from_numpy(idx).cuda())
            got = h.alloc_batch(sd, out=dst)
        elif mode == "step":
            got = h.step(table, sd, idx=torch.from_numpy(idx).cuda(), out=dst)
        else:
            got = h.step(torch.from_numpy(offs.astype(np.int64)).cuda(), sd, out=dst)
        o.free_batch(offs.view(np.uint64))
        want = o.alloc_batch(sz)
        assert np.array_equal(got.cpu().numpy().view(np.uint64), want), (policy, micro, bi)
    st, ost = h.stats(), o.stats()
    for k in COUNTERS:
        assert st[k] == ost[k], (k, st[k], ost[k])
