"""Trace generator: determinism and workload shape."""
import numpy as np

import tracegen as tg


def _collect(cfg, ops):
    return [(f.copy(), s.copy(), first) for f, s, first in tg.Trace(cfg, total_ops=ops)]


def test_same_seed_same_trace():
    for c in (1, 2, 3, 4):
        a = _collect(tg.CONFIGS[c], 20000)
        b = _collect(tg.CONFIGS[c], 20000)
        assert len(a) == len(b)
        for (f1, s1, x1), (f2, s2, x2) in zip(a, b):
            assert np.array_equal(f1, f2) and np.array_equal(s1, s2) and x1 == x2


def test_batch_model_shape():
    cfg = tg.CONFIGS[3]
    bs = _collect(cfg, 3 * cfg.batch)
    assert len(bs) == 3
    assert len(bs[0][0]) == 0 and len(bs[0][1]) == cfg.batch          # first batch: no frees
    nf = round(cfg.batch * cfg.rho_num / cfg.rho_den)
    assert len(bs[1][0]) == nf and len(bs[1][1]) == cfg.batch - nf
    s = np.concatenate([b[1] for b in bs])
    assert s.min() >= 16 and s.max() < 4096
    # octave-uniform: each octave [2^e, 2^(e+1)) gets ~1/8 of the draws
    h = np.bincount(np.floor(np.log2(s.astype(np.float64))).astype(int) - 4, minlength=8)
    assert np.all(np.abs(h / h.sum() - 1 / 8) < 0.01)
    # frees are distinct ids of earlier allocs
    f = np.concatenate([b[0] for b in bs])
    assert len(np.unique(f)) == len(f)


def test_buddy_sizes():
    bs = _collect(tg.CONFIGS[4], 70000)
    s = np.concatenate([b[1] for b in bs])
    k = np.log2(s.astype(np.float64))
    assert np.all(k == np.round(k)) and k.min() >= 8 and k.max() <= 24
    # mean exactly 64 KiB by construction (weights 2^floor((24-k)/2))
    assert abs(s.mean() / 65536 - 1) < 0.05


def test_slot_model_cut_rule():
    """Config 1: a batch never frees an id allocated in the same batch (reading C24)."""
    cfg = tg.CONFIGS[1]
    ops = 0
    for f, s, first in tg.Trace(cfg):
        assert np.all(f < first)
        ops += len(f) + len(s)
    assert ops == 1000
