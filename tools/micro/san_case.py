"""Dev: a few small batches through the micro path and through the general path's onesweep sort /
single-pass scan (for compute-sanitizer).  Usage: python tools/micro/san_case.py [micro|general]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["HEAP_MICRO"] = "1" if (sys.argv[1:] or ["micro"])[0] == "micro" else "0"
import tracegen as tg
from oracle import OracleL
from paper_2405_07079_b200 import Heap
for pol in (tg.FIRST_FIT, tg.NEXT_FIT, tg.BEST_FIT, tg.TLSF):
    cfg = tg.custom(pol, 1 << 20, 16, 300, rho=(1, 2), total_ops=3000, sizes=(4, 12), idx=33)
    h = Heap(cfg.arena_bytes, cfg.align, pol, 2048, 300)
    h.set_graphs(False)
    o = OracleL(cfg.arena_bytes, cfg.align, pol)
    idm = np.full(4000, (1 << 64) - 1, dtype=np.uint64)
    for f, s, first in tg.Trace(cfg):
        offs = idm[f.astype(np.int64)]
        h.free_batch(torch.from_numpy(offs.view(np.int64)).cuda()); o.free_batch(offs)
        out = h.alloc_batch(torch.from_numpy(s.view(np.int64)).cuda()).cpu().numpy().view(np.uint64)
        assert np.array_equal(out, o.alloc_batch(s)), pol
        idm[first:first + len(s)] = out
print("san case ok")
