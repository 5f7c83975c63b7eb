"""Dev: small batches through this session's kernels for compute-sanitizer: best fit's speculative
engine (and, with argv[1] == 'cls', the class-indexed one), binary buddies (shared-memory top-down,
k_bud_scatter), heap_step / heap_free_batch_handles on a single-launch and a general heap.
Usage: python tools/micro/san_case2.py [spec|cls|buddy|step]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
mode = (sys.argv[1:] or ["spec"])[0]
if mode == "cls":
    os.environ["HEAP_BF_FLAT"] = "3"
import tracegen as tg
from oracle import OracleL
from paper_2405_07079_b200 import Heap

def run(pol, arena, batch, ops, sizes, kind=0, micro="0", step=False):
    os.environ["HEAP_MICRO"] = micro
    cfg = tg.custom(pol, arena, 16, batch, rho=(1, 2), total_ops=ops, sizes=sizes, size_kind=kind, idx=34)
    h = Heap(cfg.arena_bytes, cfg.align, pol, 4000, batch + 8)
    h.set_graphs(False)
    o = OracleL(cfg.arena_bytes, cfg.align, pol)
    table = torch.full((ops + 8,), -1, dtype=torch.int64, device="cuda")
    for f, s, first in tg.Trace(cfg):
        idx = torch.from_numpy(f.astype(np.int64)).cuda()
        offs = table[idx].cpu().numpy().view(np.uint64) if len(f) else np.zeros(0, np.uint64)
        sd = torch.from_numpy(s.view(np.int64)).cuda()
        if step:
            out = h.step(table, sd, idx=idx, out=table[first:first + len(s)])
        else:
            h.free_batch_handles(table, idx)
            out = h.alloc_batch(sd, out=table[first:first + len(s)])
        o.free_batch(offs)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), o.alloc_batch(s)), (pol, mode)
    print("ok", pol, mode)

if mode in ("spec", "cls"):
    run(tg.BEST_FIT, 256 << 20, 512, 6000, (4, 20))
    run(tg.BEST_FIT, 1 << 14, 64, 3000, (4, 10))
elif mode == "buddy":
    run(tg.BUDDY, 1 << 30, 1024, 12000, (8, 20), kind=1)
else:
    run(tg.FIRST_FIT, 1 << 20, 64, 3000, (4, 12), micro="1", step=True)
    run(tg.TLSF, 1 << 20, 64, 3000, (4, 12), micro="0", step=True)
print("san case2 ok")
