"""Dev tool: replay a small case batch by batch against Oracle-L, stop at the first mismatch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tracegen as tg  # noqa: E402
from oracle import OracleL  # noqa: E402
from paper_2405_07079_b200 import Heap  # noqa: E402

pol = int(sys.argv[1]); arena = int(sys.argv[2]); batch = int(sys.argv[3]); ops = int(sys.argv[4])
cfg = tg.custom(pol, arena, 16, batch, rho=(1, 2), total_ops=ops, sizes=(4, 10), idx=60 + pol)
h = Heap(arena, 16, pol, 1 << 15, batch)
o = OracleL(arena, 16, pol)
idm = np.full(ops + 1, (1 << 64) - 1, dtype=np.uint64)
for bi, (f, s, first) in enumerate(tg.Trace(cfg)):
    offs = idm[f.astype(np.int64)]
    print("batch", bi, "nf", len(f), "na", len(s), flush=True)
    h.free_batch(torch.from_numpy(offs.view(np.int64)).cuda())
    torch.cuda.synchronize()
    print("  freed; counters", h.debug_counters()[:3], flush=True)
    out = h.alloc_batch(torch.from_numpy(s.view(np.int64)).cuda()).cpu().numpy().view(np.uint64).copy()
    torch.cuda.synchronize()
    print("  alloc; counters", h.debug_counters()[:3], "stats err", h.stats()["error_flags"], flush=True)
    o.free_batch(offs)
    want = o.alloc_batch(s)
    if not np.array_equal(out, want):
        bad = np.flatnonzero(out != want)
        print("MISMATCH at", bad[:10], "gpu", out[bad[:5]], "want", want[bad[:5]], "r", s[bad[:5]])
        fp, lp = o.export()
        print("oracle free blocks (units):", (fp[:40] // 16).tolist())
        break
    idm[first:first + len(s)] = out
print("done")
