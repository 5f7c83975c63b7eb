"""Dev tool: replay one custom case with the wilderness split and report the first mismatch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tracegen as tg  # noqa: E402
from oracle import OracleL  # noqa: E402
from paper_2405_07079_b200 import Heap  # noqa: E402

pol, arena, batch, ops, a, b, rn, rd, idx = (int(x) for x in sys.argv[1:10])
graphs = len(sys.argv) < 11 or sys.argv[10] != "direct"
cfg = tg.custom(pol, arena, 16, batch, rho=(rn, rd), total_ops=ops, sizes=(a, b), idx=idx)
h = Heap(arena, 16, pol, max(1 << 15, 8 * batch), batch)
h.set_graphs(graphs)
o = OracleL(arena, 16, pol)
idm = np.full(ops + 1, (1 << 64) - 1, dtype=np.uint64)
for bi, (f, s, first) in enumerate(tg.Trace(cfg)):
    offs = idm[f.astype(np.int64)]
    h.free_batch(torch.from_numpy(offs.view(np.int64)).cuda())
    out = h.alloc_batch(torch.from_numpy(s.view(np.int64)).cuda()).cpu().numpy().view(np.uint64).copy()
    torch.cuda.synchronize()
    c = h.debug_counters()
    o.free_batch(offs)
    want = o.alloc_batch(s)
    print("batch", bi, "nf", len(f), "na", len(s), "split batches", c[14], "engine flag", c[2], flush=True)
    if not np.array_equal(out, want):
        bad = np.flatnonzero(out != want)
        print("MISMATCH n", len(bad), "at", bad[:10].tolist())
        print(" gpu ", [hex(int(x)) for x in out[bad[:10]]])
        print(" want", [int(x) // 16 for x in want[bad[:10]]], "r", s[bad[:10]].tolist())
        fp, lp = o.export()
        print(" oracle free blocks after (units):", (fp[:60] // 16).tolist())
        break
    idm[first:first + len(s)] = out
print("done")
