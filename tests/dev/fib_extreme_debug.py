"""Dev: replay the 2^32-unit Fibonacci edge case one request per batch against Oracle-L, printing
the first divergence of the free sets."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import OracleL  # noqa: E402
from paper_2405_07079_b200 import Heap  # noqa: E402

arena, align = 1 << 36, 16
sizes = [1 << 35, 16, 4096, 1 << 30, 3 << 20, 1 << 34, 16]
h, o = Heap(arena, align, 10, 1 << 10, 1 << 10), OracleL(arena, align, 10)
for i, s in enumerate(sizes):
    g = h.alloc_batch(torch.tensor([s], dtype=torch.int64, device="cuda")).cpu().numpy().view(np.uint64)
    w = o.alloc_batch([s])
    gf, gl = [x.numpy().view(np.uint64) for x in h.export()]
    of, ol = o.export()
    print(i, s, "gpu", int(g[0]) // 16, "oracle", int(w[0]) // 16, "free sets equal", np.array_equal(gf, of))
    if not np.array_equal(gf, of):
        a = {tuple(int(v) // 16 for v in p) for p in gf}
        b = {tuple(int(v) // 16 for v in p) for p in of}
        print("  gpu only:", sorted(a - b)[:10])
        print("  oracle only:", sorted(b - a)[:10])
        break
print("fib K roots:", [tuple(int(v) // 16 for v in p) for p in OracleL(arena, align, 10).export()[0]])
