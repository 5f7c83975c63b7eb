"""Dev tool: sweep small SEGFIT_LIFO cases on the GPU against Oracle-L; for each failing case
save (config, batch index, sizes, gpu out, oracle out) to gpurun_out/lifo_hunt/ for offline
analysis.  Usage: PYTHONPATH=. python tests/dev/lifo_hunt.py [max_cases]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tracegen as tg  # noqa: E402
from oracle import OracleL  # noqa: E402
from paper_2405_07079_b200 import Heap  # noqa: E402

OUT = os.path.join("gpurun_out", "lifo_hunt")
os.makedirs(OUT, exist_ok=True)


def run(arena, batch, ops, sizes, rho, idx):
    cfg = tg.custom(6, arena, 16, batch, rho=rho, total_ops=ops, sizes=sizes, idx=idx)
    h = Heap(arena, 16, 6, 1 << 15, batch)
    o = OracleL(arena, 16, 6)
    idm = np.full(ops + 1, (1 << 64) - 1, dtype=np.uint64)
    for bi, (f, s, first) in enumerate(tg.Trace(cfg)):
        offs = idm[f.astype(np.int64)]
        h.free_batch(torch.from_numpy(offs.view(np.int64)).cuda())
        out = h.alloc_batch(torch.from_numpy(s.view(np.int64)).cuda()).cpu().numpy().view(np.uint64).copy()
        o.free_batch(offs)
        want = o.alloc_batch(s)
        if not np.array_equal(out, want):
            bad = np.flatnonzero(out != want)
            return dict(batch=bi, nbad=int(len(bad)), first=int(bad[0]), gpu=out, want=want, sizes=s)
        idm[first:first + len(s)] = out
    return None


cases = []
rng = np.random.default_rng(5)
cases.append((1 << 24, 3000, 40000, (4, 14), (2, 5), 66))
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60):
    arena = 1 << int(rng.integers(14, 21))
    batch = int(rng.choice([8, 32, 33, 64, 100, 300, 1000]))
    ops = int(min(40000, batch * 12))
    lo = 4
    hi = int(rng.integers(6, 12))
    cases.append((arena, batch, ops, (lo, hi), (1, int(rng.integers(2, 5))), 100 + i))

summary = []
for c in cases:
    r = run(*c)
    line = dict(case=list(map(str, c)), fail=None)
    if r is not None:
        line["fail"] = dict(batch=r["batch"], nbad=r["nbad"], first=r["first"])
        np.savez(os.path.join(OUT, f"case_{c[5]}.npz"), gpu=r["gpu"], want=r["want"], sizes=r["sizes"])
    summary.append(line)
    print(json.dumps(line), flush=True)
with open(os.path.join(OUT, "summary.json"), "w") as f:
    json.dump(summary, f, indent=1)
