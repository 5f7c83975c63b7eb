"""Steady-state measurement (dev tool, GPU): config 5 run through batches 0..LAST on the production
path (batch graphs), the late window FIRST..LAST timed one batch per step exactly as bench.py times
its steps (L2 flushed before each, CUDA events on the heap's stream), and every returned offset of
every batch compared with Oracle-L.  The paper separates warm-up from steady state
(PAPER.md:516,530); bench.py times batches 5..24, this times a late window of the same trace.

Usage: python tools/steady_state.py [FIRST LAST]   (default 80 84) -> one JSON line on stdout."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen as tg  # noqa: E402
from oracle import OracleL  # noqa: E402
from paper_2405_07079_b200 import Heap  # noqa: E402

first_t = int(sys.argv[1]) if len(sys.argv) > 1 else 80
last_t = int(sys.argv[2]) if len(sys.argv) > 2 else 84
cfg = tg.CONFIGS[5]
nb = last_t + 1
dev = torch.device("cuda", 0)
h = Heap(cfg.arena_bytes, cfg.align, cfg.policy, cfg.max_live, cfg.batch, device=dev)
o = OracleL(cfg.arena_bytes, cfg.align, cfg.policy)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
idmap = torch.full((cfg.batch * nb + 1,), -1, dtype=torch.int64, device=dev)
omap = np.full(cfg.batch * nb + 1, (1 << 64) - 1, dtype=np.uint64)
step_ms, ops, mism, o_s, o_ops = [], 0, None, 0.0, 0
for bi, (f, s, first) in enumerate(tg.Trace(cfg, total_ops=cfg.batch * nb)):
    fd = torch.from_numpy(f.astype(np.int64)).to(dev)
    sd = torch.from_numpy(s.view(np.int64)).to(dev)
    timed = bi >= first_t
    if timed:
        flush.fill_(bi & 255)
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
    h.free_batch(idmap[fd] if len(f) else fd)
    out = h.alloc_batch(sd, out=idmap[first:first + len(s)])
    if timed:
        e.record()
        torch.cuda.synchronize()
        step_ms.append(a.elapsed_time(e))
        ops += len(f) + len(s)
    g = out.cpu().numpy().view(np.uint64)
    offs = omap[f.astype(np.int64)]
    t0 = time.perf_counter()
    o.free_batch(offs)
    want = o.alloc_batch(s)
    if timed:
        o_s += time.perf_counter() - t0
        o_ops += len(f) + len(s)
    if mism is None and not np.array_equal(g, want):
        j = int(np.flatnonzero(g != want)[0])
        mism = {"batch": bi, "request": j}
    omap[first:first + len(s)] = want
st = h.stats()
t = sum(step_ms)
print(json.dumps({
    "tool": "tools/steady_state.py", "workload": "config 5 (TLSF, 64 GiB arena, 1M-request batches)",
    "window": f"batches {first_t}..{last_t} of one trace (bench.py times 5..24)",
    "value": ops / (t / 1e3), "unit": "ops/s", "ms_per_step": t / len(step_ms), "step_ms": step_ms,
    "oracle_same_batches": o_ops / o_s, "vs_oracle": (ops / (t / 1e3)) / (o_ops / o_s),
    "parity": {"checked": f"every returned offset of batches 0..{last_t}", "ok": mism is None, "first_mismatch": mism},
    "heap": {"n_live": st["n_live"], "n_free": st["n_free"], "error_flags": st["error_flags"]},
}))
