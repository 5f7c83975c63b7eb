"""Dev: micro-kernel phase clocks (MICRO_TIMING build) per batch on config 1."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tracegen as tg
from paper_2405_07079_b200 import Heap
cfg = tg.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
bs = list(tg.Trace(cfg, total_ops=(cfg.batch * 40 if cfg.model == 0 else None)))[:40]
h = Heap(cfg.arena_bytes, cfg.align, cfg.policy, cfg.max_live, max(cfg.batch, 1000))
idm = torch.full((sum(len(b[1]) for b in bs) + 1,), -1, dtype=torch.int64, device="cuda")
prev = h.debug_counters()
names = {16: "f.load", 17: "f.classify", 18: "f.sort", 19: "f.lookup", 20: "f.compact", 21: "f.merge+write",
         22: "a.load", 23: "a.engine", 24: "a.compact", 25: "a.finish"}
tot = {k: 0 for k in names}
nf = na = 0
for i, (f, s, first) in enumerate(bs):
    fd = torch.from_numpy(f.astype(np.int64)).cuda()
    h.free_batch(idm[fd] if len(f) else fd)
    idm[first:first + len(s)] = h.alloc_batch(torch.from_numpy(s.view(np.int64)).cuda())
    c = h.debug_counters()
    if i >= 5:
        for k in names: tot[k] += c[k] - prev[k]
        nf += len(f); na += len(s)
    prev = c
nb = len(bs) - 5
print(f"batches {nb}, avg frees {nf/nb:.1f} allocs {na/nb:.1f}, F={h.stats()['n_free']}")
for k, v in names.items(): print(f"{v:14s} {tot[k]/nb:9.0f} cycles/batch")
