"""Dev: k_alloc_levels phase clocks (BUDDY_TIMING build) on config 4."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tracegen as tg
from paper_2405_07079_b200 import Heap
cfg = tg.CONFIGS[4]
nb = 12
bs = list(tg.Trace(cfg, total_ops=cfg.batch * nb))[:nb]
h = Heap(cfg.arena_bytes, cfg.align, cfg.policy, cfg.max_live, cfg.batch)
idm = torch.full((sum(len(b[1]) for b in bs) + 1,), -1, dtype=torch.int64, device="cuda")
prev = None
for i, (f, s, first) in enumerate(bs):
    if i == 4: prev = h.debug_counters()
    fd = torch.from_numpy(f.astype(np.int64)).cuda()
    h.free_batch(idm[fd] if len(f) else fd)
    idm[first:first + len(s)] = h.alloc_batch(torch.from_numpy(s.view(np.int64)).cuda())
c = h.debug_counters()
d = [(a - b) / (nb - 4) for a, b in zip(c, prev)]
print("alloc levels cycles/batch: bottom-up %.0f  top-down %.0f  lists %.0f" % (d[20], d[21], d[22]))
print("bottom-up per level:", " ".join(f"{t}:{d[t]:.0f}" for t in range(20)))
