"""Dev: k_bf_spec_engine phase clocks (BF_TIMING build) on config 2."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tracegen as tg
from paper_2405_07079_b200 import Heap
cfg = tg.CONFIGS[2]
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 24
bs = list(tg.Trace(cfg, total_ops=cfg.batch * nb))[:nb]
h = Heap(cfg.arena_bytes, cfg.align, cfg.policy, cfg.max_live, cfg.batch)
idm = torch.full((sum(len(b[1]) for b in bs) + 1,), -1, dtype=torch.int64, device="cuda")
prev = None
for i, (f, s, first) in enumerate(bs):
    if i == nb // 2: prev = h.debug_counters()
    fd = torch.from_numpy(f.astype(np.int64)).cuda()
    h.free_batch(idm[fd] if len(f) else fd)
    idm[first:first + len(s)] = h.alloc_batch(torch.from_numpy(s.view(np.int64)).cuda())
c = h.debug_counters()
d = [(a - b) for a, b in zip(c, prev)]
ch = max(d[8], 1)
names = ["search", "dirty", "sort", "survivors", "remainders"]
print(f"chunks {d[8]}, {d[9]/ch:.1f} requests/chunk; cycles per chunk: " + "  ".join(f"{n} {d[16 + j]/ch:.0f}" for j, n in enumerate(names)))
