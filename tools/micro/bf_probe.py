"""Dev: k_bf_cls_engine phase clocks (BF_TIMING build) on config 2: build, search, delete,
remainder search, remainder insert, write-back — cycles per batch and per request."""
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
prev, na = None, 0
for i, (f, s, first) in enumerate(bs):
    if i == nb // 2: prev = h.debug_counters()
    if i >= nb // 2: na += len(s)
    fd = torch.from_numpy(f.astype(np.int64)).cuda()
    h.free_batch(idm[fd] if len(f) else fd)
    idm[first:first + len(s)] = h.alloc_batch(torch.from_numpy(s.view(np.int64)).cuda())
c = h.debug_counters()
st = h.stats()
d = [(a - b) for a, b in zip(c, prev)]
k = nb - nb // 2
names = ["build", "search", "delete", "rsearch", "insert", "writeback"]
print(f"batches {nb//2}..{nb-1}: {na/k:.0f} allocs/batch, n_free now {st.get('n_free')}")
print("cycles/batch: " + "  ".join(f"{n} {d[16 + j]/k:.0f}" for j, n in enumerate(names)))
print("cycles/request: " + "  ".join(f"{n} {d[16 + j]/na:.0f}" for j, n in enumerate(names[1:5], 1)))
if d[9]:
    print(f"speculative chunks: {d[8]/k:.0f}/batch, {d[9]/max(d[8],1):.1f} requests per chunk")
