"""Dev tool: per-tag device time (heap_profile_*) over a few batches of a config."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen as tg  # noqa: E402
from paper_2405_07079_b200 import Heap  # noqa: E402
from paper_2405_07079_b200._native import NTAGS  # noqa: E402

c, _, pol = sys.argv[1].partition(":"); c = int(c); nb = int(sys.argv[2])   # "c" or "c:policy"
cfg = tg.CONFIGS[c]
if pol:
    cfg = tg.Config(cfg.idx, cfg.name, int(pol), cfg.arena_bytes, cfg.align, cfg.model, cfg.batch, cfg.rho_num,
                    cfg.rho_den, cfg.total_ops, cfg.size_kind, cfg.a, cfg.b, n_slots=cfg.n_slots, max_live=cfg.max_live)
bs = list(tg.Trace(cfg, total_ops=cfg.batch * nb if cfg.model == 0 else None))[:nb]
h = Heap(cfg.arena_bytes, cfg.align, cfg.policy, cfg.max_live, max(cfg.batch, 1000))
idm = torch.full((sum(len(b[1]) for b in bs) + 1,), -1, dtype=torch.int64, device="cuda")
half = nb // 2
for i, (f, s, first) in enumerate(bs):
    if i == half:
        torch.cuda.synchronize()
        h.profile((1 << NTAGS) - 1)
        h.profile_read()
    fd = torch.from_numpy(f.astype(np.int64)).cuda()
    sd = torch.from_numpy(s.view(np.int64)).cuda()
    h.free_batch(idm[fd] if len(f) else fd)
    idm[first:first + len(s)] = h.alloc_batch(sd)
p = h.profile_read()
tot = sum(v[0] for v in p.values())
for k, (ms, n) in sorted(p.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:20s} {ms / (nb - half):9.3f} ms/batch  {n // (nb - half):4d} launches/batch  {ms / tot:6.1%}")
