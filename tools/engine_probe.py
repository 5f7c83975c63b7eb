"""Dev probe: per-batch alloc-engine diagnostics on a config (GPU).  Not part of the product."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen as tg  # noqa: E402
from paper_2405_07079_b200 import Heap  # noqa: E402

cfg = tg.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
h = Heap(cfg.arena_bytes, cfg.align, cfg.policy, cfg.max_live, cfg.batch)
idmap = torch.full((cfg.batch * nb + 1,), -1, dtype=torch.int64, device="cuda")
prev = h.debug_counters()
h.profile(1 << 9)
for bi, (f, s, first) in enumerate(tg.Trace(cfg, total_ops=cfg.batch * nb)):
    fd = torch.from_numpy(f.astype(np.int64)).cuda()
    sd = torch.from_numpy(s.view(np.int64)).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.free_batch(idmap[fd] if len(f) else fd)
    out = h.alloc_batch(sd)
    idmap[first:first + len(s)] = out
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    c = h.debug_counters()
    d = [a - b for a, b in zip(c, prev)]
    prev = c
    eng = h.profile_read().get("engine", (0, 0))[0]
    st = h.stats()
    na = len(s)
    print(f"b{bi} na={na} F={st['n_free']} step={dt*1e3:.1f}ms engine={eng:.1f}ms chunks={d[0]} "
          f"commit={na/max(d[0],1):.1f} rounds/chunk={d[3]/max(d[0],1):.2f} qsteps/round={d[4]/max(d[3],1):.2f} "
          f"reaims={d[1]} cyc/chunk spec={d[5]/max(d[0],1):.0f} dirty={d[6]/max(d[0],1):.0f} "
          f"cls={d[7]/max(d[0],1):.0f}(store {d[11]/max(d[0],1):.0f} refills {d[12]} maxlane_refill_cyc/chunk {d[13]/max(d[0],1):.0f}) arr={d[8]/max(d[0],1):.0f} delmin={d[9]} visits={d[10]} ovf_inserts={d[15]} cls_split pop={d[16]/max(d[0],1):.0f} rcsr={d[17]/max(d[0],1):.0f} rovf={d[18]/max(d[0],1):.0f} gather={d[19]/max(d[0],1):.0f} fail={c[2]}", flush=True)
