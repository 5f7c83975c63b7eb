"""Dev probe: per-batch diagnostics of the sequential TLSF engine (engine_seq.cuh) on a config
(GPU).  Not part of the product.  Usage: python tools/seq_probe.py CFG NBATCH"""
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
h.profile(0xFFFF)
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
    prof = h.profile_read()
    eng = prof.get("engine", (0, 0))[0]
    st = h.stats()
    na = len(s)
    cyc = d[5]
    if os.environ.get("HEAP_ENGINE", "") != "seq":
        ch = max(d[0], 1)
        print(f"b{bi} na={na} engine={eng:.2f}ms chunks={d[0]} commit/chunk={na/ch:.1f} cyc/chunk spec={d[5]/ch:.0f} "
              f"dirty={d[6]/ch:.0f} cls={d[7]/ch:.0f} arr={d[8]/ch:.0f} store={d[11]/ch:.0f} | req={d[9]} waits={d[12]} "
              f"waitcyc/chunk={d[13]/ch:.0f} ins={d[15]} helper_msgs={d[10]} err={c[2]}", flush=True)
        continue
    print(f"b{bi} na={na} F={st['n_free']} step={dt*1e3:.1f}ms engine={eng:.2f}ms cyc/req={cyc/max(na,1):.0f} "
          f"pops={d[0]} arr={d[1]} req={d[3]} ins={d[4]} waits={d[7]} waitcyc={d[6]} ({d[6]/max(cyc,1)*100:.1f}%) "
          f"merges={d[8]} gives={d[9]} helper_msgs={d[10]} err={c[2]} "
          f"cyc: load={d[11]/max(na,1):.0f} serve={d[12]/max(na,1):.0f} pop={d[13]/max(na,1):.0f} arr={d[15]/max(na,1):.0f} "
          f"rest={(cyc-d[11]-d[12]-d[13]-d[15])/max(na,1):.0f} "
          f"prof={ {k: round(v[0], 2) for k, v in prof.items()} }", flush=True)
