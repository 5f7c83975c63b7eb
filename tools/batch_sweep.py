"""SURVEY.md §8(d) batch-size sweep on the config-5 generator (TLSF, 64 GiB, LU8[16,4096), 60/40):
device-time ops/s and the payload-roofline fraction (64 B per alloc + 88 B per free, the
survey's minimum-traffic model) per batch size.  Timed: the 4th..6th batch of each run."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen as tg  # noqa: E402
from paper_2405_07079_b200 import Heap  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
base = tg.CONFIGS[5]
for B in [int(x) for x in (sys.argv[1:] or ["65536", "262144", "1048576", "4194304"])]:
    cfg = tg.Config(5, f"cfg5-B{B}", base.policy, base.arena_bytes, base.align, 0, B, base.rho_num, base.rho_den,
                    B * 6, 0, base.a, base.b, max_live=max(base.max_live, 4 * B))
    bs = list(tg.Trace(cfg))
    h = Heap(cfg.arena_bytes, cfg.align, cfg.policy, cfg.max_live, B)
    idm = torch.full((sum(len(b[1]) for b in bs) + 1,), -1, dtype=torch.int64, device="cuda")
    t_ms, ops, byts = 0.0, 0, 0
    for i, (f, s, first) in enumerate(bs):
        fd = torch.from_numpy(f.astype(np.int64)).cuda()
        sd = torch.from_numpy(s.view(np.int64)).cuda()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.free_batch(idm[fd] if len(f) else fd)
        idm[first:first + len(s)] = h.alloc_batch(sd)
        e.record()
        torch.cuda.synchronize()
        if i >= 3:
            t_ms += a.elapsed_time(e)
            ops += len(f) + len(s)
            byts += 64 * len(s) + 88 * len(f)
    gbs = byts / (t_ms / 1e3) / 1e9
    print(f"B={B:>8d}  {ops / (t_ms / 1e3):.3e} ops/s  {t_ms / 3:.2f} ms/batch  payload {gbs:.2f} GB/s "
          f"= {gbs / peak:.5f} of measured HBM", flush=True)
    del h
    torch.cuda.empty_cache()
