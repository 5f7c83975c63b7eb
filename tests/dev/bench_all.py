"""Dev tool: device-time throughput of every BASELINE config (a few batches each) vs the oracle.
Arguments: config ids, optionally "c:p" to run config c's trace under policy p."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tracegen as tg  # noqa: E402
from oracle import OracleL  # noqa: E402
from paper_2405_07079_b200 import Heap  # noqa: E402

NB = {1: 30, 2: 60, 3: 40, 4: 40, 5: 6}
for arg in (sys.argv[1:] or ["1", "2", "3", "4", "5"]):
    c, _, pol = arg.partition(":")
    c = int(c)
    cfg = tg.CONFIGS[c]
    if pol:
        cfg = tg.Config(cfg.idx, f"{cfg.name}-as-{tg.POLICY_NAME[int(pol)]}", int(pol), cfg.arena_bytes, cfg.align,
                        cfg.model, cfg.batch, cfg.rho_num, cfg.rho_den, cfg.total_ops, cfg.size_kind, cfg.a, cfg.b,
                        n_slots=cfg.n_slots, max_live=cfg.max_live)
    nb = NB[c]
    bs = list(tg.Trace(cfg, total_ops=cfg.batch * nb if cfg.model == 0 else None))[:nb]
    h = Heap(cfg.arena_bytes, cfg.align, cfg.policy, cfg.max_live, max(cfg.batch, 1000))
    idm = torch.full((sum(len(b[1]) for b in bs) + 1,), -1, dtype=torch.int64, device="cuda")
    dev = [(torch.from_numpy(f.astype(np.int64)).cuda(), torch.from_numpy(s.view(np.int64)).cuda(), first) for f, s, first in bs]
    torch.cuda.synchronize()
    half = len(dev) // 2
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ops = 0
    for i, (f, s, first) in enumerate(dev):
        if i == half:
            torch.cuda.synchronize()
            ev0.record()
        h.free_batch(idm[f] if f.numel() else f)
        out = h.alloc_batch(s)
        idm[first:first + s.numel()] = out
        if i >= half:
            ops += f.numel() + s.numel()
    ev1.record()
    torch.cuda.synchronize()
    g_ms = ev0.elapsed_time(ev1)
    o = OracleL(cfg.arena_bytes, cfg.align, cfg.policy)
    om = np.full(sum(len(b[1]) for b in bs) + 1, (1 << 64) - 1, dtype=np.uint64)
    ot, oops = 0.0, 0
    for i, (f, s, first) in enumerate(bs):
        offs = om[f.astype(np.int64)]
        t0 = time.perf_counter()
        o.free_batch(offs)
        out = o.alloc_batch(s)
        if i >= half:
            ot += time.perf_counter() - t0
            oops += len(f) + len(s)
        om[first:first + len(s)] = out
    print(f"cfg{c} {cfg.name}: gpu {ops / g_ms * 1e3:.3e} ops/s ({g_ms / (len(dev) - half):.3f} ms/batch)  "
          f"oracle {oops / ot:.3e} ops/s  ratio {ops / g_ms * 1e3 / (oops / ot):.1f}x", flush=True)
