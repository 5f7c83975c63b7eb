import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import tracegen as tg
from paper_2405_07079_b200 import Heap
c4 = tg.CONFIGS[4]
cfg = tg.Config(c4.idx, "x", 10, c4.arena_bytes, c4.align, c4.model, c4.batch, c4.rho_num, c4.rho_den, c4.batch*12, c4.size_kind, c4.a, c4.b, max_live=c4.max_live)
h = Heap(cfg.arena_bytes, cfg.align, 10, cfg.max_live, cfg.batch)
idm = torch.full((cfg.batch*12+1,), -1, dtype=torch.int64, device="cuda")
prev = h.debug_counters()
for bi,(f,s,first) in enumerate(tg.Trace(cfg)):
    fd = torch.from_numpy(f.astype(np.int64)).cuda(); sd = torch.from_numpy(s.view(np.int64)).cuda()
    h.free_batch(idm[fd] if len(f) else fd); idm[first:first+len(s)] = h.alloc_batch(sd)
    c = h.debug_counters(); d=[a-b for a,b in zip(c,prev)]; prev=c; na=len(s)
    print(f"b{bi} na={na} cyc/req={d[0]/na:.0f} ins/req={d[3]/na:.2f} cyc/ins={d[1]/max(d[3],1):.0f} shift/ins={d[4]/max(d[3],1):.1f} refills={d[6]}", flush=True)
