"""Dev: bench.py's per-config side measurement for the given configs (GPU)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import tracegen as tg
dev = torch.device("cuda:0")
flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
NB = {1: 0, 2: 60, 3: 24, 4: 24}
for c in (int(x) for x in (sys.argv[1:] or ["1", "2", "3", "4"])):
    r = bench.run_config(tg.CONFIGS[c], NB[c], dev, flush)
    print(c, json.dumps({k: r[k] for k in ("device_ops_s", "ms_per_batch", "oracle_ops_s", "vs_oracle", "parity_ok", "timing")}), flush=True)
