"""Dev tool: HEAP_PARTIAL_FREE throughput on a config-3-shaped trace (TLSF, 4 GiB, 64K-request
batches, 40% frees) where half of the frees are tail frees, beside the same heap
without the flag on the unmodified trace, and Oracle-L on the same batches.

Pass 1 (untimed) replays the trace once on the GPU heap to fix every batch's free offsets (the
tail deltas are seeded; offsets come from the heap's own results, which the parity tests prove
equal to the oracle's).  Pass 2 replays the recorded batches on a fresh heap with CUDA events
(device time of the second half); the free-lookup tag's time per launch gives the resolve +
apply kernels' share.  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tracegen as tg  # noqa: E402
from oracle import OracleL  # noqa: E402
from paper_2405_07079_b200 import HEAP_PARTIAL_FREE, Heap  # noqa: E402

NB = int(sys.argv[1]) if len(sys.argv) > 1 else 40
base = tg.CONFIGS[3]
rng = np.random.default_rng(2405)


def record(flag):
    """One untimed pass: per batch (free offsets, sizes)."""
    h = Heap(base.arena_bytes, base.align, base.policy | flag, base.max_live, 2 * base.batch)
    units, out_batches = {}, []
    idm = np.full(base.batch * NB + 1, (1 << 64) - 1, dtype=np.uint64)
    for bi, (fids, sizes, first) in enumerate(tg.Trace(base, total_ops=base.batch * NB)):
        offs = idm[fids.astype(np.int64)].copy()
        if flag:
            z = np.array([units.get(int(i), 1) for i in fids], dtype=np.int64)
            tail = (rng.random(len(fids)) < 0.5) & (z > 1) & (offs != np.uint64((1 << 64) - 1))
            d = 1 + (rng.random(len(fids)) * np.maximum(z - 1, 1)).astype(np.int64)
            offs[tail] += (d[tail] * base.align).astype(np.uint64)
        h.free_batch(torch.from_numpy(offs.view(np.int64)).cuda())
        out = h.alloc_batch(torch.from_numpy(sizes.view(np.int64)).cuda()).cpu().numpy().view(np.uint64)
        idm[first:first + len(sizes)] = out
        for k, s in enumerate(sizes):
            units[first + k] = -(-int(s) // base.align)
        out_batches.append((offs, sizes))
    h.close()
    return out_batches


def timed(flag, batches):
    h = Heap(base.arena_bytes, base.align, base.policy | flag, base.max_live, 2 * base.batch)
    dev = [(torch.from_numpy(f.view(np.int64)).cuda(), torch.from_numpy(s.view(np.int64)).cuda()) for f, s in batches]
    half = len(dev) // 2
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ops = 0
    for i, (f, s) in enumerate(dev):
        if i == half:
            torch.cuda.synchronize()
            ev0.record()
        h.free_batch(f)
        h.alloc_batch(s)
        if i >= half:
            ops += f.numel() + s.numel()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    # per-tag device time over two more replays of the last batches (direct launches)
    h2 = Heap(base.arena_bytes, base.align, base.policy | flag, base.max_live, 2 * base.batch)
    for i, (f, s) in enumerate(dev):
        if i == half:
            h2.profile(1 << 3)          # HEAP_TAG_LOOKUP: the lookup / resolve + apply kernels
        h2.free_batch(f)
        h2.alloc_batch(s)
    prof = h2.profile_read()
    st = h.stats()
    h.close()
    h2.close()
    return ops / ms * 1e3, ms / (len(dev) - half), prof, st


def oracle_rate(flag, batches):
    o = OracleL(base.arena_bytes, base.align, base.policy | flag)
    half, t, ops = len(batches) // 2, 0.0, 0
    for i, (f, s) in enumerate(batches):
        t0 = time.perf_counter()
        o.free_batch(f)
        o.alloc_batch(s)
        if i >= half:
            t += time.perf_counter() - t0
            ops += len(f) + len(s)
    return ops / t, o.stats()


res = {}
for name, flag in (("partial", HEAP_PARTIAL_FREE), ("plain", 0)):
    b = record(flag)
    v, ms, prof, st = timed(flag, b)
    ov, ost = oracle_rate(flag, b)
    lk = prof.get("table_lookup", (0.0, 0))
    res[name] = {"ops_per_s": v, "ms_per_batch": ms, "oracle_ops_per_s": ov, "ratio": v / ov,
                 "lookup_ms_per_launch_group": lk[0] / max(len(b) - len(b) // 2, 1),
                 "frees_ok": st["frees_ok"], "frees_double": st["frees_double"],
                 "frees_invalid": st["frees_invalid"], "oracle_counters_equal":
                 all(st[k] == ost[k] for k in ("frees_ok", "frees_double", "frees_invalid", "allocs_ok"))}
print(json.dumps({"workload": f"cfg3-shaped TLSF 4 GiB, {NB} batches of 65536, half the frees tail frees",
                  **res}))
