"""heap_stats_allgather: the statistics collective of the multi-GPU path (DESIGN.md
§9), through the library's own NCCL communicator.  One GPU is available, so the communicator has one
rank: the gathered record must equal the heap's local heap_stats after a few batches, and the
collective must run asynchronously on the heap's stream (graph-captured batches included)."""
import numpy as np
import pytest
import torch

import tracegen as tg
from paper_2405_07079_b200 import Heap, nccl_comm_destroy, nccl_comm_init, nccl_comm_init_all, nccl_unique_id
from paper_2405_07079_b200._native import HeapStats

FIELDS = [n for n, _ in HeapStats._fields_]


def _run_some_batches(h, cfg, nb):
    idmap = torch.full((cfg.batch * nb + 1,), -1, dtype=torch.int64, device="cuda")
    for bi, (f, s, first) in enumerate(tg.Trace(cfg, total_ops=cfg.batch * nb)):
        fd = torch.from_numpy(f.astype(np.int64)).cuda()
        h.free_batch(idmap[fd] if len(f) else fd)
        idmap[first:first + len(s)] = h.alloc_batch(torch.from_numpy(s.view(np.int64)).cuda())


@pytest.mark.gpu
@pytest.mark.parametrize("init", ["all", "rank"])
def test_stats_allgather_one_rank(init):
    torch.cuda.set_device(0)
    if init == "all":
        comm = nccl_comm_init_all([0])[0]
    else:
        comm = nccl_comm_init(1, nccl_unique_id(), 0)
    try:
        for pol in (tg.TLSF, tg.BUDDY, tg.BEST_FIT):
            cfg = tg.custom(pol, 1 << 24, 256 if pol == tg.BUDDY else 16, 2048, total_ops=8192,
                            sizes=(8, 16) if pol == tg.BUDDY else (4, 12), size_kind=1 if pol == tg.BUDDY else 0,
                            idx=90 + pol)
            h = Heap(cfg.arena_bytes, cfg.align, pol, 1 << 14, 2048)
            _run_some_batches(h, cfg, 4)
            out = torch.full((1, 16), -7, dtype=torch.int64, device="cuda")
            h.stats_allgather(comm, out)
            torch.cuda.synchronize()
            local = h.stats()
            got = {n: int(v) for n, v in zip(FIELDS, out[0].cpu().tolist())}
            for n in FIELDS:
                assert got[n] == local[n], (pol, n, got[n], local[n])
            assert got["allocs_ok"] > 0 and got["live_bytes"] + got["free_bytes"] == cfg.arena_bytes
            h.close()
    finally:
        nccl_comm_destroy(comm)
