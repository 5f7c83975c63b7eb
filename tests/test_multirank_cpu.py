"""Multi-rank host logic on CPU (gloo, world size 2): per-rank independent heaps (replicas),
the statistics all-gather that is the path's only collective, and the whole-job aggregation
bench.py uses (max over ranks of time, sum over ranks of ops).  The per-rank heap here is the
oracle (no GPU on this box); the GPU path runs the same code under torchrun with NCCL."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import tracegen as tg
from oracle import OracleL
from tests.helpers import IdMap, replay

FIELDS = 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = tg.custom(tg.TLSF, 1 << 20, 16, 256, rho=(2, 5), total_ops=3000, idx=5)
    t = tg.Trace(cfg, rank=rank)
    h = OracleL(cfg.arena_bytes, cfg.align, cfg.policy)
    ops = [0]

    def on_batch(bi, offs, sizes, out):
        ops[0] += len(offs) + len(sizes)
    replay(h, t, IdMap(4096), on_batch=on_batch)
    st = h.stats()
    local = torch.tensor([st[k] for k in st], dtype=torch.int64)
    gathered = bench.gather_stats(local, world)
    t_max, ops_all = bench.aggregate(float(rank + 1), ops[0], world, torch.device("cpu"))
    q.put((rank, local.numpy(), gathered.numpy(), t_max, ops_all, ops[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_gather_and_aggregate():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    locals_ = [r[1] for r in res]
    # independent replicas: different traces give different heaps
    assert not np.array_equal(locals_[0], locals_[1])
    for rank, local, gathered, t_max, ops_all, ops in res:
        assert gathered.shape == (world, FIELDS)
        for r in range(world):
            assert np.array_equal(gathered[r], locals_[r])      # gathered row r == rank r's stats
        assert t_max == float(world)                             # max over ranks
        assert ops_all == sum(x[5] for x in res)                 # sum over ranks


def test_bench_line_helpers():
    """bench.py's derived fields: the payload roofline (64 B per alloc, 88 B per
    free, 73.6 B per op at the 60/40 mix) and the engine-chain summary of heap_debug_counters."""
    pr = bench._payload_roofline(1e6)
    assert abs(pr["bytes_per_op"] - 73.6) < 1e-9
    assert abs(pr["achieved"] - 0.0736) < 1e-12
    assert abs(pr["frac"] - pr["achieved"] / pr["peak"]) < 1e-15
    dc = [0] * 32
    dc[0], dc[3], dc[5], dc[6], dc[8], dc[11], dc[9], dc[15] = 10, 10, 2000, 1000, 2500, 100, 7, 9
    dc[16], dc[17], dc[18] = 350, 850, 2300
    ec = bench._engine_chain(dc, 190, tg.TLSF)
    assert ec["chunks"] == 10 and ec["committed_per_chunk"] == 19.0 and ec["rounds_per_chunk"] == 1.0
    assert ec["cycles_per_chunk"]["refill_overflow"] == 230.0 and ec["cycles_per_chunk"]["dirty_check"] == 100.0
    assert ec["overflow_extractions"] == 7 and ec["overflow_inserts"] == 9
    dc[5] = 0                                # a production build: no phase clocks
    assert isinstance(bench._engine_chain(dc, 190, tg.TLSF)["cycles_per_chunk"], str)
    assert bench._engine_chain(dc, 190, tg.BUDDY) is None
    assert bench._engine_chain([0] * 32, 190, tg.TLSF) is None
