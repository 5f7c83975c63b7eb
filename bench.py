#!/usr/bin/env python
"""bench.py — throughput of the batched device heap on BASELINE.json's headline workload.

Workload: BASELINE config 5 per GPU — TLSF, 64 GiB arena (2^32 units of
16 B), batches of 1,048,576 requests with a 60/40 alloc/free mix, sizes LU8[16 B, 4 KiB).
A *step* is one canonical batch through the whole hot path: id -> offset gather of the
batch's frees, heap_free_batch (classify, sort, block-table delete, merge, coalesce) and
heap_alloc_batch (normalise, class index, exact engine, compaction, block-table insert),
plus the NCCL all-gather of heap statistics when N > 1.

``value`` = submitted alloc+free requests of all ranks / max-over-ranks device time of the
K timed steps (inputs resident in HBM, L2 flushed between steps).  ``e2e`` = the same
metric through the C ABI with host buffers: pinned-host -> device copies of the step's
offsets and sizes and the device -> host copy of its results inside the timed region.

``--impl reference`` times the CPU oracle (oracle/, the tier's reference arm) on the same
workload, one batch per step, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import tracegen as tg  # noqa: E402

METRIC = "alloc+free ops/sec per GPU and 8-GPU aggregate vs cudaMalloc/cudaMallocAsync"
UNIT = "ops/s"

# Algorithmic bytes per processed unit for each kernel group: what the step
# must move at minimum with the 8-byte ABI words and 8/16-byte metadata records.
#   unit "alloc": one alloc request; "free": one free request; "elem": one element of the
#   tag's own array per launch (sort: keys+payload of a pass; merge/coalesce/compact: blocks)
TAG_BYTES = {
    # SURVEY.md 8(d)'s per-op payload model for the two phases' dominant kernels: an alloc moves
    # size 8 + offset 8 + table slot 16 + chosen free entry 16 + remainder 16 = 64 B; a free moves
    # offset 8 + slot read 16 + tombstone 16 + coalesced entry 16 + two neighbour reads 32 = 88 B
    "engine": ("alloc", 64),
    "table_lookup": ("free", 88),
    "finish": ("alloc", 8 + 8 + 8 + 8),             # r, offset in; bytes out; table slot write
    "alloc_prep": ("alloc", 8 + 8 + 4),             # size in; r, class out
    "classify": ("free", 8 + 4 + 4),                # offset in; key, flag out
}
# HEAP_HYBRID (pool.cuh): its tags name different kernels
TAG_BYTES_HYBRID = {
    "engine": ("alloc", 4 + 8 + 1),                 # k_select: request index in, offset out, ~1 B of bitmap
    "classify": ("free", 8 + 4 + 8 + 4),            # k_free: offset in, flag out, bitmap word r/w, superblock count
    "alloc_prep": ("alloc", 8 + 4 + 4),             # k_keys: size in, key + index out
    "sort": ("alloc", 2 * (4 + 4)),                 # one counting-sort pass: key + index in and out
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=5)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-batches", type=int, default=0, help="0 = auto")
    p.add_argument("--no-arena", action="store_true", help="do not allocate the arena tensor")
    p.add_argument("--no-driver-baselines", action="store_true")
    p.add_argument("--driver-max-ops", type=int, default=2_000_000)
    p.add_argument("--dist-backend", default="nccl", help=argparse.SUPPRESS)
    p.add_argument("--dev-share-gpu", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--no-per-config", action="store_true", help="skip the configs 1-4 side measurements")
    p.add_argument("--no-hybrid", action="store_true",
                   help="skip the extra HEAP_HYBRID measurement on the same trace")
    return p.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def aggregate(t_ms, ops, world, dev):
    """Whole-job numbers: max over ranks of the device time, sum over ranks of the ops."""
    if world == 1:
        return t_ms, ops
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "gloo":
        dev = "cpu"
    tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    oo = torch.tensor([ops], dtype=torch.int64, device=dev)
    dist.all_reduce(oo, op=dist.ReduceOp.SUM)
    return float(tt.item()), int(oo.item())


def gather_stats(local, world):
    """All-gather of the 16 x u64 heap statistics (the path's only collective)."""
    if world == 1:
        return local.view(1, -1)
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "gloo":            # CPU tests and the one-GPU dev mode
        parts = [torch.empty_like(local.cpu()) for _ in range(world)]
        dist.all_gather(parts, local.cpu())
        return torch.stack(parts).to(local.device)
    out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local)
    return out.view(world, -1)


def make_trace(cfg, rank, nbatches):
    t = tg.Trace(cfg, rank=rank, total_ops=cfg.batch * nbatches)
    return [b for b in t]


# ------------------------------------------------------------------ clocks ----
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 7:
                    rows.append(parts)
        finally:
            os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        load = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(tag):
    """Per-launch DRAM bytes of the tag's dominant kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(tag)
    except Exception:
        return None


def cpu_info():
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def oracle_replay(cfg, batches, warmup, gpu_outs=None, core=None):
    """Oracle-L (1 host thread, pinned to `core` if given) over every batch of the trace: the
    canonical free batch then the alloc batch, timed on batches warmup.. (the GPU's timed window),
    and every returned offset compared with gpu_outs[bi] (the GPU's results, HEAP_NULL as -1)."""
    from oracle import OracleL
    if core is not None:
        try:
            os.sched_setaffinity(0, {core % (os.cpu_count() or 1)})
        except (AttributeError, OSError):
            pass
    o = OracleL(cfg.arena_bytes, cfg.align, cfg.policy)
    n_alloc = sum(len(b[1]) for b in batches) + 1
    omap = np.full(n_alloc, (1 << 64) - 1, dtype=np.uint64)
    t, ops, mism, checked = 0.0, 0, None, 0
    for bi, (fids, sizes, first) in enumerate(batches):
        offs = omap[fids.astype(np.int64)]
        t0 = time.perf_counter()
        o.free_batch(offs)
        out = o.alloc_batch(sizes)
        dt = time.perf_counter() - t0
        if bi >= warmup:
            t += dt
            ops += len(fids) + len(sizes)
        if gpu_outs is not None and bi < len(gpu_outs):
            g = gpu_outs[bi].view(np.uint64)
            if mism is None and not np.array_equal(g, out):
                j = int(np.flatnonzero(g != out)[0])
                mism = {"batch": bi, "request": j, "gpu": int(g[j]), "oracle": int(out[j])}
            checked += 1
        omap[first:first + len(sizes)] = out
    return {"value": ops / t if t > 0 else None, "ops": ops, "seconds": t, "mismatch": mism,
            "checked_batches": checked, "state": o.stats()}


# --------------------------------------------------------------- reference ----
def run_reference(args, cfg):
    from oracle import OracleL
    nb = args.warmup + args.steps
    batches = make_trace(cfg, 0, nb)
    h = OracleL(cfg.arena_bytes, cfg.align, cfg.policy)
    idmap = np.full(cfg.batch * nb + 1, tg.HEAP_NULL if hasattr(tg, "HEAP_NULL") else (1 << 64) - 1, dtype=np.uint64)
    t_total, ops = 0.0, 0
    for bi, (fids, sizes, first) in enumerate(batches):
        offs = idmap[fids.astype(np.int64)]
        t0 = time.perf_counter()
        h.free_batch(offs)
        out = h.alloc_batch(sizes)
        dt = time.perf_counter() - t0
        idmap[first:first + len(sizes)] = out
        if bi >= args.warmup:
            t_total += dt
            ops += len(fids) + len(sizes)
    value = ops / t_total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (tracegen, seed 2405070790+1000c+r)",
        "config": {"workload": cfg.name, "policy": "tlsf", "arena_bytes": cfg.arena_bytes,
                   "align": cfg.align, "batch": cfg.batch, "alloc_free_mix": "60/40",
                   "sizes": "LU8[16,4096)", "batches": f"{args.warmup}..{nb - 1} of the trace"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"config {cfg.idx} batches {args.warmup}..{nb - 1} ({ops} ops), Oracle-L, 1 thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- ours ----
def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2405_07079_b200 import Heap, heap_stats_async, nccl_comm_init, nccl_unique_id
    from paper_2405_07079_b200._native import NTAGS

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    nb = args.warmup + args.steps
    batches = make_trace(cfg, rank, nb)
    n_alloc_total = sum(len(b[1]) for b in batches) + 1
    dev_batches = [(torch.from_numpy(f.astype(np.int64)).to(dev), torch.from_numpy(s.view(np.int64)).to(dev), first)
                   for f, s, first in batches]
    max_live = cfg.max_live
    arena = None
    if not args.no_arena:
        try:   # the arena the offsets index into; the heap never touches it
            arena = torch.empty(cfg.arena_bytes, dtype=torch.uint8, device=dev)
        except RuntimeError:
            arena = None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stats_dev = torch.zeros(16, dtype=torch.int64, device=dev)
    stats_all = torch.zeros(16 * world, dtype=torch.int64, device=dev) if world > 1 else None
    gloo = world > 1 and dist.get_backend() == "gloo"
    comm = None
    if world > 1 and not gloo:
        # the library's own NCCL communicator (heap_stats_allgather): rank 0's unique id travels
        # over the process group once, outside any timed region
        uid = torch.tensor(list(nccl_unique_id()) if rank == 0 else [0] * 128, dtype=torch.uint8, device=dev)
        dist.broadcast(uid, 0)
        comm = nccl_comm_init(world, bytes(uid.cpu().tolist()), rank)

    def run_device(h, idmap, outbuf, b, stream_stats=True):
        fids, sizes, first = b
        na = sizes.numel()
        # heap_step: frees by handle (offsets idmap[fids], looked up by the library), then the allocs
        h.step(idmap, sizes, idx=fids, out=idmap[first:first + na])
        if world > 1 and stream_stats:
            if gloo:      # CPU tests / one-GPU dev mode: NCCL cannot put two ranks on one GPU
                heap_stats_async(h.handle, stats_dev)
                stats_all.copy_(gather_stats(stats_dev, world).view(-1))
            else:         # heap_stats_allgather: ncclAllGather of the 128-byte records
                h.stats_allgather(comm, stats_all.view(world, 16))

    # ---------------- device-resident run ----------------
    def device_run(policy, profile, keep_outs=False):
        """W warm-up + K timed steps on a fresh heap.  profile=False: the production path (batch
        graphs), timed for `value`; profile=True: direct launches bracketed by per-tag events
        (heap_profile_*), used only for the kernel shares and the roofline."""
        h = Heap(cfg.arena_bytes, cfg.align, policy, max_live, cfg.batch, device=dev)
        idmap = torch.full((n_alloc_total,), -1, dtype=torch.int64, device=dev)
        outbuf = None                 # results go straight into idmap (the handle table)
        outs = []
        for b in dev_batches[:args.warmup]:
            run_device(h, idmap, outbuf, b)
            if keep_outs:
                outs.append(idmap[b[2]:b[2] + b[1].numel()].cpu().numpy())
        torch.cuda.synchronize()
        if profile:
            h.profile((1 << NTAGS) - 1)
            h.profile_read()
        l0 = h.launch_count()
        dc0 = h.debug_counters()
        sampler = ClockSampler(local_rank)
        sampler.start()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        ops = 0
        for k, b in enumerate(dev_batches[args.warmup:]):
            flush.fill_(k & 255)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev[k][0].record()
            run_device(h, idmap, outbuf, b)
            ev[k][1].record()
            torch.cuda.synchronize()
            ops += b[0].numel() + b[1].numel()
            if keep_outs:      # outside the timed region: the step's results, for the parity check
                outs.append(idmap[b[2]:b[2] + b[1].numel()].cpu().numpy())
        torch.cuda.synchronize()
        clocks = sampler.stop()
        launches = h.launch_count() - l0
        dc = [a - b for a, b in zip(h.debug_counters(), dc0)]
        prof = h.profile_read() if profile else None
        h.profile(0)
        step_ms = [a.elapsed_time(e) for a, e in ev]
        t_ms = sum(step_ms)
        st = h.stats()
        t_max, ops_all = aggregate(t_ms, ops, world, dev)
        del h
        torch.cuda.empty_cache()
        return dict(value=ops_all / (t_max / 1e3), t_ms=t_ms, t_max=t_max, step_ms=step_ms, prof=prof,
                    launches=launches, st=st, clocks=clocks, dc=dc, outs=outs)

    R = device_run(cfg.policy, False, keep_outs=True)
    value, t_ms, t_max, step_ms, launches, st, clocks = (R[k] for k in (
        "value", "t_ms", "t_max", "step_ms", "launches", "st", "clocks"))
    engine_chain = _engine_chain(R["dc"], sum(len(b[1]) for b in batches[args.warmup:]), cfg.policy)
    RP = device_run(cfg.policy, True)
    prof, t_ms_prof = RP["prof"], RP["t_ms"]

    # ---------------- e2e through the C ABI with host buffers ----------------
    e2e = None
    if not args.no_e2e:
        h = Heap(cfg.arena_bytes, cfg.align, cfg.policy, max_live, cfg.batch, device=dev)
        hmap = np.full(n_alloc_total, -1, dtype=np.int64)
        pin_off = torch.empty(cfg.batch, dtype=torch.int64).pin_memory()
        pin_sz = torch.empty(cfg.batch, dtype=torch.int64).pin_memory()
        pin_out = torch.empty(cfg.batch, dtype=torch.int64).pin_memory()
        d_off = torch.empty(cfg.batch, dtype=torch.int64, device=dev)
        d_sz = torch.empty(cfg.batch, dtype=torch.int64, device=dev)
        e_ms, e_ops, h2d, d2h = 0.0, 0, 0, 0
        for bi, (fids, sizes, first) in enumerate(batches):
            nf, na = len(fids), len(sizes)
            pin_off[:nf].numpy()[:] = hmap[fids.astype(np.int64)]
            pin_sz[:na].numpy()[:] = sizes.view(np.int64)
            flush.fill_(bi & 255)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            d_off[:nf].copy_(pin_off[:nf], non_blocking=True)
            d_sz[:na].copy_(pin_sz[:na], non_blocking=True)
            h.free_batch(d_off[:nf])
            out = h.alloc_batch(d_sz[:na])
            pin_out[:na].copy_(out, non_blocking=True)
            e.record()
            torch.cuda.synchronize()
            hmap[first:first + na] = pin_out[:na].numpy()
            if bi >= args.warmup:
                e_ms += a.elapsed_time(e)
                e_ops += nf + na
                h2d += 8 * (nf + na)
                d2h += 8 * na
        e_ms, e_ops_all = aggregate(e_ms, e_ops, world, dev)
        e2e = {"value": e_ops_all / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps}
        del h

    # ---------------- roofline of the dominant kernel group ----------------
    def roofline(prof, t_ms, table):
        dom = max(prof.items(), key=lambda kv: kv[1][0]) if prof else None
        shares = {k: round(v[0] / max(t_ms, 1e-9), 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}
        if not dom:
            return None, shares
        tag, (ms, nl) = dom
        peak, peak_src = measured_peak_hbm()
        unit, bpu = table.get(tag, ("alloc", 64))
        n_units = sum(len(b[1]) if unit == "alloc" else len(b[0]) for b in batches[args.warmup:])
        per_launch_bytes = bpu * n_units / max(nl, 1)
        avg_s = ms / max(nl, 1) / 1e3
        achieved = per_launch_bytes / avg_s / 1e9
        return ({"bound": "hbm", "kernel": tag, "achieved": achieved, "peak": peak, "unit": "GB/s",
                 "frac": achieved / peak, "traffic": ncu_traffic(tag) if table is TAG_BYTES else None,
                 "peak_source": peak_src, "bytes_per_launch": per_launch_bytes, "avg_launch_ms": avg_s * 1e3},
                shares)

    roof, shares = roofline(prof, t_ms_prof, TAG_BYTES)

    # ---------------- the same trace on the §5.3 hybrid (pools below a page + TLSF) ----------------
    hyb = None
    if not args.no_hybrid and cfg.policy != tg.HYBRID:
        H = device_run(tg.HYBRID, False)
        HP = device_run(tg.HYBRID, True)
        hroof, hshares = roofline(HP["prof"], HP["t_ms"], TAG_BYTES_HYBRID)
        hyb = {"policy": "hybrid", "value": H["value"], "unit": UNIT, "ms_per_step": H["t_max"] / args.steps,
               "gpu_launches": H["launches"], "roofline": hroof, "kernel_shares": hshares,
               "ms_per_step_profiled": HP["t_max"] / args.steps,
               "heap": {"n_live": H["st"]["n_live"], "allocs_failed": H["st"]["allocs_failed"],
                        "error_flags": H["st"]["error_flags"]},
               "note": "same trace and timing protocol; every request of this workload is below a page, "
                       "so the bitmask pools serve it (DESIGN.md C26) — a different allocator, not the headline"}

    # ---------------- driver-allocator baselines (the paper's comparison) ----------------
    drv = None
    if rank == 0 and not args.no_driver_baselines:
        import baselines
        drv = {}
        for name, mode in (("cudaMalloc", 0), ("cudaMallocAsync", 1)):
            try:
                r = baselines.replay(mode, batches, max_ops=args.driver_max_ops, max_seconds=60.0)
            except Exception as e:  # never lose the main line over a baseline
                r = {"error": str(e)[:200]}
            r["sample"] = (f"config {cfg.idx} batches from 0, same per-batch op order, 1 host thread, "
                           f"capped at {args.driver_max_ops} ops / 60 s")
            drv[name] = r

    # ---------------- CPU oracle: the same timed batches, and parity of every result ----------------
    # Each rank replays its own trace with Oracle-L on its own host core (pinned), after the GPU
    # runs; cpu_baseline = sum of ops / max time over ranks.  The oracle's outputs
    # are compared with every offset the production run returned, warm-up and timed batches alike.
    cpu, parity = None, None
    if not args.no_cpu_baseline:
        orc = oracle_replay(cfg, batches, args.warmup, R["outs"], core=local_rank if world > 1 else None)
        c_s, c_ops = aggregate(orc["seconds"] * 1e3, orc["ops"], world, dev)
        bad = orc["mismatch"] is not None
        if world > 1:
            import torch.distributed as dist
            fl = torch.tensor([1 if bad else 0], dtype=torch.int64, device="cpu" if gloo else dev)
            dist.all_reduce(fl)
            bad = int(fl.item()) > 0
        parity = {"checked": f"batches 0..{nb - 1} (warm-up and timed), every returned offset, every rank",
                  "ok": not bad, "first_mismatch_rank0": orc["mismatch"]}
        cpu = {"value": c_ops / (c_s / 1e3), "unit": UNIT, "cores": world, "kind": "oracle",
               "sample": (f"config {cfg.idx} batches {args.warmup}..{nb - 1} ({c_ops} ops over {world} rank(s)) - "
                          f"the GPU's timed batches - replayed by Oracle-L, 1 pinned host thread per rank"),
               **cpu_info()}

    # ---------------- the other configs: device vs oracle on the same batches ----------------
    per_config = None
    if rank == 0 and world == 1 and not args.no_per_config and cfg.idx == 5:
        per_config = {}
        for cid, nbc in ((1, 0), (2, 60), (3, 24), (4, 24)):
            try:
                per_config[tg.CONFIGS[cid].name] = run_config(tg.CONFIGS[cid], nbc, dev, flush)
            except Exception as e:   # never lose the headline line over a side measurement
                per_config[tg.CONFIGS[cid].name] = {"error": str(e)[:200]}

    valid = st["error_flags"] == 0 and (parity is None or parity["ok"])
    if rank == 0:
        line = {
            "valid": valid,
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (tracegen, seed 2405070790+1000c+r; per-rank independent traces)",
            "config": {"workload": cfg.name, "policy": tg.POLICY_NAME.get(cfg.policy, str(cfg.policy)), "arena_bytes": cfg.arena_bytes,
                       "align": cfg.align, "batch": cfg.batch, "alloc_free_mix": "60/40",
                       "sizes": "LU8[16,4096)", "timed_batches": f"{args.warmup}..{nb - 1}",
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"replicas x{world} (independent heaps, NCCL all-gather of heap_stats)",
                       "arena_allocated": arena is not None},
            "gpu_launches": launches,
            "roofline": roof,
            "kernel_shares": shares,
            "cpu_baseline": cpu,
            "parity": parity,
            "per_config": per_config,
            "driver_baselines": drv,
            "hybrid_same_trace": hyb,
            "e2e": e2e,
            "clocks": clocks,
            "heap": {"n_live": st["n_live"], "n_free": st["n_free"], "allocs_failed": st["allocs_failed"],
                     "error_flags": st["error_flags"]},
            "step_ms": [round(x, 3) for x in step_ms],
            "batch_latency_ms": {"p50": float(np.percentile(step_ms, 50)), "p99": float(np.percentile(step_ms, 99))},
            # SURVEY.md 8(d) payload model: 64 B per alloc, 88 B per free -> 73.6 B per op at 60/40
            "payload_roofline": _payload_roofline(value),
            # the TLSF engine is one warp's dependent chain: its structure
            "engine_chain": engine_chain,
        }
        print(json.dumps(line), flush=True)


def run_config(cfg, nbatches, dev, flush, warmup=3):
    """One BASELINE config as a side measurement (not the headline): W warm-up batches and the rest
    timed on the device (batch graphs, CUDA events, L2 flushed between steps), the same batches
    through Oracle-L on one host thread, every returned offset compared."""
    import torch
    from paper_2405_07079_b200 import Heap
    batches = make_trace(cfg, 0, nbatches) if nbatches else [b for b in tg.Trace(cfg)]
    warmup = min(warmup, len(batches) - 1)
    n_alloc = sum(len(b[1]) for b in batches) + 1
    h = Heap(cfg.arena_bytes, cfg.align, cfg.policy, cfg.max_live, max(max(len(b[1]), len(b[0])) for b in batches) or 1,
             device=dev)
    idmap = torch.full((n_alloc,), -1, dtype=torch.int64, device=dev)
    outs, t_ms, ops = [], 0.0, 0
    staged = [(torch.from_numpy(f.astype(np.int64)).to(dev), torch.from_numpy(s.view(np.int64)).to(dev), first)
              for f, s, first in batches]
    # warm-up batches run eagerly; the timed window is captured as ONE CUDA graph (the library launches
    # directly under capture) and replayed once, so small batches are timed without host issue gaps
    # frees by handle (heap_free_batch_handles): the id -> offset lookup happens inside the library's
    # free (fused into the kernel on single-launch heaps), as the oracle's host-side lookup sits
    # outside its own timing
    # (heap_step: the free batch then the alloc batch in one call — one launch on a single-launch heap)
    for bi, (fd, sd, first) in enumerate(staged[:warmup]):
        h.step(idmap, sd, idx=fd, out=idmap[first:first + len(sd)])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for fd, sd, first in staged[warmup:]:
            h.step(idmap, sd, idx=fd, out=idmap[first:first + len(sd)])
    flush.fill_(1)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    t_ms = a.elapsed_time(e)
    del g
    for bi, (fd, sd, first) in enumerate(staged):
        outs.append(idmap[first:first + len(sd)].cpu().numpy())
        if bi >= warmup:
            ops += len(fd) + len(sd)
    st = h.stats()
    del h
    orc = oracle_replay(cfg, batches, warmup, outs)
    dev_v = ops / (t_ms / 1e3)
    n_free = sum(len(b[0]) for b in batches[warmup:])
    n_al = sum(len(b[1]) for b in batches[warmup:])
    peak, src = measured_peak_hbm()
    pay = (64 * n_al + 88 * n_free) / (t_ms / 1e3) / 1e9
    return {"policy": tg.POLICY_NAME.get(cfg.policy), "batches": f"{warmup}..{len(batches) - 1} timed of {len(batches)}",
            "device_ops_s": dev_v, "ms_per_batch": t_ms / max(len(batches) - warmup, 1),
            "timing": ("the timed batches captured as one CUDA graph and replayed once (device time, no host "
                       "gaps, no L2 flush between batches)"),
            "oracle_ops_s": orc["value"], "vs_oracle": dev_v / orc["value"] if orc["value"] else None,
            "parity_ok": orc["mismatch"] is None and st["error_flags"] == 0, "mismatch": orc["mismatch"],
            "payload_roofline": {"achieved": pay, "peak": peak, "unit": "GB/s", "frac": pay / peak,
                                 "peak_source": src, "bytes": "64 B/alloc + 88 B/free (SURVEY.md 8(d))"}}


def _engine_chain(dc, n_alloc, policy):
    """TLSF/SEGFIT alloc-engine structure over the timed steps, from heap_debug_counters
    (engine_tlsf.cuh): chunks of 32 candidate requests, requests committed per chunk,
    speculation rounds per chunk, and the engine's cycles per chunk by phase."""
    if policy not in (tg.TLSF, tg.SEGFIT) or not dc or dc[0] == 0:
        return None
    ch = dc[0]
    out = {"allocs": n_alloc, "chunks": ch, "committed_per_chunk": n_alloc / ch,
           "rounds_per_chunk": dc[3] / ch, "overflow_inserts": dc[15], "overflow_extractions": dc[9]}
    if dc[5]:   # phase clocks exist only in an ENGINE_TIMING build (off in production: 0.4 % cost)
        out["cycles_per_chunk"] = {"speculation": dc[5] / ch, "dirty_check": dc[6] / ch,
                                   "class_update_pops": dc[16] / ch, "refill_csr": dc[17] / ch,
                                   "refill_overflow": dc[18] / ch, "arrivals": dc[8] / ch, "stores": dc[11] / ch}
    else:
        out["cycles_per_chunk"] = ("ENGINE_TIMING build only: tools/engine_probe.py, "
                                   "profiles/r02_engine_study.md")
    return out


def _payload_roofline(ops_per_s):
    bpo = 0.6 * 64 + 0.4 * 88
    peak, src = measured_peak_hbm()
    ach = ops_per_s * bpo / 1e9
    return {"bytes_per_op": bpo, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "peak_source": src}


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.dev_share_gpu:        # dev only: run every rank on GPU 0 (tests the N > 1 logic on one GPU)
        local_rank = 0
    cfg = tg.CONFIGS[args.config]
    if args.impl == "reference":
        # the reference arm is the CPU oracle: rank 0 alone runs it, no GPU and no process group
        if rank == 0:
            run_reference(args, cfg)
        return
    if args.dev_share_gpu:
        args.dist_backend = "gloo"    # NCCL refuses two ranks on one GPU
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(args.dist_backend)
    run_ours(args, cfg, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
