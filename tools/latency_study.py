"""SURVEY §8(f) f1 study: batch-size-1 latency and fragmentation on the paper's malloc-large
shape (Fig. 3/4 analogue).  Not part of the product path; needs a GPU.

Workload (DESIGN.md §9 reading): the mimalloc malloc-large pattern the paper adapted — a slot
model (tracegen model 1) over N_SLOTS slots: pick a uniform slot, free its block if occupied,
allocate a new one of LU8[1 KiB, 16 MiB) bytes — for N_OPS ops.  The same op sequence runs
through (a) this library's C ABI one request per call (SEGFIT_LIFO = the paper's Alg. 4/5
allocator, and TLSF), (b) cudaMalloc/cudaFree, (c) cudaMallocAsync/cudaFreeAsync + sync.

Usage: python tools/latency_study.py [out.json]
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import baselines  # noqa: E402
import tracegen as tg  # noqa: E402
from paper_2405_07079_b200 import Heap  # noqa: E402
from paper_2405_07079_b200 import heap as H  # noqa: E402

N_SLOTS, N_OPS, ARENA, ALIGN = 100, 6000, 8 << 30, 256
SRC = os.path.join(ROOT, "tools", "latency_study.cu")
LIB = os.path.join(ROOT, "tools", "liblatency_study.so")


def build():
    pkg = os.path.join(ROOT, "paper_2405_07079_b200")
    subprocess.check_call(["nvcc", "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared",
                           "-I", os.path.join(ROOT, "include"), "-o", LIB, SRC, "-L", pkg, "-lheap",
                           f"-Xlinker=-rpath={pkg}", "-cudart", "shared"])
    return ctypes.CDLL(LIB)


def op_list():
    cfg = tg.custom(tg.SEGFIT_LIFO, ARENA, ALIGN, 2, total_ops=N_OPS, sizes=(10, 24), model=1,
                    n_slots=N_SLOTS, idx=95)
    kind, arg = [], []
    for f, s, _ in tg.Trace(cfg):
        for i in f:
            kind.append(0); arg.append(int(i))
        for z in s:
            kind.append(1); arg.append(int(z))
    return np.array(kind, np.uint8), np.array(arg, np.uint64)


def live_bytes(kind, arg, align=1):
    sizes, live, cur = [], np.zeros(len(kind), np.uint64), 0
    for j, (k, a) in enumerate(zip(kind, arg)):
        if k:
            z = -(-int(a) // align) * align
            sizes.append(z); cur += z
        else:
            cur -= sizes[int(a)]
        live[j] = cur
    return live


def summarise(lat, kind, used, live, warm=200):
    out = {}
    for name, m in (("alloc", kind == 1), ("free", kind == 0)):
        x = lat[m] / 1e3
        xs = lat[m][warm // 2:] / 1e3
        out[name] = {"n": int(m.sum()), "p50_us": float(np.median(x)), "p99_us": float(np.percentile(x, 99)),
                     "max_us": float(x.max()), "mean_us": float(x.mean()),
                     "steady_p50_us": float(np.median(xs)), "first_op_us": float(x[0])}
    half = len(kind) // 2
    frag = 1.0 - live[half:].astype(np.float64) / np.maximum(used[half:].astype(np.float64), 1)
    out["fragmentation_second_half"] = {"mean": float(frag.mean()), "max": float(frag.max())}
    return out


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join("gpurun_out", "latency_study.json")
    kind, arg = op_list()
    live = live_bytes(kind, arg)
    L = build()
    res = {"workload": f"slot model (malloc-large shape): {N_SLOTS} slots, {len(kind)} ops, "
                       f"LU8[1 KiB, 16 MiB) bytes, seed {tg.custom(6, ARENA, ALIGN, 2, idx=95).seed(0)}",
           "arena_bytes": ARENA, "align": ALIGN, "gpu": torch.cuda.get_device_name(0), "arms": {}}
    series = {"live": live[::10].tolist()}
    for pol in (tg.SEGFIT_LIFO, tg.TLSF):
        h = Heap(ARENA, ALIGN, pol, 4096, 2)
        n = len(kind)
        lat = np.zeros(n); lv = np.zeros(n, np.uint64); hw = np.zeros(n, np.uint64)
        fail = ctypes.c_uint64(0)
        dp = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))  # noqa: E731
        s = torch.cuda.current_stream()
        rc = L.heap_latency(h.handle, ctypes.c_void_p(s.cuda_stream), ctypes.c_uint64(n), dp(kind, ctypes.c_uint8),
                            dp(arg, ctypes.c_uint64), dp(lat, ctypes.c_double), dp(lv, ctypes.c_uint64),
                            dp(hw, ctypes.c_uint64), ctypes.byref(fail))
        assert rc == 0, rc
        assert np.array_equal(lv, live_bytes(kind, arg, ALIGN)), "heap live bytes differ from the trace's"
        name = H.POLICY_NAMES[pol]
        res["arms"][name] = summarise(lat, kind, hw, live)
        res["arms"][name]["failed"] = int(fail.value)
        res["arms"][name]["launches_per_op"] = h.launch_count() / n
        series[name + "_hwm"] = hw[::10].tolist()
        h.close()
        del h
        torch.cuda.empty_cache()
    for mode, name in ((0, "cudaMalloc"), (1, "cudaMallocAsync")):
        torch.cuda.synchronize()
        fr, tot = torch.cuda.mem_get_info()
        base = tot - fr                     # the process's device memory before the replay
        lat, used, fail = baselines.replay_latency(mode, kind, arg)
        prov = np.maximum(used.astype(np.int64) - base, 0).astype(np.uint64)
        res["arms"][name] = summarise(lat, kind, prov, live)
        res["arms"][name]["failed"] = fail
        series[name + "_used"] = prov[::10].tolist()
    for a in res["arms"].values():
        print(json.dumps(a))
    os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    with open(out_path.replace(".json", "_series.json"), "w") as f:
        json.dump(series, f)


if __name__ == "__main__":
    main()
