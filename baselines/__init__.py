"""Driver-allocator baselines (the paper's comparison) for bench.py.

Not part of the product path.  ``replay(mode, batches)`` replays the same per-batch op order
with cudaMalloc/cudaFree (mode 0) or cudaMallocAsync/cudaFreeAsync (mode 1)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cudamalloc_replay.cu")
_LIB = os.path.join(_HERE, "libcudamalloc_replay.so")


def build(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["nvcc", "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared",
                               "-cudart", "shared", "-o", _LIB, _SRC])
    return _LIB


def replay(mode, batches, max_ops=10**6, max_seconds=60.0):
    """batches: list of (free_ids, sizes, first_alloc_id) from tracegen.  Returns dict."""
    L = ctypes.CDLL(build())
    u64p = ctypes.POINTER(ctypes.c_uint64)
    fo = np.zeros(len(batches) + 1, dtype=np.uint64)
    ao = np.zeros(len(batches) + 1, dtype=np.uint64)
    for i, (f, s, first) in enumerate(batches):
        fo[i + 1] = fo[i] + len(f)
        ao[i + 1] = ao[i] + len(s)
        assert first == ao[i]
    fids = np.ascontiguousarray(np.concatenate([b[0] for b in batches]).astype(np.uint64))
    sizes = np.ascontiguousarray(np.concatenate([b[1] for b in batches]).astype(np.uint64))
    ops, fail = ctypes.c_uint64(0), ctypes.c_uint64(0)
    sec = ctypes.c_double(0)
    L.replay.restype = ctypes.c_int
    rc = L.replay(mode, len(batches), fo.ctypes.data_as(u64p), fids.ctypes.data_as(u64p),
                  ao.ctypes.data_as(u64p), sizes.ctypes.data_as(u64p), ctypes.c_uint64(max_ops),
                  ctypes.c_double(max_seconds), ctypes.byref(ops), ctypes.byref(sec), ctypes.byref(fail))
    if rc != 0:
        return {"error": f"replay rc {rc}"}
    return {"value": ops.value / sec.value if sec.value else None, "unit": "ops/s", "ops": ops.value,
            "seconds": sec.value, "failed": fail.value,
            "capped": bool(ops.value < int(ao[-1] + fo[-1]))}


def replay_latency(mode, kind, arg):
    """Per-op host latency (ns) and process device-memory use after each op for the
    batch-size-1 study.  kind: uint8 [n] (0 free id / 1 alloc bytes), arg: uint64 [n]."""
    L = ctypes.CDLL(build())
    kind = np.ascontiguousarray(kind, dtype=np.uint8)
    arg = np.ascontiguousarray(arg, dtype=np.uint64)
    n = len(kind)
    lat = np.zeros(n, dtype=np.float64)
    used = np.zeros(n, dtype=np.uint64)
    fail = ctypes.c_uint64(0)
    L.replay_latency.restype = ctypes.c_int
    rc = L.replay_latency(mode, ctypes.c_uint64(n), kind.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                          arg.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                          lat.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                          used.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), ctypes.byref(fail))
    if rc != 0:
        raise RuntimeError(f"replay_latency rc {rc}")
    return lat, used, int(fail.value)
