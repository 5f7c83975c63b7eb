"""Seeded synthetic malloc/free traces shared by the oracle side and the CUDA side.

This module is the ONLY code both sides use.  It draws request
sizes and which live ids are freed; it contains none of the allocator's
arithmetic.  The workload recipe is SURVEY.md §8(d) / DESIGN.md §4:

* PRNG: SplitMix64 seeding xoshiro256**, ``seed(c, r) = 2405070790 + 1000 c + r``.
* sizes ``LU8[2^a, 2^b)`` (octave-uniform) or buddy orders with weights
  ``2^floor((b-k)/2)``; the paper's own workload is "blocks 1kB and 16MB in size"
  allocated and freed "randomly ... several thousand times".
* batch model (configs 2-5) and slot model (config 1, SPEC.md:497-505 shape).

Ids are abstract: the j-th alloc request of the trace has id j whether or not it
succeeds; a failed alloc's id maps to HEAP_NULL, so its later free is a null
no-op and the trace stays allocator-independent.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tracegen.c")
_LIB = os.path.join(_HERE, "libtracegen.so")

HEAP_NULL = (1 << 64) - 1

# policy ids (numbers only; the meaning lives in include/heap.h and oracle/)
FIRST_FIT, BEST_FIT, SEGFIT, TLSF, BUDDY, SEGFIT_LIFO, HYBRID, NEXT_FIT, DOUBLE_BUDDY, FIB_BUDDY = range(1, 11)
POLICY_NAME = {1: "first_fit", 2: "best_fit", 3: "segfit", 4: "tlsf", 5: "buddy", 6: "segfit_lifo", 7: "hybrid", 8: "next_fit", 9: "double_buddy",
               10: "fib_buddy"}


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config (index = position in ``configs``)."""
    idx: int
    name: str
    policy: int
    arena_bytes: int
    align: int
    model: int          # 0 batch model, 1 slot model
    batch: int          # B
    rho_num: int
    rho_den: int
    total_ops: int
    size_kind: int      # 0 LU8, 1 buddy orders
    a: int
    b: int
    n_slots: int = 0
    max_live: int = 0   # metadata capacity the bench/tests provision

    def seed(self, rank: int = 0) -> int:
        return 2405070790 + 1000 * self.idx + rank


# BASELINE.json "configs" (0-based here; SURVEY.md §8(d) numbers them 1..5)
CONFIGS = {
    1: Config(1, "cfg1-firstfit-1MiB", FIRST_FIT, 1 << 20, 16, 1, 0, 1, 2, 1000, 0, 4, 12,
              n_slots=1000, max_live=1 << 12),
    2: Config(2, "cfg2-bestfit-256MiB", BEST_FIT, 256 << 20, 16, 0, 4096, 1, 2, 10**6, 0, 4, 20,
              max_live=1 << 14),
    3: Config(3, "cfg3-tlsf-4GiB", TLSF, 4 << 30, 16, 0, 65536, 2, 5, 10**7, 0, 4, 12,
              max_live=3 << 20),
    4: Config(4, "cfg4-buddy-16GiB", BUDDY, 1 << 34, 256, 0, 65536, 1, 2, 10**7, 1, 8, 24,
              max_live=1 << 18),
    5: Config(5, "cfg5-tlsf-64GiB", TLSF, 1 << 36, 16, 0, 1 << 20, 2, 5, 10**8, 0, 4, 12,
              max_live=24 << 20),
}


def _build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(_build())
        u64 = ctypes.c_uint64
        L.tg_create.restype = ctypes.c_void_p
        L.tg_create.argtypes = [ctypes.c_int, u64, u64, u64, u64, u64, ctypes.c_int, u64, u64, u64]
        L.tg_destroy.argtypes = [ctypes.c_void_p]
        L.tg_next_batch.restype = ctypes.c_int
        L.tg_next_batch.argtypes = [ctypes.c_void_p, u64, ctypes.c_void_p, ctypes.POINTER(u64),
                                    ctypes.c_void_p, ctypes.POINTER(u64), ctypes.POINTER(u64)]
        L.tg_n_live.restype = u64
        L.tg_n_live.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


class Trace:
    """Iterator over canonical batches ``(free_ids, sizes, first_alloc_id)``.

    ``free_ids`` are uint64 ids of earlier allocs (in draw order; the canonical
    free order is by address and is the allocator's business), ``sizes`` are raw
    byte sizes (uint64) in request order; alloc ids are ``first_alloc_id + j``.
    """

    def __init__(self, cfg: Config, rank: int = 0, total_ops: int | None = None,
                 batch: int | None = None):
        self.cfg = cfg
        self.batch = batch if batch is not None else cfg.batch
        ops = cfg.total_ops if total_ops is None else total_ops
        if cfg.model == 0:
            self.max_n = max(self.batch, 1)
        else:   # slot model: `batch` caps a batch's ops (2 = one step per batch)
            self.max_n = max(batch, 1) if batch is not None else max(ops, 1)
        L = lib()
        self._h = L.tg_create(cfg.model, cfg.seed(rank), self.batch, cfg.rho_num, cfg.rho_den,
                              ops, cfg.size_kind, cfg.a, cfg.b, cfg.n_slots)
        self._fids = np.zeros(self.max_n, dtype=np.uint64)
        self._sizes = np.zeros(self.max_n, dtype=np.uint64)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().tg_destroy(h)
            self._h = None

    def next_batch(self):
        nf = ctypes.c_uint64(0)
        na = ctypes.c_uint64(0)
        first = ctypes.c_uint64(0)
        ok = lib().tg_next_batch(self._h, self.max_n, self._fids.ctypes.data, ctypes.byref(nf),
                                 self._sizes.ctypes.data, ctypes.byref(na), ctypes.byref(first))
        if not ok:
            return None
        return (self._fids[: nf.value].copy(), self._sizes[: na.value].copy(), first.value)

    def __iter__(self):
        while True:
            b = self.next_batch()
            if b is None:
                return
            yield b

    def n_live(self) -> int:
        return int(lib().tg_n_live(self._h))


def custom(policy: int, arena_bytes: int, align: int, batch: int, rho=(1, 2), total_ops=1000,
           sizes=(4, 12), size_kind=0, model=0, n_slots=0, idx=90, max_live=1 << 12) -> Config:
    """A small ad-hoc config for parity tests (same generator, other shapes)."""
    return Config(idx, f"custom-{idx}", policy, arena_bytes, align, model, batch, rho[0], rho[1],
                  total_ops, size_kind, sizes[0], sizes[1], n_slots=n_slots, max_live=max_live)
