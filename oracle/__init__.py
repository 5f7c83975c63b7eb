"""Oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product
package ``paper_2405_07079_b200`` never imports, links or executes it, and the
two share no code.

* ``OracleL`` — ctypes wrapper over ``oracle_l.cpp`` (plain single-threaded C++
  with std::map/std::set; every function cites its PAPER.md passage).
* ``oracle_b`` — structurally different brute-force allocator over a unit
  bitmap (pure Python/numpy; tiny heaps and config 1).

Parity status of each function is listed in DESIGN.md §5 ("pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_l.cpp")
_LIB = os.path.join(_HERE, "liboracle_l.so")

HEAP_NULL = (1 << 64) - 1
STATS_FIELDS = ("arena_bytes", "align", "live_bytes", "free_bytes", "n_live", "n_free",
                "largest_free", "high_water_end", "allocs_ok", "allocs_failed", "frees_ok",
                "frees_invalid", "frees_double", "frees_null", "metadata_bytes", "error_flags")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u64, vp = ctypes.c_uint64, ctypes.c_void_p
        L.oracle_create.restype = vp
        L.oracle_create.argtypes = [u64, u64, ctypes.c_int]
        L.oracle_destroy.argtypes = [vp]
        L.oracle_free_batch.argtypes = [vp, vp, u64]
        L.oracle_alloc_batch.argtypes = [vp, vp, u64, vp]
        L.oracle_stats.argtypes = [vp, vp]
        L.oracle_export.argtypes = [vp, vp, u64, vp, u64, vp]
        L.oracle_insert_class.restype = u64
        L.oracle_insert_class.argtypes = [u64, ctypes.c_int]
        L.oracle_search_class.restype = u64
        L.oracle_search_class.argtypes = [u64, ctypes.c_int]
        _lib = L
    return _lib


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


class OracleL:
    """Oracle-L heap: ``free_batch(offsets)``, ``alloc_batch(sizes) -> offsets``."""

    def __init__(self, arena_bytes: int, align: int, policy: int):
        self._h = lib().oracle_create(arena_bytes, align, policy)
        if not self._h:
            raise ValueError("oracle_create: invalid arguments")
        self.arena_bytes, self.align, self.policy = arena_bytes, align, policy

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().oracle_destroy(h)
            self._h = None

    def free_batch(self, offsets) -> None:
        a = _u64(offsets)
        lib().oracle_free_batch(self._h, a.ctypes.data, a.size)

    def alloc_batch(self, sizes) -> np.ndarray:
        a = _u64(sizes)
        out = np.empty(a.size, dtype=np.uint64)
        lib().oracle_alloc_batch(self._h, a.ctypes.data, a.size, out.ctypes.data)
        return out

    def stats(self) -> dict:
        o = np.zeros(16, dtype=np.uint64)
        lib().oracle_stats(self._h, o.ctypes.data)
        return {k: int(v) for k, v in zip(STATS_FIELDS, o)}

    def export(self):
        """(free_pairs[nf,2], live_pairs[nl,2]) in bytes, sorted by start."""
        counts = np.zeros(2, dtype=np.uint64)
        lib().oracle_export(self._h, None, 0, None, 0, counts.ctypes.data)
        nf, nl = int(counts[0]), int(counts[1])
        fp = np.zeros((max(nf, 1), 2), dtype=np.uint64)
        lp = np.zeros((max(nl, 1), 2), dtype=np.uint64)
        lib().oracle_export(self._h, fp.ctypes.data, nf, lp.ctypes.data, nl, counts.ctypes.data)
        return fp[:nf], lp[:nl]


def insert_class(u: int, L: int) -> int:
    return int(lib().oracle_insert_class(u, L))


def search_class(u: int, L: int) -> int:
    return int(lib().oracle_search_class(u, L))
