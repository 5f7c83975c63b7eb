"""Thin ctypes binding over libheap.so (include/heap.h).  Argument marshalling only.

Every step of a batch runs in the library's sm_100a kernels; this module never
computes allocator results itself and has no CPU fallback: if ``libheap.so`` is
missing or no CUDA device is present, it raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
LIB_PATH = os.path.join(_HERE, os.environ.get("HEAP_DEV_LIB", "libheap.so"))  # dev override: debug build
SRC_DIR = os.path.join(_HERE, "csrc")
HEADER = os.path.join(ROOT, "include", "heap.h")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def nccl_dirs():
    """The image's NCCL (2.28, the copy torch loads): include and lib directories."""
    import nvidia.nccl
    base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) \
        else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return [os.path.join(SRC_DIR, f) for f in sorted(os.listdir(SRC_DIR))
            if f.endswith((".cu", ".cuh"))] + [HEADER]


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libheap.so for sm_100a (nvcc cross-compiles; no GPU needed)."""
    newest = max(os.path.getmtime(p) for p in sources())
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    inc, libdir = nccl_dirs()
    cmd = ["nvcc", *NVCC_FLAGS, "-I", inc, "-o", LIB_PATH + ".tmp", os.path.join(SRC_DIR, "heap.cu"),
           "-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath," + libdir]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


class HeapStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "arena_bytes", "align", "live_bytes", "free_bytes", "n_live", "n_free", "largest_free",
        "high_water_end", "allocs_ok", "allocs_failed", "frees_ok", "frees_invalid",
        "frees_double", "frees_null", "metadata_bytes", "error_flags")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


EXPORTS = ("heap_workspace_bytes", "heap_create", "heap_destroy", "heap_free_batch", "heap_free_batch_handles", "heap_step",
           "heap_alloc_batch", "heap_stats_async", "heap_stats", "heap_export",
           "heap_launch_count", "heap_set_graphs", "heap_profile_enable", "heap_profile_read", "heap_tag_name",
           "heap_debug_counters", "heap_stats_allgather", "heap_nccl_unique_id", "heap_nccl_comm_init",
           "heap_nccl_comm_init_all", "heap_nccl_comm_destroy", "heap_strerror")
NTAGS = 16

_lib = None


def lib():
    """Load libheap.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        u64, vp, i32 = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        L.heap_workspace_bytes.restype = ctypes.c_size_t
        L.heap_workspace_bytes.argtypes = [u64, u64, i32, u64, u64]
        L.heap_create.restype = i32
        L.heap_create.argtypes = [u64, u64, i32, u64, u64, vp, ctypes.c_size_t, vp, ctypes.POINTER(vp)]
        L.heap_destroy.restype = i32
        L.heap_destroy.argtypes = [vp]
        L.heap_free_batch.restype = i32
        L.heap_free_batch.argtypes = [vp, vp, u64, vp]
        L.heap_free_batch_handles.restype = i32
        L.heap_free_batch_handles.argtypes = [vp, vp, u64, vp, u64, vp]
        L.heap_step.restype = i32
        L.heap_step.argtypes = [vp, vp, vp, u64, u64, vp, vp, u64, vp]
        L.heap_alloc_batch.restype = i32
        L.heap_alloc_batch.argtypes = [vp, vp, vp, u64, vp]
        L.heap_stats_async.restype = i32
        L.heap_stats_async.argtypes = [vp, vp, vp]
        L.heap_stats.restype = i32
        L.heap_stats.argtypes = [vp, ctypes.POINTER(HeapStats), vp]
        L.heap_export.restype = i32
        L.heap_export.argtypes = [vp, vp, u64, vp, u64, ctypes.POINTER(u64), vp]
        L.heap_launch_count.restype = u64
        L.heap_launch_count.argtypes = [vp]
        L.heap_set_graphs.restype = i32
        L.heap_set_graphs.argtypes = [vp, i32]
        L.heap_profile_enable.restype = i32
        L.heap_profile_enable.argtypes = [vp, u64]
        L.heap_profile_read.restype = i32
        L.heap_profile_read.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(u64)]
        L.heap_debug_counters.restype = i32
        L.heap_debug_counters.argtypes = [vp, ctypes.POINTER(u64), i32, vp]
        L.heap_tag_name.restype = ctypes.c_char_p
        L.heap_tag_name.argtypes = [i32]
        L.heap_strerror.restype = ctypes.c_char_p
        L.heap_strerror.argtypes = [i32]
        L.heap_stats_allgather.restype = i32
        L.heap_stats_allgather.argtypes = [vp, vp, vp, vp]
        L.heap_nccl_unique_id.restype = i32
        L.heap_nccl_unique_id.argtypes = [ctypes.c_char_p]
        L.heap_nccl_comm_init.restype = i32
        L.heap_nccl_comm_init.argtypes = [ctypes.POINTER(vp), i32, ctypes.c_char_p, i32]
        L.heap_nccl_comm_init_all.restype = i32
        L.heap_nccl_comm_init_all.argtypes = [ctypes.POINTER(vp), i32, ctypes.POINTER(i32)]
        L.heap_nccl_comm_destroy.restype = i32
        L.heap_nccl_comm_destroy.argtypes = [vp]
        _lib = L
    return _lib


class HeapError(RuntimeError):
    def __init__(self, fn: str, code: int):
        super().__init__(f"{fn} failed: {code} ({lib().heap_strerror(code).decode()})")
        self.code = code


def check(fn: str, code: int) -> int:
    if code != 0:
        raise HeapError(fn, code)
    return code
