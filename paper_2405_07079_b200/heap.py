"""Python binding with the C-ABI's names (include/heap.h) plus a small ``Heap`` wrapper.

PyTorch only provides device memory (the workspace tensor, request/result tensors)
and streams.  Offsets and sizes are passed as int64 tensors whose bits are read as
uint64 by the library (HEAP_NULL = -1 as int64).
"""
from __future__ import annotations

import ctypes

import torch

from . import _native
from ._native import HeapStats, check, lib

HEAP_FIRST_FIT, HEAP_BEST_FIT, HEAP_SEGFIT, HEAP_TLSF, HEAP_BUDDY, HEAP_SEGFIT_LIFO, HEAP_HYBRID = 1, 2, 3, 4, 5, 6, 7
HEAP_NEXT_FIT, HEAP_DOUBLE_BUDDY, HEAP_FIB_BUDDY = 8, 9, 10
HEAP_PARTIAL_FREE = 0x100   # policy flag: partial (tail) deallocation (include/heap.h)
HEAP_NULL = (1 << 64) - 1
HEAP_NULL_I64 = -1
POLICY_NAMES = {1: "first_fit", 2: "best_fit", 3: "segfit", 4: "tlsf", 5: "buddy", 6: "segfit_lifo", 7: "hybrid", 8: "next_fit", 9: "double_buddy",
                10: "fib_buddy"}


def _stream_handle(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _dev_ptr(t: torch.Tensor, name: str) -> int:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype not in (torch.int64, torch.uint64) or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous int64/uint64 tensor")
    return t.data_ptr()


# ---- same names as the C ABI ----
def heap_workspace_bytes(arena_bytes: int, align: int, policy: int, max_live_blocks: int,
                         max_batch: int) -> int:
    return int(lib().heap_workspace_bytes(arena_bytes, align, policy, max_live_blocks, max_batch))


def heap_create(arena_bytes: int, align: int, policy: int, max_live_blocks: int, max_batch: int,
                workspace: torch.Tensor, stream=None) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    check("heap_create", lib().heap_create(arena_bytes, align, policy, max_live_blocks, max_batch,
                                           workspace.data_ptr(), workspace.numel() * workspace.element_size(),
                                           _stream_handle(stream), ctypes.byref(h)))
    return h


def heap_destroy(h) -> None:
    check("heap_destroy", lib().heap_destroy(h))


def heap_free_batch(h, offsets: torch.Tensor, stream=None) -> None:
    n = offsets.numel()
    check("heap_free_batch", lib().heap_free_batch(h, _dev_ptr(offsets, "offsets") if n else None, n,
                                                   _stream_handle(stream)))


def heap_free_batch_handles(h, table: torch.Tensor, idx: torch.Tensor, stream=None) -> None:
    n = idx.numel()
    check("heap_free_batch_handles",
          lib().heap_free_batch_handles(h, _dev_ptr(table, "table") if n else None, table.numel(),
                                        _dev_ptr(idx, "idx") if n else None, n, _stream_handle(stream)))


def heap_step(h, offsets: torch.Tensor, idx: torch.Tensor | None, sizes: torch.Tensor, out_offsets: torch.Tensor,
              stream=None) -> None:
    nf = idx.numel() if idx is not None else offsets.numel()
    na = sizes.numel()
    if out_offsets.numel() < na:
        raise ValueError("out_offsets too small")
    check("heap_step", lib().heap_step(
        h, _dev_ptr(offsets, "offsets") if nf else None, _dev_ptr(idx, "idx") if (idx is not None and nf) else None,
        offsets.numel(), nf, _dev_ptr(sizes, "sizes") if na else None,
        _dev_ptr(out_offsets, "out_offsets") if na else None, na, _stream_handle(stream)))


def heap_alloc_batch(h, sizes: torch.Tensor, out_offsets: torch.Tensor, stream=None) -> None:
    n = sizes.numel()
    if out_offsets.numel() < n:
        raise ValueError("out_offsets too small")
    check("heap_alloc_batch", lib().heap_alloc_batch(
        h, _dev_ptr(sizes, "sizes") if n else None, _dev_ptr(out_offsets, "out_offsets") if n else None,
        n, _stream_handle(stream)))


def heap_stats_async(h, d_out: torch.Tensor, stream=None) -> None:
    """Write the 16 x u64 statistics into a CUDA int64/uint64 tensor of 16 elements."""
    check("heap_stats_async", lib().heap_stats_async(h, _dev_ptr(d_out, "d_out"), _stream_handle(stream)))


def heap_stats_allgather(h, comm: int, d_all: torch.Tensor, stream=None) -> None:
    """NCCL all-gather of every rank's 128-byte statistics into d_all (CUDA int64, nranks x 16)."""
    check("heap_stats_allgather", lib().heap_stats_allgather(h, ctypes.c_void_p(comm), _dev_ptr(d_all, "d_all"),
                                                             _stream_handle(stream)))


def nccl_unique_id() -> bytes:
    """128 opaque bytes identifying a new NCCL communicator (create on one rank, share)."""
    buf = ctypes.create_string_buffer(128)
    check("heap_nccl_unique_id", lib().heap_nccl_unique_id(buf))
    return buf.raw


def nccl_comm_init(nranks: int, uid: bytes, rank: int) -> int:
    """This rank's NCCL communicator (on the current CUDA device); returns the handle."""
    comm = ctypes.c_void_p()
    check("heap_nccl_comm_init", lib().heap_nccl_comm_init(ctypes.byref(comm), nranks, uid, rank))
    return int(comm.value)


def nccl_comm_init_all(devices) -> list:
    """One communicator per device of this process (single-process multi-GPU)."""
    n = len(devices)
    comms = (ctypes.c_void_p * n)()
    devs = (ctypes.c_int * n)(*devices)
    check("heap_nccl_comm_init_all", lib().heap_nccl_comm_init_all(comms, n, devs))
    return [int(c) for c in comms]


def nccl_comm_destroy(comm: int) -> None:
    check("heap_nccl_comm_destroy", lib().heap_nccl_comm_destroy(ctypes.c_void_p(comm)))


def heap_stats(h, stream=None) -> dict:
    st = HeapStats()
    rc = lib().heap_stats(h, ctypes.byref(st), _stream_handle(stream))
    d = st.as_dict()
    d["rc"] = rc
    return d


def heap_export(h, stream=None):
    """Returns (free_pairs, live_pairs) as CPU int64 tensors [n, 2] of (start, size) bytes."""
    counts = (ctypes.c_uint64 * 2)()
    check("heap_export", lib().heap_export(h, None, 0, None, 0, counts, _stream_handle(stream)))
    nf, nl = int(counts[0]), int(counts[1])
    dev = torch.device("cuda", torch.cuda.current_device())
    fp = torch.empty((max(nf, 1), 2), dtype=torch.int64, device=dev)
    lp = torch.empty((max(nl, 1), 2), dtype=torch.int64, device=dev)
    check("heap_export", lib().heap_export(h, fp.data_ptr(), nf, lp.data_ptr(), nl, counts,
                                           _stream_handle(stream)))
    return fp[:nf].cpu(), lp[:nl].cpu()


def heap_launch_count(h) -> int:
    return int(lib().heap_launch_count(h))


def heap_set_graphs(h, enable: bool) -> None:
    check("heap_set_graphs", lib().heap_set_graphs(h, 1 if enable else 0))


def heap_profile_enable(h, tag_mask: int) -> None:
    check("heap_profile_enable", lib().heap_profile_enable(h, tag_mask))


def heap_profile_read(h) -> dict:
    """{tag_name: (milliseconds, launches)} accumulated since the last read (synchronises)."""
    ms = (ctypes.c_double * _native.NTAGS)()
    cnt = (ctypes.c_uint64 * _native.NTAGS)()
    check("heap_profile_read", lib().heap_profile_read(h, ms, cnt))
    return {heap_tag_name(t): (ms[t], int(cnt[t])) for t in range(_native.NTAGS) if cnt[t]}


def heap_tag_name(tag: int) -> str:
    return lib().heap_tag_name(tag).decode()


def heap_strerror(code: int) -> str:
    return lib().heap_strerror(code).decode()


class Heap:
    """Owns the workspace tensor and the handle; every call enqueues on ``stream``."""

    def __init__(self, arena_bytes: int, align: int, policy: int, max_live_blocks: int,
                 max_batch: int, device=None, stream=None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2405_07079_b200.Heap needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device if device is not None else "cuda")
        self.arena_bytes, self.align, self.policy = arena_bytes, align, policy
        self.max_live, self.max_batch = max_live_blocks, max_batch
        self.stream = stream
        nbytes = heap_workspace_bytes(arena_bytes, align, policy, max_live_blocks, max_batch)
        if nbytes == 0:
            raise ValueError("invalid heap arguments")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        # heap_create reads the current device (SM count, kernel attributes): make it ours
        with torch.cuda.device(self.device):
            self._h = heap_create(arena_bytes, align, policy, max_live_blocks, max_batch, self.workspace,
                                  self._stream())
        self._out = torch.empty(max_batch, dtype=torch.int64, device=self.device)

    def _stream(self):
        return self.stream if self.stream is not None else torch.cuda.current_stream(self.device)

    def close(self):
        if getattr(self, "_h", None):
            torch.cuda.synchronize(self.device)
            heap_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def free_batch(self, offsets: torch.Tensor) -> None:
        with torch.cuda.device(self.device):
            heap_free_batch(self._h, offsets, self._stream())

    def free_batch_handles(self, table: torch.Tensor, idx: torch.Tensor) -> None:
        """Free the offsets table[idx[i]] (int64 tensors; an index >= table.numel() frees nothing):
        a caller keeping its blocks in a handle table frees them without a separate gather."""
        with torch.cuda.device(self.device):
            heap_free_batch_handles(self._h, table, idx, self._stream())

    def step(self, offsets: torch.Tensor, sizes: torch.Tensor, idx: torch.Tensor | None = None,
             out: torch.Tensor | None = None) -> torch.Tensor:
        """One canonical batch: free `offsets` (or, with `idx`, the handles offsets[idx]), then
        allocate `sizes`; returns the offsets as alloc_batch does (`out` may be a slice of the
        handle table)."""
        n = sizes.numel()
        with torch.cuda.device(self.device):
            dst = self._out[:n] if out is None else out[:n]
            heap_step(self._h, offsets, idx, sizes, dst, self._stream())
            return dst.clone() if out is None else dst

    def alloc_batch(self, sizes: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Serve a batch of sizes (bytes) in request order; returns the offsets (HEAP_NULL as -1).

        Without ``out`` the result is a fresh tensor the caller owns.  With ``out`` (int64, at least
        ``sizes.numel()`` elements) the offsets are written there and ``out[:n]`` is returned: the
        zero-copy path for callers that manage their own result buffers."""
        n = sizes.numel()
        with torch.cuda.device(self.device):
            if out is None:
                heap_alloc_batch(self._h, sizes, self._out[:n], self._stream())
                return self._out[:n].clone()
            heap_alloc_batch(self._h, sizes, out[:n], self._stream())
            return out[:n]

    def stats(self) -> dict:
        with torch.cuda.device(self.device):
            return heap_stats(self._h, self._stream())

    def export(self):
        with torch.cuda.device(self.device):
            return heap_export(self._h, self._stream())

    def stats_allgather(self, comm: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """Every rank's statistics (int64 [nranks, 16], heap_stats_t field order) through NCCL;
        collective over comm, asynchronous on the heap's stream."""
        with torch.cuda.device(self.device):
            if out is None:
                raise ValueError("pass out = torch.empty((nranks, 16), dtype=torch.int64, device=heap.device)")
            heap_stats_allgather(self._h, comm, out, self._stream())
            return out

    def launch_count(self) -> int:
        return heap_launch_count(self._h)

    def set_graphs(self, enable: bool) -> None:
        heap_set_graphs(self._h, enable)

    def profile(self, tag_mask: int) -> None:
        heap_profile_enable(self._h, tag_mask)

    def profile_read(self) -> dict:
        return heap_profile_read(self._h)

    def debug_counters(self) -> list:
        out = (ctypes.c_uint64 * 32)()
        with torch.cuda.device(self.device):
            check("heap_debug_counters", lib().heap_debug_counters(self._h, out, 32, _stream_handle(self._stream())))
        return [int(x) for x in out]
