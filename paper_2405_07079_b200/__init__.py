"""paper_2405_07079_b200 — a B200-native batched device heap with out-of-band metadata.

arXiv 2405.07079 ("Host-Based Allocators for Device Memory") poses an allocator that may
never read the memory it manages.  This package services whole
batches of malloc/free requests against such a heap with sm_100a kernels behind the C ABI
in include/heap.h; the Python layer only marshals arguments.
"""
from .heap import (HEAP_BEST_FIT, HEAP_BUDDY, HEAP_FIRST_FIT, HEAP_NULL, HEAP_NULL_I64, HEAP_SEGFIT,
                   HEAP_SEGFIT_LIFO, HEAP_HYBRID, HEAP_NEXT_FIT, HEAP_DOUBLE_BUDDY, HEAP_FIB_BUDDY, HEAP_PARTIAL_FREE,
                   HEAP_TLSF, POLICY_NAMES, Heap, heap_alloc_batch, heap_create, heap_destroy,
                   heap_export, heap_free_batch, heap_free_batch_handles, heap_step, heap_launch_count, heap_profile_enable, heap_set_graphs,
                   heap_profile_read, heap_tag_name, heap_stats, heap_stats_async,
                   heap_strerror, heap_workspace_bytes, heap_stats_allgather, nccl_unique_id, nccl_comm_init,
                   nccl_comm_init_all, nccl_comm_destroy)

__all__ = ["Heap", "heap_workspace_bytes", "heap_create", "heap_destroy", "heap_free_batch", "heap_free_batch_handles", "heap_step",
           "heap_alloc_batch", "heap_stats_async", "heap_stats", "heap_export", "heap_launch_count", "heap_set_graphs",
           "heap_strerror", "heap_stats_allgather", "nccl_unique_id", "nccl_comm_init", "nccl_comm_init_all",
           "nccl_comm_destroy", "heap_profile_enable", "heap_profile_read", "heap_tag_name", "HEAP_FIRST_FIT", "HEAP_BEST_FIT", "HEAP_SEGFIT", "HEAP_TLSF", "HEAP_BUDDY", "HEAP_SEGFIT_LIFO", "HEAP_HYBRID", "HEAP_NEXT_FIT", "HEAP_DOUBLE_BUDDY",
           "HEAP_PARTIAL_FREE", "HEAP_FIB_BUDDY",
           "HEAP_NULL", "HEAP_NULL_I64", "POLICY_NAMES"]
