/*
 * heap.h — C ABI of libheap: a batched, device-resident heap whose metadata lives out of
 * band (arXiv 2405.07079, "Host-Based Allocators for Device Memory").
 *
 * The problem statement: an allocator manages an arena it may never
 * read, so no boundary tags; all block metadata lives elsewhere.  Here
 * the arena is any device range the caller owns (e.g. a torch tensor); the library returns
 * byte OFFSETS into it and never dereferences the arena.  The metadata (block table, free
 * arrays, class indices) lives in a caller-provided device WORKSPACE and is maintained by
 * sm_100a kernels, one batch of requests per call.
 *
 * Semantics of a batch (BASELINE.json north_star):
 *   heap_free_batch  - every offset is classified against the batch-start state; the valid
 *                      live block starts are freed as if one by one in ascending address
 *                      order, each coalescing with its free neighbours (Alg. 2 PAPER.md:214-236,
 *                      Alg. 5; buddy merge PAPER.md:118).
 *   heap_alloc_batch - requests are served as if one by one in request order under the
 *                      policy (first/best fit PAPER.md:87-88, Alg. 3 :298-317; segregated fit
 *                      Alg. 4 :327-369 with the bitmap/ffs fallback :440; TLSF :444-458; binary
 *                      buddy :111-125); each choice splits the block from its low end (Alg. 1
 *                      :173-184).  Results are bit-exact with the CPU oracle (oracle/).
 *
 * Conventions
 *   - Every pointer argument is DEVICE memory unless its name starts with h_.
 *   - Calls are asynchronous and ordered on the given stream (cudaStream_t; 0 = legacy
 *     default stream).  Request arrays must stay valid until the stream passes the call.
 *     One heap must be used from one stream at a time; there is no internal locking.
 *   - Per-request failures are data, not return codes: a failed alloc (size 0, larger
 *     than the arena, or no candidate block) yields HEAP_NULL and changes nothing; a free
 *     of HEAP_NULL is a no-op; a free of anything that is not a live block start is
 *     skipped and counted (frees_invalid / frees_double).  Partial (interior) frees are
 *     opt-in per heap with the HEAP_PARTIAL_FREE policy flag (below); without it an interior
 *     offset is invalid (C6).
 *   - Metadata capacity overflow inside a batch (more live blocks than max_live_blocks)
 *     cannot be reported synchronously: it sets error_flags and the next heap_stats()
 *     returns HEAP_ECAPACITY.  The heap state after such a batch is unspecified.
 *   - Units: sizes are rounded up to a multiple of align; arena_bytes / align must be
 *     <= 2^32 (C20).
 */
#ifndef LIBHEAP_HEAP_H
#define LIBHEAP_HEAP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct heap heap_t;
/* ABI-compatible with cudaStream_t; declared opaquely so this header needs no CUDA headers */
typedef struct CUstream_st *heap_stream_t;
/* NCCL communicator handle, declared exactly as nccl.h does (so either header may come first) */
typedef struct ncclComm *ncclComm_t;

/* policies: which free block an alloc takes (lowest key wins; DESIGN.md §2 table) */
enum heap_policy {
    HEAP_FIRST_FIT = 1, /* lowest-address block with size >= r */
    HEAP_BEST_FIT = 2,  /* min (size, address) over size >= r             PAPER.md:87, Alg. 3 */
    HEAP_SEGFIT = 3,    /* power-of-two bins, request bin = ceil(log2 r),
                           block bin = floor(log2 size), address order    Alg. 4/5 */
    HEAP_TLSF = 4,      /* two-level bins (32 linear sub-bins per power
                           of two), min (bin, address) over bin >= search PAPER.md:447-458 */
    HEAP_BUDDY = 5,     /* binary buddy, min order then address; align is
                           the minimum block */
    HEAP_SEGFIT_LIFO = 6, /* the paper's segregated fit verbatim: power-of-two
                           bins as stacks — an alloc pops the head (most recent
                           push) of the first nonempty bin >= ceil(log2 r); frees
                           and split remainders are pushed at the head      Alg. 4/5 */
    HEAP_HYBRID = 7,    /* §5.3 hybrid: requests of 0 < s < 4096 B
                           take the LOWEST free slot of a bitmask object pool
                           (§3.2) of align*2^j-byte objects, the
                           smallest that holds s; a full pool and every other
                           request use a TLSF heap.  Layout (C26): the
                           pools share the first half of the arena evenly, each a
                           whole number of 4 KiB pages; the TLSF heap covers the rest.
                           A pool offset frees iff it is an allocated slot start.
                           heap_stats: n_free counts maximal runs of free pool slots
                           plus TLSF free blocks; largest_free is the TLSF heap's.
                           heap_export lists pool runs / objects, then TLSF blocks.
                           max_live_blocks bounds the TLSF heap's live blocks only. */
    HEAP_NEXT_FIT = 8,  /* first fit resumed at a rover: the first
                           block with start >= rover and size >= r, else the first
                           from address 0; the rover is the end of the last
                           allocation; frees leave it alone (C27) */
    HEAP_DOUBLE_BUDDY = 9, /* double buddies: a binary buddy heap of
                           align-sized units on [0, A) and one of 3*align-sized units
                           (blocks 3*2^k*align) on [A, arena) holding
                           floor(arena / 6 align) units; a request of r units goes to
                           the heap with the smaller class, 2^ceil(log2 r) or
                           3*2^ceil(log2 ceil(r/3)) units, with no fallback
                           (C28).  Offsets past A must be whole 3-units.
                           max_live_blocks bounds each heap's live blocks. */
    HEAP_FIB_BUDDY = 10 /* Fibonacci buddies: block sizes 1, 2, 3, 5,
                           8, ... units (S_k = S_{k-1} + S_{k-2}); a block splits into
                           its low part of the previous size and its high part of the
                           size before (2 = 1 + 1); the arena is the greedy
                           (Zeckendorf) sum of Fibonacci roots.  A request of r units
                           takes the smallest nonempty class whose size is >= r,
                           lowest address, split keeping the low part; a free merges
                           a block with its split-tree sibling while that is free
                           (C30).  Per alloc batch at most 1024 split
                           leftovers of one class may be created (else
                           HEAP_ECAPACITY). */
};

/* Policy flag (OR into policy): partial (tail) deallocation, "freeing the last 2kB of a 10kB
 * block ... the in-use block will be shrunk" (Alg. 2 :205-212 searches the used
 * list for the block CONTAINING the address).  Valid with HEAP_FIRST_FIT, HEAP_BEST_FIT,
 * HEAP_SEGFIT, HEAP_TLSF and HEAP_NEXT_FIT (heap_create returns HEAP_EINVAL otherwise).  In a
 * free batch an offset inside a live block frees from that offset to the block's end (the
 * whole block when it is the start); per live block of the batch-start state the LOWEST such
 * offset of the batch frees and every other offset inside the block (copies included) counts
 * as frees_double; an offset in free memory that is not a free block's start stays
 * frees_invalid (C29).  The shrunk block keeps its start; heap_export reports its
 * new size.  Costs one bit per arena unit of workspace (a live-start bitmap with summaries). */
#define HEAP_PARTIAL_FREE 0x100

#define HEAP_NULL UINT64_MAX /* failed alloc; no-op in a free batch (offset 0 is valid, C18) */

enum heap_error {
    HEAP_OK = 0,
    HEAP_EINVAL = -1,    /* bad argument (align not a power of two, arena not a multiple of
                            align, arena/align > 2^32, n > max_batch, NULL handle, ...) */
    HEAP_ENOMEM = -2,    /* workspace too small or host allocation failed */
    HEAP_ECAPACITY = -3, /* a batch overflowed a metadata capacity (sticky, see above) */
    HEAP_ECUDA = -4,     /* a CUDA call failed */
    HEAP_ENCCL = -5      /* an NCCL call failed (heap_stats_allgather, heap_nccl_*) */
};

/* 16 x u64 = 128 bytes; byte quantities unless noted */
typedef struct heap_stats {
    uint64_t arena_bytes, align;
    uint64_t live_bytes, free_bytes;   /* live + free == arena (conservation, I2) */
    uint64_t n_live, n_free;           /* live blocks, free blocks */
    uint64_t largest_free;             /* size of the largest free block */
    uint64_t high_water_end;           /* max over all successful allocs of offset + size */
    uint64_t allocs_ok, allocs_failed; /* failed = OOM + zero size + oversize */
    uint64_t frees_ok, frees_invalid, frees_double, frees_null;
    uint64_t metadata_bytes;           /* device workspace bytes the heap occupies */
    uint64_t error_flags;              /* bit 0: live-block capacity, bit 1: table full,
                                          bit 2: free-array capacity, bit 3: engine watchdog,
                                          bit 4: live-start bitmap and table disagree */
} heap_stats_t;

/* Bytes of device workspace heap_create needs for these capacities.
 *   max_live_blocks: upper bound on simultaneously live blocks (sizes the block table and
 *                    the free-block arrays); max_batch: largest n of a single batch call.
 * Returns 0 for invalid arguments. */
size_t heap_workspace_bytes(uint64_t arena_bytes, uint64_t align, int policy,
                            uint64_t max_live_blocks, uint64_t max_batch);

/* Create a heap over [0, arena_bytes) (offsets), all free: one free block,
 * or for HEAP_BUDDY the greedy decomposition into maximal aligned power-of-two blocks.
 * d_workspace (>= heap_workspace_bytes(...) bytes, 256-byte aligned) is caller-owned and
 * must outlive the heap; initialisation kernels are enqueued on s.  *h_out receives the
 * host handle (the only memory the library owns).
 * Environment (read here; for ablation and for testing both paths — results are identical either
 * way): HEAP_WILD_SPLIT=0 turns off the TLSF/SEGFIT wilderness split (the alloc engine then
 * carries the top class's single member like any other piece); HEAP_BF_FLAT=1 / 2 / 3 runs
 * BEST_FIT one request at a time on one flat sorted key array / the blocked chunk list / the
 * class-indexed chunk list instead of the speculative 32-request chunks; HEAP_ENGINE_WARPS=1 / 3
 * runs the TLSF/SEGFIT engine on one warp / three warps (warp 1 also refilling the classes without
 * arrivals, warp 2 gathering candidates) instead of two; HEAP_MICRO=0 keeps small heaps
 * (FIRST/NEXT/BEST fit, SEGFIT, TLSF with max_live_blocks + 1 <= 4160, arena_bytes / align < 2^32,
 * max_batch <= 4096) off the single-launch path (one 512-thread CTA per batch, micro.cuh);
 * HEAP_BUDDY_LEVELS=1 runs the binary-buddy free phase level by level instead of in parallel
 * form; HEAP_PDL=0 launches without programmatic dependent launch. */
int heap_create(uint64_t arena_bytes, uint64_t align, int policy, uint64_t max_live_blocks,
                uint64_t max_batch, void *d_workspace, size_t workspace_bytes,
                heap_stream_t s, heap_t **h_out);

/* Release the host handle.  Does not free the workspace (caller-owned).  The caller must
 * make sure no enqueued work of this heap is still pending on a stream. */
int heap_destroy(heap_t *h);

/* Free a batch of n offsets (bytes).  0 <= n <= max_batch. */
int heap_free_batch(heap_t *h, const uint64_t *d_offsets, uint64_t n, heap_stream_t s);

/* The same batch by handle: offset i is d_table[d_idx[i]] (device arrays; d_table holds
 * table_len offsets, e.g. the results of earlier heap_alloc_batch calls, HEAP_NULL allowed; an
 * index >= table_len frees nothing and counts as a null free).  Identical to heap_free_batch on the
 * gathered offsets (Alg. 2); a single-launch heap reads them inside its free
 * kernel, other heaps gather them first (one extra launch).  0 <= n <= max_batch;
 * HEAP_EINVAL on a null heap or null arrays with n > 0. */
int heap_free_batch_handles(heap_t *h, const uint64_t *d_table, uint64_t table_len, const uint64_t *d_idx,
                            uint64_t n, heap_stream_t s);

/* One canonical batch (BASELINE north_star: the frees, then the allocs in request order) in one
 * call: heap_free_batch(d_offsets, nf) — or, when d_idx is not NULL, heap_free_batch_handles(
 * d_offsets as the table of table_len handles, d_idx, nf) — followed by heap_alloc_batch(d_sizes,
 * d_out, na), with exactly their results.  A single-launch heap runs both phases in ONE kernel
 * (micro.cuh k_micro_step); other heaps issue the two batches.  d_out may alias the handle table:
 * the frees are read before any result is written.  0 <= nf, na <= max_batch; HEAP_EINVAL on a
 * null heap or null arrays with a nonzero count. */
int heap_step(heap_t *h, const uint64_t *d_offsets, const uint64_t *d_idx, uint64_t table_len, uint64_t nf,
              const uint64_t *d_sizes, uint64_t *d_out_offsets, uint64_t na, heap_stream_t s);

/* Allocate a batch of n requests: d_sizes[i] bytes -> d_out_offsets[i] (byte offset into the
 * arena, or HEAP_NULL).  0 <= n <= max_batch.  d_out_offsets must not alias d_sizes. */
int heap_alloc_batch(heap_t *h, const uint64_t *d_sizes, uint64_t *d_out_offsets, uint64_t n,
                     heap_stream_t s);

/* Enqueue a reduction of the heap's statistics into d_out (device, 128 bytes).  No host
 * synchronisation; this is what an NCCL all-gather of statistics consumes. */
int heap_stats_async(heap_t *h, heap_stats_t *d_out, heap_stream_t s);

/* heap_stats_async + copy to h_out + stream synchronise.  Returns HEAP_ECAPACITY if a
 * capacity error flag is set (h_out is still filled). */
int heap_stats(heap_t *h, heap_stats_t *h_out, heap_stream_t s);

/* Multi-GPU statistics.  The paper's model is one host allocator
 * per device heap (§1): heaps do not shard, so N GPUs run N independent heaps and
 * the only cross-GPU traffic is their statistics.  heap_stats_allgather enqueues this rank's
 * heap_stats_async into the heap's workspace and an ncclAllGather of the 128-byte records over
 * comm, on stream s (no host synchronisation): d_all (device, nranks x 128 bytes) receives rank
 * r's statistics at d_all[r].  Collective: every rank of comm must call it (with its own heap) in
 * the same order.  Returns HEAP_EINVAL for NULL arguments, HEAP_ENCCL if NCCL fails. */
int heap_stats_allgather(heap_t *h, ncclComm_t comm, heap_stats_t *d_all, heap_stream_t s);

/* NCCL plumbing for callers without a communicator (the library links the image's NCCL 2.28):
 *   heap_nccl_unique_id: 128 opaque bytes into h_id (rank 0 creates it and shares it, e.g. over
 *     torch.distributed);
 *   heap_nccl_comm_init: *h_comm = this rank's communicator of nranks (current CUDA device);
 *   heap_nccl_comm_init_all: ndev communicators for devices h_devs[0..ndev) of this process
 *     (single-process multi-GPU, no bootstrap network; ndev = 1 gives a 1-rank communicator);
 *   heap_nccl_comm_destroy.  All return HEAP_OK or HEAP_ENCCL (HEAP_EINVAL for NULL pointers). */
int heap_nccl_unique_id(uint8_t *h_id);
int heap_nccl_comm_init(ncclComm_t *h_comm, int nranks, const uint8_t *h_id, int rank);
int heap_nccl_comm_init_all(ncclComm_t *h_comms, int ndev, const int *h_devs);
int heap_nccl_comm_destroy(ncclComm_t comm);

/* Export the state for parity checks: free blocks and live blocks as (start, size) byte
 * pairs sorted by start, into device arrays of cap_free / cap_live pairs (2 x u64 each).
 * h_counts[0] = #free blocks, h_counts[1] = #live blocks (true counts even if they exceed
 * the capacities, in which case only the first cap pairs are written).  Synchronises s. */
int heap_export(heap_t *h, uint64_t *d_free_pairs, uint64_t cap_free, uint64_t *d_live_pairs,
                uint64_t cap_live, uint64_t *h_counts, heap_stream_t s);

/* Number of kernel launches this heap has enqueued so far (for the bench's gpu_launches);
 * kernels run inside a batch graph count individually. */
uint64_t heap_launch_count(const heap_t *h);

/* Batch graphs (default: enabled).  When enabled, heap_free_batch / heap_alloc_batch run each
 * batch as ONE CUDA-graph launch: the first call per (operation, internal ping-pong state)
 * captures the batch's kernels once (a few ms); later calls of any n patch the request count
 * and the request/result copies (staged through the workspace) and relaunch.  Semantics and
 * results are identical to direct launches.  Direct launches are used instead while tracing is
 * enabled (heap_profile_enable) or when the stream is itself being captured.  enable = 0
 * switches to direct launches.  Returns HEAP_EINVAL for a NULL handle. */
int heap_set_graphs(heap_t *h, int enable);

/* Per-kernel timing (tracing).  Kernels are grouped by tag (HEAP_TAG_*); for every tag whose
 * bit is set in tag_mask, each launch is bracketed by two CUDA events on its stream.
 * heap_profile_read synchronises those events, adds each tag's summed milliseconds and launch
 * count into h_ms[tag] / h_launches[tag] (arrays of HEAP_NTAGS), and forgets the records.
 * tag_mask = 0 disables (the default); enabling costs two event records per bracketed launch. */
enum heap_tag {
    HEAP_TAG_CLASSIFY = 0, HEAP_TAG_SCAN = 1, HEAP_TAG_SORT = 2, HEAP_TAG_LOOKUP = 3,
    HEAP_TAG_COMPACT = 4, HEAP_TAG_MERGE = 5, HEAP_TAG_COALESCE = 6, HEAP_TAG_ALLOC_PREP = 7,
    HEAP_TAG_INDEX = 8, HEAP_TAG_ENGINE = 9, HEAP_TAG_FINISH = 10, HEAP_TAG_REBUILD = 11,
    HEAP_TAG_BUDDY_FREE = 12, HEAP_TAG_BUDDY_ALLOC = 13, HEAP_TAG_MISC = 14,
    HEAP_TAG_MICRO = 15, HEAP_NTAGS = 16
};
int heap_profile_enable(heap_t *h, uint64_t tag_mask);
/* Copy the alloc engine's cumulative diagnostic counters (n <= 32 u64: chunks, re-aimed
 * requests, invariant-failure flag, replay rounds, leader steps, cycle counts per engine
 * phase) to h_out.  Synchronises s.  For tuning and tests; values are implementation-defined. */
int heap_debug_counters(heap_t *h, uint64_t *h_out, int n, heap_stream_t s);
int heap_profile_read(heap_t *h, double *h_ms, uint64_t *h_launches);
const char *heap_tag_name(int tag);

const char *heap_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif /* LIBHEAP_HEAP_H */
