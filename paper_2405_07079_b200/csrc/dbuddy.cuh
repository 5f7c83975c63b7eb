// dbuddy.cuh — HEAP_DOUBLE_BUDDY: double buddies ("two heaps with staggered
// class sizes, e.g. one heap with sizes of 2, 4, 8, ... and another with 3, 6, 12, ...").
//
// Reading C28: a binary buddy heap of align-sized units on [0, A_bytes) and one of
// 3*align-sized units on [A_bytes, arena), the latter holding floor(arena / 6 align) units.  A
// request of r units goes to the heap whose class is smaller — 2^ceil(log2 r) units or
// 3 * 2^ceil(log2 ceil(r/3)) units (never equal) — with no fallback.  Both heaps are the binary
// buddy machinery of buddy.cuh (exactly parallel, L6); this file only splits a batch into the
// two heaps' sub-batches (request order kept in each) and puts the results back.
#pragma once
#include "common.cuh"

namespace dbl {

struct Ctr {
    u64 nreq, nA, nB;
    u64 frees_null, frees_invalid;
    u64 scan_total;
};

// frees: HEAP_NULL and offsets past A_bytes that are not a whole number of 3-units are settled
// here; the rest become each heap's own offsets (binary: bytes; 3-unit heap: unit index)
__global__ void k_free_split(const u64 *__restrict__ offs, u64 n, const u64 *n_in, u64 A_bytes, u64 u3, int has3,
                             u32 *__restrict__ fa, u32 *__restrict__ fb, u64 *__restrict__ va, u64 *__restrict__ vb,
                             Ctr *c) {
    PDL_ENTRY();
    if (n_in) n = *n_in;
    if (blockIdx.x == 0 && threadIdx.x == 0) c->nreq = n;
    u64 nnull = 0, ninv = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 o = offs[i];
        u32 a = 0, b = 0;
        if (o == HEAP_NULL_U64) nnull++;
        else if (o < A_bytes) { a = 1; va[i] = o; }
        else if (!has3 || (o - A_bytes) % u3) ninv++;
        else { b = 1; vb[i] = (o - A_bytes) / u3; }
        fa[i] = a;
        fb[i] = b;
    }
    nnull = warp_sum64(nnull);
    ninv = warp_sum64(ninv);
    if (lane_id() == 0) {
        if (nnull) atomicAdd(&c->frees_null, nnull);
        if (ninv) atomicAdd(&c->frees_invalid, ninv);
    }
}

// allocs: the class choice; the 3-unit heap is asked for ceil(r/3) of its units
__global__ void k_alloc_split(const u64 *__restrict__ sizes, u64 n, const u64 *n_in, int alog2, u64 A_u, int has3,
                              u32 *__restrict__ fa, u32 *__restrict__ fb, u64 *__restrict__ va, u64 *__restrict__ vb,
                              Ctr *c) {
    PDL_ENTRY();
    if (n_in) n = *n_in;
    if (blockIdx.x == 0 && threadIdx.x == 0) c->nreq = n;
    const u64 amask = (1ull << alog2) - 1;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 s = sizes[i];
        const u64 r = (s >> alog2) + ((s & amask) != 0);
        bool three = false;
        u64 q = 0;
        if (s != 0 && r <= A_u && has3) {
            q = (r + 2) / 3;
            const u64 two = (r <= 1) ? 1 : (1ull << (64 - __clzll(r - 1)));
            const u64 p3 = (q <= 1) ? 1 : (1ull << (64 - __clzll(q - 1)));
            three = 3 * p3 < two;
        }
        fa[i] = three ? 0u : 1u;
        fb[i] = three ? 1u : 0u;
        if (three) vb[i] = q; else va[i] = s;
    }
}

__global__ void k_compact_idx(const u64 *__restrict__ v, const u32 *__restrict__ flags, const u32 *__restrict__ pos,
                              const u64 *n_dev, u64 *__restrict__ out, u32 *__restrict__ idx) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        if (flags[i]) { out[pos[i]] = v[i]; if (idx) idx[pos[i]] = (u32)i; }
}

__global__ void k_scatter(const u64 *__restrict__ res, const u32 *__restrict__ idx, const u64 *n_dev, u64 base,
                          u64 mul, u64 *__restrict__ out) {
    PDL_ENTRY();
    const u64 n = *n_dev;
    for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (u64)gridDim.x * blockDim.x) {
        const u64 o = res[k];
        out[idx[k]] = (o == HEAP_NULL_U64) ? HEAP_NULL_U64 : base + o * mul;
    }
}

// export of the 3-unit heap: (unit, units) -> bytes past A_bytes
__global__ void k_pairs_to_bytes(u64 *pairs, u64 n, u64 base, u64 mul) {
    PDL_ENTRY();
    for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (u64)gridDim.x * blockDim.x) {
        pairs[2 * k] = base + pairs[2 * k] * mul;
        pairs[2 * k + 1] *= mul;
    }
}

// heap_stats of the pair (reading C28): sums; sizes of the 3-unit heap scaled to bytes
__global__ void k_stats(const heap_stats_t *a, const heap_stats_t *b, int has3, const Ctr *c, u64 arena, u64 align,
                        u64 A_bytes, u64 meta, heap_stats_t *out) {
    PDL_ENTRY();
    const u64 u3 = 3 * align;
    heap_stats_t z = {};
    const heap_stats_t *bb = has3 ? b : &z;
    const u64 live = a->live_bytes + bb->live_bytes * u3;
    out->arena_bytes = arena;
    out->align = align;
    out->live_bytes = live;
    out->free_bytes = arena - live;
    out->n_live = a->n_live + bb->n_live;
    out->n_free = a->n_free + bb->n_free;
    const u64 lb = bb->largest_free * u3;
    out->largest_free = a->largest_free > lb ? a->largest_free : lb;
    const u64 hb = bb->high_water_end ? A_bytes + bb->high_water_end * u3 : 0;
    out->high_water_end = a->high_water_end > hb ? a->high_water_end : hb;
    out->allocs_ok = a->allocs_ok + bb->allocs_ok;
    out->allocs_failed = a->allocs_failed + bb->allocs_failed;
    out->frees_ok = a->frees_ok + bb->frees_ok;
    out->frees_invalid = a->frees_invalid + bb->frees_invalid + c->frees_invalid;
    out->frees_double = a->frees_double + bb->frees_double;
    out->frees_null = a->frees_null + bb->frees_null + c->frees_null;
    out->metadata_bytes = meta;
    out->error_flags = a->error_flags | bb->error_flags;
}

}  // namespace dbl
