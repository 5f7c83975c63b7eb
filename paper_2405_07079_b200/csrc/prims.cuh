// prims.cuh — device-wide primitives with device-resident element counts:
// exclusive scan / stream compaction, LSD radix sort (8-bit digits, stable), merge path.
//
// Every kernel reads its element count from a u64 in device memory and walks tiles with
// a grid-stride loop, so the host never has to synchronise to size a launch.
#pragma once
#include "common.cuh"

namespace prims {

constexpr int NT = 256;        // threads per CTA
constexpr int IPT = 8;         // items per thread
constexpr int TILE = NT * IPT; // 2048 elements per tile

__host__ __device__ inline u64 ntiles_of(u64 n) { return (n + TILE - 1) / TILE; }

// ---------------------------------------------------------------- scan (u32) ----
// pass 1: per-tile sums
__global__ void __launch_bounds__(NT) k_scan_reduce(const u32 *__restrict__ in, const u64 *n_dev,
                                                    u32 *__restrict__ tile_sums) {
    __shared__ u64 sm[33];
    const u64 n = *n_dev, nt = ntiles_of(n);
    for (u64 t = blockIdx.x; t < nt; t += gridDim.x) {
        u64 base = t * TILE;
        u64 s = 0;
#pragma unroll
        for (int i = 0; i < IPT; i++) {
            u64 idx = base + (u64)i * NT + threadIdx.x;
            if (idx < n) s += in[idx];
        }
        s = block_sum64<NT>(s, sm);
        if (threadIdx.x == 0) tile_sums[t] = (u32)s;
    }
}

// pass 2: one CTA scans the tile sums in place (exclusive) and writes the grand total
__global__ void __launch_bounds__(1024) k_scan_tiles(u32 *tile_sums, const u64 *n_dev, u64 *total) {
    __shared__ u32 sm[33];
    const u64 nt = ntiles_of(*n_dev);
    u32 carry = 0;
    for (u64 base = 0; base < nt; base += 1024) {
        u64 idx = base + threadIdx.x;
        u32 v = idx < nt ? tile_sums[idx] : 0;
        u32 tot;
        u32 ex = block_excl_scan<1024>(v, sm, &tot);
        if (idx < nt) tile_sums[idx] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

// pass 3: per-tile exclusive scan plus the tile's offset
__global__ void __launch_bounds__(NT) k_scan_down(const u32 *__restrict__ in, u32 *__restrict__ out,
                                                  const u64 *n_dev, const u32 *__restrict__ tile_sums) {
    __shared__ u32 sm[33];
    __shared__ u32 stage[TILE];
    const u64 n = *n_dev, nt = ntiles_of(n);
    for (u64 t = blockIdx.x; t < nt; t += gridDim.x) {
        u64 base = t * TILE;
#pragma unroll
        for (int i = 0; i < IPT; i++) {   // coalesced load into smem
            u64 idx = base + (u64)i * NT + threadIdx.x;
            stage[i * NT + threadIdx.x] = idx < n ? in[idx] : 0;
        }
        __syncthreads();
        u32 v[IPT], s = 0;
#pragma unroll
        for (int i = 0; i < IPT; i++) { v[i] = stage[threadIdx.x * IPT + i]; s += v[i]; }
        u32 tot;
        u32 ex = block_excl_scan<NT>(s, sm, &tot) + tile_sums[t];
#pragma unroll
        for (int i = 0; i < IPT; i++) { stage[threadIdx.x * IPT + i] = ex; ex += v[i]; }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IPT; i++) {
            u64 idx = base + (u64)i * NT + threadIdx.x;
            if (idx < n) out[idx] = stage[i * NT + threadIdx.x];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ radix sort ----
// Stable LSD pass on digit (key >> shift) & 255.  hist layout: hist[d * ntiles + t].
template <typename K>
__global__ void __launch_bounds__(NT) k_rs_hist(const K *__restrict__ keys, const u64 *n_dev, int shift,
                                                u32 *__restrict__ hist, u64 *n_hist) {
    __shared__ u32 h[256];
    const u64 n = *n_dev, nt = ntiles_of(n);
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_hist = 256 * nt;
    for (u64 t = blockIdx.x; t < nt; t += gridDim.x) {
        h[threadIdx.x] = 0;
        __syncthreads();
        u64 base = t * TILE;
#pragma unroll
        for (int i = 0; i < IPT; i++) {
            u64 idx = base + (u64)i * NT + threadIdx.x;
            if (idx < n) atomicAdd(&h[(u32)(keys[idx] >> shift) & 255u], 1u);
        }
        __syncthreads();
        hist[(u64)threadIdx.x * nt + t] = h[threadIdx.x];
        __syncthreads();
    }
}

template <typename K, bool HV>
__global__ void __launch_bounds__(NT) k_rs_scatter(const K *__restrict__ kin, const u32 *__restrict__ vin,
                                                   K *__restrict__ kout, u32 *__restrict__ vout,
                                                   const u64 *n_dev, int shift,
                                                   const u32 *__restrict__ hscan) {
    __shared__ u32 run[256];
    __shared__ u32 wcnt[NT / 32][257];
    const u64 n = *n_dev, nt = ntiles_of(n);
    const int w = threadIdx.x >> 5;
    for (u64 t = blockIdx.x; t < nt; t += gridDim.x) {
        run[threadIdx.x] = 0;
        u64 base = t * TILE;
        for (int q = 0; q < IPT; q++) {
            u64 idx = base + (u64)q * NT + threadIdx.x;
            bool valid = idx < n;
            K key = valid ? kin[idx] : (K)0;
            u32 val = (HV && valid) ? vin[idx] : 0u;
            u32 d = valid ? ((u32)(key >> shift) & 255u) : 256u;
#pragma unroll
            for (int j = 0; j < NT / 32; j++) wcnt[j][threadIdx.x] = 0;
            __syncthreads();
            u32 peers = __match_any_sync(FULLMASK, d);
            u32 rank = __popc(peers & lanemask_lt());
            if (rank == 0 && valid) wcnt[w][d] = __popc(peers);
            __syncthreads();
            {
                u32 s = run[threadIdx.x];
#pragma unroll
                for (int j = 0; j < NT / 32; j++) {
                    u32 c = wcnt[j][threadIdx.x];
                    wcnt[j][threadIdx.x] = s;
                    s += c;
                }
                run[threadIdx.x] = s;
            }
            __syncthreads();
            if (valid) {
                u32 pos = hscan[(u64)d * nt + t] + wcnt[w][d] + rank;
                kout[pos] = key;
                if (HV) vout[pos] = val;
            }
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------ merge path ----
// Merge two start-sorted SoA arrays (start, end) of lengths *na, *nb into out (length
// na + nb).  Starts are distinct (disjoint blocks), ties go to a.
constexpr int MIPT = 8;
__global__ void __launch_bounds__(NT) k_merge(const u64 *__restrict__ as, const u64 *__restrict__ ae,
                                              const u64 *na_dev, const u64 *__restrict__ bs,
                                              const u64 *__restrict__ be, const u64 *nb_dev,
                                              u64 *__restrict__ os, u64 *__restrict__ oe, u64 *total,
                                              const u32 *__restrict__ at = nullptr,
                                              const u32 *__restrict__ bt = nullptr, u32 *__restrict__ ot = nullptr) {
    // at/bt/ot: optional per-block payload merged alongside (push stamps of SEGFIT_LIFO)
    const u64 na = *na_dev, nb = *nb_dev, n = na + nb;
    if (blockIdx.x == 0 && threadIdx.x == 0 && total) *total = n;
    const u64 nchunks = (n + MIPT - 1) / MIPT;
    for (u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += (u64)gridDim.x * blockDim.x) {
        u64 diag = c * MIPT;
        u64 lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
        while (lo < hi) {
            u64 mid = (lo + hi) >> 1;
            if (as[mid] <= bs[diag - mid - 1]) lo = mid + 1; else hi = mid;
        }
        u64 i = lo, j = diag - lo;
#pragma unroll
        for (int k = 0; k < MIPT; k++) {
            u64 o = diag + k;
            if (o >= n) break;
            bool take_a = (j >= nb) || (i < na && as[i] <= bs[j]);
            if (take_a) { os[o] = as[i]; oe[o] = ae[i]; if (ot) ot[o] = at[i]; i++; }
            else { os[o] = bs[j]; oe[o] = be[j]; if (ot) ot[o] = bt[j]; j++; }
        }
    }
}

}  // namespace prims
