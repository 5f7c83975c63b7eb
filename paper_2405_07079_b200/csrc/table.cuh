// table.cuh — the block table: an address-keyed open-addressing hash table that holds what a
// boundary tag would (the block's size), out of band (§3.3).
//
// B200 design (differs from the paper's chained 6-word entries):
//   * one 8-byte slot per live block: (key << 32) | (size_units - 1), key = offset / align;
//     free-list links and prev_adj are not needed because free blocks live in sorted arrays;
//   * linear probing over 32-byte sectors (4 slots): a probe is one sector read by a 2-lane tile
//     (16 B per lane), match/empty found with one warp ballot, 16 keys per warp.  Round 1 probed
//     whole 128-byte lines with 8-lane tiles; the sector probe cut config 5's lookup kernel from
//     41 to 25 us (ncu) but not its DRAM bytes (~126 B per free either way: a random access fills a
//     128-byte L2 line from HBM);
//   * delete writes a TOMBSTONE; insert reuses the first EMPTY-or-TOMBSTONE slot of the first
//     line that has one (CAS); lookup stops at the first line containing an EMPTY slot, which
//     is sound because slots only become EMPTY again in a full rebuild.
// Slot placement may depend on CAS order; lookups do not, so results are deterministic.
#pragma once
#include "common.cuh"

namespace table {

constexpr u64 EMPTY = 0xFFFFFFFFFFFFFFFFull;
constexpr u64 TOMB = 0xFFFFFFFFFFFFFFFEull;
constexpr int TILE_LANES = 2;   // lanes per key
constexpr int KPW = 32 / TILE_LANES;   // keys per warp
constexpr int LINE = 4;         // slots per probed 32-byte sector (2 per lane)

__device__ __forceinline__ u64 pack(u64 key, u64 size_units) { return (key << 32) | (size_units - 1); }
__device__ __forceinline__ bool is_live(u64 s) { return s < TOMB; }
__device__ __forceinline__ u64 slot_key(u64 s) { return s >> 32; }
__device__ __forceinline__ u64 slot_size(u64 s) { return (s & 0xFFFFFFFFull) + 1; }

__device__ __forceinline__ u64 home_line(u64 key, u64 mask) {
    u64 h = (key + 1) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31;
    return (h & mask) & ~(u64)(LINE - 1);
}

// Tile-cooperative lookup (and optional replacement of the slot found: TOMB deletes, a packed
// value updates the size; EMPTY leaves it).  All 32 lanes of the warp call it; lanes of an
// inactive group pass active = false.  Returns the live slot value found (EMPTY if the key is
// absent) on every lane of the group.
__device__ u64 lookup(u64 *__restrict__ slots, u64 mask, u64 key, bool active, u64 repl, u64 max_lines) {
    const u32 lane = lane_id(), sub = lane & (TILE_LANES - 1), g = lane / TILE_LANES;
    const u32 gmask = ((1u << TILE_LANES) - 1u) << (g * TILE_LANES);
    u64 line = active ? home_line(key, mask) : 0;
    u64 result = EMPTY;
    bool done = !active;
    for (u64 p = 0;; p++) {
        if (!__any_sync(FULLMASK, !done)) break;
        bool m0 = false, m1 = false, empty = false;
        ulonglong2 v = make_ulonglong2(EMPTY, EMPTY);
        if (!done) {
            v = *reinterpret_cast<const ulonglong2 *>(slots + line + 2 * sub);
            m0 = is_live(v.x) && slot_key(v.x) == key;
            m1 = is_live(v.y) && slot_key(v.y) == key;
            empty = (v.x == EMPTY) || (v.y == EMPTY);
        }
        u32 bm = __ballot_sync(FULLMASK, m0 || m1) & gmask;
        u32 be = __ballot_sync(FULLMASK, empty) & gmask;
        if (!done) {
            if (bm) {
                if (lane == (u32)(__ffs(bm) - 1)) {
                    result = m0 ? v.x : v.y;
                    if (repl != EMPTY) slots[line + 2 * sub + (m0 ? 0 : 1)] = repl;
                }
                done = true;
            } else if (be || p + 1 >= max_lines) {
                done = true;
            } else {
                line = (line + LINE) & mask;
            }
        }
    }
    u64 r = result;
#pragma unroll
    for (int o = 1; o < TILE_LANES; o <<= 1) {
        u64 t = __shfl_xor_sync(FULLMASK, r, o);
        r = (t != EMPTY) ? t : r;
    }
    return r;
}

// Tile-cooperative insert of a key that is known to be absent.  Returns, on the lane that
// performed the successful CAS: +1 if it consumed an EMPTY slot, -1 if a TOMBSTONE; 0 on the
// other lanes; 2 on lane sub==0 if no slot was found within max_lines (table full).
__device__ int insert(u64 *__restrict__ slots, u64 mask, u64 key, u64 size_units, bool active,
                      u64 max_lines) {
    const u32 lane = lane_id(), sub = lane & (TILE_LANES - 1), g = lane / TILE_LANES;
    const u32 gmask = ((1u << TILE_LANES) - 1u) << (g * TILE_LANES);
    const u64 nv = active ? pack(key, size_units) : 0;
    u64 line = active ? home_line(key, mask) : 0;
    bool done = !active;
    int ret = 0;
    for (u64 p = 0;;) {
        if (!__any_sync(FULLMASK, !done)) break;
        bool c0 = false, c1 = false;
        ulonglong2 v = make_ulonglong2(0, 0);
        if (!done) {
            v = __ldcg(reinterpret_cast<const ulonglong2 *>(slots + line + 2 * sub));   // L2: sees racing CASes
            c0 = (v.x >= TOMB);
            c1 = (v.y >= TOMB);
        }
        u32 bc = __ballot_sync(FULLMASK, c0 || c1) & gmask;
        u32 src = (!done && bc) ? (u32)(__ffs(bc) - 1) : lane;
        int ok = 0;
        if (!done && bc && lane == src) {
            int which = c0 ? 0 : 1;
            u64 old = which ? v.y : v.x;
            u64 prev = atomicCAS(&slots[line + 2 * sub + which], old, nv);
            if (prev == old) { ok = 1; ret = (old == EMPTY) ? 1 : -1; }
        }
        ok = __shfl_sync(FULLMASK, ok, src);
        if (!done) {
            if (bc) {
                if (ok) done = true;          // else: lost a race, re-read the same line
            } else if (++p >= max_lines) {
                done = true;
                if (sub == 0) ret = 2;
            } else {
                line = (line + LINE) & mask;
            }
        }
    }
    return ret;
}

}  // namespace table
