// latency_study.cu — batch-size-1 driver for the SURVEY §8(f) f1 study (PAPER.md:505-518,
// Fig. 3/4 analogue).  Not part of the product: it calls the public C ABI (include/heap.h) the
// way a host program would use a host-side allocator — one request per call, the result read
// back before the next call — and records each call's host wall time.
//
// ops[j] = (kind, arg): kind 0 = free of alloc id `arg`, kind 1 = alloc of `arg` bytes (alloc ids
// in order).  Per op: the request word is copied from pinned host memory, the batch call runs
// with n = 1, an alloc's offset is copied back, and the stream is synchronised (all timed).
// After the op (untimed) heap_stats gives live bytes and the high-water end — the arena extent
// that has to be physically backed, this heap's "provisioned" memory.
#include <chrono>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "heap.h"

extern "C" int heap_latency(heap_t *h, void *stream, uint64_t nops, const uint8_t *kind,
                            const uint64_t *arg, double *lat_ns, uint64_t *live, uint64_t *hwm,
                            uint64_t *fail_out) {
    cudaStream_t s = (cudaStream_t)stream;
    uint64_t nalloc = 0;
    for (uint64_t j = 0; j < nops; j++) nalloc += kind[j];
    std::vector<uint64_t> off(nalloc, HEAP_NULL);
    uint64_t *hbuf = nullptr, *dbuf = nullptr;
    if (cudaMallocHost(&hbuf, 2 * sizeof(uint64_t)) != cudaSuccess) return -1;
    if (cudaMalloc(&dbuf, 2 * sizeof(uint64_t)) != cudaSuccess) return -1;
    uint64_t next = 0, fail = 0;
    heap_stats_t st;
    for (uint64_t j = 0; j < nops; j++) {
        auto t0 = std::chrono::steady_clock::now();
        int rc;
        if (kind[j] == 0) {
            hbuf[0] = off[arg[j]];
            off[arg[j]] = HEAP_NULL;
            cudaMemcpyAsync(dbuf, hbuf, 8, cudaMemcpyHostToDevice, s);
            rc = heap_free_batch(h, dbuf, 1, (heap_stream_t)s);
            cudaStreamSynchronize(s);
        } else {
            hbuf[0] = arg[j];
            cudaMemcpyAsync(dbuf, hbuf, 8, cudaMemcpyHostToDevice, s);
            rc = heap_alloc_batch(h, dbuf, dbuf + 1, 1, (heap_stream_t)s);
            cudaMemcpyAsync(hbuf + 1, dbuf + 1, 8, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            off[next++] = hbuf[1];
            if (hbuf[1] == HEAP_NULL) fail++;
        }
        lat_ns[j] = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
        if (rc != HEAP_OK) return -2;
        if (heap_stats(h, &st, (heap_stream_t)s) != HEAP_OK) return -3;
        live[j] = st.live_bytes;
        hwm[j] = st.high_water_end;
    }
    cudaFreeHost(hbuf);
    cudaFree(dbuf);
    *fail_out = fail;
    return 0;
}
