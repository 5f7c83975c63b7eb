// cudamalloc_replay.cu — the paper's comparison system: the same per-batch
// op order replayed with the driver allocator, one call per request from one host thread.
// Not part of the product path; bench.py loads it to report the baselines beside our numbers.
//
//   mode 0: cudaMalloc / cudaFree          (the paper's baseline)
//   mode 1: cudaMallocAsync / cudaFreeAsync on one stream, default pool, release threshold max
//
// Input: the trace flattened over batches: for batch b, frees free_ids[fo[b] .. fo[b+1]) then
// allocs of sizes[ao[b] .. ao[b+1]) with ids ao[b] + j.  A failed alloc's id maps to NULL and its
// free is cudaFree(NULL).  Stops after max_ops requests or max_seconds.  Returns the number of
// requests replayed and their wall time (host clock, final device synchronise included).
#include <chrono>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

extern "C" int replay(int mode, uint64_t nbatches, const uint64_t *fo, const uint64_t *free_ids,
                      const uint64_t *ao, const uint64_t *sizes, uint64_t max_ops, double max_seconds,
                      uint64_t *ops_done, double *seconds, uint64_t *failed) {
    std::vector<void *> ptr(ao[nbatches], nullptr);
    cudaStream_t s = nullptr;
    if (mode == 1) {
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return -1;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return -1;
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaDeviceSynchronize();
    uint64_t ops = 0, fail = 0;
    auto t0 = std::chrono::steady_clock::now();
    double el = 0;
    for (uint64_t b = 0; b < nbatches && ops < max_ops; b++) {
        for (uint64_t j = fo[b]; j < fo[b + 1] && ops < max_ops; j++, ops++) {
            void *p = ptr[free_ids[j]];
            if (mode == 0) cudaFree(p);
            else if (p) cudaFreeAsync(p, s);
            ptr[free_ids[j]] = nullptr;
        }
        for (uint64_t j = ao[b]; j < ao[b + 1] && ops < max_ops; j++, ops++) {
            void *p = nullptr;
            cudaError_t e = (mode == 0) ? cudaMalloc(&p, sizes[j]) : cudaMallocAsync(&p, sizes[j], s);
            if (e != cudaSuccess) { p = nullptr; fail++; cudaGetLastError(); }
            ptr[j] = p;
        }
        el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > max_seconds) break;
    }
    if (mode == 1) cudaStreamSynchronize(s);
    cudaDeviceSynchronize();
    el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *ops_done = ops;
    *seconds = el;
    *failed = fail;
    // release everything so the process can continue
    for (void *p : ptr)
        if (p) { if (mode == 0) cudaFree(p); else cudaFreeAsync(p, s); }
    if (mode == 1) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    cudaDeviceSynchronize();
    return 0;
}

// Per-op latency replay for the batch-size-1 study (Fig. 3/4 analogue).
// ops[j] = (kind, arg): kind 0 = free of alloc id `arg`, kind 1 = alloc of `arg` bytes (ids are
// assigned to allocs in order).  lat_ns[j] = host wall time of the one driver call (cudaFree /
// cudaMalloc; the async pair is followed by a stream synchronise so the op has completed).
// used[j] = device memory in use by the process after op j (cudaMemGetInfo total - free), the
// "provisioned" figure of Fig. 4; it is sampled outside the timed call.
extern "C" int replay_latency(int mode, uint64_t nops, const uint8_t *kind, const uint64_t *arg,
                              double *lat_ns, uint64_t *used, uint64_t *fail_out) {
    uint64_t nalloc = 0;
    for (uint64_t j = 0; j < nops; j++) nalloc += kind[j];
    std::vector<void *> ptr(nalloc, nullptr);
    cudaStream_t s = 0;
    if (mode == 1) {
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return -1;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return -1;
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaDeviceSynchronize();
    uint64_t next = 0, fail = 0;
    for (uint64_t j = 0; j < nops; j++) {
        auto t0 = std::chrono::steady_clock::now();
        if (kind[j] == 0) {
            void *p = ptr[arg[j]];
            ptr[arg[j]] = nullptr;
            if (mode == 0) cudaFree(p);
            else { if (p) cudaFreeAsync(p, s); cudaStreamSynchronize(s); }
        } else {
            void *p = nullptr;
            cudaError_t e = (mode == 0) ? cudaMalloc(&p, arg[j]) : cudaMallocAsync(&p, arg[j], s);
            if (mode == 1) cudaStreamSynchronize(s);
            if (e != cudaSuccess) { p = nullptr; fail++; cudaGetLastError(); }
            ptr[next++] = p;
        }
        lat_ns[j] = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        used[j] = (uint64_t)(tot - fr);
    }
    for (void *p : ptr)
        if (p) { if (mode == 0) cudaFree(p); else cudaFreeAsync(p, s); }
    if (mode == 1) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    cudaDeviceSynchronize();
    *fail_out = fail;
    return 0;
}
