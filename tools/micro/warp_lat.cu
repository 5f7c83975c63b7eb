// tools/micro/warp_lat.cu — dev microbenchmark (not product): dependent-chain latency of the warp
// primitives the TLSF engine is built from, one warp alone on the SM (the engine's situation).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/warp_lat tools/micro/warp_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned int u32;
typedef unsigned long long u64;
#define N 4096
__global__ void k(u32 *out, long long *cyc, u32 seed, const u32 *g) {
    __shared__ u32 sm[1024];
    const u32 lane = threadIdx.x;
    for (int i = lane; i < 1024; i += 32) sm[i] = (i * 7 + 1) & 1023;
    __syncwarp();
    u32 x = seed + lane;
    long long t0, t1;
    int slot = 0;
#define TIME(name, body) { __syncwarp(); t0 = clock64(); for (int i = 0; i < N; i++) { body; } t1 = clock64(); cyc[slot++] = (t1 - t0); }
    TIME("lds", x = sm[x & 1023]);
    TIME("shfl", x = __shfl_sync(0xffffffffu, x, x & 31));
    TIME("ballot", x = __ballot_sync(0xffffffffu, x & (1u << lane)) + lane);
    TIME("match_any", x = __match_any_sync(0xffffffffu, x & 7) + x);
    TIME("redux_min", x = __reduce_min_sync(0xffffffffu, x) + lane);
    TIME("any", x += __any_sync(0xffffffffu, x == 12345u));
    TIME("ffs", x = __ffs(x) + x);
    TIME("popc_lanemask", x = __popc(x & ((1u << lane) - 1)) + x);
    TIME("imad", x = x * 3 + 1);
    TIME("ldg_l1", x = g[x & 1023]);
    TIME("ldg_cg", x = __ldcg(&g[(x & 1023)]));
    TIME("atoms_or", x = atomicOr(&sm[x & 1023], 1u) & 1023);
    TIME("sts_lds", { sm[lane] = x; x = sm[(lane + 1) & 31]; });
    TIME("syncwarp_lds", { __syncwarp(); x = sm[x & 1023]; });
    out[lane] = x;
}
int main() {
    u32 *out, *g; long long *cyc;
    cudaMalloc(&out, 128); cudaMalloc(&cyc, 64 * 8); cudaMalloc(&g, 4096 * 4);
    u32 h[4096]; for (int i = 0; i < 4096; i++) h[i] = (i * 13 + 5) & 1023;
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; rep++) k<<<1, 32>>>(out, cyc, 1, g);
    cudaDeviceSynchronize();
    long long c[64]; cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    const char *names[] = {"lds", "shfl", "ballot+iadd", "match_any+iadd", "redux_min+iadd", "any+iadd", "ffs+iadd",
                           "popc(and lanemask)+iadd", "imad", "ldg_l1", "ldg_cg(L2)", "atoms_or", "sts+lds", "syncwarp+lds"};
    for (int i = 0; i < 14; i++) printf("%-26s %.1f cyc/iter\n", names[i], (double)c[i] / N);
    return 0;
}
