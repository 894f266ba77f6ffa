// Microbenchmark: L2 atomic throughput for the tile-binning design decision
// (RED vs ATOM-with-return into ~255K per-tile counters, 60M pairs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
// splat i (random screen position) covers a 3x1 run of tiles
__device__ __forceinline__ uint32_t tile_of(uint32_t i, uint32_t ntiles) {
    const uint32_t s = i / 3, k = i % 3;
    return (hash32(s) % (ntiles - 3)) + k;
}
__global__ void k_red(uint32_t n, uint32_t ntiles, uint32_t *cnt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd(&cnt[tile_of(i, ntiles)], 1u);
}
__global__ void k_atom(uint32_t n, uint32_t ntiles, uint32_t *cur, uint32_t *out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t t = tile_of(i, ntiles);
        const uint32_t p = atomicAdd(&cur[t], 1u);
        out[(size_t)t * 300 + (p % 300)] = i;
    }
}
__global__ void k_plain(uint32_t n, uint32_t ntiles, uint32_t *out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[(size_t)tile_of(i, ntiles) * 300 + (i % 300)] = i;
}
int main() {
    const uint32_t n = 60000000, ntiles = 255000;
    uint32_t *cnt, *out;
    cudaMalloc(&cnt, ntiles * 4);
    cudaMalloc(&out, (size_t)ntiles * 300 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; rep++) {
        float ms;
        cudaMemset(cnt, 0, ntiles * 4);
        cudaEventRecord(a);
        k_red<<<148 * 8, 256>>>(n, ntiles, cnt);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("RED  60M: %.3f ms (%.1f G/s)\n", ms, n / ms / 1e6);
        cudaMemset(cnt, 0, ntiles * 4);
        cudaEventRecord(a);
        k_atom<<<148 * 8, 256>>>(n, ntiles, cnt, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("ATOM 60M + store: %.3f ms (%.1f G/s)\n", ms, n / ms / 1e6);
        cudaEventRecord(a);
        k_plain<<<148 * 8, 256>>>(n, ntiles, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("plain scattered store 60M: %.3f ms\n", ms);
    }
    return 0;
}
