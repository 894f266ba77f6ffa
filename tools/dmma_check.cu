// dmma_check.cu -- does the fp64 tensor-core MMA (mma.sync m8n8k4 f64) round
// like a chain of fused multiply-adds in k order?  And how fast is it on
// this part?  (Decides whether k_sh_accumulate may use it: the oracle's
// normal equations are sequential fma chains over the views.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_check tools/dmma_check.cu
//   ./dmma_check
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b, double c0,
                                     double c1) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
        : "=d"(d0), "=d"(d1)
        : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// A: 8x4 row-major, B: 4x8 (element (k, n) at B[k * 8 + n]), C/D: 8x8 row-major.
__global__ void k_mma(const double *A, const double *B, const double *C, double *D, int reps) {
    const int lane = threadIdx.x;
    const int t = blockIdx.x;
    const double *a = A + 32 * t, *b = B + 32 * t, *c = C + 64 * t;
    double *d = D + 64 * t;
    const double av = a[(lane >> 2) * 4 + (lane & 3)];
    const double bv = b[(lane & 3) * 8 + (lane >> 2)];
    double c0 = c[(lane >> 2) * 8 + (lane & 3) * 2], c1 = c[(lane >> 2) * 8 + (lane & 3) * 2 + 1];
    for (int r = 0; r < reps; r++) dmma(c0, c1, av, bv, c0, c1);
    d[(lane >> 2) * 8 + (lane & 3) * 2] = c0;
    d[(lane >> 2) * 8 + (lane & 3) * 2 + 1] = c1;
}

// throughput: independent accumulators per warp
__global__ void k_mma_rate(double *out, int iters) {
    const int lane = threadIdx.x & 31;
    double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
    double c[8][2];
    for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) dmma(c[i][0], c[i][1], a, b, c[i][0], c[i][1]);
    }
    double s = 0;
    for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fma_rate(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
    double c[16];
    for (int i = 0; i < 16; i++) c[i] = 0.0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) c[i] = fma(a, b, c[i]);
    }
    double s = 0;
    for (int i = 0; i < 16; i++) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static double rnd(uint64_t &s) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    const double u = (double)(s >> 11) * (1.0 / 9007199254740992.0);
    const int e = (int)(s % 41) - 20;  // wide magnitudes to expose rounding
    return (u - 0.5) * std::ldexp(1.0, e);
}

int main() {
    const int T = 1 << 16;
    double *A, *B, *C, *D;
    cudaMallocManaged(&A, sizeof(double) * 32 * T);
    cudaMallocManaged(&B, sizeof(double) * 32 * T);
    cudaMallocManaged(&C, sizeof(double) * 64 * T);
    cudaMallocManaged(&D, sizeof(double) * 64 * T);
    uint64_t s = 88172645463325252ull;
    for (int i = 0; i < 32 * T; i++) A[i] = rnd(s), B[i] = rnd(s);
    for (int i = 0; i < 64 * T; i++) C[i] = rnd(s);
    k_mma<<<T, 32>>>(A, B, C, D, 1);
    cudaDeviceSynchronize();
    long seq = 0, rev = 0, pair = 0, total = 0;
    for (int t = 0; t < T; t++)
        for (int i = 0; i < 8; i++)
            for (int j = 0; j < 8; j++) {
                const double *a = A + 32 * t + 4 * i;
                const double *b = B + 32 * t;
                const double c = C[64 * t + 8 * i + j];
                double f = c;  // fma chain k = 0..3
                for (int k = 0; k < 4; k++) f = std::fma(a[k], b[k * 8 + j], f);
                double r = c;  // k = 3..0
                for (int k = 3; k >= 0; k--) r = std::fma(a[k], b[k * 8 + j], r);
                // pairwise: (a0b0 + a1b1) + (a2b2 + a3b3) + c, each product exact-ish via fma
                double p01 = std::fma(a[1], b[8 + j], a[0] * b[j]);
                double p23 = std::fma(a[3], b[24 + j], a[2] * b[16 + j]);
                double p = c + (p01 + p23);
                const double g = D[64 * t + 8 * i + j];
                seq += g == f;
                rev += g == r;
                pair += g == p;
                total++;
            }
    printf("{\"entries\": %ld, \"equal_fma_chain_k_ascending\": %ld, \"equal_fma_chain_k_descending\": %ld, \"equal_pairwise\": %ld}\n",
           total, seq, rev, pair);
    // rates
    double *out;
    cudaMalloc(&out, sizeof(double) * 148 * 8 * 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    k_mma_rate<<<148 * 8, 256>>>(out, 16);
    cudaEventRecord(e0);
    k_mma_rate<<<148 * 8, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mma_fma = 148.0 * 8 * 8 * (double)iters * 8 * 256;  // warps * iters * 8 mma * 256 FMA
    printf("{\"dmma_TFMA_per_s\": %.2f}\n", mma_fma / (ms * 1e-3) / 1e12);
    k_fma_rate<<<148 * 8, 256>>>(out, 16);
    cudaEventRecord(e0);
    k_fma_rate<<<148 * 8, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fma_n = 148.0 * 8 * 256 * (double)iters * 16;
    printf("{\"dfma_TFMA_per_s\": %.2f}\n", fma_n / (ms * 1e-3) / 1e12);
    return 0;
}
