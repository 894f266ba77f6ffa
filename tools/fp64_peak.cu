// Measured FP64 DFMA throughput of this B200 (the roofline denominator of the
// fp64 rasterizer / SH kernels): 148 SMs x full occupancy, 16 independent FMA
// chains per thread, timed with CUDA events after a warm-up.  Prints JSON.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_dfma(double *out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 16; i++) s += x[i];
    if (s == 12345.678) out[0] = s;  // keep the work
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double *out;
    cudaMalloc(&out, 8);
    const int blocks = sms * 8, threads = 256, iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; r++) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double fmas = (double)blocks * threads * iters * 16;
    const double rate = fmas / (best * 1e-3) / 1e12;
    printf("{\"fp64_fma_tera_per_s\": %.4f, \"fp64_tflops\": %.4f, \"sms\": %d, "
           "\"clock_rate_khz\": %d, \"nominal_fma_tera_per_s_at_1965\": %.4f, "
           "\"how\": \"%d blocks x %d threads x %d iters x 16 independent DFMA chains, best of 10, "
           "CUDA events\"}\n",
           rate, 2 * rate, sms, clk, sms * 64 * 1.965e9 / 1e12, blocks, threads, iters);
    return 0;
}
