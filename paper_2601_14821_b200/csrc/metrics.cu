// metrics.cu -- image-quality metrics on the device:
// the MSE behind psnr (metrics.py:24-30) and the windowed SSIM (:33-52) of
// two (H, W, 3) float64 renders, both clamped to [0, 1] first.
//
// SSIM follows the reference's scipy formulation: per channel, the five
// moment images (a, b, a*a, b*b, a*b) are blurred by gaussian_filter (sigma
// 1.5, truncate 3.5 -> radius 5, mode 'reflect' = half-sample symmetric),
// axis 0 then axis 1, each 1-D pass restating scipy's symmetric correlate1d
// (centre tap, then the tap pairs from the outermost in); the SSIM map is
// averaged over the border-cropped interior [5, H-5) x [5, W-5), and the
// three channel means are averaged.  Reductions use fixed-order block
// partials, so results are run-to-run identical.
#include "common.cuh"
#include "raster.cuh"

namespace potr {

constexpr int kSsimRadius = 5;
constexpr double kSsimC1 = 0.01 * 0.01;
constexpr double kSsimC2 = 0.03 * 0.03;
constexpr int kMetricBlocks = 296;  // 2 x 148 SMs, fixed so the sum order is too
constexpr int kMetricThreads = 256;

__device__ __forceinline__ double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }

// mode='reflect': (d c b a | a b c d | d c b a)
__device__ __forceinline__ int reflect(int i, int n) {
    if (n == 1) return 0;
    while (i < 0 || i >= n) i = i < 0 ? -i - 1 : 2 * n - i - 1;
    return i;
}

__device__ __forceinline__ double block_sum(double v, double *red) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += red[i];
    __syncthreads();
    return t;
}

// Per-block partial sums of the clamped squared difference.
__global__ void __launch_bounds__(kMetricThreads) k_sq_diff(int64_t m, const double *__restrict__ a,
                                                            const double *__restrict__ b,
                                                            double *__restrict__ partial) {
    __shared__ double red[kMetricThreads / 32];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = clamp01(a[i]) - clamp01(b[i]);
        s += d * d;
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// Axis-0 (vertical) pass of the five moments of channel ch.
__global__ void k_ssim_vertical(int W, int H, int ch, const double *__restrict__ a,
                                const double *__restrict__ b, const double *__restrict__ w,
                                double *__restrict__ mom) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= W) return;
    double q[5];
    auto load = [&](int yy, double *v) {
        const int64_t p = ((int64_t)reflect(yy, H) * W + x) * 3 + ch;
        const double va = clamp01(a[p]), vb = clamp01(b[p]);
        v[0] = va;
        v[1] = vb;
        v[2] = va * va;
        v[3] = vb * vb;
        v[4] = va * vb;
    };
    double c[5];
    load(y, c);
#pragma unroll
    for (int k = 0; k < 5; k++) q[k] = c[k] * w[kSsimRadius];
    for (int j = kSsimRadius; j >= 1; j--) {
        double lo[5], hi[5];
        load(y - j, lo);
        load(y + j, hi);
#pragma unroll
        for (int k = 0; k < 5; k++) q[k] += (hi[k] + lo[k]) * w[kSsimRadius - j];
    }
    const int64_t plane = (int64_t)W * H, p = (int64_t)y * W + x;
#pragma unroll
    for (int k = 0; k < 5; k++) mom[k * plane + p] = q[k];
}

// Axis-1 (horizontal) pass, the SSIM map, and per-block partial sums over the
// cropped interior.
__global__ void __launch_bounds__(kMetricThreads) k_ssim_horizontal(
    int W, int H, const double *__restrict__ mom, const double *__restrict__ w,
    double *__restrict__ partial) {
    __shared__ double red[kMetricThreads / 32];
    const int pad = kSsimRadius;
    const int64_t cw = W - 2 * pad, chh = H - 2 * pad;
    const int64_t m = cw > 0 && chh > 0 ? cw * chh : 0;
    const int64_t plane = (int64_t)W * H;
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int y = pad + (int)(i / cw), x = pad + (int)(i % cw);
        double q[5];
        const int64_t row = (int64_t)y * W;
#pragma unroll
        for (int k = 0; k < 5; k++) q[k] = mom[k * plane + row + x] * w[kSsimRadius];
        for (int j = kSsimRadius; j >= 1; j--) {
            const int xl = reflect(x - j, W), xr = reflect(x + j, W);
#pragma unroll
            for (int k = 0; k < 5; k++)
                q[k] += (mom[k * plane + row + xr] + mom[k * plane + row + xl]) * w[kSsimRadius - j];
        }
        const double mu_a = q[0], mu_b = q[1];
        const double var_a = q[2] - mu_a * mu_a, var_b = q[3] - mu_b * mu_b;
        const double cov = q[4] - mu_a * mu_b;
        s += ((2 * mu_a * mu_b + kSsimC1) * (2 * cov + kSsimC2)) /
             ((mu_a * mu_a + mu_b * mu_b + kSsimC1) * (var_a + var_b + kSsimC2));
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_sum_partials(int nparts, const double *__restrict__ partial, double *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double t = 0.0;
    for (int i = 0; i < nparts; i++) t += partial[i];
    *out = t;
}

// out[0] = sum of clamped squared differences, out[1 + ch] = sum of the
// cropped SSIM map of channel ch (NaN-free; an empty crop gives 0).
cudaError_t launch_image_compare(int W, int H, const double *a, const double *b,
                                 const double *gauss_w, double *mom, double *partial, double *out,
                                 cudaStream_t st) {
    const int64_t m = (int64_t)W * H * 3;
    k_sq_diff<<<kMetricBlocks, kMetricThreads, 0, st>>>(m, a, b, partial);
    k_sum_partials<<<1, 32, 0, st>>>(kMetricBlocks, partial, out);
    for (int ch = 0; ch < 3; ch++) {
        dim3 g((W + 127) / 128, H);
        k_ssim_vertical<<<g, 128, 0, st>>>(W, H, ch, a, b, gauss_w, mom);
        k_ssim_horizontal<<<kMetricBlocks, kMetricThreads, 0, st>>>(W, H, mom, gauss_w,
                                                                     partial + kMetricBlocks);
        k_sum_partials<<<1, 32, 0, st>>>(kMetricBlocks, partial + kMetricBlocks, out + 1 + ch);
    }
    return cudaGetLastError();
}

int image_compare_partials() { return 2 * kMetricBlocks; }

}  // namespace potr
