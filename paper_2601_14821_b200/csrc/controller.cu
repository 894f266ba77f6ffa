// controller.cu -- device half of the pruning controller (pruning.py:57-111):
// the removal priority m(dMSE / dMSE_MAX) of every candidate as an
// order-preserving 64-bit key, sorted by the library's stable radix sort
// (sort.cu) == np.argsort(mapping_m(...), kind="stable").
#include "common.cuh"
#include "raster.cuh"

namespace potr {

// mapping_m (pruning.py:57-66) with numpy's operation order: x = dm / max
// (IEEE division), xn = min(x, 0), neg = (sqrt(1 - (2 a) xn) - 1) / a,
// m = x >= 0 ? x : neg.  The library is built with --fmad=false, so nothing
// is contracted.  The key maps the double to an unsigned integer with the
// same total order (-0 folded onto +0, NaN last as in np.argsort).
__global__ void k_removal_keys(int64_t n, const double *__restrict__ dm,
                               const int64_t *__restrict__ idx, double dmax, double two_a,
                               double a, uint64_t *__restrict__ keys) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = dm[idx ? idx[i] : i] / dmax;
    const double xn = x < 0.0 ? x : 0.0;
    const double neg = (sqrt(1.0 - two_a * xn) - 1.0) / a;
    double m = x >= 0.0 ? x : neg;
    if (m == 0.0) m = 0.0;  // -0 -> +0: equal keys, stable order decides
    uint64_t b = (uint64_t)__double_as_longlong(m);
    if (m != m) b = 0x7ff8000000000000ull;  // every NaN after +inf
    keys[i] = (b >> 63) ? ~b : (b | (1ull << 63));
}

cudaError_t launch_removal_keys(int64_t n, const double *dm, const int64_t *idx, double dmax,
                                double a, uint64_t *keys, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    // numpy: 2.0 * a * xn evaluates (2.0 * a) first (a Python float)
    k_removal_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, dm, idx, dmax, 2.0 * a, a,
                                                                keys);
    return cudaGetLastError();
}

__global__ void k_iota64(int64_t n, int64_t *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

cudaError_t launch_iota64(int64_t n, int64_t *out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_iota64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, out);
    return cudaGetLastError();
}

}  // namespace potr
