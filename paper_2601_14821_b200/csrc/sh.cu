// sh.cu -- kernel (e): training-free SH recompute (compaction.py:89-243).
//
// The reference builds, per splat, Y = basis * w and C = YCoCg(basis . sh^T) * w
// over the cameras that see it (compaction.py:89-107) and then only ever uses
// Y^T Y and Y^T C (sparsify :110-124, ridge :127-148).  So the GPU never
// materialises Y: k_sh_accumulate streams the (S, N) per-camera importances
// once and accumulates, per splat, the 16x16 Gram matrix G (136 unique
// entries) and the 16x3 right-hand sides B in fp64 registers -- eight lanes
// per splat, each owning rows {g, 15-g} -- in camera order, exactly the
// summation order of the reference's row loop.  k_sh_solve then does the
// parallel-column sparsification, the two-pass ridge (Cholesky, with the
// reference's 1e-10 jitter retry and RidgeError semantics) and the DC
// fallback for unseen splats, one thread per splat.
//
// Precision: fp64.  The north-star suggested fp32 solves; the reference's own
// lambda sweep (tests/test_compaction.py:310-319, lambda down to 1e-9) makes
// these 16x16 systems far too ill-conditioned for fp32 to meet the 1e-4
// coefficient tolerance, and B200 runs fp64 at half the fp32 rate.
#include "common.cuh"
#include "raster.cuh"

namespace potr {

__device__ __forceinline__ int tri(int i, int j) { return i * 16 - (i * (i - 1)) / 2 + (j - i); }

// compaction.py:19-28
__constant__ double kRgbToYcocg[9] = {0.25, 0.5, 0.25, 0.5, 0.0, -0.5, -0.25, 0.5, -0.25};
__constant__ double kYcocgToRgb[9] = {1.0, 1.0, -1.0, 1.0, 0.0, 1.0, 1.0, -1.0, -1.0};

__global__ void __launch_bounds__(256) k_sh_accumulate(potr_splats sp, int ncam,
                                                       const double *__restrict__ eyes,
                                                       const double *__restrict__ cam_imp,
                                                       double *__restrict__ neq) {
    const int64_t n = sp.n;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k = gid >> 3;
    const int g = threadIdx.x & 7;
    const unsigned gmask = 0xffu << (threadIdx.x & 24);
    const bool active = k < n;
    const int64_t kk = active ? k : 0;
    if (n == 0) return;
    const double px = sp.positions[3 * kk], py = sp.positions[3 * kk + 1],
                 pz = sp.positions[3 * kk + 2];
    const int ch = g < 3 ? g : 0;
    double shc[16];
#pragma unroll
    for (int i = 0; i < 16; i++) shc[i] = sp.sh[48 * kk + ch * 16 + i];
    const int ra = g, rb = 15 - g;
    double ga[16], gb[16], ba[3], bb[3];
#pragma unroll
    for (int j = 0; j < 16; j++) ga[j] = gb[j] = 0.0;
#pragma unroll
    for (int c = 0; c < 3; c++) ba[c] = bb[c] = 0.0;
    int seen = 0;
    for (int s = 0; s < ncam; s++) {
        const double w = active ? cam_imp[(int64_t)s * n + k] : 0.0;
        if (!(w > 0.0)) continue;  // compaction.py:97 seen = w > 0
        double d0 = px - eyes[3 * s], d1 = py - eyes[3 * s + 1], d2 = pz - eyes[3 * s + 2];
        double nrm = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        double y[16];
        sh_basis16(d0 / nrm, d1 / nrm, d2 / nrm, y);
        double col = 0.0;
#pragma unroll
        for (int i = 0; i < 16; i++) col += y[i] * shc[i];
        double c0 = __shfl_sync(gmask, col, 0, 8);
        double c1 = __shfl_sync(gmask, col, 1, 8);
        double c2 = __shfl_sync(gmask, col, 2, 8);
        double cw[3];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            double yc = c0 * kRgbToYcocg[c * 3] + c1 * kRgbToYcocg[c * 3 + 1] +
                        c2 * kRgbToYcocg[c * 3 + 2];
            cw[c] = yc * w;
        }
        double yw[16];
#pragma unroll
        for (int i = 0; i < 16; i++) yw[i] = y[i] * w;
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int i = 0; i < 16; i++) {
            a = (i == ra) ? yw[i] : a;
            b = (i == rb) ? yw[i] : b;
        }
#pragma unroll
        for (int j = 0; j < 16; j++) {
            ga[j] += a * yw[j];
            gb[j] += b * yw[j];
        }
#pragma unroll
        for (int c = 0; c < 3; c++) {
            ba[c] += a * cw[c];
            bb[c] += b * cw[c];
        }
        seen++;
    }
    if (!active) return;
#pragma unroll
    for (int j = 0; j < 16; j++) {
        if (j >= ra) neq[(int64_t)tri(ra, j) * n + k] += ga[j];
        if (j >= rb) neq[(int64_t)tri(rb, j) * n + k] += gb[j];
    }
#pragma unroll
    for (int c = 0; c < 3; c++) {
        neq[(int64_t)(136 + ra * 3 + c) * n + k] += ba[c];
        neq[(int64_t)(136 + rb * 3 + c) * n + k] += bb[c];
    }
    if (g == 0) neq[(int64_t)184 * n + k] += (double)seen;
}

// Upper Cholesky of the m x m principal block, packed with tri() (LAPACK
// dpotrf 'U' semantics: a pivot <= 0 or NaN fails).
__device__ int chol_upper(double *A, int m) {
    for (int j = 0; j < m; j++) {
        double ajj = A[tri(j, j)];
        for (int k = 0; k < j; k++) ajj -= A[tri(k, j)] * A[tri(k, j)];
        if (!(ajj > 0.0)) return j + 1;
        ajj = sqrt(ajj);
        A[tri(j, j)] = ajj;
        for (int c = j + 1; c < m; c++) {
            double v = A[tri(j, c)];
            for (int k = 0; k < j; k++) v -= A[tri(k, j)] * A[tri(k, c)];
            A[tri(j, c)] = v / ajj;
        }
    }
    return 0;
}

// dpotrs: U^T y = b, U x = y
__device__ void chol_solve(const double *U, int m, double *b) {
    for (int i = 0; i < m; i++) {
        double v = b[i];
        for (int k = 0; k < i; k++) v -= U[tri(k, i)] * b[k];
        b[i] = v / U[tri(i, i)];
    }
    for (int i = m - 1; i >= 0; i--) {
        double v = b[i];
        for (int k = i + 1; k < m; k++) v -= U[tri(i, k)] * b[k];
        b[i] = v / U[tri(i, i)];
    }
}

// _solve_channel (compaction.py:127-148) on the normal equations.
// Returns 0 ok, 1 ok after jitter, -1 RidgeError.
__device__ int solve_channel(const double *G, const double *B, int ch, const bool *mask,
                             double lam, double *out) {
    int cols[16];
    int m = 0;
    for (int i = 0; i < 16; i++)
        if (mask[i]) cols[m++] = i;
    double A[136], Asave[136], b[16];
    for (int i = 0; i < m; i++) {
        for (int j = i; j < m; j++) A[tri(i, j)] = G[tri(cols[i], cols[j])];
        A[tri(i, i)] += (cols[i] == 0) ? 0.0 : lam;
        b[i] = B[cols[i] * 3 + ch];
    }
    for (int i = 0; i < m; i++)
        for (int j = i; j < m; j++) Asave[tri(i, j)] = A[tri(i, j)];
    int status = 0;
    if (chol_upper(A, m)) {
        for (int i = 0; i < m; i++)
            for (int j = i; j < m; j++) A[tri(i, j)] = Asave[tri(i, j)];
        for (int i = 0; i < m; i++) A[tri(i, i)] += 1e-10;
        if (chol_upper(A, m)) return -1;
        status = 1;
    }
    chol_solve(A, m, b);
    for (int i = 0; i < 16; i++) out[i] = 0.0;
    for (int i = 0; i < m; i++) out[cols[i]] = b[i];
    return status;
}

__device__ void coeffs_convert(const double *M, const double *in, double *out) {
    for (int i = 0; i < 3; i++)
        for (int c = 0; c < 16; c++) {
            double acc = 0.0;
            for (int j = 0; j < 3; j++) acc += M[i * 3 + j] * in[j * 16 + c];
            out[i * 16 + c] = acc;
        }
}

__global__ void __launch_bounds__(128) k_sh_solve(potr_splats sp, const double *__restrict__ neq,
                                                  double lambda_y, double par_thr,
                                                  double zero_thr, double *__restrict__ rgb_out,
                                                  double *__restrict__ ycocg_out,
                                                  int8_t *__restrict__ status_out) {
    const int64_t n = sp.n;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double *sh = sp.sh + 48 * k;
    double rgb[48], yc[48];
    int status = 0;
    if (neq[(int64_t)184 * n + k] == 0.0) {
        // _fallback_dc (compaction.py:161-166) over the 26 cube probes (:32-37)
        double acc[3] = {0.0, 0.0, 0.0};
        for (int i = -1; i <= 1; i++)
            for (int j = -1; j <= 1; j++)
                for (int q = -1; q <= 1; q++) {
                    if (i == 0 && j == 0 && q == 0) continue;
                    double nrm = sqrt((double)(i * i) + (double)(j * j) + (double)(q * q));
                    double basis[16];
                    sh_basis16(i / nrm, j / nrm, q / nrm, basis);
                    for (int c = 0; c < 3; c++) {
                        double col = 0.0;
                        for (int t = 0; t < 16; t++) col += basis[t] * sh[c * 16 + t];
                        acc[c] += col;
                    }
                }
        for (int i = 0; i < 48; i++) rgb[i] = 0.0;
        for (int c = 0; c < 3; c++) rgb[c * 16] = acc[c] / 26.0 / kShDC;
        coeffs_convert(kRgbToYcocg, rgb, yc);
        status = 3;
    } else {
        double G[136], B[48];
        for (int e = 0; e < 136; e++) G[e] = neq[(int64_t)e * n + k];
        for (int e = 0; e < 48; e++) B[e] = neq[(int64_t)(136 + e) * n + k];
        // sparsify_parallel_columns (compaction.py:110-124)
        double norms[16];
        for (int i = 0; i < 16; i++) norms[i] = sqrt(G[tri(i, i)]);
        bool mask[16];
        for (int i = 0; i < 16; i++) mask[i] = (i == 0);
        for (int i = 1; i < 16; i++) {
            if (norms[i] == 0.0) continue;
            bool par = false;
            for (int j = 0; j < i; j++) {
                if (!mask[j]) continue;
                double gij = j < i ? G[tri(j, i)] : G[tri(i, j)];
                double cs = fabs(gij) / (norms[i] * norms[j]);
                if (cs > par_thr) par = true;
            }
            mask[i] = !par;
        }
        const double lam[3] = {lambda_y, 3.0 * lambda_y, 3.0 * lambda_y};
        for (int ch = 0; ch < 3 && status != 2; ch++) {
            double first[16];
            int rc = solve_channel(G, B, ch, mask, lam[ch], first);
            if (rc < 0) {
                status = 2;
                break;
            }
            if (rc > 0) status = 1;
            bool m2[16];
            for (int i = 0; i < 16; i++) m2[i] = mask[i] && !(i > 0 && fabs(first[i]) < zero_thr);
            rc = solve_channel(G, B, ch, m2, lam[ch], yc + ch * 16);
            if (rc < 0) {
                status = 2;
                break;
            }
            if (rc > 0) status = 1;
        }
        if (status == 2) {
            for (int i = 0; i < 48; i++) rgb[i] = sh[i];
            coeffs_convert(kRgbToYcocg, rgb, yc);
        } else {
            coeffs_convert(kYcocgToRgb, yc, rgb);
        }
    }
    for (int i = 0; i < 48; i++) {
        rgb_out[48 * k + i] = rgb[i];
        ycocg_out[48 * k + i] = yc[i];
    }
    status_out[k] = (int8_t)status;
}

cudaError_t launch_sh_accumulate(const potr_splats &sp, int ncam, const double *eyes_dev,
                                 const double *cam_imp, double *neq, cudaStream_t st) {
    if (sp.n == 0) return cudaSuccess;
    int64_t threads = sp.n * 8;
    k_sh_accumulate<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(sp, ncam, eyes_dev, cam_imp,
                                                                        neq);
    return cudaGetLastError();
}

cudaError_t launch_sh_solve(const potr_splats &sp, const double *neq, double lambda_y,
                            double par_thr, double zero_thr, double *rgb, double *ycocg,
                            int8_t *status, cudaStream_t st) {
    if (sp.n == 0) return cudaSuccess;
    k_sh_solve<<<(unsigned)((sp.n + 127) / 128), 128, 0, st>>>(sp, neq, lambda_y, par_thr,
                                                                zero_thr, rgb, ycocg, status);
    return cudaGetLastError();
}

}  // namespace potr
