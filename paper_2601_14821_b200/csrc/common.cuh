// common.cuh -- shared constants, device math and the per-view splat record.
//
// Arithmetic is float64 and the library is compiled with --fmad=false so the
// order of every multiply/add matches the reference's numpy/numba code
// (which never contracts to FMA); the few places where the reference itself
// runs through an FMA kernel (OpenBLAS dgemm, rasterizer.py:65) use explicit
// fma() to reproduce it.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/potr_b200.h"
#include "exp_table.h"

namespace potr {

// Bounds checks of a debug build (-DPOTR_CHECKS; compute-sanitizer is not
// available on this pool): a violated check fails the launch with a device
// assert.  Compiled out otherwise.
#ifdef POTR_CHECKS
#include <cassert>
#define POTR_CHECK(cond) assert(cond)
#else
#define POTR_CHECK(cond) ((void)0)
#endif

// rasterizer.py:22-26
constexpr double kAlphaFloor = 1.0 / 255.0;
constexpr double kAlphaCap = 0.999;
constexpr double kTTerminate = 1e-4;
constexpr double kNearClip = 0.01;
constexpr double kCovDilation = 0.3;

// sh.py:11-18
constexpr double kShDC = 0.28209479177387814;
constexpr double kShC1 = 0.4886025119029199;
constexpr double kShC2_0 = 1.0925484305920792;
constexpr double kShC2_1 = -1.0925484305920792;
constexpr double kShC2_2 = 0.31539156525252005;
constexpr double kShC2_3 = -1.0925484305920792;
constexpr double kShC2_4 = 0.5462742152960396;
constexpr double kShC3_0 = -0.5900435899266435;
constexpr double kShC3_1 = 2.890611442640554;
constexpr double kShC3_2 = -0.4570457994644658;
constexpr double kShC3_3 = 0.3731763325901154;
constexpr double kShC3_4 = -0.4570457994644658;
constexpr double kShC3_5 = 1.445305721320277;
constexpr double kShC3_6 = -0.5900435899266435;

// Tile geometry of the rasterizer: 8x4-pixel tiles, one warp per tile (lane =
// pixel), so a tile's front-to-back walk needs no block barrier and every
// listed splat overlaps the warp's pixels.
constexpr int kTileW = 8;
constexpr int kTileH = 4;
constexpr int kTileWLog2 = 3;
constexpr int kTileHLog2 = 2;
constexpr int kRasterWarps = 4;  // warps (= independent tile workers) per CTA

// Prefilter margin on the Gaussian exponent: power < log(floor/o) - margin
// guarantees o*exp(power) < floor for any exp with < 1e-12 relative error,
// so the full-precision exp is evaluated only where the floor test could pass.
constexpr double kPowerMargin = 1e-9;

__constant__ double kExpTable[64][2] = POTR_EXP_TABLE_INIT;

// exp_neg's scalar constants in the constant bank: DFMA/DMUL/DADD take them
// as c[][] operands, so the hot loops do not rematerialise 64-bit immediates
// (two UMOVs each) on every iteration.
__constant__ double kExpK[8] = {POTR_EXP_INV_STEP, POTR_EXP_SHIFT, -POTR_EXP_STEP_HI,
                                -POTR_EXP_STEP_LO, POTR_EXP_C2, POTR_EXP_C3,
                                POTR_EXP_C4, POTR_EXP_C5};

// The compositing thresholds, for the same reason (DSETP takes c[][] operands).
__constant__ double kCompositeK[3] = {kAlphaCap, kAlphaFloor, kTTerminate};

// 1/d for d in [0.01, 1]: the MUFU approximation refined by two Newton steps
// (relative error below 2^-52; not correctly rounded, which the removal
// scores' 1e-4 tolerance does not need).
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// exp(x) for the Gaussian exponent after the ALPHA_FLOOR prefilter
// (x in [log(ALPHA_FLOOR), 0]).  Table-driven (2^(j/64) double-double, held
// in shared memory) with a degree-5 Estrin polynomial: 11 FP64 operations and
// a 6-deep dependency chain instead of the libdevice exp's ~19 / 17, at
// < 0.82 ulp (tests/test_exp.py; the reference's glibc exp is ~0.5 ulp).
// 16-byte shared load from a 32-bit shared-window address held in a register.
__device__ __forceinline__ double2 lds_double2(unsigned addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}

// tab_s: shared-window address of the 64-entry table (kExpTable copied to
// shared memory by the caller).
__device__ __forceinline__ double exp_neg(double x, unsigned tab_s) {
    const double t = fma(x, kExpK[0], kExpK[1]);
    const double k = t - kExpK[1];
    const int ki = __double2loint(t);
    double r = fma(k, kExpK[2], x);
    r = fma(k, kExpK[3], r);
    const double r2 = r * r;
    const double a = fma(r, kExpK[5], kExpK[4]);
    const double b = fma(r, kExpK[7], kExpK[6]);
    const double q = fma(r2, b, a);
    const double p = fma(r2, q, r);
    const double2 T = lds_double2(tab_s + ((unsigned)(ki & 63) << 4));
    const double res = fma(T.x, p, T.y) + T.x;
    return __hiloint2double(__double2hiint(res) + (ki >> 6) * (1 << 20), __double2loint(res));
}

// Per-view splat record, 96 bytes, written by the preprocess kernel and read
// per (tile, splat) pair by the rasterizer.
// Six 16-byte fields: the exponent and its prefilter need the first three,
// a composited sample the last two; the duplicate kernel's cull test reads
// only the first 64 bytes (two sectors).
struct __align__(16) SplatRec {
    double mx, my;      // mean2d
    double ha, ib;      // conic (a, b, c) = (c, -b, a) / det (rasterizer.py:149-154): ha = -a/2
    double hc, pthr;    // hc = -c/2; pthr = log(ALPHA_FLOOR / opac) - margin
    int32_t x0, x1, y0, y1;  // clipped pixel bbox (:135-148), inclusive
    double opac, cr;    // opacity, compositing colour clamped at 0 (:100-110)
    double cg, cb;
};
static_assert(sizeof(SplatRec) == 96, "SplatRec must stay 96 bytes");

// sh.py:23-51 -- the 16 real SH bases, 3DGS signs.
__device__ __forceinline__ void sh_basis16(double x, double y, double z, double *o) {
    double xx = x * x, yy = y * y, zz = z * z;
    double xy = x * y, yz = y * z, xz = x * z;
    o[0] = kShDC;
    o[1] = -kShC1 * y;
    o[2] = kShC1 * z;
    o[3] = -kShC1 * x;
    o[4] = kShC2_0 * xy;
    o[5] = kShC2_1 * yz;
    o[6] = kShC2_2 * (2.0 * zz - xx - yy);
    o[7] = kShC2_3 * xz;
    o[8] = kShC2_4 * (xx - yy);
    o[9] = kShC3_0 * y * (3.0 * xx - yy);
    o[10] = kShC3_1 * xy * z;
    o[11] = kShC3_2 * y * (4.0 * zz - xx - yy);
    o[12] = kShC3_3 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    o[13] = kShC3_4 * x * (4.0 * zz - xx - yy);
    o[14] = kShC3_5 * z * (xx - yy);
    o[15] = kShC3_6 * x * (xx - 3.0 * yy);
}

// Device-side camera (same layout as potr_camera).
struct Cam {
    double eye[3];
    double rot[9];
    double fx, fy, cx, cy;
    int32_t width, height;
};
static_assert(sizeof(Cam) == sizeof(potr_camera), "camera layout");

// Views processed together by one pipeline round (one preprocess, one scan,
// one duplicate, one tile sort, one persistent raster launch).
constexpr int kMaxViewBatch = 8;

struct CamBatch {
    Cam cam[kMaxViewBatch];
};

struct Proj {
    double mx, my, a, b, c, depth, radius;
    bool valid;
};

// Tile rows of a drawn (splat, view) entry as the preprocess culled them, so
// the duplicate kernel need not redo the ellipse test: rows [ty0, ty0 + nrows),
// tile columns [c[2r], c[2r+1]] of the first kSpanRows rows (c0 > c1: culled
// row).  Entries with more rows are recomputed from the record.
constexpr int kSpanRows = 3;
struct __align__(16) TileSpan {
    uint16_t ty0, nrows;
    uint16_t c[2 * kSpanRows];
};
static_assert(sizeof(TileSpan) == 16, "TileSpan must stay 16 bytes");

// View-independent per-splat terms, computed once per call (k_splat_prep)
// and read by the preprocess of every view batch.
struct __align__(16) SplatPrep {
    double S[9];  // Sigma, all nine entries (the sums are not exactly symmetric)
    double pthr;  // log(ALPHA_FLOOR / opacity) - margin
};
static_assert(sizeof(SplatPrep) == 80, "SplatPrep must stay 80 bytes");

// Sigma = R diag(s^2) R^T (rasterizer.py:75-76, quat_to_rotmat :40-53).
__device__ __forceinline__ void splat_sigma(const double *__restrict__ s,
                                            const double *__restrict__ q, double *S) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    double R[9];
    R[0] = 1 - 2 * (y * y + z * z);
    R[1] = 2 * (x * y - w * z);
    R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);
    R[4] = 1 - 2 * (x * x + z * z);
    R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);
    R[7] = 2 * (y * z + w * x);
    R[8] = 1 - 2 * (x * x + y * y);
    double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int k = 0; k < 3; k++) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 3; j++) acc += R[i * 3 + j] * s2[j] * R[k * 3 + j];
            S[i * 3 + k] = acc;
        }
}

// project_splats for one splat given its Sigma (rasterizer.py:64-97).  The
// sums follow numpy's einsum order term by term; in J V J^T the terms with a
// structural zero of J are dropped (adding them changes nothing but the sign
// of an exact zero).
__device__ __forceinline__ Proj project_sigma(const double *__restrict__ p,
                                              const double *__restrict__ S, const Cam &cam) {
    const double *W = cam.rot;
    double d0 = p[0] - cam.eye[0], d1 = p[1] - cam.eye[1], d2 = p[2] - cam.eye[2];
    // (positions - eye) @ W.T: OpenBLAS accumulates with FMA in index order.
    double t0 = fma(d2, W[2], fma(d1, W[1], d0 * W[0]));
    double t1 = fma(d2, W[5], fma(d1, W[4], d0 * W[3]));
    double t2 = fma(d2, W[8], fma(d1, W[7], d0 * W[6]));
    Proj o;
    o.valid = t2 > kNearClip;
    double safe_z = o.valid ? t2 : 1.0;
    double inv_z = 1.0 / safe_z;
    o.mx = cam.fx * t0 * inv_z + cam.cx;
    o.my = cam.fy * t1 * inv_z + cam.cy;
    // Sigma_view = W Sigma W^T, entry (i, l) = sum_j sum_k W_ij S_jk W_lk
    double V[9];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int l = 0; l < 3; l++) {
            if (i == 1 && l == 0) continue;  // unused by J V J^T
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 3; j++)
#pragma unroll
                for (int k = 0; k < 3; k++) acc += W[i * 3 + j] * S[j * 3 + k] * W[l * 3 + k];
            V[i * 3 + l] = acc;
        }
    const double j00 = cam.fx * inv_z, j02 = -cam.fx * t0 * inv_z * inv_z;
    const double j11 = cam.fy * inv_z, j12 = -cam.fy * t1 * inv_z * inv_z;
    // cov = J V J^T with J = [[j00, 0, j02], [0, j11, j12]]
    double c00 = 0.0, c01 = 0.0, c11 = 0.0;
    c00 += j00 * V[0] * j00;
    c00 += j00 * V[2] * j02;
    c00 += j02 * V[6] * j00;
    c00 += j02 * V[8] * j02;
    c01 += j00 * V[1] * j11;
    c01 += j00 * V[2] * j12;
    c01 += j02 * V[7] * j11;
    c01 += j02 * V[8] * j12;
    c11 += j11 * V[4] * j11;
    c11 += j11 * V[5] * j12;
    c11 += j12 * V[7] * j11;
    c11 += j12 * V[8] * j12;
    o.a = c00 + kCovDilation;
    o.b = c01;
    o.c = c11 + kCovDilation;
    double mid = 0.5 * (o.a + o.c);
    double det = o.a * o.c - o.b * o.b;
    double disc = mid * mid - det;
    double lam_max = mid + sqrt(disc > 0.0 ? disc : 0.0);
    o.radius = 3.0 * sqrt(lam_max);
    o.depth = t2;
    o.valid = o.valid && (o.mx >= -o.radius) && (o.mx <= cam.width + o.radius);
    o.valid = o.valid && (o.my >= -o.radius) && (o.my <= cam.height + o.radius);
    return o;
}

__device__ __forceinline__ Proj project_one(const double *__restrict__ p,
                                            const double *__restrict__ s,
                                            const double *__restrict__ q, const Cam &cam) {
    double S[9];
    splat_sigma(s, q, S);
    return project_sigma(p, S, cam);
}

// splat_colors for one splat (rasterizer.py:100-110): SH at the unit
// direction eye -> centre, clamped at zero, no +0.5 offset.
__device__ __forceinline__ void splat_color(const double *__restrict__ p,
                                            const double *__restrict__ sh, const Cam &cam,
                                            double *rgb) {
    double d0 = p[0] - cam.eye[0], d1 = p[1] - cam.eye[1], d2 = p[2] - cam.eye[2];
    double norm = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    if (norm == 0.0) norm = 1.0;
    double basis[16];
    sh_basis16(d0 / norm, d1 / norm, d2 / norm, basis);
    const double2 *sh2 = reinterpret_cast<const double2 *>(sh);
#pragma unroll
    for (int ch = 0; ch < 3; ch++) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            double2 v = __ldg(sh2 + ch * 8 + i);
            acc += v.x * basis[2 * i];
            acc += v.y * basis[2 * i + 1];
        }
        rgb[ch] = acc > 0.0 ? acc : 0.0;
    }
}

}  // namespace potr
