// raster.cu -- the prune-score pass on sm_100a: kernels (a)-(d).  All work is
// done for a batch of up to 8 equal-size views at a time, in "slot space":
// once per call the splats are ordered by the Morton code of their centres
// (k_morton + radix sort, sort.cu) and copied in that order with their view-independent
// terms (k_splat_slots), so that the records a tile reads are close together
// in HBM; slots map back to splat indices where results leave (raster.cuh).
//
//  (a) k_preprocess: one thread per (slot, view): EWA projection, cov2d,
//      radius, clipped bbox, conic, SH colour, compact depth key, culled tile
//      rows and count (rasterizer.py:56-110, :135-154)
//  (b) depth order: radix sort (sort.cu) of the 32-bit hi part of the depth key +
//      k_depth_fixup (runs of equal hi ordered by the full key, exact ties by
//      splat index) == np.argsort(kind="stable") (:248-250); scan of the
//      counts in depth order, k_duplicate (pairs in depth order, tiles culled
//      by the prefilter ellipse), stable radix sort on 16-bit tile keys,
//      k_tile_ranges: every tile gets its splats in (tile, depth, id) order.
//  (c)+(d) k_raster    persistent warps, one warp per 8x4-pixel tile (lane =
//      pixel).  Pass 1 composites front to back with the reference's exact
//      per-pixel rules (:159-201), each lane walking only the chunk entries
//      whose bbox and prefilter ellipse reach its pixel; the replay revisits
//      the composited samples and evaluates the closed-form removal delta
//      PD = a/(1-a) (P_K - P_i - T c) (:232-243), dSE = sum_ch PD^2 +
//      2 PD (c - c_t) (:333) and T*alpha (:228), adding them per (tile,
//      splat) slot in a fixed lane order -- no floating-point atomics, so
//      scores are bit-reproducible.
//  k_splat_reduce / k_view_accumulate / k_mse_reduce: per splat, its slots in
//      tile order, divided by P / 3P, added in camera order (:226-230, :334,
//      :340-347).
#include "common.cuh"
#include "raster.cuh"
#include "sort.cuh"

#ifndef POTR_RASTER_MIN_BLOCKS
#define POTR_RASTER_MIN_BLOCKS 8
#endif

namespace potr {

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

static inline unsigned grid_for(int64_t n, int block) {
    return (unsigned)((n + block - 1) / block);
}

// ---------------------------------------------------------------------------
// (a) preprocess

// Tile culling: the tile columns [*c0, *c1] of tile row ty whose pixel centres
// can pass the exp prefilter (power >= pthr) of record r.  The region
// power >= pthr is the ellipse q(d) = ia dx^2 + 2 ib dx dy + ic dy^2 <= R,
// R = -2 pthr; over the row's band of pixel-centre dy its x extent is
// [min g, max f] with f, g = (-ib dy +- sqrt(ia R - det dy^2)) / ia, concave /
// convex in dy with extrema at dy = -+ ib sqrt(R / (det ic)), clamped to the
// band.  A margin on R and on the pixel bounds keeps the cut conservative
// against rounding, so a culled (tile, splat) pair holds no sample that the
// rasterizer would composite: renders and records are bit-identical with or
// without it (scores up to the add order of the per-(tile, splat) sums).
// Near-degenerate conics keep the full bbox row.
constexpr double kCullMarginPower = 1e-6;
constexpr double kCullMarginPixel = 1e-3;  // covers the fp32 sqrt below (|x| < 1e4 px)

// The per-splat part of the test, computed once per (splat, view).
struct CullEllipse {
    double mx, my, b, inv_a, aR, det, ymax, sdy;
    int x0, x1, y0, y1;
    bool none, full;  // none: no sample passes; full: degenerate conic, keep the bbox rows
};

__device__ __forceinline__ CullEllipse cull_ellipse(const SplatRec &r) {
    CullEllipse e;
    e.mx = r.mx, e.my = r.my, e.b = r.ib;
    e.x0 = r.x0, e.x1 = r.x1, e.y0 = r.y0, e.y1 = r.y1;
    const double R = -2.0 * (r.pthr - kCullMarginPower);
    e.none = !(R > 0.0) || r.x0 > r.x1;  // pthr >= margin > 0 >= power: nothing passes
    const double a = -2.0 * r.ha, c = -2.0 * r.hc;
    e.det = a * c - e.b * e.b;
    e.full = !(a > 1e-280 && c > 1e-280 && a < 1e280 && c < 1e280 && e.det > 1e-4 * (a * c) &&
               e.det > 1e-280 && isfinite(R) && isfinite(e.det));
    // conservative use only (margins far above 1e-16): Newton reciprocals
    e.inv_a = rcp_nr(a);
    e.aR = a * R;
    const double inv_det = rcp_nr(e.det);
    e.ymax = sqrt(R * a * inv_det);
    e.sdy = e.b * sqrt(R * inv_det * rcp_nr(c));
    return e;
}

__device__ __forceinline__ bool row_span(const CullEllipse &e, int ty, int *c0, int *c1) {
    const int py0 = max(ty * kTileH, e.y0), py1 = min(ty * kTileH + kTileH - 1, e.y1);
    if (py0 > py1 || e.none) return false;
    int px0 = e.x0, px1 = e.x1;
    if (!e.full) {
        const double d0 = (double)py0 + 0.5 - e.my, d1 = (double)py1 + 0.5 - e.my;
        const double lo = fmax(d0, -e.ymax), hi = fmin(d1, e.ymax);
        if (lo > hi + kCullMarginPixel) return false;
        const double ya = fmin(fmax(-e.sdy, lo), hi), yb = fmin(fmax(e.sdy, lo), hi);
        const double sa = (double)sqrtf((float)fmax(e.aR - e.det * ya * ya, 0.0));
        const double sb = (double)sqrtf((float)fmax(e.aR - e.det * yb * yb, 0.0));
        const double xmax = (sa - e.b * ya) * e.inv_a;
        const double xmin = (-sb - e.b * yb) * e.inv_a;
        const double e0 = ceil(e.mx + xmin - 0.5 - kCullMarginPixel);
        const double e1 = floor(e.mx + xmax - 0.5 + kCullMarginPixel);
        if (e0 > (double)px0) px0 = e0 > (double)px1 ? px1 + 1 : (int)e0;
        if (e1 < (double)px1) px1 = e1 < (double)px0 ? px0 - 1 : (int)e1;
        if (px0 > px1) return false;
    }
    *c0 = px0 >> kTileWLog2;
    *c1 = px1 >> kTileWLog2;
    return true;
}

// One thread per (splat, view) of the batch; the views of a splat are adjacent
// threads, so its attributes come from one cache line fetch.
__global__ void k_splat_prep(int64_t n, const double *__restrict__ scales,
                             const double *__restrict__ rotations,
                             const double *__restrict__ opacities, SplatPrep *__restrict__ prep) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double scl[3], rot[4];
#pragma unroll
    for (int i = 0; i < 3; i++) scl[i] = scales[3 * k + i];
#pragma unroll
    for (int i = 0; i < 4; i++) rot[i] = rotations[4 * k + i];
    SplatPrep p;
    splat_sigma(scl, rot, p.S);
    p.pthr = log(kAlphaFloor / opacities[k]) - kPowerMargin;
    prep[k] = p;
}

// The splats in record-slot order (raster.cuh spatial_order): slot r holds
// splat perm[r]'s position, SH, opacity and view-independent terms, so the
// per-batch preprocess reads and writes contiguously in slot order.
__global__ void k_splat_slots(int64_t n, potr_splats sp, const int32_t *__restrict__ perm,
                              double *__restrict__ pos, double *__restrict__ sh,
                              double *__restrict__ opac, SplatPrep *__restrict__ prep) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int64_t k = perm[r];
    double scl[3], rot[4];
#pragma unroll
    for (int i = 0; i < 3; i++) {
        pos[3 * r + i] = sp.positions[3 * k + i];
        scl[i] = sp.scales[3 * k + i];
    }
#pragma unroll
    for (int i = 0; i < 4; i++) rot[i] = sp.rotations[4 * k + i];
    if (sh) {  // null: the SH rows follow with k_slot_sh (still uploading)
        const double2 *src = reinterpret_cast<const double2 *>(sp.sh + 48 * k);
        double2 *dst = reinterpret_cast<double2 *>(sh + 48 * r);
#pragma unroll 8
        for (int i = 0; i < 24; i++) dst[i] = src[i];
    }
    const double o = sp.opacities[k];
    opac[r] = o;
    SplatPrep p;
    splat_sigma(scl, rot, p.S);
    p.pthr = log(kAlphaFloor / o) - kPowerMargin;
    prep[r] = p;
}

cudaError_t launch_splat_slots(const potr_splats &sp, const int32_t *perm, double *pos, double *sh,
                               double *opac, SplatPrep *prep, cudaStream_t st) {
    if (sp.n == 0) return cudaSuccess;
    k_splat_slots<<<(unsigned)((sp.n + 127) / 128), 128, 0, st>>>(sp.n, sp, perm, pos, sh, opac,
                                                                  prep);
    return cudaGetLastError();
}

// The SH rows in slot order: one 16-byte piece per thread (coalesced writes).
__global__ void k_slot_sh(int64_t n, const double *__restrict__ sh_in,
                          const int32_t *__restrict__ perm, double *__restrict__ sh) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * 24) return;
    const int64_t r = i / 24, q = i - r * 24;
    const int64_t k = perm[r];
    reinterpret_cast<double2 *>(sh)[i] = reinterpret_cast<const double2 *>(sh_in)[k * 24 + q];
}

cudaError_t launch_slot_sh(int64_t n, const double *sh_in, const int32_t *perm, double *sh,
                           cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_slot_sh<<<grid_for(n * 24, 256), 256, 0, st>>>(n, sh_in, perm, sh);
    return cudaGetLastError();
}

// The colours of a batch's drawn records, after a preprocess without them
// (colors = 0).  Same thread layout as the preprocess (the views of a splat in
// adjacent threads: one SH row fetch serves them all) and the same products
// as its splat_color; each drawn record's (opac, cr) (cg, cb) sector is
// rewritten whole.
__global__ void __launch_bounds__(128) k_batch_colors(int64_t n, int nview,
                                                      const double *__restrict__ pos,
                                                      const double *__restrict__ sh,
                                                      const double *__restrict__ opac,
                                                      CamBatch cams, SplatRec *__restrict__ rec) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * nview) return;
    const int64_t k = t / nview;
    const int v = (int)(t - k * nview);
    const int64_t g = (int64_t)v * n + k;
    SplatRec &r = rec[g];
    const int2 xs = *reinterpret_cast<const int2 *>(&r.x0);
    if (xs.x > xs.y) return;  // not drawn (the preprocess left x0 > x1)
    double p[3], rgb[3];
#pragma unroll
    for (int j = 0; j < 3; j++) p[j] = __ldg(pos + 3 * k + j);
    splat_color(p, sh + 48 * k, cams.cam[v], rgb);
    double2 *f = reinterpret_cast<double2 *>(&r.opac);
    f[0] = make_double2(__ldg(opac + k), rgb[0]);
    f[1] = make_double2(rgb[1], rgb[2]);
}

cudaError_t launch_batch_colors(int64_t n, int nview, const double *pos, const double *sh,
                                const double *opac, const CamBatch &cams, SplatRec *rec,
                                cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_batch_colors<<<grid_for(n * nview, 128), 128, 0, st>>>(n, nview, pos, sh, opac, cams, rec);
    return cudaGetLastError();
}

cudaError_t launch_splat_prep(const potr_splats &sp, SplatPrep *prep, cudaStream_t st) {
    if (sp.n == 0) return cudaSuccess;
    k_splat_prep<<<(unsigned)((sp.n + 127) / 128), 128, 0, st>>>(sp.n, sp.scales, sp.rotations,
                                                                 sp.opacities, prep);
    return cudaGetLastError();
}

#ifndef POTR_PRE_MIN_BLOCKS
#define POTR_PRE_MIN_BLOCKS 8  // 64 regs: 42.5 ms per C3 step (43.8 at 7, 44.9 at 9, 57.8 at 10)
#endif
#define POTR_PRE_BOUNDS __launch_bounds__(128, POTR_PRE_MIN_BLOCKS)
// colors: 0 leaves the records' colours to launch_batch_colors (the SH rows
// are still being uploaded while the batch is binned)
__global__ void POTR_PRE_BOUNDS k_preprocess(potr_splats sp, const SplatPrep *__restrict__ prep,
                                             CamBatch cams, int nview, int tiles_x,
                                             int all_colors, int colors, int cull, DepthKey dk,
                                             SplatRec *__restrict__ rec,
                                             TileSpan *__restrict__ spans,
                                             uint64_t *__restrict__ key,
                                             int32_t *__restrict__ cnt,
                                             unsigned long long *counters) {
    const int64_t n = sp.n;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * nview) return;
    const int64_t k = t / nview;
    const int v = (int)(t - k * nview);
    const Cam &cam = cams.cam[v];
    const int64_t g = (int64_t)v * n + k;
    double pos[3], Sig[9];
#pragma unroll
    for (int i = 0; i < 3; i++) pos[i] = __ldg(sp.positions + 3 * k + i);
    const double2 *pp = reinterpret_cast<const double2 *>(prep + k);
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const double2 v = __ldg(pp + i);
        Sig[2 * i] = v.x;
        Sig[2 * i + 1] = v.y;
    }
    const double2 v4 = __ldg(pp + 4);
    Sig[8] = v4.x;
    const double pthr = v4.y;
    const Proj pr = project_sigma(pos, Sig, cam);
    int32_t c = 0;
    uint64_t kk = dk.compact ? ((uint64_t)v << dk.nbits) | dk.sentinel : ~0ull;
    if (pr.valid) {
        // depth > 0.01 > 0: its IEEE bits are monotone in depth
        const uint64_t bits = (uint64_t)__double_as_longlong(pr.depth);
        if (dk.compact) {
            // batch-wide key: view in the high bits, depth bits relative to a
            // bound of the scene's depth range below (exact, order preserving)
            uint64_t rel = bits >= dk.lo_bits ? bits - dk.lo_bits : 0ull;
            if (bits < dk.lo_bits || rel >= dk.sentinel) {
                *dk.overflow = 1;
                rel = rel >= dk.sentinel ? dk.sentinel - 1 : rel;
            }
            kk = ((uint64_t)v << dk.nbits) | rel;
            // the invalid sentinel's hi part is reserved for invalid splats
            if (dk.shift && (rel >> dk.shift) == (dk.sentinel >> dk.shift)) *dk.overflow = 1;
        } else {
            kk = bits;
        }
    }
    // the depth key leaves now (it is final; no register holds it below)
    key[g] = kk;
    if (dk.shift) dk.khi[g] = (uint32_t)(kk >> dk.shift);
    if (pr.valid) {
        const int W = cam.width, H = cam.height;
        double x0 = floor(pr.mx - pr.radius), x1 = ceil(pr.mx + pr.radius);
        double y0 = floor(pr.my - pr.radius), y1 = ceil(pr.my + pr.radius);
        if (x0 < 0) x0 = 0;
        if (y0 < 0) y0 = 0;
        if (x1 > W - 1) x1 = W - 1;
        if (y1 > H - 1) y1 = H - 1;
        const double det = pr.a * pr.c - pr.b * pr.b;
        const bool draw = !(x0 > x1 || y0 > y1) && det > 0.0;
        if (draw || all_colors) {
            // the geometry half of the record and the tile rows first, the
            // colour last: the conic is dead before the SH evaluation needs
            // its registers
            SplatRec r;
            r.mx = pr.mx;
            r.my = pr.my;
            // -0.5 * (a dx^2 + c dy^2) == ha dx^2 + hc dy^2 exactly (power-of-two scale)
            r.ha = -0.5 * (pr.c / det);
            r.ib = -pr.b / det;
            r.hc = -0.5 * (pr.a / det);
            r.pthr = pthr;  // log(kAlphaFloor / o) - kPowerMargin, from k_splat_prep
            r.x0 = (int32_t)x0;
            r.x1 = (int32_t)x1;
            r.y0 = (int32_t)y0;
            r.y1 = (int32_t)y1;
            if (!draw) r.x0 = 1, r.x1 = 0;  // empty: never drawn
            double2 *rf = reinterpret_cast<double2 *>(rec + g);
            rf[0] = make_double2(r.mx, r.my);
            rf[1] = make_double2(r.ha, r.ib);
            rf[2] = make_double2(r.hc, r.pthr);
            reinterpret_cast<int4 *>(rec + g)[3] = make_int4(r.x0, r.x1, r.y0, r.y1);
            if (draw) {
                const int ty0 = r.y0 >> kTileHLog2, ty1 = r.y1 >> kTileHLog2;
                const int bx0 = r.x0 >> kTileWLog2, bx1 = r.x1 >> kTileWLog2;
                TileSpan sp_;
                sp_.ty0 = (uint16_t)ty0;
                sp_.nrows = (uint16_t)(ty1 - ty0 + 1);
                CullEllipse ce;
                if (cull) ce = cull_ellipse(r);
                for (int ty = ty0; ty <= ty1; ty++) {
                    int t0 = bx0, t1 = bx1;
                    if (cull && !row_span(ce, ty, &t0, &t1)) t0 = 1, t1 = 0;
                    c += t1 - t0 + 1;
                    if (ty - ty0 < kSpanRows) {
                        sp_.c[2 * (ty - ty0)] = (uint16_t)t0;
                        sp_.c[2 * (ty - ty0) + 1] = (uint16_t)t1;
                    }
                }
                spans[g] = sp_;
            }
            double rgb[3] = {0.0, 0.0, 0.0};
            if (colors) {
                // the centre again (an L1 hit): not held across the rows
                double pc[3];
#pragma unroll
                for (int i = 0; i < 3; i++) pc[i] = __ldg(sp.positions + 3 * k + i);
                splat_color(pc, sp.sh + 48 * k, cam, rgb);
            }
            rf[4] = make_double2(__ldg(sp.opacities + k), rgb[0]);
            rf[5] = make_double2(rgb[1], rgb[2]);
        }
        if (draw) {
            if (counters)  // E: pixels the reference loop visits (rasterizer.py:159-161)
                atomicAdd(&counters[0], (unsigned long long)((x1 - x0 + 1.0) * (y1 - y0 + 1.0)));
        }
    }
    if (!pr.valid && all_colors) {  // an invalid splat's colour output is 0 (records mode)
        SplatRec r;
        memset(&r, 0, sizeof(r));
        r.x0 = 1, r.x1 = 0;
        rec[g] = r;
    }
    cnt[g] = c;
}

// project_splats / splat_colors dump for parity tests (potr_project).
__global__ void k_project_dump(potr_splats sp, Cam cam, double *mean2d, double *cov2d,
                               double *depth, double *radius, uint8_t *valid, double *colors) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= sp.n) return;
    Proj pr = project_one(sp.positions + 3 * k, sp.scales + 3 * k, sp.rotations + 4 * k, cam);
    mean2d[2 * k] = pr.mx;
    mean2d[2 * k + 1] = pr.my;
    cov2d[3 * k] = pr.a;
    cov2d[3 * k + 1] = pr.b;
    cov2d[3 * k + 2] = pr.c;
    depth[k] = pr.depth;
    radius[k] = pr.radius;
    valid[k] = pr.valid ? 1 : 0;
    if (colors) splat_color(sp.positions + 3 * k, sp.sh + 48 * k, cam, colors + 3 * k);
}

// ---------------------------------------------------------------------------
// (b) binning

// Batch arrays are view-major: element (v, i) at v*n + i.

// Emit the (tile, splat) pairs of every drawn splat, walking splats in depth
// order so a stable sort on the tile key yields (tile, depth, id) order.
// Views are sorted in groups of `sb`; a pair's key is its tile index inside
// its group, (v % sb) * ntiles + ty * tiles_x + tx, which fits 16 bits
// whenever sb * ntiles <= 65536 (halving the sort's key traffic).
template <typename KeyT>
__global__ void k_duplicate(int64_t total, int64_t n, const int32_t *__restrict__ ids,
                            const int64_t *__restrict__ offs, const SplatRec *__restrict__ rec,
                            const TileSpan *__restrict__ spans, int tiles_x, int ntiles, int sb,
                            int cull, KeyT *__restrict__ tkey, int32_t *__restrict__ dup_id,
                            int32_t *__restrict__ dup_rank) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int64_t o = offs[i];
    const int64_t e = offs[i + 1];
    if (o == e) return;
    const int64_t v = i / n;
    const int32_t g = ids[i];
    const uint32_t tbase0 = (uint32_t)((v % sb) * ntiles);
    const int32_t rank = (int32_t)(i - v * n);
    const TileSpan s = spans[g];
    if (s.nrows <= kSpanRows) {  // the preprocess's rows: no record read, no recompute
        for (int r = 0; r < s.nrows; r++) {
            const int ty = s.ty0 + r;
            for (int tx = s.c[2 * r]; tx <= (int)s.c[2 * r + 1]; tx++) {
                POTR_CHECK(o < e && tx < tiles_x);
                tkey[o] = (KeyT)(tbase0 + (uint32_t)(ty * tiles_x + tx));
                dup_id[o] = g;
                if (dup_rank) dup_rank[o] = rank;
                o++;
            }
        }
        return;
    }
    const SplatRec &R = rec[g];
    const int tx0 = R.x0 >> kTileWLog2, tx1 = R.x1 >> kTileWLog2;
    const int ty0 = R.y0 >> kTileHLog2, ty1 = R.y1 >> kTileHLog2;
    const uint32_t tbase = (uint32_t)((v % sb) * ntiles);
    CullEllipse ce;
    if (cull) ce = cull_ellipse(R);
    for (int ty = ty0; ty <= ty1; ty++) {
        int c0 = tx0, c1 = tx1;
        if (cull && !row_span(ce, ty, &c0, &c1)) continue;
        for (int tx = c0; tx <= c1; tx++) {
            POTR_CHECK(o < e && tx < tiles_x);
            tkey[o] = (KeyT)(tbase + (uint32_t)(ty * tiles_x + tx));
            dup_id[o] = g;
            if (dup_rank) dup_rank[o] = (int32_t)(i - v * n);
            o++;
        }
    }
}

// Tile [start, end) ranges of the sorted pairs of one sort group (pairs
// [j0, j0 + K) carrying group-local keys; tile index = tbase + key).  skey
// points at the group's slice.  The sorted (slot, record) pairs come straight
// out of the sort (radix_sort_packed).
template <typename KeyT>
__global__ void k_tile_ranges(int64_t j0, int64_t K, const KeyT *__restrict__ skey,
                              int2 *__restrict__ rng, int tbase) {
    // eight consecutive sorted keys per thread (one predecessor load)
    constexpr int kPer = 8;
    const int64_t jb = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kPer;
    if (jb >= K) return;
    uint32_t k[kPer];
#pragma unroll
    for (int q = 0; q < kPer; q++) k[q] = jb + q < K ? (uint32_t)skey[jb + q] : 0xffffffffu;
    uint32_t prev = jb > 0 ? (uint32_t)skey[jb - 1] : 0xffffffffu;
    const uint32_t after = jb + kPer < K ? (uint32_t)skey[jb + kPer] : 0xffffffffu;
#pragma unroll
    for (int q = 0; q < kPer; q++) {
        const int64_t jj = jb + q;
        if (jj >= K) break;
        const uint32_t t = k[q];
        const uint32_t nxt = q + 1 < kPer ? k[q + 1] : after;
        if (jj == 0 || prev != t) rng[tbase + t].x = (int)(j0 + jj);
        if (jj == K - 1 || nxt != t) rng[tbase + t].y = (int)(j0 + jj + 1);
        prev = t;
    }
}

// ---------------------------------------------------------------------------
// (c)+(d) tile rasterizer and removal-effect pass

// Per-warp staging.  A chunk is 32 consecutive pairs of the tile's list; its
// records are held field-major (six 16-byte fields x 32 entries) so lanes that
// read different entries hit different banks.  Two buffers: the next chunk
// streams in with cp.async while the current one is composited.
#ifndef POTR_MASK_CHUNKS
#define POTR_MASK_CHUNKS 16
#endif
constexpr int kMaskChunks = POTR_MASK_CHUNKS;  // chunks per tile whose per-lane contribution masks are kept

struct ChunkBuf {
    double2 f[6][32];  // (mx,my) (ha,ib) (hc,pthr) bbox(int4) (opac,cr) (cg,cb)
    int32_t dup[32];
};

#ifndef POTR_CHUNK_BUFFERS
#define POTR_CHUNK_BUFFERS 1
#endif
// 1: single-buffered chunks; at 8 CTAs x 4 warps per SM the other warps hide
// the copy (measured faster at C3 than double buffering at 6 CTAs per SM)
constexpr int kChunkBufs = POTR_CHUNK_BUFFERS;

#ifndef POTR_ACC_SPLIT
#define POTR_ACC_SPLIT 2
#endif
// Lane groups with their own accumulator row: groups of lanes adding to the
// same entry are split by half-warp, halving the serial rounds.
constexpr int kAccSplit = POTR_ACC_SPLIT;

struct WarpSmem {
    ChunkBuf buf[kChunkBufs];
    unsigned cmask[kMaskChunks][32];  // pass-1 contribution mask of each lane, per chunk
    double2 acc[kAccSplit][32];       // per-entry (dSE, T*alpha) sums of the current chunk,
                                      // one row per lane group (summed in row order)
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// The lane's slice of a chunk: pair index and splat id.
struct ChunkIds {
    int32_t d, id;
    bool valid;
};

__device__ __forceinline__ ChunkIds fetch_ids(const RasterArgs &a, int cbase, int end, int lane) {
    ChunkIds c;
    const int j = cbase + lane;
    c.valid = j < end;
    const int2 p = c.valid ? a.pair[j] : make_int2(0, 0);
    POTR_CHECK(!c.valid || (p.x >= 0 && p.y >= 0));
    c.d = p.x;
    c.id = p.y;
    return c;
}

// Start the async copy of a chunk's records into buffer `b`; always commits a
// group so wait_group counts stay uniform.
__device__ __forceinline__ void issue_chunk(const RasterArgs &a, ChunkBuf &B, const ChunkIds &c,
                                            int lane) {
    if (c.valid) {
        const char *src = reinterpret_cast<const char *>(a.rec + c.id);
#pragma unroll
        for (int q = 0; q < 6; q++) cp_async16(&B.f[q][lane], src + 16 * q);
        B.dup[lane] = c.d;
    }
    cp_async_commit();
}

__device__ __forceinline__ int4 bbox_of(const ChunkBuf &B, int e) {
    return *reinterpret_cast<const int4 *>(&B.f[3][e]);
}

#ifndef POTR_PIXEL_CULL
#define POTR_PIXEL_CULL 1
#endif

// Pixel culling of one entry over the tile: the columns [c0, c1] (tile-local,
// already clipped to the bbox) of each bbox row whose pixel centre can pass
// the exp prefilter (power >= pthr), as a 32-bit tile mask.  The same
// ellipse and margins as the tile culling (cull_ellipse / row_span), at a
// single pixel-centre dy per row, so it is conservative: every sample the
// rasterizer would composite keeps its bit and renders stay bit-identical.
__device__ __forceinline__ unsigned ellipse_rows(const ChunkBuf &B, int e, int ox, int oy,
                                                 int c0, int c1, int r0, int r1) {
    const double2 m = B.f[0][e], ab = B.f[1][e], cp = B.f[2][e];
    const double R = -2.0 * (cp.y - kCullMarginPower);
    const double a = -2.0 * ab.x, c = -2.0 * cp.x, b = ab.y;
    const double det = a * c - b * b;
    const bool full = !(a > 1e-280 && c > 1e-280 && a < 1e280 && c < 1e280 &&
                        det > 1e-4 * (a * c) && det > 1e-280 && isfinite(R) && isfinite(det));
    const unsigned cols = (0xFFu >> (7 - c1)) & (0xFFu << c0);
    if (full) {
        const unsigned rows = (0xFFFFFFFFu >> (8 * (3 - r1))) & (0xFFFFFFFFu << (8 * r0));
        return (cols * 0x01010101u) & rows;
    }
    if (!(R > 0.0)) return 0u;
    // The rows in fp32, in tile-local coordinates (small magnitudes), off the
    // FP64 pipe: a R is widened by 4e-6 relative (far above the fp32 rounding
    // of D's two terms, ~2e-7) and the pixel bounds by 1e-2 px plus 1e-5 of
    // the magnitudes involved (the fp32 rounding of the interval is ~3e-7 of
    // them), so the mask stays a superset of the pixels whose centre can pass
    // the exact fp64 prefilter; floor / ceil are single rounding conversions.
    const float faR = (float)(a * R) * (1.0f + 4e-6f);
    const float fdet = (float)det, fb = (float)b;
    const float finv_a = 1.0f / (float)a;
    const float mxl = (float)(m.x - (double)ox - 0.5);  // pixel k is in when k - mxl in [xmin, xmax]
    const float dy0 = (float)((double)oy + 0.5 - m.y);
    unsigned w = 0u;
    for (int r = r0; r <= r1; r++) {
        const float dy = dy0 + (float)r;
        const float D = faR - fdet * dy * dy;
        if (D < 0.0f) continue;
        const float sq = sqrtf(D), t = fb * dy;
        const float xmax = (sq - t) * finv_a, xmin = (-sq - t) * finv_a;
        const float mg = 1e-2f + 1e-5f * (fabsf(xmax) + fabsf(xmin) + fabsf(mxl));
        const int k0 = max(__float2int_ru(mxl + xmin - mg), c0);
        const int k1 = min(__float2int_rd(mxl + xmax + mg), c1);
        if (k0 <= k1) w |= ((0xFFu >> (7 - k1)) & (0xFFu << k0)) << (8 * r);
    }
    return w;
}

// Entries of this chunk whose clipped bbox (rasterizer.py:135-148) contains
// the lane's pixel (and, with POTR_PIXEL_CULL, whose prefilter ellipse can
// reach it).  Lane e turns entry e into the 32-bit set of tile pixels it
// covers (bit c + 8r <-> lane c + 8r, the lane's pixel); a 32x32 bit
// transpose over the warp then hands every lane its per-entry bits.  Must be
// called by the whole warp.
__device__ __forceinline__ unsigned live_mask(const ChunkBuf &B, int cnt, int ox, int oy,
                                              int lane) {
    unsigned w = 0u;
    if (lane < cnt) {
        const int4 bb = bbox_of(B, lane);
        const int c0 = max(bb.x - ox, 0), c1 = min(bb.y - ox, kTileW - 1);
        const int r0 = max(bb.z - oy, 0), r1 = min(bb.w - oy, kTileH - 1);
        if (c0 <= c1 && r0 <= r1) {
            if (POTR_PIXEL_CULL) {
                w = ellipse_rows(B, lane, ox, oy, c0, c1, r0, r1);
            } else {
                const unsigned cols = (0xFFu >> (7 - c1)) & (0xFFu << c0);
                const unsigned rows = (0xFFFFFFFFu >> (8 * (3 - r1))) & (0xFFFFFFFFu << (8 * r0));
                w = (cols * 0x01010101u) & rows;
            }
        }
    }
    // transpose: swap the off-diagonal j x j blocks, j = 16, 8, 4, 2, 1
    const unsigned FULL = 0xffffffffu;
#pragma unroll
    for (int j = 16, k = 0; j > 0; j >>= 1, k++) {
        const unsigned hm = k == 0 ? 0xFFFF0000u : k == 1 ? 0xFF00FF00u : k == 2 ? 0xF0F0F0F0u
                          : k == 3 ? 0xCCCCCCCCu : 0xAAAAAAAAu;
        const unsigned y = __shfl_xor_sync(FULL, w, j);
        w = (lane & j) ? ((w & hm) | ((y & hm) >> j)) : ((w & ~hm) | ((y & ~hm) << j));
    }
    return w;
}

// rasterizer.py:165-171 for entry e at this lane's pixel: the Gaussian exponent
// with the exp prefilter, then alpha capped at ALPHA_CAP.  Returns false when
// alpha < ALPHA_FLOOR (the sample is skipped and T is untouched).
__device__ __forceinline__ bool eval_alpha(const ChunkBuf &B, int e, double pxc, double pyc,
                                           unsigned tab, double &alpha) {
    const double2 m = B.f[0][e], ab = B.f[1][e], cp = B.f[2][e];
    const double dx = pxc - m.x, dy = pyc - m.y;
    // -0.5 * (a dx dx + c dy dy) - b dx dy, with the -0.5 folded into ha, hc
    const double power = (ab.x * dx * dx + cp.x * dy * dy) - ab.y * dx * dy;
    if (power < cp.y) return false;  // o*exp(power) < ALPHA_FLOOR for certain
    alpha = B.f[4][e].x * exp_neg(power, tab);
    if (alpha > kCompositeK[0]) alpha = kCompositeK[0];
    return !(alpha < kCompositeK[1]);
}

// eval_alpha for a sample pass 1 already composited (its tests passed): the
// same arithmetic, so the same bits, without the tests.
__device__ __forceinline__ double known_alpha(const ChunkBuf &B, int e, double pxc, double pyc,
                                              unsigned tab) {
    const double2 m = B.f[0][e], ab = B.f[1][e], cp = B.f[2][e];
    const double dx = pxc - m.x, dy = pyc - m.y;
    const double power = (ab.x * dx * dx + cp.x * dy * dy) - ab.y * dx * dy;
    const double alpha = B.f[4][e].x * exp_neg(power, tab);
    return alpha > kCompositeK[0] ? kCompositeK[0] : alpha;
}

// Deterministic segmented sum over the lanes that hold the same key: pointer
// jumping along each group's members in lane order leaves the group total in
// its lowest lane.  The add order depends only on group membership.
__device__ __forceinline__ bool group_sum(int key, double &v0, double &v1) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
#ifndef POTR_BALLOT_GROUPS
    const unsigned peers = __match_any_sync(FULL, key);
#else
    // keys are entry indices 0..31 (valid) or 32+lane (singletons): five
    // ballots on the key bits give every valid lane its group
    const bool grouped = key < 32;
    unsigned peers = __ballot_sync(FULL, grouped);
#pragma unroll
    for (int bit = 0; bit < 5; bit++) {
        const bool kb = (key >> bit) & 1;
        const unsigned x = __ballot_sync(FULL, kb);
        peers &= kb ? x : ~x;
    }
    if (!grouped) peers = 1u << lane;
#endif
    const unsigned above = peers & ~((2u << lane) - 1u);
    int nxt = above ? __ffs(above) - 1 : -1;
    const int gmax = __reduce_max_sync(FULL, (unsigned)__popc(peers));
    for (int span = 1; span < gmax; span <<= 1) {
        const int src = nxt >= 0 ? nxt : lane;
        const double t0 = __shfl_sync(FULL, v0, src);
        const double t1 = __shfl_sync(FULL, v1, src);
        const int n2 = __shfl_sync(FULL, nxt, src);
        if (nxt >= 0) {
            v0 += t0;
            v1 += t1;
            nxt = n2;
        }
    }
    return (peers & ((1u << lane) - 1u)) == 0u;  // this lane leads its group
}

// S.acc[key] += (v0, v1) for every lane with a valid key (< 32), in a fixed
// order: per key, the lanes of the group add in lane order.  Small groups
// (the common case: ~5 lanes at the C3 shape) do that directly, one rank per
// round; large ones reduce first with group_sum.  Either way the result
// depends only on the keys and values, never on scheduling.
#ifndef POTR_REPLAY_FMA
#define POTR_REPLAY_FMA 1
#endif

#ifndef POTR_SERIAL_GROUPS
#define POTR_SERIAL_GROUPS 8
#endif
constexpr int kSerialGroups = POTR_SERIAL_GROUPS;

__device__ __forceinline__ void accumulate(WarpSmem &S, int key, double v0, double v1) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int row = lane / (32 / kAccSplit);  // kAccSplit in {1, 2, 4}
    const unsigned peers = __match_any_sync(FULL, key + 64 * row);
    const int gmax = __reduce_max_sync(FULL, (unsigned)__popc(peers));
    if (gmax <= kSerialGroups) {
        const int rank = __popc(peers & ((1u << lane) - 1u));
        for (int r = 0; r < gmax; r++) {
            if (rank == r && key < 32) {
                double2 t = S.acc[row][key];
                t.x += v0;
                t.y += v1;
                S.acc[row][key] = t;
            }
            __syncwarp();
        }
        return;
    }
    if (group_sum(key + 64 * row, v0, v1) && key < 32) {
        S.acc[row][key].x += v0;
        S.acc[row][key].y += v1;
    }
}

// MODE: kRender     pass 1 only, writes image/trans
//       kImportance pass 1, then the replay accumulating T*alpha slots
//       kScore      pass 1, then the replay with the removal effect (targets)
//       kRecords    pass 1, appending every contribution record
//
// Persistent warps pull 8x4-pixel tiles from an atomic counter; a tile's
// result depends only on its own list, so the schedule does not change bits.
// Pass 1 is a per-lane walk: each lane visits only the chunk entries whose
// bbox holds its pixel, in list (depth) order, compositing exactly as the
// reference (rasterizer.py:159-201), and records which entries it composited.
// The replay visits exactly those (lane, entry) samples again, evaluates the
// closed-form removal delta (forward form, :232-243), dSE (:333) and T*alpha
// (:228), and sums them per (tile, splat) with group_sum.
template <int MODE>
__global__ void __launch_bounds__(32 * kRasterWarps, POTR_RASTER_MIN_BLOCKS) k_raster(RasterArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem &S = reinterpret_cast<WarpSmem *>(smem_raw)[threadIdx.x >> 5];
    __shared__ double2 tab[64];
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    for (int i = threadIdx.x; i < 64; i += blockDim.x)
        tab[i] = make_double2(kExpTable[i][0], kExpTable[i][1]);
    __syncthreads();
    // the table's shared address, opaque so it stays in one register
    unsigned tab_s = (unsigned)__cvta_generic_to_shared(tab);
    asm volatile("" : "+r"(tab_s));

    for (;;) {
        int tile = 0;
        if (lane == 0) tile = atomicAdd(a.tile_counter, 1);
        tile = __shfl_sync(FULL, tile, 0);
        if (tile >= a.ntiles) return;

        POTR_CHECK(tile >= 0 && tile < a.ntiles);
        const int view = tile / a.ntiles_view;
        const int vt = tile - view * a.ntiles_view;
        const int tx = vt % a.tiles_x, ty = vt / a.tiles_x;
        const int px = tx * kTileW + (lane & 7), py = ty * kTileH + (lane >> 3);
        const double *target = a.target[view];
        double *image = a.image[view];
        double *trans = a.trans[view];
        const bool inside = px < a.width && py < a.height;
        const int64_t pix = (int64_t)py * a.width + px;
        const int2 range = a.ranges[tile];
        const int start = range.x, end = range.y > range.x ? range.y : range.x;
        const double pxc = (double)px + 0.5, pyc = (double)py + 0.5;

        // ---- pass 1: per-lane front-to-back compositing -------------------
        double T = 1.0, P0 = 0.0, P1 = 0.0, P2 = 0.0;
        bool done = !inside;
        int stop = start;  // chunks [start, stop) were walked
        if (start < end && !__all_sync(FULL, done)) {
            ChunkIds next = fetch_ids(a, start, end, lane);
            if (kChunkBufs == 2) {
                issue_chunk(a, S.buf[0], next, lane);
                next = fetch_ids(a, start + 32, end, lane);
            }
            int b = 0;
            for (int base = start; base < end; base += 32, b ^= kChunkBufs - 1) {
                if (kChunkBufs == 2) {
                    issue_chunk(a, S.buf[(b ^ 1) & (kChunkBufs - 1)], next, lane);
                    next = fetch_ids(a, base + 64, end, lane);
                    cp_async_wait<1>();
                } else {
                    issue_chunk(a, S.buf[0], next, lane);
                    next = fetch_ids(a, base + 32, end, lane);
                    cp_async_wait<0>();
                }
                __syncwarp();
                const ChunkBuf &B = S.buf[b];
                const int cnt = min(32, end - base);
                unsigned m = live_mask(B, cnt, px - (lane & 7), py - (lane >> 3), lane);
                if (done) m = 0u;
                unsigned cm = 0u;
                unsigned n_live = 0u;
                while (m) {
                    const int e = __ffs(m) - 1;
                    m &= m - 1u;
                    n_live++;
                    double alpha;
                    if (!eval_alpha(B, e, pxc, pyc, tab_s, alpha)) continue;
                    cm |= 1u << e;
                    if (MODE == kRecords) {
                        unsigned long long slot = atomicAdd(a.rec_counter, 1ull);
                        if ((int64_t)slot < a.rec_capacity) {
                            a.rec_key[slot] =
                                ((uint64_t)(uint32_t)a.dup_rank[B.dup[e]] << 32) | (uint64_t)(uint32_t)pix;
                            a.rec_alpha[slot] = alpha;
                            a.rec_t[slot] = T;
                            a.rec_p[3 * slot] = P0;
                            a.rec_p[3 * slot + 1] = P1;
                            a.rec_p[3 * slot + 2] = P2;
                        }
                    }
                    const double c0 = B.f[4][e].y;
                    const double2 c12 = B.f[5][e];
                    const double w = T * alpha;
                    P0 += w * c0;
                    P1 += w * c12.x;
                    P2 += w * c12.y;
                    T = T * (1.0 - alpha);
                    if (T < kCompositeK[2]) {  // every later sample is skipped (:162-164)
                        done = true;
                        m = 0u;
                    }
                }
                if (a.counters) {
                    const unsigned lv = __reduce_add_sync(FULL, n_live);
                    const unsigned ct = __reduce_add_sync(FULL, (unsigned)__popc(cm));
                    if (lane == 0) {
                        atomicAdd(&a.counters[1], (unsigned long long)lv);
                        atomicAdd(&a.counters[2], (unsigned long long)ct);
                    }
                }
                const int ci = (base - start) >> 5;
                if (ci < kMaskChunks) S.cmask[ci][lane] = cm;
                stop = base + 32;
                __syncwarp();
                if (__all_sync(FULL, done)) break;
            }
            cp_async_wait<0>();
            __syncwarp();
            if (stop > end) stop = end;
        }

        if (MODE == kRender || MODE == kRecords) {
            if (inside && image) {
                image[3 * pix] = P0;
                image[3 * pix + 1] = P1;
                image[3 * pix + 2] = P2;
            }
            if (inside && trans) trans[pix] = T;
            continue;
        }

        // ---- replay: removal effect / importance (rasterizer.py:226-243, :322-336)
        const double PK0 = P0, PK1 = P1, PK2 = P2;
        double dr0 = 0.0, dr1 = 0.0, dr2 = 0.0;
        if (MODE == kScore) {
            double se = 0.0;
            if (inside && !a.self_target) {  // self target: c - c_t = 0 exactly
                dr0 = PK0 - target[3 * pix];
                dr1 = PK1 - target[3 * pix + 1];
                dr2 = PK2 - target[3 * pix + 2];
                se = dr0 * dr0 + dr1 * dr1 + dr2 * dr2;
            }
            se = warp_sum(se);
            if (lane == 0) a.tile_se[tile] = se;
        }
        if (inside && image) {
            image[3 * pix] = PK0;
            image[3 * pix + 1] = PK1;
            image[3 * pix + 2] = PK2;
        }
        if (inside && trans) trans[pix] = T;
        // the replay carries Q = P_K - P_i (the colour still to come) and 2 dr
        P0 = PK0, P1 = PK1, P2 = PK2;
        dr0 = 2.0 * dr0, dr1 = 2.0 * dr1, dr2 = 2.0 * dr2;
        T = 1.0;
        int written = start;
        if (start < stop) {
            ChunkIds next = fetch_ids(a, start, end, lane);
            if (kChunkBufs == 2) {
                issue_chunk(a, S.buf[0], next, lane);
                next = fetch_ids(a, start + 32, end, lane);
            }
            int b = 0;
            for (int base = start; base < stop; base += 32, b ^= kChunkBufs - 1) {
                if (kChunkBufs == 2) {
                    issue_chunk(a, S.buf[(b ^ 1) & (kChunkBufs - 1)], next, lane);
                    next = fetch_ids(a, base + 64, end, lane);
                } else {
                    issue_chunk(a, S.buf[0], next, lane);
                    next = fetch_ids(a, base + 32, end, lane);
                }
#pragma unroll
                for (int q = 0; q < kAccSplit; q++) S.acc[q][lane] = make_double2(0.0, 0.0);
                if (kChunkBufs == 2) cp_async_wait<1>();
                else cp_async_wait<0>();
                __syncwarp();
                const ChunkBuf &B = S.buf[b];
                const int cnt = min(32, end - base);
                const int ci = (base - start) >> 5;
                // One composited sample of entry e: the removal delta, dSE and
                // T*alpha; P carries the colour still to come.
                auto removal = [&](int e, double alpha, double &dse, double &timp) {
                    const double c0 = B.f[4][e].y;
                    const double2 c12 = B.f[5][e];
                    const double w = T * alpha;
                    if (MODE == kScore) {
                        // prune_deltas, forward form: a/(1-a) * (P_K - P_i - T c),
                        // dSE = |pd|^2 + 2 pd . dr (rasterizer.py:232-243, :333).
                        // Scores only (1e-4 contract), so fused multiply-adds;
                        // alpha, T and T*alpha keep the reference's rounding.
                        const double f = alpha * rcp_nr(1.0 - alpha);
                        if (POTR_REPLAY_FMA) {
                            const double pd0 = f * fma(-T, c0, P0);
                            const double pd1 = f * fma(-T, c12.x, P1);
                            const double pd2 = f * fma(-T, c12.y, P2);
                            dse = pd0 * (pd0 + dr0);
                            dse = fma(pd1, pd1 + dr1, dse);
                            dse = fma(pd2, pd2 + dr2, dse);
                            P0 = fma(-w, c0, P0);
                            P1 = fma(-w, c12.x, P1);
                            P2 = fma(-w, c12.y, P2);
                        } else {
                            const double pd0 = f * (P0 - T * c0);
                            const double pd1 = f * (P1 - T * c12.x);
                            const double pd2 = f * (P2 - T * c12.y);
                            dse = pd0 * (pd0 + dr0);
                            dse = dse + pd1 * (pd1 + dr1);
                            dse = dse + pd2 * (pd2 + dr2);
                            P0 -= w * c0;
                            P1 -= w * c12.x;
                            P2 -= w * c12.y;
                        }
                    }
                    timp = w;
                    T = T * (1.0 - alpha);
                };
                if (ci < kMaskChunks) {
                    // pass 1's masks: exactly the composited samples, none after
                    // termination (T evolves bit for bit as in pass 1), so
                    // neither the alpha tests nor the T test are repeated
                    unsigned m = S.cmask[ci][lane];
                    while (__any_sync(FULL, m != 0u)) {
                        int key = 32 + lane;
                        double dse = 0.0, timp = 0.0;
                        if (m) {
                            const int e = __ffs(m) - 1;
                            m &= m - 1u;
                            key = e;
                            removal(e, known_alpha(B, e, pxc, pyc, tab_s), dse, timp);
                        }
                        accumulate(S, key, dse, timp);
                    }
                } else {
                    // beyond the kept masks the samples are re-decided exactly as
                    // in pass 1; T < T_TERMINATE here iff pass 1 had stopped
                    unsigned m = live_mask(B, cnt, px - (lane & 7), py - (lane >> 3), lane);
                    if (!inside || T < kCompositeK[2]) m = 0u;
                    while (__any_sync(FULL, m != 0u)) {
                        int key = 32 + lane;
                        double dse = 0.0, timp = 0.0;
                        if (m) {
                            const int e = __ffs(m) - 1;
                            m &= m - 1u;
                            double alpha;
                            if (eval_alpha(B, e, pxc, pyc, tab_s, alpha)) {
                                key = e;
                                removal(e, alpha, dse, timp);
                                if (T < kCompositeK[2]) m = 0u;
                            }
                        }
                        accumulate(S, key, dse, timp);
                    }
                }
                __syncwarp();
                if (lane < cnt) {
                    POTR_CHECK(B.dup[lane] >= 0);
                    double2 t = S.acc[0][lane];
#pragma unroll
                    for (int q = 1; q < kAccSplit; q++) t.x += S.acc[q][lane].x, t.y += S.acc[q][lane].y;
                    a.partial[B.dup[lane]] = t;
                }
                written = base + cnt;
                __syncwarp();
            }
            cp_async_wait<0>();
            __syncwarp();
        }
        for (int j = written + lane; j < end; j += 32)
            a.partial[a.pair[j].x] = make_double2(0.0, 0.0);
    }
}

// Per (view, splat): sum of its (tile, splat) slots in tile order
// (deterministic), normalised by P and 3P (rasterizer.py:230, :334).  A warp
// takes 32 consecutive (view, rank) entries, whose slots are one contiguous
// range: it stages that range in shared memory with coalesced loads, then
// each lane sums its own entry's slots in order.
constexpr int kReduceStage = 256;  // slots staged per warp

__global__ void __launch_bounds__(256) k_splat_reduce(int64_t total, int64_t n,
                                                      const int32_t *__restrict__ ids,
                                                      const int64_t *__restrict__ offs,
                                                      const double2 *__restrict__ partial,
                                                      double P, const int32_t *__restrict__ perm,
                                                      double2 *__restrict__ vals) {
    __shared__ double2 stage[8][kReduceStage];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i0 = ((int64_t)blockIdx.x * 8 + w) * 32;
    if (i0 >= total) return;
    const int64_t i = i0 + lane;
    const bool act = i < total;
    const int64_t o = act ? offs[i] : 0, e = act ? offs[i + 1] : 0;
    // the output index: the entry's record (slot space stays slot space; the
    // view accumulation maps slots to splats)
    const int64_t g = act ? ids[i] : 0;
    const int64_t base = __shfl_sync(0xffffffffu, o, 0);
    const int64_t last = total - i0 < 32 ? total - i0 - 1 : 31;
    const int64_t top = __shfl_sync(0xffffffffu, e, (int)last);
    double dse = 0.0, imp = 0.0;
    if (top - base <= kReduceStage) {
        for (int64_t j = base + lane; j < top; j += 32) stage[w][j - base] = partial[j];
        __syncwarp();
        for (int64_t j = o; j < e; j++) {
            const double2 x = stage[w][j - base];
            dse += x.x;
            imp += x.y;
        }
    } else {
        for (int64_t j = o; j < e; j++) {
            const double2 x = partial[j];
            dse += x.x;
            imp += x.y;
        }
    }
    if (!act) return;
    // one 16-byte scatter per (view, splat): (I_k(s), dMSE_k(s)), by splat id
    // (perm: slot -> splat), so the view accumulation reads coalesced
    int64_t out = g;
    if (perm) {
        const int64_t v = g / n;
        out = v * n + perm[g - v * n];
    }
    vals[out] = make_double2(imp / P, dse / (P * 3.0));
}

// Camera-ordered accumulation over the views of the batch (rasterizer.py:343-347),
// writing the camera_importance rows on the way (all accesses coalesced, by
// splat id: k_splat_reduce scattered the per-view sums by splat id).
__global__ void k_view_accumulate(int64_t n, int nview, const double2 *__restrict__ vals,
                                  double *__restrict__ cam_imp_rows, double *__restrict__ imp_acc,
                                  double *__restrict__ dmse_acc, double *__restrict__ dmse_rows) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double ia = imp_acc[k];
    double da = dmse_acc ? dmse_acc[k] : 0.0;
    for (int v = 0; v < nview; v++) {
        const double2 x = vals[(int64_t)v * n + k];  // by splat id (k_splat_reduce)
        if (cam_imp_rows) cam_imp_rows[(int64_t)v * n + k] = x.x;
        if (dmse_rows) dmse_rows[(int64_t)v * n + k] = x.y;
        ia += x.x;
        da += x.y;
    }
    imp_acc[k] = ia;
    if (dmse_acc) dmse_acc[k] = da;
}

// Per view (one block each), the sum of its tiles' squared errors in a fixed
// order; mse(s) = sum / 3P (:335).  k_mse_accumulate then adds the views to
// the camera-ordered accumulator (:347).
__global__ void k_mse_reduce(int ntiles, const double *__restrict__ tile_se, double P,
                             double *__restrict__ mse_view) {
    __shared__ double red[32];
    const int v = blockIdx.x;
    double s = 0.0;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s += tile_se[(int64_t)v * ntiles + t];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
        mse_view[v] = t / (P * 3.0);
    }
}

__global__ void k_mse_accumulate(int nview, const double *__restrict__ mse_view,
                                 double *__restrict__ mse_acc, double *__restrict__ mse_rows) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double a = mse_acc[0];
    for (int v = 0; v < nview; v++) {
        a += mse_view[v];
        if (mse_rows) mse_rows[v] = mse_view[v];
    }
    mse_acc[0] = a;
}

__global__ void k_finalize(int64_t n, double S, double *imp, double *dmse, double *mse) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) {
        imp[k] = imp[k] / S;
        if (dmse) dmse[k] = dmse[k] / S;
    }
    if (k == 0 && mse) mse[0] = mse[0] / S;
}

// records mode: gather the sorted records into the caller's arrays
__global__ void k_records_gather(int64_t m, const uint64_t *__restrict__ skey,
                                 const int32_t *__restrict__ sidx, const int32_t *__restrict__ ids,
                                 const double *__restrict__ ra, const double *__restrict__ rt,
                                 const double *__restrict__ rp, int64_t *splat_ids,
                                 int64_t *pixels, double *alphas, double *trans_at,
                                 double *partials, const int32_t *__restrict__ perm) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    uint64_t k = skey[i];
    int32_t s = sidx[i];
    const int32_t g = ids[(int64_t)(k >> 32)];  // one view: slot
    splat_ids[i] = perm ? perm[g] : g;
    pixels[i] = (int64_t)(k & 0xffffffffu);
    alphas[i] = ra[s];
    trans_at[i] = rt[s];
    partials[3 * i] = rp[3 * (int64_t)s];
    partials[3 * i + 1] = rp[3 * (int64_t)s + 1];
    partials[3 * i + 2] = rp[3 * (int64_t)s + 2];
}

// Records mode preprocesses with all_colors: every splat has a record, with
// zero colour when it is invalid (rasterizer.py:252-254 leaves those at 0).
__global__ void k_colors_from_rec(int64_t n, const SplatRec *__restrict__ rec,
                                  const int32_t *__restrict__ mpos, double *colors) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const SplatRec &r = rec[mpos ? mpos[k] : k];
    colors[3 * k] = r.cr;
    colors[3 * k + 1] = r.cg;
    colors[3 * k + 2] = r.cb;
}

__global__ void k_tile_offsets(int ntiles, const int2 *__restrict__ rng, int64_t K,
                               int64_t *__restrict__ out) {
    // tiles are sorted ascending, so offset(t) = first pair index of a tile >= t
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    if (t == ntiles) {
        out[t] = K;
        return;
    }
    int64_t o = K;
    for (int u = t; u < ntiles; u++) {
        if (rng[u].y > rng[u].x) {
            o = rng[u].x;
            break;
        }
    }
    out[t] = o;
}

__global__ void k_tile_splats(int64_t K, const int2 *__restrict__ pair,
                              const int32_t *__restrict__ mperm, int32_t *__restrict__ out) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < K) out[j] = mperm ? mperm[pair[j].y] : pair[j].y;  // one view: slot = rank
}

__global__ void k_order_out(int64_t nv, const int32_t *__restrict__ ids,
                            const int32_t *__restrict__ perm, int64_t *__restrict__ out) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nv) out[r] = perm ? perm[ids[r]] : ids[r];  // one view: slot -> splat
}

__global__ void k_count_valid(int64_t n, const uint64_t *__restrict__ skey, uint64_t invalid,
                              unsigned long long *__restrict__ out) {
    // sorted keys: valid ones first; find the boundary
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    bool v = skey[r] != invalid;
    bool next_v = (r + 1 < n) ? (skey[r + 1] != invalid) : false;
    if (v && !next_v) *out = (unsigned long long)(r + 1);
}

// ---------------------------------------------------------------------------
// host-side launchers (called from capi.cu)


size_t raster_smem_bytes() { return sizeof(WarpSmem) * kRasterWarps; }

cudaError_t launch_preprocess(const potr_splats &sp, const SplatPrep *prep, const CamBatch &cams,
                              int nview,
                              int tiles_x, int all_colors, int colors, int cull, const DepthKey &dk,
                              SplatRec *rec, TileSpan *spans, uint64_t *key, int32_t *cnt,
                              unsigned long long *counters, cudaStream_t st) {
    if (sp.n == 0) return cudaSuccess;
    k_preprocess<<<grid_for(sp.n * nview, 128), 128, 0, st>>>(sp, prep, cams, nview, tiles_x,
                                                               all_colors, colors, cull, dk, rec,
                                                               spans, key, cnt, counters);
    return cudaGetLastError();
}

cudaError_t launch_project_dump(const potr_splats &sp, const Cam &cam, double *mean2d,
                                double *cov2d, double *depth, double *radius, uint8_t *valid,
                                double *colors, cudaStream_t st) {
    if (sp.n == 0) return cudaSuccess;
    k_project_dump<<<grid_for(sp.n, 128), 128, 0, st>>>(sp, cam, mean2d, cov2d, depth, radius,
                                                         valid, colors);
    return cudaGetLastError();
}

// Double-buffered (sort.cu): *in_alt is set when the sorted keys/values ended
// in the second buffer of each pair.
// The values are the record indices val_base + 0..n-1 (implicit in the
// first pass).
cudaError_t depth_sort(void *temp, size_t temp_bytes, uint64_t *key_a, uint64_t *key_b,
                       int32_t *val_a, int32_t *val_b, int64_t n, int end_bit, int64_t val_base,
                       bool *in_alt, cudaStream_t st) {
    return radix_sort_pairs<uint64_t, int32_t>(temp, temp_bytes, key_a, key_b, val_a, val_b, n,
                                               0, end_bit, true, in_alt, st, val_base);
}

cudaError_t depth_sort32(void *temp, size_t temp_bytes, uint32_t *key_a, uint32_t *key_b,
                         int32_t *val_a, int32_t *val_b, int64_t n, int end_bit, bool *in_alt,
                         cudaStream_t st) {
    return radix_sort_pairs<uint32_t, int32_t>(temp, temp_bytes, key_a, key_b, val_a, val_b, n,
                                               0, end_bit, true, in_alt, st);
}

cudaError_t depth_sort32_temp(int64_t n, size_t *bytes) {
    *bytes = radix_sort_temp_bytes(n, 0, 32);
    return cudaSuccess;
}

// The first position of each run of equal hi keys insertion-sorts the run's
// record ids by their full keys.  The hi sort was stable, so equal full keys
// keep record-index order (the tiebreak).
__device__ __forceinline__ void fixup_run(int64_t j, uint32_t h, int64_t total,
                                          const uint32_t *__restrict__ hi,
                                          int32_t *__restrict__ sids,
                                          const uint64_t *__restrict__ key, int *overflow,
                                          const int32_t *__restrict__ perm, int64_t n) {
    int len = 2;
    while (j + len < total && hi[j + len] == h) {
        if (++len > kFixupRun) {
            *overflow = 1;
            return;
        }
    }
    // records in slot order (perm): equal full keys order by splat index,
    // as np.argsort(kind="stable") does; a run shares its view
    int32_t id[kFixupRun];
    uint64_t kv[kFixupRun];
    for (int i = 0; i < len; i++) {
        id[i] = sids[j + i];
        kv[i] = key[id[i]];
    }
    for (int i = 1; i < len; i++) {
        const int32_t x = id[i];
        const uint64_t y = kv[i];
        const int32_t ox = perm ? perm[x % n] : x;
        int q = i - 1;
        while (q >= 0 && (kv[q] > y || (perm && kv[q] == y && perm[id[q] % n] > ox))) {
            kv[q + 1] = kv[q];
            id[q + 1] = id[q];
            q--;
        }
        kv[q + 1] = y;
        id[q + 1] = x;
    }
    for (int i = 0; i < len; i++) sids[j + i] = id[i];
}

// One sorted position per thread: coalesced loads, neighbours by shuffle (the
// kernel is a stream over the hi keys: runs are rare).
__global__ void __launch_bounds__(256) k_depth_fixup(int64_t total, const uint32_t *__restrict__ hi,
                                                     int32_t *__restrict__ sids,
                                                     const uint64_t *__restrict__ key,
                                                     uint32_t invalid_lo, uint32_t lo_mask,
                                                     int *overflow,
                                                     const int32_t *__restrict__ perm, int64_t n) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    const uint32_t c = j < total ? hi[j] : 0u;
    uint32_t prev = __shfl_up_sync(FULL, c, 1), next = __shfl_down_sync(FULL, c, 1);
    if (lane == 0) prev = j > 0 && j < total ? hi[j - 1] : ~c;
    if (lane == 31) next = j + 1 < total ? hi[j + 1] : 0u;
    if (j >= total) return;
    // a run start: differs from the previous key, equals the next one;
    // invalid splats (the sentinel) are already in record order
    if (c != prev && j + 1 < total && c == next && (c & lo_mask) != invalid_lo)
        fixup_run(j, c, total, hi, sids, key, overflow, perm, n);
}

cudaError_t launch_depth_fixup(int64_t total, const uint32_t *khi_sorted, int32_t *sids,
                               const uint64_t *key, int shift, uint64_t sentinel, int nbits,
                               int *overflow, const int32_t *perm, int64_t n, cudaStream_t st) {
    if (total < 2) return cudaSuccess;
    // hi = (view << (nbits - shift)) | depth part; the invalid sentinel's depth part
    const int dbits = nbits - shift;
    const uint32_t lo_mask = dbits >= 32 ? 0xffffffffu : ((1u << dbits) - 1u);
    const uint32_t invalid_lo = (uint32_t)(sentinel >> shift) & lo_mask;
    k_depth_fixup<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        total, khi_sorted, sids, key, invalid_lo, lo_mask, overflow, perm, n);
    return cudaGetLastError();
}

__global__ void k_gather_keys(int64_t total, const int32_t *__restrict__ sids,
                              const uint64_t *__restrict__ key, uint64_t *__restrict__ skey) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < total) skey[j] = key[sids[j]];
}

cudaError_t launch_gather_keys(int64_t total, const int32_t *sids, const uint64_t *key,
                               uint64_t *skey, cudaStream_t st) {
    if (total == 0) return cudaSuccess;
    k_gather_keys<<<grid_for(total, 256), 256, 0, st>>>(total, sids, key, skey);
    return cudaGetLastError();
}

cudaError_t depth_sort_temp(int64_t n, size_t *bytes) {
    *bytes = radix_sort_temp_bytes(n, 0, 64);
    return cudaSuccess;
}

__global__ void __launch_bounds__(256) k_bbox(int64_t n, const double *__restrict__ pos,
                                              unsigned long long *__restrict__ out) {
    // out[0..2] = ordered-int min of x,y,z; out[3..5] = ordered-int max.  Warp
    // and CTA reductions first: six global atomics per CTA (same-address
    // atomics from every thread serialised at L2: ~300 us per call before).
    __shared__ unsigned long long red[8][6];
    unsigned long long mn[3] = {~0ull, ~0ull, ~0ull}, mx[3] = {0ull, 0ull, 0ull};
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int i = 0; i < 3; i++) {
            const long long b = __double_as_longlong(pos[3 * k + i]);
            // total order on doubles as unsigned integers
            const unsigned long long u = b < 0 ? ~(unsigned long long)b
                                               : ((unsigned long long)b | (1ull << 63));
            mn[i] = u < mn[i] ? u : mn[i];
            mx[i] = u > mx[i] ? u : mx[i];
        }
    }
#pragma unroll
    for (int i = 0; i < 3; i++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn[i], o);
            const unsigned long long b = __shfl_xor_sync(0xffffffffu, mx[i], o);
            mn[i] = a < mn[i] ? a : mn[i];
            mx[i] = b > mx[i] ? b : mx[i];
        }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
        for (int i = 0; i < 3; i++) red[w][i] = mn[i], red[w][3 + i] = mx[i];
    __syncthreads();
    if (threadIdx.x < 6) {
        const int i = threadIdx.x;
        unsigned long long v = red[0][i];
        for (int q = 1; q < (int)(blockDim.x >> 5); q++)
            v = i < 3 ? (red[q][i] < v ? red[q][i] : v) : (red[q][i] > v ? red[q][i] : v);
        if (i < 3) atomicMin(&out[i], v);
        else atomicMax(&out[i], v);
    }
}

// Spatial record order: a 30-bit Morton code of each splat centre within the
// scene bounds (10 bits per axis; non-finite coordinates go to cell 0).
__global__ void k_morton(int64_t n, const double *__restrict__ pos, double lx, double ly,
                         double lz, double sx, double sy, double sz, uint32_t *__restrict__ code) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double lo[3] = {lx, ly, lz}, sc[3] = {sx, sy, sz};
    uint32_t c = 0u;
#pragma unroll
    for (int i = 0; i < 3; i++) {
        double q = (pos[3 * k + i] - lo[i]) * sc[i];
        q = q >= 0.0 ? (q < 1023.0 ? q : 1023.0) : 0.0;  // NaN -> 0
        uint32_t u = (uint32_t)q;
        // spread the 10 bits three apart
        u = (u | (u << 16)) & 0x030000FFu;
        u = (u | (u << 8)) & 0x0300F00Fu;
        u = (u | (u << 4)) & 0x030C30C3u;
        u = (u | (u << 2)) & 0x09249249u;
        c |= u << i;
    }
    code[k] = c;
}

__global__ void k_scatter_rank(int64_t n, const int32_t *__restrict__ perm,
                               int32_t *__restrict__ pos) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) pos[perm[r]] = (int32_t)r;
}

cudaError_t spatial_order_temp(int64_t n, size_t *bytes) {
    *bytes = radix_sort_temp_bytes(n, 0, 30);
    return cudaSuccess;
}

// perm = splats by Morton code (stable: ties by index), rank = perm^-1.
// code / code_sorted are the key pair, perm / rank the value pair.
cudaError_t spatial_order(void *temp, size_t temp_bytes, int64_t n, const double *pos,
                          const double lo[3], const double hi[3], uint32_t *code,
                          uint32_t *code_sorted, int32_t *perm, int32_t *rank, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    double sc[3];
    for (int i = 0; i < 3; i++) {
        const double ext = hi[i] - lo[i];
        sc[i] = ext > 0.0 && ext < 1e300 ? 1024.0 / ext : 0.0;
    }
    k_morton<<<grid_for(n, 256), 256, 0, st>>>(n, pos, lo[0], lo[1], lo[2], sc[0], sc[1], sc[2],
                                               code);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    bool alt = false;
    e = radix_sort_pairs<uint32_t, int32_t>(temp, temp_bytes, code, code_sorted, perm, rank, n, 0,
                                            30, true, &alt, st);
    if (e != cudaSuccess) return e;
    if (alt) {
        e = cudaMemcpyAsync(perm, rank, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
    }
    k_scatter_rank<<<grid_for(n, 256), 256, 0, st>>>(n, perm, rank);
    return cudaGetLastError();
}

cudaError_t launch_bbox(int64_t n, const double *pos, unsigned long long *out, cudaStream_t st) {
    unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
    cudaError_t e = cudaMemcpyAsync(out, init, sizeof(init), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess || n == 0) return e;
    k_bbox<<<296, 256, 0, st>>>(n, pos, out);
    return cudaGetLastError();
}

// offs[0] = 0, offs[i + 1] = sum of cnt[ids[j]] for j <= i (sort.cu: the
// counts are gathered in depth order by the scan itself).
cudaError_t scan_counts(void *temp, size_t temp_bytes, const int32_t *ids, const int32_t *cnt,
                        int64_t *offs, int64_t total, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(offs, 0, sizeof(int64_t), st);
    if (e != cudaSuccess || total == 0) return e;
    return inclusive_sum_gather(temp, temp_bytes, ids, cnt, offs + 1, total, st);
}
cudaError_t scan_temp(int64_t n, size_t *bytes) {
    *bytes = scan_temp_bytes(n);
    return cudaSuccess;
}

cudaError_t launch_duplicate(int64_t total, int64_t n, const int32_t *ids, const int64_t *offs,
                             const SplatRec *rec, const TileSpan *spans, int tiles_x, int ntiles,
                             int sb, bool key16, int cull, void *tkey, int32_t *dup_id,
                             int32_t *dup_rank, cudaStream_t st) {
    if (total == 0) return cudaSuccess;
    if (key16)
        k_duplicate<uint16_t><<<grid_for(total, 256), 256, 0, st>>>(
            total, n, ids, offs, rec, spans, tiles_x, ntiles, sb, cull, (uint16_t *)tkey, dup_id,
            dup_rank);
    else
        k_duplicate<uint32_t><<<grid_for(total, 256), 256, 0, st>>>(
            total, n, ids, offs, rec, spans, tiles_x, ntiles, sb, cull, (uint32_t *)tkey, dup_id,
            dup_rank);
    return cudaGetLastError();
}

static int bits_for(int ntiles) {
    int b = 1;
    while ((1 << b) < ntiles) b++;
    return b;
}

// Stable sort of one sort group's pairs by tile key.  Pair j0 + i enters as
// (slot = j0 + i, record = dup_id[i]) and leaves, in (tile, depth) order, as
// the rasterizer's one 8-byte fetch.  Double-buffered over (tkey, tkey_alt) x
// (pair, pair_alt); *in_alt tells where the result is.
cudaError_t tile_sort(void *temp, size_t temp_bytes, bool key16, void *tkey, void *tkey_alt,
                      const int32_t *dup_id, int64_t j0, int2 *pair, int2 *pair_alt, int64_t K,
                      int nkeys, bool *in_alt, cudaStream_t st) {
    *in_alt = false;
    if (K == 0) return cudaSuccess;
    if (key16)
        return radix_sort_packed<uint16_t>(temp, temp_bytes, (uint16_t *)tkey,
                                           (uint16_t *)tkey_alt, dup_id, j0, pair, pair_alt, K, 0,
                                           bits_for(nkeys), in_alt, st);
    return radix_sort_packed<uint32_t>(temp, temp_bytes, (uint32_t *)tkey, (uint32_t *)tkey_alt,
                                       dup_id, j0, pair, pair_alt, K, 0, bits_for(nkeys), in_alt,
                                       st);
}

cudaError_t tile_sort_temp(int64_t K, int nkeys, bool key16, size_t *bytes) {
    (void)key16;
    *bytes = radix_sort_temp_bytes(K, 0, bits_for(nkeys));
    return cudaSuccess;
}

cudaError_t records_sort_temp(int64_t m, size_t *bytes) {
    *bytes = radix_sort_temp_bytes(m, 0, 64);
    return cudaSuccess;
}

cudaError_t records_sort(void *temp, size_t temp_bytes, uint64_t *key, uint64_t *key_alt,
                         int32_t *sidx, int32_t *sidx_alt, int64_t m, bool *in_alt,
                         cudaStream_t st) {
    return radix_sort_pairs<uint64_t, int32_t>(temp, temp_bytes, key, key_alt, sidx, sidx_alt, m,
                                               0, 64, true, in_alt, st);
}

cudaError_t launch_tile_ranges(int64_t j0, int64_t K, bool key16, const void *skey, int2 *rng,
                               int tbase, cudaStream_t st) {
    if (K == 0) return cudaSuccess;
    const unsigned g = grid_for((K + 7) / 8, 256);
    if (key16)
        k_tile_ranges<uint16_t><<<g, 256, 0, st>>>(j0, K, (const uint16_t *)skey, rng, tbase);
    else
        k_tile_ranges<uint32_t><<<g, 256, 0, st>>>(j0, K, (const uint32_t *)skey, rng, tbase);
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_raster_t(const RasterArgs &a, cudaStream_t st) {
    const size_t smem = raster_smem_bytes();
    static int grid = 0;
    if (grid == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_raster<MODE>,
                                                              32 * kRasterWarps, smem);
        if (e != cudaSuccess) return e;
        grid = sms * (per_sm > 0 ? per_sm : 1);  // persistent: fill every SM exactly
    }
    k_raster<MODE><<<grid, 32 * kRasterWarps, raster_smem_bytes(), st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_raster(int mode, const RasterArgs &a, int ntiles, cudaStream_t st) {
    if (ntiles == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.tile_counter, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    switch (mode) {
        case kRender: return launch_raster_t<kRender>(a, st);
        case kImportance: return launch_raster_t<kImportance>(a, st);
        case kScore: return launch_raster_t<kScore>(a, st);
        case kRecords: return launch_raster_t<kRecords>(a, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_splat_reduce(int64_t total, int64_t n, const int32_t *ids, const int64_t *offs,
                                const double2 *partial, double P, const int32_t *perm,
                                double2 *vals, cudaStream_t st) {
    if (total == 0) return cudaSuccess;
    k_splat_reduce<<<grid_for(total, 256), 256, 0, st>>>(total, n, ids, offs, partial, P, perm,
                                                         vals);
    // (one warp per 32 entries, 8 warps per block: grid_for(total, 256) blocks)
    return cudaGetLastError();
}

cudaError_t launch_view_accumulate(int64_t n, int nview, const double2 *vals,
                                   double *cam_imp_rows, double *imp_acc, double *dmse_acc,
                                   double *dmse_rows, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_view_accumulate<<<grid_for(n, 256), 256, 0, st>>>(n, nview, vals, cam_imp_rows, imp_acc,
                                                         dmse_acc, dmse_rows);
    return cudaGetLastError();
}

cudaError_t launch_mse_reduce(int nview, int ntiles, double *tile_se, double P,
                              double *mse_acc, double *mse_rows, cudaStream_t st) {
    k_mse_reduce<<<nview, 1024, 0, st>>>(ntiles, tile_se, P, tile_se + (int64_t)nview * ntiles);
    k_mse_accumulate<<<1, 32, 0, st>>>(nview, tile_se + (int64_t)nview * ntiles, mse_acc,
                                       mse_rows);
    return cudaGetLastError();
}

cudaError_t launch_finalize(int64_t n, int S, double *imp, double *dmse, double *mse,
                            cudaStream_t st) {
    int64_t m = n > 0 ? n : 1;
    k_finalize<<<grid_for(m, 256), 256, 0, st>>>(n, (double)S, imp, dmse, mse);
    return cudaGetLastError();
}

cudaError_t launch_records_gather(int64_t m, const uint64_t *skey, const int32_t *sidx,
                                  const int32_t *ids, const double *ra, const double *rt,
                                  const double *rp, int64_t *splat_ids, int64_t *pixels,
                                  double *alphas, double *trans_at, double *partials,
                                  const int32_t *perm, cudaStream_t st) {
    if (m == 0) return cudaSuccess;
    k_records_gather<<<grid_for(m, 256), 256, 0, st>>>(m, skey, sidx, ids, ra, rt, rp, splat_ids,
                                                        pixels, alphas, trans_at, partials, perm);
    return cudaGetLastError();
}

cudaError_t launch_colors_from_rec(int64_t n, const SplatRec *rec, const int32_t *mpos,
                                  double *colors, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_colors_from_rec<<<grid_for(n, 256), 256, 0, st>>>(n, rec, mpos, colors);
    return cudaGetLastError();
}

cudaError_t launch_bin_outputs(int64_t n, const uint64_t *skey, uint64_t invalid,
                               const int32_t *sids,
                               unsigned long long *nvalid_dev, int64_t *order, int ntiles,
                               const int2 *rng, int64_t K, int64_t *tile_offsets,
                               const int2 *pair, int32_t *tile_splats, const int32_t *mperm,
                               cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(nvalid_dev, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    if (n > 0) {
        k_count_valid<<<grid_for(n, 256), 256, 0, st>>>(n, skey, invalid, nvalid_dev);
        k_order_out<<<grid_for(n, 256), 256, 0, st>>>(n, sids, mperm, order);
    }
    if (tile_offsets) k_tile_offsets<<<grid_for(ntiles + 1, 128), 128, 0, st>>>(ntiles, rng, K,
                                                                               tile_offsets);
    if (tile_splats && K > 0)
        k_tile_splats<<<grid_for(K, 256), 256, 0, st>>>(K, pair, mperm, tile_splats);
    return cudaGetLastError();
}

}  // namespace potr
