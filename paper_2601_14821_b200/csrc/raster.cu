// raster.cu -- the prune-score pass on sm_100a: kernels (a)-(d).
//
//  (a) k_preprocess    project + cov2d + radius + clipped bbox + conic + SH
//                      colour + fp64 depth key, one thread per splat
//                      (rasterizer.py:56-110, :135-154)
//  (b) k_gather_counts / k_duplicate / k_tile_ranges around two CUB onesweep
//      radix sorts: a stable sort of the fp64 depth bits (ties keep ascending
//      splat id == np.argsort(kind="stable"), :248-250), then a stable sort of
//      the per-(tile, splat) duplicates on the tile id, giving every tile its
//      splats in (tile, depth, id) order.
//  (c)+(d) k_raster    one CTA per 16x16 tile; splat batches staged in shared
//      memory; front-to-back compositing with the reference's exact per-pixel
//      rules (:159-201); a second walk over the same batches evaluates the
//      closed-form removal delta PD = a/(1-a) (P_K - P_i - T c) (:232-243),
//      dSE = sum_ch PD^2 + 2 PD (c - c_t) (:333) and T*alpha (:228); warps
//      reduce per splat with shuffles and the 8 warps combine in a fixed
//      order into one slot per (tile, splat) pair -- no floating-point
//      atomics, so scores are bit-reproducible.
//  k_splat_reduce      per splat, sums its pair slots in tile order, divides
//                      by P / 3P and adds into the camera-ordered accumulators
//                      (:226-230, :334, :340-347).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "raster.cuh"

#ifndef POTR_RASTER_MIN_BLOCKS
#define POTR_RASTER_MIN_BLOCKS 6
#endif

namespace potr {

// ---------------------------------------------------------------------------
// (a) preprocess

__global__ void __launch_bounds__(256) k_preprocess(potr_splats sp, Cam cam, int tiles_x,
                                                     int all_colors, SplatRec *__restrict__ rec,
                                                     uint64_t *__restrict__ key,
                                                     int32_t *__restrict__ cnt,
                                                     unsigned long long *counters) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= sp.n) return;
    Proj pr = project_one(sp.positions + 3 * k, sp.scales + 3 * k, sp.rotations + 4 * k, cam);
    int32_t c = 0;
    uint64_t kk = ~0ull;
    if (pr.valid) {
        kk = (uint64_t)__double_as_longlong(pr.depth);  // depth > 0.01: bits are monotone
        const int W = cam.width, H = cam.height;
        double x0 = floor(pr.mx - pr.radius), x1 = ceil(pr.mx + pr.radius);
        double y0 = floor(pr.my - pr.radius), y1 = ceil(pr.my + pr.radius);
        if (x0 < 0) x0 = 0;
        if (y0 < 0) y0 = 0;
        if (x1 > W - 1) x1 = W - 1;
        if (y1 > H - 1) y1 = H - 1;
        double det = pr.a * pr.c - pr.b * pr.b;
        bool draw = !(x0 > x1 || y0 > y1) && det > 0.0;
        if (draw || all_colors) {
            SplatRec r;
            r.mx = pr.mx;
            r.my = pr.my;
            r.ia = pr.c / det;
            r.ib = -pr.b / det;
            r.ic = pr.a / det;
            double o = sp.opacities[k];
            r.opac = o;
            double rgb[3];
            splat_color(sp.positions + 3 * k, sp.sh + 48 * k, cam, rgb);
            r.cr = rgb[0];
            r.cg = rgb[1];
            r.cb = rgb[2];
            r.pthr = log(kAlphaFloor / o) - kPowerMargin;
            r.x0 = (int32_t)x0;
            r.x1 = (int32_t)x1;
            r.y0 = (int32_t)y0;
            r.y1 = (int32_t)y1;
            if (!draw) r.x0 = 1, r.x1 = 0;  // empty: never drawn
            rec[k] = r;
        }
        if (draw) {
            int tx0 = (int)x0 >> kTileWLog2, tx1 = (int)x1 >> kTileWLog2;
            int ty0 = (int)y0 >> kTileHLog2, ty1 = (int)y1 >> kTileHLog2;
            c = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
            if (counters)  // E: pixels the reference loop visits (rasterizer.py:159-161)
                atomicAdd(&counters[0],
                          (unsigned long long)((x1 - x0 + 1.0) * (y1 - y0 + 1.0)));
        }
    }
    key[k] = kk;
    cnt[k] = c;
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

__global__ void k_gather_counts(int64_t n, const int32_t *__restrict__ ids,
                                const int32_t *__restrict__ cnt, int64_t *__restrict__ out) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) out[r] = cnt[ids[r]];
}

__global__ void k_duplicate(int64_t n, const int32_t *__restrict__ ids,
                            const int64_t *__restrict__ offs, const SplatRec *__restrict__ rec,
                            int tiles_x, uint32_t *__restrict__ tkey, int32_t *__restrict__ dup_id,
                            int32_t *__restrict__ dup_rank) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t o = offs[r], e = offs[r + 1];
    if (o == e) return;
    int32_t id = ids[r];
    const SplatRec &R = rec[id];
    int tx0 = R.x0 >> kTileWLog2, tx1 = R.x1 >> kTileWLog2;
    int ty0 = R.y0 >> kTileHLog2, ty1 = R.y1 >> kTileHLog2;
    for (int ty = ty0; ty <= ty1; ty++)
        for (int tx = tx0; tx <= tx1; tx++) {
            tkey[o] = (uint32_t)(ty * tiles_x + tx);
            dup_id[o] = id;
            if (dup_rank) dup_rank[o] = (int32_t)r;
            o++;
        }
}

// Tile [start, end) ranges of the sorted pairs, plus each sorted pair's splat
// id (so the rasterizer's chunk fetch is two loads deep, not three).
__global__ void k_tile_ranges(int64_t K, const uint32_t *__restrict__ skey,
                              const int32_t *__restrict__ perm, const int32_t *__restrict__ dup_id,
                              int32_t *__restrict__ sid, int2 *__restrict__ rng) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= K) return;
    sid[j] = dup_id[perm[j]];
    uint32_t t = skey[j];
    if (j == 0 || skey[j - 1] != t) rng[t].x = (int)j;
    if (j == K - 1 || skey[j + 1] != t) rng[t].y = (int)(j + 1);
}

__global__ void k_iota(int64_t n, int32_t *out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)i;
}

// ---------------------------------------------------------------------------
// (c)+(d) tile rasterizer and removal-effect pass

// Per-warp staging: two chunk buffers so the next chunk's records stream in
// with cp.async while the current one is composited.
constexpr int kChunkBitsCap = 128;  // chunks per tile whose contribution bits are kept

struct WarpSmem {
    SplatRec rec[2][32];
    int32_t dup[2][32];
    // score mode: bit e of cbits[c] = entry e of chunk c composited somewhere
    // in pass 1; pass 2 visits only those (others leave T and P unchanged)
    unsigned cbits[kChunkBitsCap];
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

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

// One sample of rasterizer.py:162-171 for this lane's pixel: returns true when
// the splat composites here (alpha >= ALPHA_FLOOR), with the capped alpha.
__device__ __forceinline__ bool sample_alpha(const SplatRec &R, double pxc, double pyc, bool live,
                                             const double2 *tab, double &alpha) {
    if (!live) return false;
    double dx = pxc - R.mx, dy = pyc - R.my;
    double power = -0.5 * (R.ia * dx * dx + R.ic * dy * dy) - R.ib * dx * dy;
    if (power < R.pthr) return false;  // o*exp(power) < ALPHA_FLOOR for certain
    alpha = R.opac * exp_neg(power, tab);
    if (alpha > kAlphaCap) alpha = kAlphaCap;
    return !(alpha < kAlphaFloor);
}

// The lane's slice of a chunk: pair index, splat id (and depth rank).
struct ChunkIds {
    int32_t d, id;
    bool valid;
};

template <int MODE>
__device__ __forceinline__ ChunkIds fetch_ids(const RasterArgs &a, int cbase, int end, int lane) {
    ChunkIds c;
    const int j = cbase + lane;
    c.valid = j < end;
    c.d = c.valid ? a.perm[j] : 0;
    c.id = c.valid ? a.sid[j] : 0;
    return c;
}

// Start the async copy of a chunk's records into buffer `b`; always commits a
// group so wait_group counts stay uniform.
template <int MODE>
__device__ __forceinline__ void issue_chunk(const RasterArgs &a, WarpSmem &S, int b,
                                            const ChunkIds &c, int lane) {
    if (c.valid) {
        const char *src = reinterpret_cast<const char *>(a.rec + c.id);
        char *dst = reinterpret_cast<char *>(&S.rec[b][lane]);
#pragma unroll
        for (int q = 0; q < (int)(sizeof(SplatRec) / 16); q++) cp_async16(dst + 16 * q, src + 16 * q);
        S.dup[b][lane] = c.d;
    }
    cp_async_commit();
}

// MODE: kRender     forward only, writes image/trans
//       kImportance forward with per-pair T*alpha slots (no targets)
//       kScore      forward, then the removal-effect walk with targets
//       kRecords    forward, appending every contribution record
//
// Persistent: each warp pulls 8x4 tiles from an atomic counter until none are
// left; a tile's result depends only on its own list, so the schedule does not
// affect the output bits.  Each pass walks the tile's list in 32-pair chunks
// through a two-stage cp.async pipeline.
template <int MODE>
__global__ void __launch_bounds__(32 * kRasterWarps, POTR_RASTER_MIN_BLOCKS) k_raster(RasterArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem &S = reinterpret_cast<WarpSmem *>(smem_raw)[threadIdx.x >> 5];
    double2 *tab = reinterpret_cast<double2 *>(smem_raw + sizeof(WarpSmem) * kRasterWarps);
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    for (int i = threadIdx.x; i < 64; i += blockDim.x)
        tab[i] = make_double2(kExpTable[i][0], kExpTable[i][1]);
    __syncthreads();

    for (;;) {
        int tile = 0;
        if (lane == 0) tile = atomicAdd(a.tile_counter, 1);
        tile = __shfl_sync(FULL, tile, 0);
        if (tile >= a.ntiles) return;

        const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
        const int px = tx * kTileW + (lane & 7), py = ty * kTileH + (lane >> 3);
        const bool inside = px < a.width && py < a.height;
        const int64_t pix = (int64_t)py * a.width + px;
        const int2 range = a.ranges[tile];
        const int start = range.x, end = range.y > range.x ? range.y : range.x;
        const double pxc = (double)px + 0.5, pyc = (double)py + 0.5;

        // ---- pass 1: front-to-back compositing (rasterizer.py:159-201) ----
        double T = 1.0, P0 = 0.0, P1 = 0.0, P2 = 0.0;
        bool done = !inside;
        int stop = start;      // entries [start, stop) were walked
        int written = start;   // importance slots written up to here
        if (start < end && !__all_sync(FULL, done)) {
            issue_chunk<MODE>(a, S, 0, fetch_ids<MODE>(a, start, end, lane), lane);
            ChunkIds next = fetch_ids<MODE>(a, start + 32, end, lane);
            int b = 0;
            for (int base = start; base < end; base += 32, b ^= 1) {
                issue_chunk<MODE>(a, S, b ^ 1, next, lane);
                next = fetch_ids<MODE>(a, base + 64, end, lane);
                cp_async_wait<1>();
                __syncwarp();
                const int cnt = min(32, end - base);
                double my_imp = 0.0;
                unsigned cbits = 0u;
                int e = 0;
                while (e < cnt) {
                    const SplatRec &R = S.rec[b][e];
                    const bool live =
                        !done && px >= R.x0 && px <= R.x1 && py >= R.y0 && py <= R.y1;
                    double alpha = 0.0;
                    const bool contrib = sample_alpha(R, pxc, pyc, live, tab, alpha);
                    if (a.counters) {
                        unsigned lv = __ballot_sync(FULL, live);
                        unsigned ct = __ballot_sync(FULL, contrib);
                        if (lane == 0) {
                            atomicAdd(&a.counters[1], (unsigned long long)__popc(lv));
                            atomicAdd(&a.counters[2], (unsigned long long)__popc(ct));
                        }
                    }
                    double timp = 0.0;
                    if (contrib) {
                        if (MODE == kRecords) {
                            unsigned long long slot = atomicAdd(a.rec_counter, 1ull);
                            if ((int64_t)slot < a.rec_capacity) {
                                a.rec_key[slot] = ((uint64_t)(uint32_t)a.dup_rank[S.dup[b][e]] << 32) |
                                                  (uint64_t)(uint32_t)pix;
                                a.rec_alpha[slot] = alpha;
                                a.rec_t[slot] = T;
                                a.rec_p[3 * slot] = P0;
                                a.rec_p[3 * slot + 1] = P1;
                                a.rec_p[3 * slot + 2] = P2;
                            }
                        }
                        const double w = T * alpha;
                        timp = w;
                        P0 += w * R.cr;
                        P1 += w * R.cg;
                        P2 += w * R.cb;
                        T = T * (1.0 - alpha);
                        done = T < kTTerminate;
                    }
                    if (MODE == kImportance && __any_sync(FULL, contrib)) {
                        const double s = warp_sum(timp);
                        if (lane == e) my_imp = s;
                    }
                    if (MODE == kScore && __any_sync(FULL, contrib)) cbits |= 1u << e;
                    e++;
                    if (__all_sync(FULL, done)) break;
                }
                stop = base + e;
                if (MODE == kScore && lane == 0 && ((base - start) >> 5) < kChunkBitsCap)
                    S.cbits[(base - start) >> 5] = cbits;
                if (MODE == kImportance) {
                    if (lane < cnt) a.partial[S.dup[b][lane]] = make_double2(0.0, my_imp);
                    written = base + cnt;
                }
                __syncwarp();
                if (__all_sync(FULL, done)) break;
            }
            cp_async_wait<0>();
            __syncwarp();
        }

        if (MODE != kScore) {
            if (inside && a.image) {
                a.image[3 * pix] = P0;
                a.image[3 * pix + 1] = P1;
                a.image[3 * pix + 2] = P2;
            }
            if (inside && a.trans) a.trans[pix] = T;
            if (MODE == kImportance)  // pairs after the early-out contribute nothing
                for (int j = written + lane; j < end; j += 32)
                    a.partial[a.perm[j]] = make_double2(0.0, 0.0);
            continue;
        }

        // ---- pass 2: removal effect (rasterizer.py:232-243, :322-336) -----
        const double PK0 = P0, PK1 = P1, PK2 = P2;
        double dr0 = 0.0, dr1 = 0.0, dr2 = 0.0, se = 0.0;
        if (inside) {
            dr0 = PK0 - a.target[3 * pix];
            dr1 = PK1 - a.target[3 * pix + 1];
            dr2 = PK2 - a.target[3 * pix + 2];
            se = dr0 * dr0 + dr1 * dr1 + dr2 * dr2;
            if (a.image) {
                a.image[3 * pix] = PK0;
                a.image[3 * pix + 1] = PK1;
                a.image[3 * pix + 2] = PK2;
            }
            if (a.trans) a.trans[pix] = T;
        }
        se = warp_sum(se);
        if (lane == 0) a.tile_se[tile] = se;
        T = 1.0;
        P0 = P1 = P2 = 0.0;
        done = !inside;
        if (start < stop) {
            issue_chunk<MODE>(a, S, 0, fetch_ids<MODE>(a, start, end, lane), lane);
            ChunkIds next = fetch_ids<MODE>(a, start + 32, end, lane);
            int b = 0;
            for (int base = start; base < stop; base += 32, b ^= 1) {
                issue_chunk<MODE>(a, S, b ^ 1, next, lane);
                next = fetch_ids<MODE>(a, base + 64, end, lane);
                cp_async_wait<1>();
                __syncwarp();
                const int cnt = min(32, end - base);
                const int lim = min(cnt, stop - base);
                const int ci = (base - start) >> 5;
                unsigned todo = ci < kChunkBitsCap ? S.cbits[ci] : 0xffffffffu;
                if (lim < 32) todo &= (1u << lim) - 1u;
                double my_dse = 0.0, my_imp = 0.0;
                while (todo) {
                    const int e = __ffs(todo) - 1;
                    todo &= todo - 1u;
                    const SplatRec &R = S.rec[b][e];
                    const bool live =
                        !done && px >= R.x0 && px <= R.x1 && py >= R.y0 && py <= R.y1;
                    double alpha = 0.0;
                    const bool contrib = sample_alpha(R, pxc, pyc, live, tab, alpha);
                    double dse = 0.0, timp = 0.0;
                    if (contrib) {
                        // prune_deltas, forward form: a/(1-a) * (P_K - P_i - T c)
                        const double f = alpha / (1.0 - alpha);
                        const double pd0 = f * (PK0 - P0 - T * R.cr);
                        const double pd1 = f * (PK1 - P1 - T * R.cg);
                        const double pd2 = f * (PK2 - P2 - T * R.cb);
                        dse = pd0 * pd0 + 2.0 * pd0 * dr0;
                        dse = dse + (pd1 * pd1 + 2.0 * pd1 * dr1);
                        dse = dse + (pd2 * pd2 + 2.0 * pd2 * dr2);
                        const double w = T * alpha;
                        timp = w;
                        P0 += w * R.cr;
                        P1 += w * R.cg;
                        P2 += w * R.cb;
                        T = T * (1.0 - alpha);
                        done = T < kTTerminate;
                    }
                    if (__any_sync(FULL, contrib)) {
                        const double s0 = warp_sum(dse);
                        const double s1 = warp_sum(timp);
                        if (lane == e) {
                            my_dse = s0;
                            my_imp = s1;
                        }
                    }
                }
                if (lane < cnt) a.partial[S.dup[b][lane]] = make_double2(my_dse, my_imp);
                written = base + cnt;
                __syncwarp();
            }
            cp_async_wait<0>();
            __syncwarp();
        }
        for (int j = written + lane; j < end; j += 32)
            a.partial[a.perm[j]] = make_double2(0.0, 0.0);
    }
}

// Per-splat sum of its (tile, splat) slots, in tile order (deterministic),
// then the per-camera normalisation and the camera-ordered accumulation.
__global__ void k_splat_reduce(int64_t n, const int32_t *__restrict__ ids,
                               const int64_t *__restrict__ offs,
                               const double2 *__restrict__ partial, double P, int64_t cam_row,
                               double *__restrict__ cam_imp, double *__restrict__ imp_acc,
                               double *__restrict__ dmse_acc) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int32_t id = ids[r];
    int64_t o = offs[r], e = offs[r + 1];
    double dse = 0.0, imp = 0.0;
    for (int64_t j = o; j < e; j++) {
        double2 v = partial[j];
        dse += v.x;
        imp += v.y;
    }
    double ci = imp / P;  // rasterizer.py:230
    if (cam_imp) cam_imp[cam_row * n + id] = ci;
    imp_acc[id] += ci;                                  // :344, :348
    if (dmse_acc) dmse_acc[id] += dse / (P * 3.0);      // :334, :346
}

// Sum of the per-tile squared errors; mse(s) = sum / 3P (:335), added to the
// camera-ordered accumulator (:347).
__global__ void k_mse_reduce(int ntiles, const double *__restrict__ tile_se, double P,
                             double *__restrict__ mse_acc) {
    __shared__ double red[32];
    double s = 0.0;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s += tile_se[t];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
        mse_acc[0] += t / (P * 3.0);
    }
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
                                 double *partials) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    uint64_t k = skey[i];
    int32_t s = sidx[i];
    splat_ids[i] = ids[(int64_t)(k >> 32)];
    pixels[i] = (int64_t)(k & 0xffffffffu);
    alphas[i] = ra[s];
    trans_at[i] = rt[s];
    partials[3 * i] = rp[3 * (int64_t)s];
    partials[3 * i + 1] = rp[3 * (int64_t)s + 1];
    partials[3 * i + 2] = rp[3 * (int64_t)s + 2];
}

__global__ void k_colors_from_rec(int64_t n, const uint64_t *__restrict__ key,
                                  const SplatRec *__restrict__ rec, double *colors) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    bool valid = key[k] != ~0ull;
    colors[3 * k] = valid ? rec[k].cr : 0.0;
    colors[3 * k + 1] = valid ? rec[k].cg : 0.0;
    colors[3 * k + 2] = valid ? rec[k].cb : 0.0;
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

__global__ void k_tile_splats(int64_t K, const int32_t *__restrict__ perm,
                              const int32_t *__restrict__ dup_id, int32_t *__restrict__ out) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < K) out[j] = dup_id[perm[j]];
}

__global__ void k_order_out(int64_t nv, const int32_t *__restrict__ ids, int64_t *__restrict__ out) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nv) out[r] = ids[r];
}

__global__ void k_count_valid(int64_t n, const uint64_t *__restrict__ skey,
                              unsigned long long *__restrict__ out) {
    // sorted keys: valid ones first; find the boundary
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    bool v = skey[r] != ~0ull;
    bool next_v = (r + 1 < n) ? (skey[r + 1] != ~0ull) : false;
    if (v && !next_v) *out = (unsigned long long)(r + 1);
}

// ---------------------------------------------------------------------------
// host-side launchers (called from capi.cu)

static inline unsigned grid_for(int64_t n, int block) {
    return (unsigned)((n + block - 1) / block);
}

size_t raster_smem_bytes() { return sizeof(WarpSmem) * kRasterWarps + 64 * sizeof(double2); }

cudaError_t launch_preprocess(const potr_splats &sp, const Cam &cam, int tiles_x, int all_colors,
                              SplatRec *rec, uint64_t *key, int32_t *cnt,
                              unsigned long long *counters, cudaStream_t st) {
    if (sp.n == 0) return cudaSuccess;
    k_preprocess<<<grid_for(sp.n, 256), 256, 0, st>>>(sp, cam, tiles_x, all_colors, rec, key, cnt,
                                                       counters);
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

cudaError_t launch_iota(int64_t n, int32_t *out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_iota<<<grid_for(n, 256), 256, 0, st>>>(n, out);
    return cudaGetLastError();
}

cudaError_t depth_sort(void *temp, size_t temp_bytes, const uint64_t *key, uint64_t *skey,
                       const int32_t *iota, int32_t *sids, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, key, skey, iota, sids, (int)n, 0, 64,
                                           st);
}

cudaError_t depth_sort_temp(int64_t n, size_t *bytes) {
    return cub::DeviceRadixSort::SortPairs((void *)nullptr, *bytes, (const uint64_t *)nullptr,
                                           (uint64_t *)nullptr, (const int32_t *)nullptr,
                                           (int32_t *)nullptr, (int)n, 0, 64);
}

cudaError_t scan_counts(void *temp, size_t temp_bytes, const int32_t *ids, const int32_t *cnt,
                        int64_t *cnt_sorted, int64_t *offs, int64_t n, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(offs, 0, sizeof(int64_t), st);
    if (e != cudaSuccess || n == 0) return e;
    k_gather_counts<<<grid_for(n, 256), 256, 0, st>>>(n, ids, cnt, cnt_sorted);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return cub::DeviceScan::InclusiveSum(temp, temp_bytes, cnt_sorted, offs + 1, (int)n, st);
}

cudaError_t scan_temp(int64_t n, size_t *bytes) {
    return cub::DeviceScan::InclusiveSum((void *)nullptr, *bytes, (const int64_t *)nullptr,
                                         (int64_t *)nullptr, (int)n);
}

cudaError_t launch_duplicate(int64_t n, const int32_t *ids, const int64_t *offs,
                             const SplatRec *rec, int tiles_x, uint32_t *tkey, int32_t *dup_id,
                             int32_t *dup_rank, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_duplicate<<<grid_for(n, 256), 256, 0, st>>>(n, ids, offs, rec, tiles_x, tkey, dup_id,
                                                   dup_rank);
    return cudaGetLastError();
}

static int bits_for(int ntiles) {
    int b = 1;
    while ((1 << b) < ntiles) b++;
    return b;
}

cudaError_t tile_sort(void *temp, size_t temp_bytes, const uint32_t *tkey, uint32_t *skey,
                      const int32_t *iota, int32_t *perm, int64_t K, int ntiles, cudaStream_t st) {
    if (K == 0) return cudaSuccess;
    return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, tkey, skey, iota, perm, (int)K, 0,
                                           bits_for(ntiles), st);
}

cudaError_t tile_sort_temp(int64_t K, int ntiles, size_t *bytes) {
    return cub::DeviceRadixSort::SortPairs((void *)nullptr, *bytes, (const uint32_t *)nullptr,
                                           (uint32_t *)nullptr, (const int32_t *)nullptr,
                                           (int32_t *)nullptr, (int)K, 0, bits_for(ntiles));
}

cudaError_t records_sort_temp(int64_t m, size_t *bytes) {
    return cub::DeviceRadixSort::SortPairs((void *)nullptr, *bytes, (const uint64_t *)nullptr,
                                           (uint64_t *)nullptr, (const int32_t *)nullptr,
                                           (int32_t *)nullptr, (int)m, 0, 64);
}

cudaError_t records_sort(void *temp, size_t temp_bytes, const uint64_t *key, uint64_t *skey,
                         const int32_t *iota, int32_t *sidx, int64_t m, cudaStream_t st) {
    if (m == 0) return cudaSuccess;
    return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, key, skey, iota, sidx, (int)m, 0, 64,
                                           st);
}

cudaError_t launch_tile_ranges(int64_t K, const uint32_t *skey, const int32_t *perm,
                               const int32_t *dup_id, int32_t *sid, int2 *rng, int ntiles,
                               cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(rng, 0, sizeof(int2) * (size_t)ntiles, st);
    if (e != cudaSuccess || K == 0) return e;
    k_tile_ranges<<<grid_for(K, 256), 256, 0, st>>>(K, skey, perm, dup_id, sid, rng);
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

cudaError_t launch_splat_reduce(int64_t n, const int32_t *ids, const int64_t *offs,
                                const double2 *partial, double P, int64_t cam_row, double *cam_imp,
                                double *imp_acc, double *dmse_acc, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_splat_reduce<<<grid_for(n, 256), 256, 0, st>>>(n, ids, offs, partial, P, cam_row, cam_imp,
                                                      imp_acc, dmse_acc);
    return cudaGetLastError();
}

cudaError_t launch_mse_reduce(int ntiles, const double *tile_se, double P, double *mse_acc,
                              cudaStream_t st) {
    k_mse_reduce<<<1, 1024, 0, st>>>(ntiles, tile_se, P, mse_acc);
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
                                  cudaStream_t st) {
    if (m == 0) return cudaSuccess;
    k_records_gather<<<grid_for(m, 256), 256, 0, st>>>(m, skey, sidx, ids, ra, rt, rp, splat_ids,
                                                        pixels, alphas, trans_at, partials);
    return cudaGetLastError();
}

cudaError_t launch_colors_from_rec(int64_t n, const uint64_t *key, const SplatRec *rec,
                                   double *colors, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_colors_from_rec<<<grid_for(n, 256), 256, 0, st>>>(n, key, rec, colors);
    return cudaGetLastError();
}

cudaError_t launch_bin_outputs(int64_t n, const uint64_t *skey, const int32_t *sids,
                               unsigned long long *nvalid_dev, int64_t *order, int ntiles,
                               const int2 *rng, int64_t K, int64_t *tile_offsets,
                               const int32_t *perm, const int32_t *dup_id, int32_t *tile_splats,
                               cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(nvalid_dev, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    if (n > 0) {
        k_count_valid<<<grid_for(n, 256), 256, 0, st>>>(n, skey, nvalid_dev);
        k_order_out<<<grid_for(n, 256), 256, 0, st>>>(n, sids, order);
    }
    if (tile_offsets) k_tile_offsets<<<grid_for(ntiles + 1, 128), 128, 0, st>>>(ntiles, rng, K,
                                                                               tile_offsets);
    if (tile_splats && K > 0)
        k_tile_splats<<<grid_for(K, 256), 256, 0, st>>>(K, perm, dup_id, tile_splats);
    return cudaGetLastError();
}

}  // namespace potr
