/*
 * potr_b200.h -- C ABI of the B200-native POTR hot path (libpotr_b200.so).
 *
 * The reference (arXiv 2601.14821, /root/reference/pkg/src/potr) is a pure
 * Python package with no FFI; its "plugin interface" for this path is the set
 * of module-level functions in rasterizer.py and compaction.py.  Each entry
 * point below replaces one of them (cited file:line); the Python host mirror
 * paper_2601_14821_b200.{rasterizer,compaction} binds these with ctypes and
 * keeps the reference's signatures, dataclasses and exceptions.
 *
 * Conventions
 *  - Plain C types only.  Arrays are float64, C-contiguous, in the reference's
 *    layouts: positions (n,3), sh (n,3,16) channel-major with coefficient 0 =
 *    DC, opacities (n), scales (n,3), rotations (n,4) wxyz, images (H,W,3).
 *  - Functions without the _host suffix take DEVICE pointers and are ordered
 *    on the context's stream (potr_set_stream; default: the legacy stream).
 *    They do not synchronize unless stated.
 *  - Every function returns 0 on success or a negative POTR_E* code; the
 *    message is available from potr_last_error(ctx).  Nothing throws across
 *    the boundary.
 *  - A context is bound to one device and is not re-entrant: use one context
 *    per host thread (one process per GPU).
 */
#ifndef POTR_B200_H
#define POTR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POTR_B200_ABI_VERSION 1

#define POTR_OK 0
#define POTR_E_ARG (-1)      /* invalid argument (maps to ValueError)     */
#define POTR_E_CUDA (-2)     /* CUDA runtime error                         */
#define POTR_E_NOMEM (-3)    /* device allocation failed                   */
#define POTR_E_CAPACITY (-4) /* caller buffer too small (records mode)     */

typedef struct potr_ctx potr_ctx;

/* scene.py:64-77 Camera.  rot = world-to-camera rows (row-major 3x3). */
typedef struct {
    double eye[3];
    double rot[9];
    double fx, fy, cx, cy;
    int32_t width, height;
} potr_camera;

/* scene.py:42-61 Splats (activated attributes), device pointers. */
typedef struct {
    int64_t n;
    const double *positions; /* (n,3)    */
    const double *sh;        /* (n,3,16) */
    const double *opacities; /* (n)      */
    const double *scales;    /* (n,3)    */
    const double *rotations; /* (n,4)    */
} potr_splats;

int potr_abi_version(void);
int potr_create(int device, potr_ctx **out);
void potr_destroy(potr_ctx *ctx);
int potr_set_stream(potr_ctx *ctx, void *cuda_stream);
int potr_synchronize(potr_ctx *ctx);
const char *potr_last_error(potr_ctx *ctx);
/* Number of kernels this context has launched so far (bench evidence). */
int64_t potr_kernel_launches(potr_ctx *ctx);

/* ---- prune-score pass ------------------------------------------------- */

/* forward_stats (rasterizer.py:311-352) / compute_delta_mse (:361-368) /
 * compute_importance (:355-358).
 *   targets: host array of ncam DEVICE pointers to (H,W,3) images, or NULL.
 *   importance (n): mean over cameras of per-camera importance.
 *   camera_importance (ncam,n): nullable.
 *   delta_mse (n) and mse (1): required iff targets != NULL.
 * Deterministic: bit-identical across runs (no floating-point atomics). */
int potr_forward_stats(potr_ctx *ctx, const potr_splats *splats, int ncam,
                       const potr_camera *cams, const double *const *targets,
                       double *importance, double *camera_importance, double *delta_mse,
                       double *mse);

/* The view-sharded building block of forward_stats (rasterizer.py:322-347):
 * scores cameras [0, ncam) and ADDS, in camera order, the un-normalised sums
 *   imp_sum[k] += I_k(s), dmse_sum[k] += dMSE_k(s), mse_sum[0] += mse(s)
 * and writes camera_importance rows (nullable).  A multi-GPU caller
 * all-reduces the sums, then calls potr_finalize_stats with the global
 * camera count. */
int potr_score_views(potr_ctx *ctx, const potr_splats *splats, int ncam,
                     const potr_camera *cams, const double *const *targets, double *imp_sum,
                     double *camera_importance, double *dmse_sum, double *mse_sum);

/* The per-view values behind those sums, for an exactly ordered multi-GPU
 * reduction: camera_importance rows (ncam, n), delta-MSE rows (ncam, n) and
 * per-view MSE (ncam) -- each already divided by P / 3P (:230, :334-335).
 * Adding the rows in camera order reproduces potr_score_views' sums bit for
 * bit.  dmse_rows / mse_rows required with targets. */
int potr_score_views_rows(potr_ctx *ctx, const potr_splats *splats, int ncam,
                          const potr_camera *cams, const double *const *targets,
                          double *camera_importance, double *dmse_rows, double *mse_rows);

/* render_targets + the first compute_delta_mse of an encode in ONE pass: the
 * targets are the renders of these very splats (pipeline.py / pruning.py:132
 * at iteration 1), so c - c_t = 0 exactly and the images are written as the
 * targets while the same walk scores them.  images: host array of ncam device
 * pointers (H, W, 3), outputs.  Sums as potr_score_views (mse_sum gets 0). */
int potr_score_views_self(potr_ctx *ctx, const potr_splats *splats, int ncam,
                          const potr_camera *cams, double *const *images, double *imp_sum,
                          double *camera_importance, double *dmse_sum, double *mse_sum);

/* rasterizer.py:348-352: divide the sums by the total camera count in place
 * (dmse_sum / mse_sum nullable). */
int potr_finalize_stats(potr_ctx *ctx, int64_t n, int total_cams, double *imp_sum,
                        double *dmse_sum, double *mse_sum);

/* render_image (rasterizer.py:270-271): image (H,W,3), trans (H,W) nullable. */
int potr_render(potr_ctx *ctx, const potr_splats *splats, const potr_camera *cam,
                double *image, double *trans);

/* render_targets (rasterizer.py:371-377): ncam views, batched; images and
 * trans are host arrays of ncam device pointers (trans nullable). */
int potr_render_batch(potr_ctx *ctx, const potr_splats *splats, int ncam,
                      const potr_camera *cams, double *const *images, double *const *trans);

/* render_with_records (rasterizer.py:246-267).  Two-call protocol: call with
 * capacity 0 to get *n_records (synchronizes), then with buffers of that
 * capacity.  Records are in the reference's order (depth order of the splat,
 * then row-major pixel).  colors (n,3): compositing colours of valid splats,
 * zero elsewhere.  All arrays device pointers. */
int potr_render_records(potr_ctx *ctx, const potr_splats *splats, const potr_camera *cam,
                        double *image, double *trans, double *colors, int64_t capacity,
                        int64_t *n_records, int64_t *splat_ids, int64_t *pixels,
                        double *alphas, double *trans_at, double *partials);

/* project_splats (rasterizer.py:56-97) + splat_colors (:100-110) for every
 * splat (colors of invalid splats are computed too).  Device outputs:
 * mean2d (n,2), cov2d (n,3), depth (n), radius (n), valid (n) uint8,
 * colors (n,3) nullable. */
int potr_project(potr_ctx *ctx, const potr_splats *splats, const potr_camera *cam,
                 double *mean2d, double *cov2d, double *depth, double *radius, uint8_t *valid,
                 double *colors);

/* Tile binning evidence: the global stable depth order of valid splats
 * (rasterizer.py:248-250) and the per-tile splat lists in (tile, depth, id)
 * order for the rasterizer's 8x4-pixel tiles (row-major tile ids).  order (n) and tile_offsets (ntiles+1) are device
 * int64 outputs; tile_splats (capacity) device int32.  *n_valid and *n_pairs
 * are host outputs (synchronizes).  tile_splats may be NULL to size. */
int potr_bin(potr_ctx *ctx, const potr_splats *splats, const potr_camera *cam,
             int64_t *order, int64_t *n_valid, int64_t *tile_offsets, int32_t *tile_splats,
             int64_t capacity, int64_t *n_pairs);

/* ---- SH recompute ------------------------------------------------------ */

/* compact_scene (compaction.py:195-243).  camera_importance (ncam,n) device.
 * Outputs rgb (n,3,16), ycocg (n,3,16) and status (n) int8:
 *   0 solved, 1 solved after the 1e-10 jitter retry (:140-145),
 *   2 RidgeError -> original coefficients kept, 3 unseen -> DC fallback.
 * rgb may be splats->sh itself (in-place update); ycocg must not overlap it. */
int potr_compact(potr_ctx *ctx, const potr_splats *splats, int ncam, const potr_camera *cams,
                 const double *camera_importance, double lambda_y, double parallel_threshold,
                 double zero_threshold, double *rgb, double *ycocg, int8_t *status);

/* The two halves of potr_compact (build_weighted_system ... compact_splat,
 * compaction.py:89-192), for sweeps (one accumulation, many solves) and
 * sharded use.
 * normal_eqs: (POTR_NEQ_STRIDE, n) entry-major:
 *   rows 0..135 = upper triangle of G = sum_s (w_s y_s)(w_s y_s)^T,
 *   rows 136..183 = B[i][c] = sum_s (w_s y_s)_i (w_s YCoCg(color_s))_c,
 *   row 184 = number of cameras with w_s > 0.
 * potr_sh_accumulate ADDS to normal_eqs (zero it first; lets a caller add
 * view shards); potr_sh_normal_equations OVERWRITES it (no zeroing pass, no
 * read of the old values).  The splat-sharded path (each rank owns a splat
 * span and all views) uses the latter. */
#define POTR_NEQ_STRIDE 185
int potr_sh_accumulate(potr_ctx *ctx, const potr_splats *splats, int ncam,
                       const potr_camera *cams, const double *camera_importance,
                       double *normal_eqs);
int potr_sh_normal_equations(potr_ctx *ctx, const potr_splats *splats, int ncam,
                             const potr_camera *cams, const double *camera_importance,
                             double *normal_eqs);
int potr_sh_solve(potr_ctx *ctx, const potr_splats *splats, const double *normal_eqs,
                  double lambda_y, double parallel_threshold, double zero_threshold,
                  double *rgb, double *ycocg, int8_t *status);

/* ---- pruning controller (pruning.py:57-111) ------------------------------ */

/* The removal order of the candidates idx[0..n) (device int64; NULL: 0..n-1):
 * np.argsort(mapping_m(delta_mse[idx] / delta_mse_max, a), kind="stable")
 * (pruning.py:80-83, :99-100), written to order (device int64, n) as splat
 * indices.  The priorities are computed with numpy's operation order and
 * IEEE division; the sort is the library's stable radix sort (ties keep the
 * candidate order, i.e. ascending index). */
int potr_removal_order(potr_ctx *ctx, int64_t n, const double *delta_mse, const int64_t *idx,
                       double delta_mse_max, double a, int64_t *order);

/* The library's stable LSD radix sort (8-bit digits, one-sweep passes) on
 * device arrays, in place: (keys, vals) ordered by key bits
 * [begin_bit, end_bit); equal keys keep their input order. */
int potr_sort_pairs_u64(potr_ctx *ctx, int64_t n, uint64_t *keys, int64_t *vals, int begin_bit,
                        int end_bit);

/* ---- image metrics (metrics.py:24-52) ------------------------------------ */

/* MSE of the [0, 1]-clamped images (psnr's, metrics.py:24-30) and mean SSIM
 * over the three channels (11-tap Gaussian window, sigma 1.5, reflect
 * borders, 5-pixel crop, K1 0.01, K2 0.03; :33-52).  a, b: device (H, W, 3)
 * float64; mse, ssim: host outputs (nullable).  Synchronizes the stream. */
int potr_image_compare(potr_ctx *ctx, int width, int height, const double *a, const double *b,
                       double *mse, double *ssim);

/* ---- codec back end (quantize.py, bitstream.py) ---------- */

/* build_octree + serialize_octree (quantize.py:98-170): positions (device,
 * n x 3), camera eyes (host, neyes x 3), tolerance max(gamma, beta * distance
 * to the nearest eye), root cube (host center[3], half; _root_cube or the
 * pinned cube), depth limit <= 24.  Writes the DFS byte stream to `stream`
 * (device, capacity bytes; n * (max_depth + 6) always suffices), its length
 * to *stream_len and the DFS order (original indices) to `order` (device,
 * int64 n).  Synchronizes. */
int potr_octree(potr_ctx *ctx, int64_t n, const double *positions, int neyes, const double *eyes,
                double beta, double gamma, const double *center, double half, int max_depth,
                uint8_t *stream, int64_t capacity, int64_t *stream_len, int64_t *order);

/* encode_attribute_streams (bitstream.py:116-155) of the splats taken in
 * `order`: ycocg (n, 3, 16), opacities, log(scales) (n, 3), rotations (n, 4),
 * all device float64 in original order.  The 55 streams (DC x3, AC x45,
 * opacity, scale x3, rotation x3) are written back to back into `out`
 * (device; 550 n bytes always suffice); their lengths to stream_lengths
 * (host int64[55]).  Synchronizes. */
int potr_attribute_streams(potr_ctx *ctx, int64_t n, const int64_t *order, const double *ycocg,
                           const double *opacities, const double *log_scales,
                           const double *rotations, double sf_sh, double sf_opacity,
                           double sf_rotation, double sf_scale, uint8_t *out, int64_t capacity,
                           int64_t *stream_lengths);

/* deserialize_octree (quantize.py:180-226): the preorder octree stream's leaf
 * centres, repeated per leaf count, in DFS order (positions, host, capacity x
 * 3) and their depths (host int32); center / half as stored in the header
 * (float32 values).  *count = splats in the stream (may exceed capacity).
 * Host code: a preorder stream's node boundaries are only known by parsing
 * it.  Errors (-1, message "octree: ..."): truncated stream, leaf with zero
 * splats, internal node below the depth limit, trailing bytes. */
int potr_octree_decode(potr_ctx *ctx, const uint8_t *stream, int64_t len, const double *center,
                       double half, int max_depth, int64_t capacity, double *positions,
                       int32_t *depths, int64_t *count);

/* decode_attribute_streams (bitstream.py:169-220) on the GPU: streams = the
 * 55 attribute streams back to back (host), their lengths (host int64[55]);
 * outputs (device, n splats in DFS order): sh (n, 3, 16) RGB, opacities,
 * scales (n, 3), rotations (n, 4) (w, x, y, z); *n_clamped = quaternions
 * outside the unit ball (clamped, as the reference warns).  Errors (-1):
 * "varint: truncated varint stream" / "varint: overlong varint" (the
 * reference's ValueError) and "integrity: <what> stream has <k> trailing
 * bytes" (IntegrityError).  Synchronizes. */
int potr_attribute_decode(potr_ctx *ctx, int64_t n, const uint8_t *streams,
                          const int64_t *stream_lengths, double sf_sh, double sf_opacity,
                          double sf_rotation, double sf_scale, double *sh, double *opacities,
                          double *scales, double *rotations, int64_t *n_clamped);

/* ---- tuning ------------------------------------------------------------- */

/* Views processed per pipeline round (1..8, default 8; env POTR_B200_VIEW_BATCH). */
#define POTR_OPT_VIEW_BATCH 1
/* Depth-sort key: 0 (default) compact batch key sorted as 32-bit hi parts with
 * runs of equal hi re-ordered by the full key; 1 raw 64-bit depth bits, one
 * sort per view; 2 the compact key sorted as 64 bits.  All give the same order. */
#define POTR_OPT_RAW_DEPTH_KEYS 2
/* 1 (default): drop (tile, splat) pairs whose tile no prefilter-passing sample
 * can reach (conservative ellipse test: renders and records bit-identical,
 * scores equal up to summation order); 0: the full bbox tile rectangle.
 * potr_bin always reports the bbox lists. */
#define POTR_OPT_TILE_CULL 3
/* 1 (default): each view's splat records are stored in the Morton order of
 * the splat centres, so a tile's records sit close together in HBM (L2 and
 * TLB locality for the rasterizer's fetches); 0: splat order.  Results are
 * bit-identical either way. */
#define POTR_OPT_SPATIAL_RECORDS 4
/* View batches binned ahead while a scoring call's SH rows are still
 * uploading (potr_upload_async), 1..8, default 6 (env POTR_B200_LOOKAHEAD);
 * each holds its own records and pair lists, bounded to half the free device
 * memory.  Results are bit-identical for every value. */
#define POTR_OPT_LOOKAHEAD 5
int potr_set_option(potr_ctx *ctx, int option, int value);

/* ---- evidence: live stage timing and work counters --------------------- */

/* Stages timed with CUDA events on the context stream while profiling. */
#define POTR_STAGE_PREPROCESS 0     /* kernel (a)                          */
#define POTR_STAGE_DEPTH_SORT 1     /* radix sort of the depth keys        */
#define POTR_STAGE_SCAN 2           /* pair-count gather + scan            */
#define POTR_STAGE_DUPLICATE 3      /* (tile, splat) pair emission         */
#define POTR_STAGE_TILE_SORT 4      /* radix sort on tile id + ranges      */
#define POTR_STAGE_RASTER 5         /* kernels (c)+(d), fused              */
#define POTR_STAGE_REDUCE 6         /* per-splat slot sums, mse            */
#define POTR_STAGE_SH_ACCUMULATE 7  /* kernel (e) normal equations         */
#define POTR_STAGE_SH_SOLVE 8       /* kernel (e) batched Cholesky         */
#define POTR_STAGE_COUNT 9

/* Enabling resets the totals; read synchronizes and returns cumulative
 * milliseconds and launch counts per stage (arrays of POTR_STAGE_COUNT). */
int potr_profile_enable(potr_ctx *ctx, int enable);
int potr_profile_read(potr_ctx *ctx, double *stage_ms, int64_t *stage_launches);

/* Work counters for the roofline's algorithmic units (off by default):
 * out[0] = bbox pixel evaluations E of the reference loop (rasterizer.py:159-166),
 * out[1] = evaluations with T >= T_TERMINATE (exp evaluated),
 * out[2] = composited contributions M, out[3] = (tile, splat) pairs.
 * Enabling resets; read synchronizes. */
int potr_counters_enable(potr_ctx *ctx, int enable);
int potr_counters_read(potr_ctx *ctx, uint64_t *out);

/* ---- host-buffer convenience (reference-facing drop-in) ---------------- */

/* Host -> device copy of `bytes` from a pageable (or any) host buffer into
 * device memory, ordered on the context stream: host threads stage chunks
 * into a pinned ring while the DMA engine moves the previous chunk.  The
 * source may be reused when the call returns. */
int potr_copy_to_device(potr_ctx *ctx, void *dst, const void *src, int64_t bytes);

/* Queues a host -> device copy of `bytes` from `src` (pinned or pageable) to
 * `dst` and returns at once; one library worker thread runs the queue in
 * order (the pinned ring for pageable sources, host threads filling it).  A
 * scoring call (potr_score_views*, potr_forward_stats) whose splats' sh is
 * the destination of the LAST queued copy waits only for the earlier ones
 * (positions before its bounds, the other attributes before its first
 * batch), bins its first view batches while the rows arrive (their geometry
 * needs no SH) and gives them their colours once the copy is done -- this is
 * how the reference's per-call upload of a fresh subset() (pruning.py:161)
 * overlaps the binning.  Every other entry point, and potr_upload_wait,
 * completes all queued copies first; each `src` must stay valid until then.
 * Replaces the reference's implicit numpy -> device transfer (no reference
 * counterpart). */
int potr_upload_async(potr_ctx *ctx, void *dst, const void *src, int64_t bytes);
/* Completes every queued potr_upload_async (the context stream is ordered
 * after them); returns the first error, if any.  No-op without any. */
int potr_upload_wait(potr_ctx *ctx);

/* forward_stats with HOST arrays in the reference layouts; copies in, runs,
 * copies out and synchronizes.  targets: host array of ncam host pointers or
 * NULL.  camera_importance nullable. */
int potr_forward_stats_host(potr_ctx *ctx, int64_t n, const double *positions, const double *sh,
                            const double *opacities, const double *scales,
                            const double *rotations, int ncam, const potr_camera *cams,
                            const double *const *targets, double *importance,
                            double *camera_importance, double *delta_mse, double *mse);

/* compact_scene with HOST arrays. */
int potr_compact_host(potr_ctx *ctx, int64_t n, const double *positions, const double *sh,
                      int ncam, const potr_camera *cams, const double *camera_importance,
                      double lambda_y, double parallel_threshold, double zero_threshold,
                      double *rgb, double *ycocg, int8_t *status);

#ifdef __cplusplus
}
#endif
#endif /* POTR_B200_H */
