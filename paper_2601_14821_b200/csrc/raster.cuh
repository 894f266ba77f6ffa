// raster.cuh -- launch interface of the prune-score kernels (raster.cu).
#pragma once

#include <string>

#include "common.cuh"

namespace potr {

enum RasterMode { kRender = 0, kImportance = 1, kScore = 2, kRecords = 3 };

struct RasterArgs {
    const SplatRec *rec;
    const int2 *pair;         // sorted pair -> (duplicate index = slot, batch record index v*n + id)
    const int32_t *dup_rank;  // duplicate index -> depth rank (records mode)
    const int2 *ranges;       // per tile [start, end) into perm
    int tiles_x, ntiles;      // ntiles: all tiles of the batch (nview * ntiles_view)
    int ntiles_view;
    int *tile_counter;        // persistent-warp work counter (zeroed per launch)
    int width, height;
    const double *target[kMaxViewBatch];  // per view (H,W,3), score mode
    double *image[kMaxViewBatch];         // per view (H,W,3), nullable
    double *trans[kMaxViewBatch];         // per view (H,W), nullable
    double2 *partial;         // per duplicate (dSE, T*alpha)
    int self_target;          // score mode: the targets are this render (dr = 0), images out
    double *tile_se;          // per tile squared error (score mode)
    // records mode
    unsigned long long *rec_counter;
    int64_t rec_capacity;
    uint64_t *rec_key;
    double *rec_alpha, *rec_t, *rec_p;
    // evidence counters (nullable): [1] live evaluations, [2] contributions
    unsigned long long *counters;
};

size_t raster_smem_bytes();

// Batch-wide depth key: (view << nbits) | (depth bits - lo_bits), exact and
// order preserving when every valid depth of the batch lies in the bound.
struct DepthKey {
    int compact;          // 0: raw 64-bit depth bits per view (per-view sorts)
    int nbits;
    uint64_t lo_bits;
    uint64_t sentinel;    // (1 << nbits) - 1: invalid splats sort last in their view
    int *overflow;        // set when a depth falls outside the bound
    // split keys (compact only): hi = key >> shift as 32 bits, sorted first;
    // ties in hi are then ordered by the full key (k_depth_fixup)
    int shift;            // 0: no split (the 64-bit key is sorted directly)
    uint32_t *khi;        // per record: key >> shift
};

cudaError_t launch_bbox(int64_t n, const double *pos, unsigned long long *out, cudaStream_t st);

// Per-splat view-independent terms (Sigma, prefilter threshold), once per call.
cudaError_t launch_splat_prep(const potr_splats &sp, SplatPrep *prep, cudaStream_t st);
cudaError_t launch_splat_slots(const potr_splats &sp, const int32_t *perm, double *pos, double *sh,
                               double *opac, SplatPrep *prep, cudaStream_t st);
// slot-ordered SH rows (k_splat_slots called with sh = null)
cudaError_t launch_slot_sh(int64_t n, const double *sh_in, const int32_t *perm, double *sh,
                           cudaStream_t st);
// colours of the drawn records of a batch binned with colors = 0
cudaError_t launch_batch_colors(int64_t n, int nview, const double *pos, const double *sh,
                                const double *opac, const CamBatch &cams, SplatRec *rec,
                                cudaStream_t st);
cudaError_t launch_preprocess(const potr_splats &sp, const SplatPrep *prep, const CamBatch &cams,
                              int nview, int tiles_x, int all_colors, int colors, int cull,
                              const DepthKey &dk,
                              SplatRec *rec, TileSpan *spans, uint64_t *key, int32_t *cnt,
                              unsigned long long *counters, cudaStream_t st);
// Spatial record layout.  Each call sorts the splats by the Morton code of
// their centres (slot r holds splat perm[r]; rank = perm^-1) and copies them
// in that order (k_splat_slots); the batch pipeline -- preprocess, depth keys,
// records, pairs -- then runs in slot space, so the records one tile reads lie
// in a few short address ranges instead of all over the view's records (L2
// and TLB locality for the rasterizer's fetches).  Slots map back to splat
// indices where results leave the pipeline (per-splat sums, records, depth
// order, tile lists), and exact depth ties are ordered by splat index in the
// run fixup, so results are bit-identical to splat order.  The 64-bit
// fallback sorts run in splat order.
cudaError_t spatial_order_temp(int64_t n, size_t *bytes);
cudaError_t spatial_order(void *temp, size_t temp_bytes, int64_t n, const double *pos,
                          const double lo[3], const double hi[3], uint32_t *code,
                          uint32_t *code_sorted, int32_t *perm, int32_t *rank, cudaStream_t st);
cudaError_t launch_project_dump(const potr_splats &sp, const Cam &cam, double *mean2d,
                                double *cov2d, double *depth, double *radius, uint8_t *valid,
                                double *colors, cudaStream_t st);
cudaError_t depth_sort_temp(int64_t n, size_t *bytes);
cudaError_t depth_sort32_temp(int64_t n, size_t *bytes);
cudaError_t depth_sort32(void *temp, size_t temp_bytes, uint32_t *key_a, uint32_t *key_b,
                         int32_t *val_a, int32_t *val_b, int64_t n, int end_bit, bool *in_alt,
                         cudaStream_t st);
// Orders every run of equal hi keys in the hi-sorted (khi_sorted, sids) by the
// full 64-bit key of its records (stable).  Runs longer than kFixupRun (or a
// valid key sharing the invalid sentinel's hi) set *overflow: the caller falls
// back to the 64-bit sort.
constexpr int kFixupRun = 64;
cudaError_t launch_depth_fixup(int64_t total, const uint32_t *khi_sorted, int32_t *sids,
                               const uint64_t *key, int shift, uint64_t sentinel, int nbits,
                               int *overflow, const int32_t *perm, int64_t n, cudaStream_t st);
cudaError_t launch_gather_keys(int64_t total, const int32_t *sids, const uint64_t *key,
                               uint64_t *skey, cudaStream_t st);
cudaError_t depth_sort(void *temp, size_t temp_bytes, uint64_t *key_a, uint64_t *key_b,
                       int32_t *val_a, int32_t *val_b, int64_t n, int end_bit, int64_t val_base,
                       bool *in_alt, cudaStream_t st);
cudaError_t scan_temp(int64_t n, size_t *bytes);
cudaError_t scan_counts(void *temp, size_t temp_bytes, const int32_t *ids, const int32_t *cnt,
                        int64_t *offs, int64_t total, cudaStream_t st);
cudaError_t launch_duplicate(int64_t total, int64_t n, const int32_t *ids, const int64_t *offs,
                             const SplatRec *rec, const TileSpan *spans, int tiles_x, int ntiles,
                             int sb, bool key16, int cull, void *tkey, int32_t *dup_id,
                             int32_t *dup_rank, cudaStream_t st);
cudaError_t tile_sort_temp(int64_t K, int nkeys, bool key16, size_t *bytes);
cudaError_t tile_sort(void *temp, size_t temp_bytes, bool key16, void *tkey, void *tkey_alt,
                      const int32_t *dup_id, int64_t j0, int2 *pair, int2 *pair_alt, int64_t K,
                      int nkeys, bool *in_alt, cudaStream_t st);
cudaError_t records_sort_temp(int64_t m, size_t *bytes);
cudaError_t records_sort(void *temp, size_t temp_bytes, uint64_t *key, uint64_t *key_alt,
                         int32_t *sidx, int32_t *sidx_alt, int64_t m, bool *in_alt,
                         cudaStream_t st);
cudaError_t launch_tile_ranges(int64_t j0, int64_t K, bool key16, const void *skey, int2 *rng,
                               int tbase, cudaStream_t st);
cudaError_t launch_raster(int mode, const RasterArgs &a, int ntiles, cudaStream_t st);
cudaError_t launch_splat_reduce(int64_t total, int64_t n, const int32_t *ids, const int64_t *offs,
                                const double2 *partial, double P, const int32_t *perm,
                                double2 *vals, cudaStream_t st);
// dmse_rows / mse_rows (nullable): the per-view values as well as their sums
cudaError_t launch_view_accumulate(int64_t n, int nview, const double2 *vals,
                                   double *cam_imp_rows, double *imp_acc, double *dmse_acc,
                                   double *dmse_rows, cudaStream_t st);
cudaError_t launch_mse_reduce(int nview, int ntiles, double *tile_se, double P,
                              double *mse_acc, double *mse_rows, cudaStream_t st);
cudaError_t launch_finalize(int64_t n, int S, double *imp, double *dmse, double *mse,
                            cudaStream_t st);
cudaError_t launch_records_gather(int64_t m, const uint64_t *skey, const int32_t *sidx,
                                  const int32_t *ids, const double *ra, const double *rt,
                                  const double *rp, int64_t *splat_ids, int64_t *pixels,
                                  double *alphas, double *trans_at, double *partials,
                                  const int32_t *perm, cudaStream_t st);
cudaError_t launch_colors_from_rec(int64_t n, const SplatRec *rec, const int32_t *mpos,
                                  double *colors, cudaStream_t st);
cudaError_t launch_bin_outputs(int64_t n, const uint64_t *skey, uint64_t invalid,
                               const int32_t *sids,
                               unsigned long long *nvalid_dev, int64_t *order, int ntiles,
                               const int2 *rng, int64_t K, int64_t *tile_offsets,
                               const int2 *pair, int32_t *tile_splats, const int32_t *mperm,
                               cudaStream_t st);

// Image metrics (metrics.cu): out[0] = sum of clamped squared differences,
// out[1..3] = per-channel sums of the cropped SSIM map.
cudaError_t launch_image_compare(int W, int H, const double *a, const double *b,
                                 const double *gauss_w, double *mom, double *partial, double *out,
                                 cudaStream_t st);
int image_compare_partials();

// Codec back end (codec.cu).  Scratch is owned by the caller (grown on demand);
// pinned: >= 64 int64 of pinned host memory.
cudaError_t run_octree(int64_t n, const double *pos, int neyes, const double *eyes_dev,
                       double beta, double gamma, const double *center, double half,
                       int max_depth, uint8_t *out, int64_t capacity, int64_t *out_len,
                       int64_t *order_out, void **scratch, size_t *scratch_cap,
                       int64_t *pinned, cudaStream_t st);
cudaError_t run_attr_streams(int64_t n, const int64_t *order, const double *ycocg,
                             const double *opac, const double *log_scales, const double *rot,
                             double sf_sh, double sf_op, double sf_rot, double sf_sc, uint8_t *out,
                             int64_t capacity, int64_t *stream_lengths, void **scratch,
                             size_t *scratch_cap, int64_t *pinned, cudaStream_t st);

// Decode side (codec.cu).  Error codes of octree_decode_host / run_attr_decode.
enum CodecDecodeError : int {
    kOctTruncated = 1,
    kOctZeroLeaf = 2,
    kOctDepth = 3,
    kOctTrailing = 4,
    kDecTruncated = 5,
    kDecOverlong = 6,
    kDecTrailing = 7,
    kDecCuda = 8,
};
// deserialize_octree's walk (host): leaf centres (positions, n x 3) and depths
// of the first `capacity` splats in DFS order; *count = splats decoded,
// *trailing = bytes left after the root.
int octree_decode_host(const uint8_t *buf, int64_t len, const double *center, double half,
                       int max_depth, int64_t capacity, double *positions, int32_t *depths,
                       int64_t *count, int64_t *trailing);
// decode_attribute_streams on the GPU: host_bytes = streams 1..55 back to back,
// sstart_host[s] = start of stream s + 1 (sstart_host[55] = total length);
// outputs on the device; *n_over = quaternions clamped to the unit ball.
int run_attr_decode(int64_t n, const uint8_t *host_bytes, const int64_t *sstart_host,
                    double sf_sh, double sf_op, double sf_sc, double sf_rot, double *sh,
                    double *opac, double *scales, double *rot, int64_t *n_over, void **scratch,
                    size_t *scratch_cap, int64_t *pinned, cudaStream_t st, std::string *err);

// Pruning controller (controller.cu): order-preserving keys of the removal
// priority m(dm[idx[i]] / dmax) (idx nullable: identity)
cudaError_t launch_removal_keys(int64_t n, const double *dm, const int64_t *idx, double dmax,
                                double a, uint64_t *keys, cudaStream_t st);
cudaError_t launch_iota64(int64_t n, int64_t *out, cudaStream_t st);

// SH recompute (sh.cu)
cudaError_t launch_sh_accumulate(const potr_splats &sp, int ncam, const double *eyes_dev,
                                 const double *cam_imp, double *neq, bool add, cudaStream_t st);
// scratch: sh_solve_scratch_bytes(n) bytes of device memory
size_t sh_solve_scratch_bytes(int64_t n);
cudaError_t launch_sh_solve(const potr_splats &sp, const double *neq, double lambda_y,
                            double par_thr, double zero_thr, double *rgb, double *ycocg,
                            int8_t *status, void *scratch, cudaStream_t st);

}  // namespace potr
