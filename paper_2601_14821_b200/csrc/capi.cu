// capi.cu -- the extern "C" boundary (include/potr_b200.h): context, grow-only
// device workspace, and the per-view orchestration of kernels (a)-(e).
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <utility>
#include <cstring>
#include <omp.h>
#include <nvtx3/nvToolsExt.h>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "raster.cuh"
#include "sort.cuh"

using namespace potr;

namespace {

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
};

}  // namespace

#ifndef POTR_SPATIAL_DEFAULT
#define POTR_SPATIAL_DEFAULT 1
#endif

struct potr_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    int64_t launches = 0;
    // per-view workspace
    // dup_id: record of each duplicated pair; pair: per tile-sorted pair
    // (slot, record); perm: the tile sort's alternate (slot, record) buffer
    DevBuf rec, key, skey, sids, cnt, offs, perm2, tkey, tskey, perm, pair, dup_id,
        dup_rank,
        partial, ranges, tile_se, temp, nvalid;
    // records mode
    DevBuf rkey, rskey, rsidx, ralpha, rt, rp, rcounter;
    // SH
    DevBuf eyes, neq;
    // host-buffer API staging
    DevBuf h_pos, h_sh, h_op, h_sc, h_rot, h_tg, h_imp, h_ci, h_dm, h_mse, h_rgb, h_yc, h_st;
    int64_t *pinned = nullptr;  // small pinned scratch for scalars
    // potr_copy_to_device: pinned staging ring for pageable host sources
#ifndef POTR_RING_BUFFERS
#define POTR_RING_BUFFERS 4
#endif
    static constexpr int kRing = POTR_RING_BUFFERS;
    void *ring[kRing] = {};
    cudaEvent_t ring_ev[kRing] = {};
    int ring_next = 0;  // the ring buffer the next chunk takes (rotates across copies)
    // live per-stage timing (CUDA events on ctx->stream) and work counters
    bool profile = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> events;
    std::vector<cudaEvent_t> event_pool;
    double stage_ms[POTR_STAGE_COUNT] = {0};
    int64_t stage_launches[POTR_STAGE_COUNT] = {0};
    bool counting = false;
    DevBuf counters;
    int64_t pairs_total = 0;
    DevBuf tile_counter, ci_v, dm_v, bbox, overflow, vidx, khi, skhi, prep, spans;
    DevBuf met_mom, met_part, met_w, met_out;  // image metrics scratch
    DevBuf sort_k, sort_v, rm_keys;            // potr_sort_pairs_u64 / potr_removal_order
    DevBuf sh_scratch;                         // SH solve size classes
    void *codec_scratch = nullptr;             // codec back end scratch
    size_t codec_cap = 0;
    DevBuf codec_eyes;
    bool depth_split = false;  // last bin_batch sorted split keys: skey not materialised
    double scene_lo[3] = {0, 0, 0}, scene_hi[3] = {0, 0, 0};  // splat position bbox
    uint64_t invalid_key0 = ~0ull;  // depth key of an invalid splat in view 0 of the last batch
    int view_batch = kMaxViewBatch;
    int depth_keys = 0;  // POTR_OPT_RAW_DEPTH_KEYS: 0 split compact, 1 raw, 2 compact 64-bit
    bool tile_cull = true;  // POTR_OPT_TILE_CULL
    bool spatial = POTR_SPATIAL_DEFAULT != 0;  // POTR_OPT_SPATIAL_RECORDS
    // spatial record order of the current call's splats and their slot-ordered
    // copy (raster.cuh spatial_order); prep: k_splat_prep in splat order
    DevBuf mperm, mrank, mcode, mcode2, slot_pos, slot_sh, slot_opac, slot_prep;
    bool spatial_ok = false;     // this call's splats have a slot order
    bool prep_ok = false;        // ctx->prep holds this call's splats
    bool batch_spatial = false;  // the last bin_batch ran in slot space
    bool slot_sh_pending = false;  // slot_sh not yet filled (SH rows still uploading)
    // potr_upload_async: host -> device copies queued FIFO on copy_stream and
    // driven by one persistent worker thread (the pinned ring for pageable
    // sources, a plain async copy for pinned ones); each records its event
    struct UploadJob {
        int64_t seq;
        void *dst;
        const void *src;
        int64_t bytes;
        cudaEvent_t ev;
    };
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t upload_after = nullptr;
    cudaEvent_t poll_ev = nullptr;  // host_wait
    std::thread upload_worker;
    std::mutex upload_mu;
    std::condition_variable upload_cv;
    std::deque<UploadJob> upload_todo;   // the worker's queue (under upload_mu)
    std::vector<UploadJob> upload_jobs;  // issued and not yet joined (caller's thread)
    std::vector<cudaEvent_t> upload_ev_pool;
    int64_t upload_issued = 0;
    int64_t upload_done = 0;  // under upload_mu
    bool upload_quit = false;  // under upload_mu
    int upload_rc = 0;         // first failure, under upload_mu
    std::string upload_err;
    bool upload_pending = false;  // upload_jobs is not empty
    // Binned batches waiting for their raster: while the SH rows upload, the
    // scoring loop bins up to `lookahead` batches ahead (colours deferred),
    // each into its own set of the buffers that binning hands to the raster
    // and reduce (the active set lives in rec / sids / offs / pair / ranges).
    static constexpr int kMaxSets = 8;
    struct BatchSet {
        DevBuf rec, sids, offs, pair, ranges;
    };
    BatchSet sets[kMaxSets];
    int active_set = 0;
    int lookahead = 6;  // POTR_B200_LOOKAHEAD
};

namespace {

int fail(potr_ctx *ctx, int code, const std::string &msg) {
    if (ctx) ctx->err = msg;
    return code;
}

#define CK(expr)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess)                                                            \
            return fail(ctx, POTR_E_CUDA,                                                 \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));              \
    } while (0)

// Launch-count bookkeeping for the bench's gpu_launches evidence.
#define LAUNCH(n_kernels, expr)    \
    do {                           \
        CK(expr);                  \
        ctx->launches += (n_kernels); \
    } while (0)

int ensure(potr_ctx *ctx, DevBuf &b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return 0;
    if (b.p) {
        cudaError_t e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return fail(ctx, POTR_E_CUDA, cudaGetErrorString(e));
        cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
    }
    size_t want = bytes + bytes / 8;  // headroom for the next, slightly larger view
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, POTR_E_NOMEM,
                    "cudaMalloc(" + std::to_string(want) + "): " + cudaGetErrorString(e));
    }
    b.cap = want;
    return 0;
}

#define ENSURE(buf, bytes)                            \
    do {                                              \
        int _rc = ensure(ctx, buf, (size_t)(bytes));  \
        if (_rc) return _rc;                          \
    } while (0)

cudaEvent_t take_event(potr_ctx *ctx) {
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// RAII-free stage bracket: begin/end record events when profiling is on.
// NVTX range names of the stages (SURVEY.md section 5 tracing): visible in
// any NVTX-aware tool; a push/pop costs nanoseconds when none is attached.
const char *const kStageNames[POTR_STAGE_COUNT] = {
    "potr:preprocess", "potr:depth_sort", "potr:scan",   "potr:duplicate",    "potr:tile_sort",
    "potr:raster",     "potr:reduce",     "potr:sh_acc", "potr:sh_solve"};

struct Stage {
    potr_ctx *ctx;
    int id;
    cudaEvent_t a = nullptr;
    bool open = true;
    Stage(potr_ctx *c, int i) : ctx(c), id(i) {
        nvtxRangePushA(kStageNames[i]);
        if (ctx->profile) {
            a = take_event(ctx);
            cudaEventRecord(a, ctx->stream);
        }
    }
    void end() {
        if (open) {
            nvtxRangePop();
            open = false;
        }
        if (ctx->profile && a) {
            cudaEvent_t b = take_event(ctx);
            cudaEventRecord(b, ctx->stream);
            ctx->events.push_back({id, {a, b}});
            a = nullptr;
        }
    }
    ~Stage() {
        if (open) nvtxRangePop();  // early return on an error path
    }
};

template <typename T>
T *P(DevBuf &b) {
    return reinterpret_cast<T *>(b.p);
}

Cam to_cam(const potr_camera &c) {
    Cam o;
    std::memcpy(&o, &c, sizeof(Cam));
    return o;
}

int check_splats(potr_ctx *ctx, const potr_splats *sp) {
    if (!sp) return fail(ctx, POTR_E_ARG, "splats is NULL");
    if (sp->n < 0 || sp->n > 0x7ffffff0LL) return fail(ctx, POTR_E_ARG, "splat count out of range");
    if (sp->n > 0 && (!sp->positions || !sp->sh || !sp->opacities || !sp->scales || !sp->rotations))
        return fail(ctx, POTR_E_ARG, "splat array pointer is NULL");
    return 0;
}

// the SH path reads only positions and sh
int check_splats_ps(potr_ctx *ctx, const potr_splats *sp) {
    if (!sp) return fail(ctx, POTR_E_ARG, "splats is NULL");
    if (sp->n < 0 || sp->n > 0x7ffffff0LL) return fail(ctx, POTR_E_ARG, "splat count out of range");
    if (sp->n > 0 && (!sp->positions || !sp->sh))
        return fail(ctx, POTR_E_ARG, "splat array pointer is NULL");
    return 0;
}

int check_cam(potr_ctx *ctx, const potr_camera *c) {
    if (!c) return fail(ctx, POTR_E_ARG, "camera is NULL");
    if (c->width <= 0 || c->height <= 0 || (int64_t)c->width * c->height > 0x7fffffffLL)
        return fail(ctx, POTR_E_ARG, "camera size out of range");
    // tile rows / columns are 16-bit in the per-entry TileSpan
    if (c->width > 65535 * kTileW || c->height > 65535 * kTileH)
        return fail(ctx, POTR_E_ARG, "camera size out of range (tile grid over 65535)");
    return 0;
}

unsigned long long *counters(potr_ctx *ctx) {
    return ctx->counting ? P<unsigned long long>(ctx->counters) : nullptr;
}

struct ViewGeom {
    int W, H, tiles_x, tiles_y, ntiles;
    double P;
};

ViewGeom geom(const potr_camera &c) {
    ViewGeom g;
    g.W = c.width;
    g.H = c.height;
    g.tiles_x = (g.W + kTileW - 1) / kTileW;
    g.tiles_y = (g.H + kTileH - 1) / kTileH;
    g.ntiles = g.tiles_x * g.tiles_y;
    g.P = (double)g.W * (double)g.H;
    return g;
}

double ordered_to_double(unsigned long long u) {
    const unsigned long long b = (u >> 63) ? (u & ~(1ull << 63)) : ~u;
    double d;
    std::memcpy(&d, &b, sizeof(d));
    return d;
}

uint64_t dbits(double d) {
    uint64_t b;
    std::memcpy(&b, &d, sizeof(b));
    return b;
}

int bits_for_tiles(int nkeys) {
    int b = 1;
    while ((1 << b) < nkeys) b++;
    return b;
}

int bitlen(uint64_t x) {
    int b = 0;
    while (x) {
        b++;
        x >>= 1;
    }
    return b;
}

// ---- uploads -------------------------------------------------------------

// The binning's host readbacks wait for the context stream.  While an upload
// is pending they poll an event instead of blocking in cudaStreamSynchronize:
// the upload worker's own CUDA calls (its ring copies) stalled behind a
// blocked synchronize, which serialised the upload with the binning.
cudaError_t host_wait(potr_ctx *ctx) {
    if (!ctx->upload_pending) return cudaStreamSynchronize(ctx->stream);
    if (!ctx->poll_ev) {
        cudaError_t e = cudaEventCreateWithFlags(&ctx->poll_ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(ctx->poll_ev, ctx->stream);
    if (e != cudaSuccess) return e;
    for (;;) {
        e = cudaEventQuery(ctx->poll_ev);
        if (e != cudaErrorNotReady) return e;
        std::this_thread::yield();
    }
}

// Pageable host -> device: chunks of kRingChunk bytes go through a ring of
// pinned buffers; host threads (OpenMP) fill chunk c + 1 while the DMA engine
// moves chunk c, so a pageable source uploads at close to the pinned PCIe
// rate instead of the driver's single-threaded staging.  Thread-safe against
// the caller's thread (potr_upload_async runs it on its own thread): touches
// only the ring and `st`, reports through *err.
#ifndef POTR_RING_CHUNK_MB
#define POTR_RING_CHUNK_MB 8  // C3 pageable: SH rows 24.2 -> 21.8 ms, geometry 7.9 -> 6.6 (32 and 16 MB measured)
#endif
constexpr size_t kRingChunk = (size_t)POTR_RING_CHUNK_MB << 20;

// Host threads filling the pinned ring: this process's share of the cores
// (torchrun's LOCAL_WORLD_SIZE processes copy at the same time on one host),
// minus `spare`, at most 16.
int ring_threads(int spare) {
    int local = 1;
    if (const char *lw = std::getenv("LOCAL_WORLD_SIZE")) local = std::atoi(lw);
    if (local < 1) local = 1;
    int t = omp_get_num_procs() / local - spare;
    return t < 1 ? 1 : t > 16 ? 16 : t;
}

int ring_copy(potr_ctx *ctx, void *dst, const void *src, int64_t bytes, cudaStream_t st,
              int threads, std::string *err) {
#define RING_CK(expr)                                                        \
    do {                                                                     \
        cudaError_t _e = (expr);                                             \
        if (_e != cudaSuccess) {                                             \
            *err = std::string(#expr) + ": " + cudaGetErrorString(_e);       \
            return POTR_E_CUDA;                                              \
        }                                                                    \
    } while (0)
    for (int r = 0; r < potr_ctx::kRing; r++) {
        if (!ctx->ring[r]) {
            RING_CK(cudaMallocHost(&ctx->ring[r], kRingChunk));
            RING_CK(cudaEventCreateWithFlags(&ctx->ring_ev[r], cudaEventDisableTiming));
        }
    }
    const char *s = reinterpret_cast<const char *>(src);
    char *d = reinterpret_cast<char *>(dst);
    // the first chunk takes the buffer after the previous copy's last one, so
    // back-to-back copies (the geometry arrays) keep filling one buffer while
    // the DMA engine drains another instead of waiting on the same buffer
    int64_t c = ctx->ring_next;
    for (int64_t off = 0; off < bytes; off += (int64_t)kRingChunk, c++) {
        const int b = (int)(c % potr_ctx::kRing);
        const int64_t len = bytes - off < (int64_t)kRingChunk ? bytes - off : (int64_t)kRingChunk;
        // the buffer's previous DMA (from this call or an earlier one) must be
        // done before it is refilled; a never-recorded event returns at once
        RING_CK(cudaEventSynchronize(ctx->ring_ev[b]));
        char *stage = reinterpret_cast<char *>(ctx->ring[b]);
        const int t_used = len < ((int64_t)1 << 20) ? 1 : threads;
#pragma omp parallel for num_threads(t_used) schedule(static)
        for (int t = 0; t < t_used; t++) {
            const int64_t a = len * t / t_used, e = len * (t + 1) / t_used;
            std::memcpy(stage + a, s + off + a, (size_t)(e - a));
        }
        RING_CK(cudaMemcpyAsync(d + off, stage, (size_t)len, cudaMemcpyHostToDevice, st));
        RING_CK(cudaEventRecord(ctx->ring_ev[b], st));
        ctx->ring_next = (int)((c + 1) % potr_ctx::kRing);
    }
#undef RING_CK
    return POTR_OK;
}

// Waits until upload `seq` (and so every earlier one: one FIFO worker, one
// copy stream) is issued, and orders the context stream after it.
int upload_wait_seq(potr_ctx *ctx, int64_t seq) {
    if (seq <= 0) return 0;
    cudaEvent_t ev = nullptr;
    for (auto &j : ctx->upload_jobs)
        if (j.seq == seq) ev = j.ev;
    int rc;
    std::string err;
    {
        std::unique_lock<std::mutex> lk(ctx->upload_mu);
        ctx->upload_cv.wait(lk, [ctx, seq] { return ctx->upload_done >= seq; });
        rc = ctx->upload_rc;
        err = ctx->upload_err;
    }
    if (rc) return fail(ctx, rc, "upload: " + err);
    if (ev) CK(cudaStreamWaitEvent(ctx->stream, ev, 0));
    return 0;
}

// The pending upload whose destination is `dst` (its seq), or 0.
int64_t upload_seq_of(potr_ctx *ctx, const void *dst) {
    for (auto &j : ctx->upload_jobs)
        if (j.dst == dst) return j.seq;
    return 0;
}

// Completes every pending potr_upload_async: the host side is done with the
// sources and the context stream is ordered after the copies.
int upload_join(potr_ctx *ctx) {
    if (ctx->upload_jobs.empty()) return 0;
    const int rc = upload_wait_seq(ctx, ctx->upload_jobs.back().seq);
    {
        // on failure the worker skips the rest: wait for it to pass them all
        std::unique_lock<std::mutex> lk(ctx->upload_mu);
        const int64_t last = ctx->upload_jobs.back().seq;
        ctx->upload_cv.wait(lk, [ctx, last] { return ctx->upload_done >= last; });
        ctx->upload_rc = 0;
        ctx->upload_err.clear();
    }
    for (auto &j : ctx->upload_jobs) ctx->upload_ev_pool.push_back(j.ev);
    ctx->upload_jobs.clear();
    ctx->upload_pending = false;
    return rc;
}

#define JOIN_UPLOAD(ctx)                   \
    do {                                   \
        int _jrc = upload_join(ctx);       \
        if (_jrc) return _jrc;             \
    } while (0)

// Makes buffer set j the active one (potr_ctx::BatchSet).
void activate_set(potr_ctx *ctx, int j) {
    if (j == ctx->active_set) return;
    auto swap_in = [ctx](potr_ctx::BatchSet &b) {
        std::swap(ctx->rec, b.rec);
        std::swap(ctx->sids, b.sids);
        std::swap(ctx->offs, b.offs);
        std::swap(ctx->pair, b.pair);
        std::swap(ctx->ranges, b.ranges);
    };
    swap_in(ctx->sets[ctx->active_set]);  // park the active set
    swap_in(ctx->sets[j]);
    ctx->active_set = j;
}

// Grows the active set's buffers to the largest capacity any set has seen, so
// sets that take turns with batches of different sizes stop reallocating (a
// cudaFree synchronizes the device, which would stall the upload overlap).
int level_active_set(potr_ctx *ctx) {
    size_t cap[5] = {0, 0, 0, 0, 0};
    for (auto &b : ctx->sets) {
        const DevBuf *d[5] = {&b.rec, &b.sids, &b.offs, &b.pair, &b.ranges};
        for (int i = 0; i < 5; i++) cap[i] = d[i]->cap > cap[i] ? d[i]->cap : cap[i];
    }
    DevBuf *a[5] = {&ctx->rec, &ctx->sids, &ctx->offs, &ctx->pair, &ctx->ranges};
    for (int i = 0; i < 5; i++) {
        if (!a[i]->cap || a[i]->cap >= cap[i]) continue;
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaFree(a[i]->p));
        a[i]->p = nullptr;
        a[i]->cap = 0;
        if (cudaMalloc(&a[i]->p, cap[i]) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, POTR_E_NOMEM, "cudaMalloc(" + std::to_string(cap[i]) + ")");
        }
        a[i]->cap = cap[i];  // exactly the largest: no headroom, no runaway growth
    }
    return 0;
}

size_t active_set_bytes(potr_ctx *ctx) {
    return ctx->rec.cap + ctx->sids.cap + ctx->offs.cap + ctx->pair.cap + ctx->ranges.cap;
}

// The view-independent splat terms (k_splat_prep) in splat order, once per
// call when a batch runs in splat order.
int ensure_prep(potr_ctx *ctx, const potr_splats &sp) {
    if (ctx->prep_ok) return 0;
    ENSURE(ctx->prep, sizeof(SplatPrep) * (sp.n > 0 ? sp.n : 1));
    Stage _st(ctx, POTR_STAGE_PREPROCESS);
    LAUNCH(1, launch_splat_prep(sp, P<SplatPrep>(ctx->prep), ctx->stream));
    _st.end();
    ctx->prep_ok = true;
    return 0;
}

// Once per call of a binning entry point: the splats' position bounds (one
// reduction + sync: they bound every view's depth range, which makes the batch
// depth key compact), then the spatial slot order and the slot-ordered splat
// copy with its view-independent terms (or those terms in splat order).
// defer_sh: the SH rows are still uploading (potr_upload_async); their slot-
// ordered copy waits for fill_slot_sh.
// pos_seq / geo_seq: pending uploads (potr_upload_async) to wait for before
// the positions are read / before the other attributes are.
int compute_scene_bounds(potr_ctx *ctx, const potr_splats &sp, bool defer_sh = false,
                         int64_t pos_seq = 0, int64_t geo_seq = 0) {
    ctx->spatial_ok = ctx->prep_ok = ctx->batch_spatial = false;
    ctx->slot_sh_pending = false;
    int wrc = upload_wait_seq(ctx, pos_seq);
    if (wrc) return wrc;
    ENSURE(ctx->bbox, 6 * sizeof(unsigned long long));
    LAUNCH(1, launch_bbox(sp.n, sp.positions, P<unsigned long long>(ctx->bbox), ctx->stream));
    CK(cudaMemcpyAsync(ctx->pinned, ctx->bbox.p, 6 * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(host_wait(ctx));
    for (int i = 0; i < 3; i++) {
        ctx->scene_lo[i] = ordered_to_double((unsigned long long)ctx->pinned[i]);
        ctx->scene_hi[i] = ordered_to_double((unsigned long long)ctx->pinned[3 + i]);
    }
    if (!ctx->spatial || sp.n == 0) {
        if ((wrc = upload_wait_seq(ctx, geo_seq))) return wrc;
        return ensure_prep(ctx, sp);
    }
    Stage _st(ctx, POTR_STAGE_PREPROCESS);
    ENSURE(ctx->mperm, sizeof(int32_t) * sp.n);
    ENSURE(ctx->mrank, sizeof(int32_t) * sp.n);
    ENSURE(ctx->mcode, sizeof(uint32_t) * sp.n);
    ENSURE(ctx->mcode2, sizeof(uint32_t) * sp.n);
    ENSURE(ctx->slot_pos, sizeof(double) * 3 * sp.n);
    ENSURE(ctx->slot_sh, sizeof(double) * 48 * sp.n);
    ENSURE(ctx->slot_opac, sizeof(double) * sp.n);
    ENSURE(ctx->slot_prep, sizeof(SplatPrep) * sp.n);
    size_t t = 0;
    CK(spatial_order_temp(sp.n, &t));
    ENSURE(ctx->temp, t);
    LAUNCH(7, spatial_order(ctx->temp.p, ctx->temp.cap, sp.n, sp.positions, ctx->scene_lo,
                            ctx->scene_hi, P<uint32_t>(ctx->mcode), P<uint32_t>(ctx->mcode2),
                            P<int32_t>(ctx->mperm), P<int32_t>(ctx->mrank), ctx->stream));
    // the other attributes: from here on (the Morton order needed positions only)
    if ((wrc = upload_wait_seq(ctx, geo_seq))) return wrc;
    LAUNCH(1, launch_splat_slots(sp, P<int32_t>(ctx->mperm), P<double>(ctx->slot_pos),
                                 defer_sh ? nullptr : P<double>(ctx->slot_sh),
                                 P<double>(ctx->slot_opac), P<SplatPrep>(ctx->slot_prep),
                                 ctx->stream));
    _st.end();
    ctx->spatial_ok = true;
    ctx->slot_sh_pending = defer_sh;
    return 0;
}

// The slot-ordered SH copy that compute_scene_bounds(defer_sh) left out.
int fill_slot_sh(potr_ctx *ctx, const potr_splats &sp) {
    if (!ctx->slot_sh_pending) return 0;
    Stage _st(ctx, POTR_STAGE_PREPROCESS);
    LAUNCH(1, launch_slot_sh(sp.n, sp.sh, P<int32_t>(ctx->mperm), P<double>(ctx->slot_sh),
                             ctx->stream));
    _st.end();
    ctx->slot_sh_pending = false;
    return 0;
}

// The last batch's slot order (slot -> splat, splat -> slot), or null when it
// ran in splat order.
const int32_t *spatial_perm(potr_ctx *ctx) {
    return ctx->batch_spatial ? P<int32_t>(ctx->mperm) : nullptr;
}
const int32_t *spatial_rank(potr_ctx *ctx) {
    return ctx->batch_spatial ? P<int32_t>(ctx->mrank) : nullptr;
}

// The compact batch depth key (raster.cuh DepthKey) from the scene bounds.
DepthKey depth_key_for(potr_ctx *ctx, const potr_camera *cams, int nview, int64_t n) {
    DepthKey dk;
    std::memset(&dk, 0, sizeof(dk));
    dk.overflow = P<int>(ctx->overflow);
    if (n == 0) return dk;
    double zmin = 1e300, zmax = -1e300;
    for (int v = 0; v < nview; v++) {
        const double *w = cams[v].rot + 6;
        double lo = 0.0, hi = 0.0;
        for (int i = 0; i < 3; i++) {
            const double a = w[i] * (ctx->scene_lo[i] - cams[v].eye[i]);
            const double b = w[i] * (ctx->scene_hi[i] - cams[v].eye[i]);
            lo += a < b ? a : b;
            hi += a < b ? b : a;
        }
        zmin = lo < zmin ? lo : zmin;
        zmax = hi > zmax ? hi : zmax;
    }
    if (!(zmax == zmax) || !(zmin == zmin)) return dk;  // NaN bounds: raw keys
    const double margin = 1e-9 * (std::fabs(zmin) + std::fabs(zmax) + 1.0);
    double lo = zmin - margin;
    if (lo < kNearClip) lo = kNearClip;
    const double hi = zmax + margin;
    if (!(hi > lo)) {
        dk.compact = 1;  // nothing can be valid: any width works
        dk.nbits = 1;
        dk.lo_bits = dbits(kNearClip);
        dk.sentinel = 1;
        return dk;
    }
    const uint64_t range = dbits(hi) - dbits(lo) + 1;
    const int nbits = bitlen(range + 1);
    const int vbits = bitlen((uint64_t)(nview - 1));
    if (nbits + vbits > 64) return dk;
    dk.compact = 1;
    dk.nbits = nbits;
    dk.lo_bits = dbits(lo);
    dk.sentinel = (nbits == 64) ? ~0ull : ((1ull << nbits) - 1);
    return dk;
}

// (a)+(b) for a batch of `nview` views of equal size: preprocess (splat
// attributes read once per batch), per-view stable depth sorts, one scan over
// all (view, rank) counts, one duplicate, one stable tile sort over batch-global
// tile keys, tile ranges.  On return *K_out holds the number of pairs.
// depth_mode: 2 split compact keys (32-bit sort + run fixup), 1 compact 64-bit
// keys, 0 raw per-view 64-bit sorts; a violated bound falls back to 0, an
// over-long run of equal hi keys to 1.
// cull: drop (tile, splat) pairs no sample of which passes the exp prefilter
// (raster.cu row_span); off for potr_bin, whose lists are the bbox lists.
// colors = false: the records' colours are left to launch_batch_colors (SH
// rows still uploading; all_colors must then be false).
int bin_batch(potr_ctx *ctx, const potr_splats &sp, const potr_camera *cams, int nview,
              bool all_colors, bool with_rank, bool cull, int64_t *K_out, int depth_mode = 2,
              bool colors = true) {
    const int64_t n = sp.n;
    const int64_t total = n * nview;
    ViewGeom g = geom(cams[0]);
    const int ntiles_b = g.ntiles * nview;
    CamBatch cb;
    std::memset(&cb, 0, sizeof(cb));
    for (int v = 0; v < nview; v++) cb.cam[v] = to_cam(cams[v]);
    ENSURE(ctx->rec, sizeof(SplatRec) * total);
    ENSURE(ctx->spans, sizeof(TileSpan) * total);
    ENSURE(ctx->key, sizeof(uint64_t) * total);
    ENSURE(ctx->skey, sizeof(uint64_t) * total);
    ENSURE(ctx->sids, sizeof(int32_t) * total);
    ENSURE(ctx->vidx, sizeof(int32_t) * total);
    ENSURE(ctx->cnt, sizeof(int32_t) * total);
    ENSURE(ctx->offs, sizeof(int64_t) * (total + 1));
    ENSURE(ctx->ranges, sizeof(int2) * ntiles_b);
    ENSURE(ctx->tile_se, sizeof(double) * (ntiles_b + kMaxViewBatch));  // + per-view MSE
    ENSURE(ctx->tile_counter, sizeof(int));
    ENSURE(ctx->overflow, 2 * sizeof(int));
    int rc = 0;
    DepthKey dk;
    std::memset(&dk, 0, sizeof(dk));
    dk.overflow = P<int>(ctx->overflow);
    const int forced = ctx->depth_keys == 1 ? 0 : ctx->depth_keys == 2 ? 1 : 2;
    if (depth_mode > forced) depth_mode = forced;
    if (depth_mode > 0) dk = depth_key_for(ctx, cams, nview, n);
    const int key_bits = dk.compact ? dk.nbits + bitlen((uint64_t)(nview - 1)) : 64;
    const bool split = dk.compact && depth_mode == 2;
    if (split) {
        ENSURE(ctx->khi, sizeof(uint32_t) * total);
        ENSURE(ctx->skhi, sizeof(uint32_t) * total);
        dk.shift = key_bits > 32 ? key_bits - 32 : 0;
        dk.khi = P<uint32_t>(ctx->khi);
    }
    ctx->depth_split = split;
    // slot space needs the split sort: its run fixup orders exact ties by splat
    // index (the 64-bit fallback sorts keep input order, i.e. slot order)
    ctx->batch_spatial = ctx->spatial_ok && split && dk.shift > 0;
    if (!ctx->batch_spatial && (rc = ensure_prep(ctx, sp))) return rc;
    potr_splats sp_b = sp;
    const SplatPrep *prep_b = P<SplatPrep>(ctx->prep);
    if (ctx->batch_spatial) {
        sp_b.positions = P<double>(ctx->slot_pos);
        sp_b.sh = P<double>(ctx->slot_sh);
        sp_b.opacities = P<double>(ctx->slot_opac);
        sp_b.scales = nullptr;     // folded into slot_prep
        sp_b.rotations = nullptr;
        prep_b = P<SplatPrep>(ctx->slot_prep);
    }
    CK(cudaMemsetAsync(ctx->overflow.p, 0, 2 * sizeof(int), ctx->stream));
    size_t t1 = 0, t2 = 0;
    CK(split ? depth_sort32_temp(total, &t1) : depth_sort_temp(total, &t1));
    CK(scan_temp(total, &t2));
    ENSURE(ctx->temp, t1 > t2 ? t1 : t2);

    {
        Stage _st(ctx, POTR_STAGE_PREPROCESS);
        LAUNCH(1, launch_preprocess(sp_b, prep_b, cb, nview, g.tiles_x, all_colors ? 1 : 0,
                                    colors ? 1 : 0, cull ? 1 : 0, dk,
                                    P<SplatRec>(ctx->rec), P<TileSpan>(ctx->spans),
                                    P<uint64_t>(ctx->key),
                                    P<int32_t>(ctx->cnt), counters(ctx),
                                    ctx->stream));
        _st.end();
    }
    {
        Stage _st(ctx, POTR_STAGE_DEPTH_SORT);
        // sorted keys / record indices end in skey / sids (buffers swapped
        // when the double-buffered sort finished in the other half)
        if (split) {  // 32-bit sort of the hi keys, then runs of equal hi by full key
            bool alt = false;
            ctx->launches += sort_launches(0, key_bits - dk.shift);
            CK(depth_sort32(ctx->temp.p, ctx->temp.cap, P<uint32_t>(ctx->khi),
                            P<uint32_t>(ctx->skhi), P<int32_t>(ctx->vidx), P<int32_t>(ctx->sids),
                            total, key_bits - dk.shift, &alt, ctx->stream));
            if (!alt) {
                std::swap(ctx->khi, ctx->skhi);
                std::swap(ctx->vidx, ctx->sids);
            }
            if (dk.shift)
                LAUNCH(1, launch_depth_fixup(total, P<uint32_t>(ctx->skhi), P<int32_t>(ctx->sids),
                                             P<uint64_t>(ctx->key), dk.shift, dk.sentinel, dk.nbits,
                                             P<int>(ctx->overflow) + 1, spatial_perm(ctx), n,
                                             ctx->stream));
        } else if (dk.compact) {  // one stable sort of the whole batch
            const int end_bit = key_bits;
            bool alt = false;
            ctx->launches += sort_launches(0, end_bit);
            CK(depth_sort(ctx->temp.p, ctx->temp.cap, P<uint64_t>(ctx->key),
                          P<uint64_t>(ctx->skey), P<int32_t>(ctx->vidx), P<int32_t>(ctx->sids),
                          total, end_bit, 0, &alt, ctx->stream));
            if (!alt) {
                std::swap(ctx->key, ctx->skey);
                std::swap(ctx->vidx, ctx->sids);
            }
        } else {  // raw 64-bit depth bits: one sort per view, all with the same
                  // pass count, so every view's result ends in the same half
            bool alt = true;
            ctx->launches += nview * sort_launches(0, 64);
            for (int v = 0; v < nview; v++)
                CK(depth_sort(ctx->temp.p, ctx->temp.cap, P<uint64_t>(ctx->key) + v * n,
                              P<uint64_t>(ctx->skey) + v * n, P<int32_t>(ctx->vidx) + v * n,
                              P<int32_t>(ctx->sids) + v * n, n, 64, (int64_t)v * n, &alt,
                              ctx->stream));
            if (!alt) {
                std::swap(ctx->key, ctx->skey);
                std::swap(ctx->vidx, ctx->sids);
            }
        }
        _st.end();
    }
    {
        Stage _st(ctx, POTR_STAGE_SCAN);
        // single-pass scan (sort.cu) gathering the counts in depth order
        ctx->launches += 1;
        CK(scan_counts(ctx->temp.p, ctx->temp.cap, P<int32_t>(ctx->sids), P<int32_t>(ctx->cnt),
                       P<int64_t>(ctx->offs), total, ctx->stream));
        _st.end();
    }
    // tile sort groups: sb views per stable sort, 16-bit keys when they fit
    const int sb_max = 65536 / g.ntiles;
    const bool key16 = sb_max >= 1;
    const int sb = key16 ? (sb_max < nview ? sb_max : nview) : nview;
    // one readback: the pair count, the key-bound flags and the pair index
    // where each sort group begins (pairs are view-major)
    CK(cudaMemcpyAsync(ctx->pinned, P<int64_t>(ctx->offs) + total, sizeof(int64_t),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(ctx->pinned + 1, ctx->overflow.p, 2 * sizeof(int), cudaMemcpyDeviceToHost,
                       ctx->stream));
    for (int v = sb; v < nview; v += sb)
        CK(cudaMemcpyAsync(&ctx->pinned[2 + v], P<int64_t>(ctx->offs) + (int64_t)v * n,
                           sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CK(host_wait(ctx));
    int flags[2];
    std::memcpy(flags, ctx->pinned + 1, sizeof(flags));
    if (dk.compact && flags[0] != 0)  // bound violated: exact raw-key fallback
        return bin_batch(ctx, sp, cams, nview, all_colors, with_rank, cull, K_out, 0, colors);
    if (split && flags[1] != 0)  // a long run of equal hi keys: 64-bit compact sort
        return bin_batch(ctx, sp, cams, nview, all_colors, with_rank, cull, K_out, 1, colors);
    const int64_t K = ctx->pinned[0];
    ctx->invalid_key0 = dk.compact ? dk.sentinel : ~0ull;
    ctx->pairs_total += K;
    if (K > 0x7fffff00LL) return fail(ctx, POTR_E_ARG, "more than 2^31 tile pairs in one batch");

    const size_t kbytes = key16 ? sizeof(uint16_t) : sizeof(uint32_t);
    ENSURE(ctx->tkey, kbytes * K);
    ENSURE(ctx->tskey, kbytes * K);
    ENSURE(ctx->perm, sizeof(int2) * K);
    ENSURE(ctx->pair, sizeof(int2) * K);
    ENSURE(ctx->dup_id, sizeof(int32_t) * K);
    ENSURE(ctx->partial, sizeof(double2) * K);
    if (with_rank) ENSURE(ctx->dup_rank, sizeof(int32_t) * K);
    size_t t3 = 0;
    CK(tile_sort_temp(K, sb * g.ntiles, key16, &t3));
    ENSURE(ctx->temp, t3);
    // pair index where each sort group begins (pairs are view-major)
    std::vector<int64_t> vstart(nview + 1, 0);
    vstart[nview] = K;
    for (int v = sb; v < nview; v += sb) vstart[v] = ctx->pinned[2 + v];

    {
        Stage _st(ctx, POTR_STAGE_DUPLICATE);
        LAUNCH(1, launch_duplicate(total, n, P<int32_t>(ctx->sids), P<int64_t>(ctx->offs),
                                   P<SplatRec>(ctx->rec), P<TileSpan>(ctx->spans), g.tiles_x,
                                   g.ntiles, sb, key16,
                                   cull ? 1 : 0, ctx->tkey.p, P<int32_t>(ctx->dup_id),
                                   with_rank ? P<int32_t>(ctx->dup_rank) : nullptr, ctx->stream));
        _st.end();
    }
    {
        Stage _st(ctx, POTR_STAGE_TILE_SORT);
        CK(cudaMemsetAsync(ctx->ranges.p, 0, sizeof(int2) * (size_t)ntiles_b, ctx->stream));
        for (int v0 = 0; v0 < nview; v0 += sb) {
            const int v1 = v0 + sb < nview ? v0 + sb : nview;
            const int64_t j0 = vstart[v0], kk = vstart[v1] - vstart[v0];
            const size_t koff = kbytes * (size_t)j0;
            bool alt = false;
            CK(tile_sort(ctx->temp.p, ctx->temp.cap, key16, (char *)ctx->tkey.p + koff,
                         (char *)ctx->tskey.p + koff, P<int32_t>(ctx->dup_id) + j0, j0,
                         P<int2>(ctx->pair) + j0, P<int2>(ctx->perm) + j0, kk, sb * g.ntiles,
                         &alt, ctx->stream));
            ctx->launches += sort_launches(0, bits_for_tiles(sb * g.ntiles));
            if (alt)  // odd pass count (few tiles, or 24-bit keys): result in the alternate
                CK(cudaMemcpyAsync(P<int2>(ctx->pair) + j0, P<int2>(ctx->perm) + j0,
                                   sizeof(int2) * (size_t)kk, cudaMemcpyDeviceToDevice,
                                   ctx->stream));
            LAUNCH(1, launch_tile_ranges(j0, kk, key16,
                                         (char *)(alt ? ctx->tskey.p : ctx->tkey.p) + koff,
                                         P<int2>(ctx->ranges), v0 * g.ntiles, ctx->stream));
        }
        _st.end();
    }
    *K_out = K;
    return 0;
}

RasterArgs raster_args(potr_ctx *ctx, const potr_camera &cam, int nview) {
    ViewGeom g = geom(cam);
    RasterArgs a;
    std::memset(&a, 0, sizeof(a));
    a.rec = P<SplatRec>(ctx->rec);
    a.pair = P<int2>(ctx->pair);
    a.dup_rank = P<int32_t>(ctx->dup_rank);
    a.ranges = P<int2>(ctx->ranges);
    a.tiles_x = g.tiles_x;
    a.ntiles_view = g.ntiles;
    a.ntiles = g.ntiles * nview;
    a.tile_counter = P<int>(ctx->tile_counter);
    a.width = g.W;
    a.height = g.H;
    a.partial = P<double2>(ctx->partial);
    a.tile_se = P<double>(ctx->tile_se);
    a.counters = counters(ctx);
    return a;
}

// Views per batch: consecutive views of the same size, at most the configured
// batch (POTR_B200_VIEW_BATCH, default kMaxViewBatch), and bounded so the
// batch workspace stays within about 12 GB.
int batch_len(potr_ctx *ctx, const potr_camera *cams, int s, int ncam, int64_t n) {
    int cap = ctx->view_batch;
    const int64_t per_view = n * (int64_t)(sizeof(SplatRec) + 48) + 64 * 1024 * 1024;
    while (cap > 1 && per_view * cap > (int64_t)12 << 30) cap--;
    int b = 1;
    while (b < cap && s + b < ncam && cams[s + b].width == cams[s].width &&
           cams[s + b].height == cams[s].height)
        b++;
    return b;
}

// A binned batch waiting for its raster (score_views_run).
struct BatchMeta {
    int set, s, nb;
    bool spatial, split, colors_pending;
    uint64_t invalid_key0;
};

// images (nullable): with targets == images the targets are this very render
// (self-target mode: the first pruning iteration of an encode, whose targets
// are the renders of the unmodified model) -- rendered and scored in one pass.
//
// When the splats' SH rows are the destination of the pending
// potr_upload_async, the loop bins up to ctx->lookahead batches ahead (their
// geometry needs no SH) while the rows arrive, each batch in its own buffer
// set, then gives them their colours and rasters them in camera order; the
// view-order accumulation, and so every result bit, is unchanged.
int score_views_run(potr_ctx *ctx, const potr_splats *sp, int ncam, const potr_camera *cams,
                    const double *const *targets, double *imp_sum, double *cam_imp,
                    double *dmse_sum, double *mse_sum, double *dmse_rows, double *mse_rows,
                    double *const *images) {
    const int64_t n = sp->n;
    // the splats' SH rows are the last pending upload: bin while they arrive
    const bool defer = n > 0 && ncam > 0 && !ctx->upload_jobs.empty() &&
                       ctx->upload_jobs.back().dst == sp->sh &&
                       ctx->upload_jobs.back().bytes >= (int64_t)sizeof(double) * 48 * n;
    if (!defer) JOIN_UPLOAD(ctx);
    int rc = compute_scene_bounds(ctx, *sp, defer, defer ? upload_seq_of(ctx, sp->positions) : 0,
                                  defer ? ctx->upload_jobs.back().seq - 1 : 0);
    if (rc) return rc;
    bool sh_ready = !defer;
    int nsets = defer ? ctx->lookahead : 1;
    if (nsets < 1) nsets = 1;
    if (nsets > potr_ctx::kMaxSets) nsets = potr_ctx::kMaxSets;
    std::vector<int> free_sets;
    for (int j = nsets - 1; j >= 0; j--) free_sets.push_back(j);
    std::deque<BatchMeta> queue;
    int s = 0;
    while (s < ncam || !queue.empty()) {
        if (s < ncam && !free_sets.empty() && (queue.empty() || !sh_ready)) {
            if ((rc = check_cam(ctx, &cams[s]))) return rc;
            const int nb = batch_len(ctx, cams, s, ncam, n);
            for (int v = 0; v < nb; v++)
                if (targets && !targets[s + v])
                    return fail(ctx, POTR_E_ARG, "target pointer is NULL");
            const int set = free_sets.back();
            free_sets.pop_back();
            activate_set(ctx, set);
            if (nsets > 1 && (rc = level_active_set(ctx))) return rc;
            int64_t K = 0;
            rc = bin_batch(ctx, *sp, cams + s, nb, false, false, ctx->tile_cull, &K, 2, sh_ready);
            if (rc) return rc;
            queue.push_back({set, s, nb, ctx->batch_spatial, ctx->depth_split, !sh_ready,
                             ctx->invalid_key0});
            s += nb;
            if (!sh_ready && queue.size() == 1 && !free_sets.empty()) {
                // bound the sets by the memory the first one took: at most
                // half of what is free now
                size_t free_b = 0, total_b = 0;
                CK(cudaMemGetInfo(&free_b, &total_b));
                const size_t per = active_set_bytes(ctx);
                const size_t more = per ? (free_b / 2) / per : free_sets.size();
                while (free_sets.size() > more) free_sets.erase(free_sets.begin());
            }
            continue;
        }
        if (!sh_ready) {
            JOIN_UPLOAD(ctx);
            if ((rc = fill_slot_sh(ctx, *sp))) return rc;
            sh_ready = true;
        }
        const BatchMeta m = queue.front();
        queue.pop_front();
        activate_set(ctx, m.set);
        ctx->batch_spatial = m.spatial;
        ctx->depth_split = m.split;
        ctx->invalid_key0 = m.invalid_key0;
        const int nb = m.nb;
        if (m.colors_pending) {
            Stage _st(ctx, POTR_STAGE_PREPROCESS);
            CamBatch cb;
            std::memset(&cb, 0, sizeof(cb));
            for (int v = 0; v < nb; v++) cb.cam[v] = to_cam(cams[m.s + v]);
            const double *pos = m.spatial ? P<double>(ctx->slot_pos) : sp->positions;
            const double *sh = m.spatial ? P<double>(ctx->slot_sh) : sp->sh;
            const double *op = m.spatial ? P<double>(ctx->slot_opac) : sp->opacities;
            LAUNCH(1, launch_batch_colors(n, nb, pos, sh, op, cb, P<SplatRec>(ctx->rec),
                                          ctx->stream));
            _st.end();
        }
        ViewGeom g = geom(cams[m.s]);
        RasterArgs a = raster_args(ctx, cams[m.s], nb);
        for (int v = 0; v < nb; v++) a.target[v] = targets ? targets[m.s + v] : nullptr;
        if (images) {
            a.self_target = 1;
            for (int v = 0; v < nb; v++) a.image[v] = images[m.s + v];
        }
        ENSURE(ctx->ci_v, sizeof(double2) * n * nb);
        {
            Stage _st(ctx, POTR_STAGE_RASTER);
            LAUNCH(1, launch_raster(targets ? kScore : kImportance, a, a.ntiles, ctx->stream));
            _st.end();
        }
        {
            Stage _st(ctx, POTR_STAGE_REDUCE);
            LAUNCH(1, launch_splat_reduce(n * nb, n, P<int32_t>(ctx->sids), P<int64_t>(ctx->offs),
                                          P<double2>(ctx->partial), g.P, spatial_perm(ctx),
                                          P<double2>(ctx->ci_v), ctx->stream));
            LAUNCH(1, launch_view_accumulate(n, nb, P<double2>(ctx->ci_v),
                                             cam_imp ? cam_imp + (int64_t)m.s * n : nullptr,
                                             imp_sum, targets ? dmse_sum : nullptr,
                                             dmse_rows ? dmse_rows + (int64_t)m.s * n : nullptr,
                                             ctx->stream));
            if (targets)
                LAUNCH(2, launch_mse_reduce(nb, g.ntiles, P<double>(ctx->tile_se), g.P, mse_sum,
                                            mse_rows ? mse_rows + m.s : nullptr, ctx->stream));
            _st.end();
        }
        free_sets.push_back(m.set);
    }
    return 0;
}

// score_views_run, which never returns with the upload it deferred to still
// pending (an early error joins it here).
int score_views_impl(potr_ctx *ctx, const potr_splats *sp, int ncam, const potr_camera *cams,
                     const double *const *targets, double *imp_sum, double *cam_imp,
                     double *dmse_sum, double *mse_sum, double *dmse_rows = nullptr,
                     double *mse_rows = nullptr, double *const *images = nullptr) {
    int rc = score_views_run(ctx, sp, ncam, cams, targets, imp_sum, cam_imp, dmse_sum, mse_sum,
                             dmse_rows, mse_rows, images);
    if (ctx->upload_pending) {
        const std::string err = ctx->err;
        const int jrc = upload_join(ctx);
        if (rc) ctx->err = err;
        else rc = jrc;
    }
    return rc;
}

}  // namespace

extern "C" {

int potr_abi_version(void) { return POTR_B200_ABI_VERSION; }

int potr_create(int device, potr_ctx **out) {
    if (!out) return POTR_E_ARG;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
        cudaGetLastError();
        return POTR_E_CUDA;
    }
    if (cudaSetDevice(device) != cudaSuccess) return POTR_E_CUDA;
    potr_ctx *ctx = new potr_ctx();
    ctx->device = device;
    if (const char *vb = std::getenv("POTR_B200_VIEW_BATCH")) {
        int b = std::atoi(vb);
        ctx->view_batch = b < 1 ? 1 : (b > kMaxViewBatch ? kMaxViewBatch : b);
    }
    if (const char *sr = std::getenv("POTR_B200_SPATIAL")) ctx->spatial = std::atoi(sr) != 0;
    if (const char *la = std::getenv("POTR_B200_LOOKAHEAD")) {
        const int v = std::atoi(la);
        ctx->lookahead = v < 1 ? 1 : (v > potr_ctx::kMaxSets ? potr_ctx::kMaxSets : v);
    }
    if (cudaMallocHost(&ctx->pinned, 64 * sizeof(int64_t)) != cudaSuccess) {
        delete ctx;
        return POTR_E_NOMEM;
    }
    *out = ctx;
    return POTR_OK;
}

void potr_destroy(potr_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    upload_join(ctx);
    if (ctx->upload_worker.joinable()) {
        {
            std::lock_guard<std::mutex> lk(ctx->upload_mu);
            ctx->upload_quit = true;
        }
        ctx->upload_cv.notify_all();
        ctx->upload_worker.join();
    }
    cudaStreamSynchronize(ctx->stream);
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
        cudaEventDestroy(ctx->upload_after);
    }
    for (cudaEvent_t e : ctx->upload_ev_pool) cudaEventDestroy(e);
    if (ctx->poll_ev) cudaEventDestroy(ctx->poll_ev);
    activate_set(ctx, 0);
    for (auto &b : ctx->sets)
        for (DevBuf *d : {&b.rec, &b.sids, &b.offs, &b.pair, &b.ranges})
            if (d->p) cudaFree(d->p);
    DevBuf *bufs[] = {&ctx->rec,     &ctx->key,     &ctx->skey,    &ctx->sids,   &ctx->cnt,
                      &ctx->offs, &ctx->perm2,   &ctx->tkey,   &ctx->tskey,
                      &ctx->pair,    &ctx->dup_id,  &ctx->dup_rank, &ctx->partial, &ctx->ranges,
                      &ctx->perm,
                      &ctx->tile_se, &ctx->temp,    &ctx->nvalid,  &ctx->rkey,   &ctx->rskey,
                      &ctx->rsidx,   &ctx->ralpha,  &ctx->rt,      &ctx->rp,     &ctx->rcounter,
                      &ctx->eyes,    &ctx->neq,     &ctx->h_pos,   &ctx->h_sh,   &ctx->h_op,
                      &ctx->h_sc,    &ctx->h_rot,   &ctx->h_tg,    &ctx->h_imp,  &ctx->h_ci,
                      &ctx->h_dm,    &ctx->h_mse,   &ctx->h_rgb,   &ctx->h_yc,   &ctx->h_st};
    for (DevBuf *b : bufs)
        if (b->p) cudaFree(b->p);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    for (int r = 0; r < potr_ctx::kRing; r++) {
        if (ctx->ring[r]) cudaFreeHost(ctx->ring[r]);
        if (ctx->ring_ev[r]) cudaEventDestroy(ctx->ring_ev[r]);
    }
    if (ctx->counters.p) cudaFree(ctx->counters.p);
    if (ctx->tile_counter.p) cudaFree(ctx->tile_counter.p);
    if (ctx->vidx.p) cudaFree(ctx->vidx.p);
    if (ctx->bbox.p) cudaFree(ctx->bbox.p);
    if (ctx->overflow.p) cudaFree(ctx->overflow.p);
    if (ctx->ci_v.p) cudaFree(ctx->ci_v.p);
    if (ctx->dm_v.p) cudaFree(ctx->dm_v.p);
    if (ctx->khi.p) cudaFree(ctx->khi.p);
    if (ctx->spans.p) cudaFree(ctx->spans.p);
    for (DevBuf *b : {&ctx->mperm, &ctx->mrank, &ctx->mcode, &ctx->mcode2, &ctx->slot_pos,
                      &ctx->slot_sh, &ctx->slot_opac, &ctx->slot_prep})
        if (b->p) cudaFree(b->p);
    for (DevBuf *b : {&ctx->met_mom, &ctx->met_part, &ctx->met_w, &ctx->met_out, &ctx->codec_eyes,
                      &ctx->sort_k, &ctx->sort_v, &ctx->rm_keys, &ctx->sh_scratch})
        if (b->p) cudaFree(b->p);
    if (ctx->codec_scratch) cudaFree(ctx->codec_scratch);
    if (ctx->prep.p) cudaFree(ctx->prep.p);
    if (ctx->skhi.p) cudaFree(ctx->skhi.p);
    for (auto &ev : ctx->events) {
        cudaEventDestroy(ev.second.first);
        cudaEventDestroy(ev.second.second);
    }
    for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
    delete ctx;
}

int potr_set_stream(potr_ctx *ctx, void *stream) {
    if (!ctx) return POTR_E_ARG;
    if (reinterpret_cast<cudaStream_t>(stream) == ctx->stream) return POTR_OK;
    JOIN_UPLOAD(ctx);
    ctx->stream = reinterpret_cast<cudaStream_t>(stream);
    return POTR_OK;
}

int potr_synchronize(potr_ctx *ctx) {
    if (!ctx) return POTR_E_ARG;
    JOIN_UPLOAD(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    return POTR_OK;
}

const char *potr_last_error(potr_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t potr_kernel_launches(potr_ctx *ctx) { return ctx ? ctx->launches : 0; }

int potr_score_views(potr_ctx *ctx, const potr_splats *splats, int ncam, const potr_camera *cams,
                     const double *const *targets, double *imp_sum, double *camera_importance,
                     double *dmse_sum, double *mse_sum) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    int rc = check_splats(ctx, splats);
    if (rc) return rc;
    if (ncam < 0 || (ncam > 0 && !cams)) return fail(ctx, POTR_E_ARG, "bad camera list");
    if (!imp_sum) return fail(ctx, POTR_E_ARG, "imp_sum is NULL");
    if (targets && (!dmse_sum || !mse_sum))
        return fail(ctx, POTR_E_ARG, "targets given without delta_mse/mse outputs");
    return score_views_impl(ctx, splats, ncam, cams, targets, imp_sum, camera_importance,
                            dmse_sum, mse_sum);
}

int potr_score_views_rows(potr_ctx *ctx, const potr_splats *splats, int ncam,
                          const potr_camera *cams, const double *const *targets,
                          double *camera_importance, double *dmse_rows, double *mse_rows) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    int rc = check_splats(ctx, splats);
    if (rc) return rc;
    if (ncam < 0 || (ncam > 0 && !cams)) return fail(ctx, POTR_E_ARG, "bad camera list");
    if (!camera_importance) return fail(ctx, POTR_E_ARG, "camera_importance is NULL");
    if (targets && (!dmse_rows || !mse_rows))
        return fail(ctx, POTR_E_ARG, "targets given without delta_mse/mse row outputs");
    const int64_t n = splats->n;
    // the sums are produced on the way and discarded
    ENSURE(ctx->dm_v, sizeof(double) * (2 * (n > 0 ? n : 1) + 1));
    double *scratch = P<double>(ctx->dm_v);
    CK(cudaMemsetAsync(scratch, 0, sizeof(double) * (2 * (n > 0 ? n : 1) + 1), ctx->stream));
    return score_views_impl(ctx, splats, ncam, cams, targets, scratch, camera_importance,
                            targets ? scratch + n : nullptr, targets ? scratch + 2 * n : nullptr,
                            dmse_rows, mse_rows);
}

int potr_score_views_self(potr_ctx *ctx, const potr_splats *splats, int ncam,
                          const potr_camera *cams, double *const *images, double *imp_sum,
                          double *camera_importance, double *dmse_sum, double *mse_sum) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    int rc = check_splats(ctx, splats);
    if (rc) return rc;
    if (ncam < 0 || (ncam > 0 && !cams)) return fail(ctx, POTR_E_ARG, "bad camera list");
    if (!imp_sum || !dmse_sum || !mse_sum) return fail(ctx, POTR_E_ARG, "NULL sum output");
    if (ncam > 0 && !images) return fail(ctx, POTR_E_ARG, "images is NULL");
    for (int v = 0; v < ncam; v++)
        if (!images[v]) return fail(ctx, POTR_E_ARG, "image pointer is NULL");
    return score_views_impl(ctx, splats, ncam, cams, images, imp_sum, camera_importance,
                            dmse_sum, mse_sum, nullptr, nullptr, images);
}

int potr_finalize_stats(potr_ctx *ctx, int64_t n, int total_cams, double *imp_sum,
                        double *dmse_sum, double *mse_sum) {
    if (!ctx || n < 0) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    LAUNCH(1, launch_finalize(n, total_cams, imp_sum, dmse_sum, mse_sum, ctx->stream));
    return POTR_OK;
}

int potr_forward_stats(potr_ctx *ctx, const potr_splats *splats, int ncam,
                       const potr_camera *cams, const double *const *targets, double *importance,
                       double *camera_importance, double *delta_mse, double *mse) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    int rc = check_splats(ctx, splats);
    if (rc) return rc;
    if (!importance) return fail(ctx, POTR_E_ARG, "importance is NULL");
    if (targets && (!delta_mse || !mse))
        return fail(ctx, POTR_E_ARG, "targets given without delta_mse/mse outputs");
    const int64_t n = splats->n;
    CK(cudaMemsetAsync(importance, 0, sizeof(double) * (n > 0 ? n : 0), ctx->stream));
    if (targets) {
        CK(cudaMemsetAsync(delta_mse, 0, sizeof(double) * (n > 0 ? n : 0), ctx->stream));
        CK(cudaMemsetAsync(mse, 0, sizeof(double), ctx->stream));
    }
    rc = potr_score_views(ctx, splats, ncam, cams, targets, importance, camera_importance,
                          delta_mse, mse);
    if (rc) return rc;
    return potr_finalize_stats(ctx, n, ncam, importance, targets ? delta_mse : nullptr,
                               targets ? mse : nullptr);
}

int potr_render_batch(potr_ctx *ctx, const potr_splats *splats, int ncam, const potr_camera *cams,
                      double *const *images, double *const *trans) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    int rc = check_splats(ctx, splats);
    if (rc) return rc;
    if (ncam < 0 || (ncam > 0 && (!cams || !images)))
        return fail(ctx, POTR_E_ARG, "bad camera / image list");
    if (ncam == 0) return POTR_OK;
    if ((rc = compute_scene_bounds(ctx, *splats))) return rc;
    for (int s = 0; s < ncam;) {
        if ((rc = check_cam(ctx, &cams[s]))) return rc;
        const int nb = batch_len(ctx, cams, s, ncam, splats->n);
        for (int v = 0; v < nb; v++)
            if (!images[s + v]) return fail(ctx, POTR_E_ARG, "image pointer is NULL");
        int64_t K = 0;
        rc = bin_batch(ctx, *splats, cams + s, nb, false, false, ctx->tile_cull, &K);
        if (rc) return rc;
        RasterArgs a = raster_args(ctx, cams[s], nb);
        for (int v = 0; v < nb; v++) {
            a.image[v] = images[s + v];
            a.trans[v] = trans ? trans[s + v] : nullptr;
        }
        {
            Stage _st(ctx, POTR_STAGE_RASTER);
            LAUNCH(1, launch_raster(kRender, a, a.ntiles, ctx->stream));
            _st.end();
        }
        s += nb;
    }
    return POTR_OK;
}

int potr_render(potr_ctx *ctx, const potr_splats *splats, const potr_camera *cam, double *image,
                double *trans) {
    if (!ctx) return POTR_E_ARG;
    if (!image) return fail(ctx, POTR_E_ARG, "image is NULL");
    return potr_render_batch(ctx, splats, 1, cam, &image, trans ? &trans : nullptr);
}

int potr_render_records(potr_ctx *ctx, const potr_splats *splats, const potr_camera *cam,
                        double *image, double *trans, double *colors, int64_t capacity,
                        int64_t *n_records, int64_t *splat_ids, int64_t *pixels, double *alphas,
                        double *trans_at, double *partials) {
    if (!ctx || !n_records) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    int rc = check_splats(ctx, splats);
    if (rc) return rc;
    if ((rc = check_cam(ctx, cam))) return rc;
    if (!image) return fail(ctx, POTR_E_ARG, "image is NULL");
    if (capacity > 0 && (!splat_ids || !pixels || !alphas || !trans_at || !partials))
        return fail(ctx, POTR_E_ARG, "record output pointer is NULL");
    const int64_t n = splats->n;
    int64_t K = 0;
    if ((rc = compute_scene_bounds(ctx, *splats))) return rc;
    rc = bin_batch(ctx, *splats, cam, 1, true, true, ctx->tile_cull, &K);
    if (rc) return rc;
    int64_t cap = capacity > 0 ? capacity : 0;
    ENSURE(ctx->rcounter, sizeof(unsigned long long));
    ENSURE(ctx->rkey, sizeof(uint64_t) * cap);
    ENSURE(ctx->ralpha, sizeof(double) * cap);
    ENSURE(ctx->rt, sizeof(double) * cap);
    ENSURE(ctx->rp, sizeof(double) * 3 * cap);
    CK(cudaMemsetAsync(ctx->rcounter.p, 0, sizeof(unsigned long long), ctx->stream));
    RasterArgs a = raster_args(ctx, *cam, 1);
    a.image[0] = image;
    a.trans[0] = trans;
    a.rec_counter = P<unsigned long long>(ctx->rcounter);
    a.rec_capacity = cap;
    a.rec_key = P<uint64_t>(ctx->rkey);
    a.rec_alpha = P<double>(ctx->ralpha);
    a.rec_t = P<double>(ctx->rt);
    a.rec_p = P<double>(ctx->rp);
    LAUNCH(1, launch_raster(kRecords, a, a.ntiles, ctx->stream));
    if (colors)
        LAUNCH(1, launch_colors_from_rec(n, P<SplatRec>(ctx->rec), spatial_rank(ctx), colors,
                                         ctx->stream));
    CK(cudaMemcpyAsync(ctx->pinned, ctx->rcounter.p, sizeof(int64_t), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const int64_t m = ctx->pinned[0];
    *n_records = m;
    if (capacity <= 0) return POTR_OK;
    if (m > capacity) return fail(ctx, POTR_E_CAPACITY, "record capacity too small");
    ENSURE(ctx->rskey, sizeof(uint64_t) * m);
    ENSURE(ctx->rsidx, sizeof(int32_t) * m);
    ENSURE(ctx->perm2, sizeof(int32_t) * m);
    size_t tb = 0;
    CK(records_sort_temp(m, &tb));
    ENSURE(ctx->temp, tb);
    bool ralt = false;
    CK(records_sort(ctx->temp.p, ctx->temp.cap, P<uint64_t>(ctx->rkey), P<uint64_t>(ctx->rskey),
                    P<int32_t>(ctx->rsidx), P<int32_t>(ctx->perm2), m, &ralt, ctx->stream));
    ctx->launches += 9;
    LAUNCH(1, launch_records_gather(m, P<uint64_t>(ralt ? ctx->rskey : ctx->rkey),
                                    P<int32_t>(ralt ? ctx->perm2 : ctx->rsidx),
                                    P<int32_t>(ctx->sids), P<double>(ctx->ralpha),
                                    P<double>(ctx->rt), P<double>(ctx->rp), splat_ids, pixels,
                                    alphas, trans_at, partials, spatial_perm(ctx), ctx->stream));
    return POTR_OK;
}

int potr_project(potr_ctx *ctx, const potr_splats *splats, const potr_camera *cam, double *mean2d,
                 double *cov2d, double *depth, double *radius, uint8_t *valid, double *colors) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    int rc = check_splats(ctx, splats);
    if (rc) return rc;
    if ((rc = check_cam(ctx, cam))) return rc;
    if (!mean2d || !cov2d || !depth || !radius || !valid)
        return fail(ctx, POTR_E_ARG, "projection output is NULL");
    LAUNCH(1, launch_project_dump(*splats, to_cam(*cam), mean2d, cov2d, depth, radius, valid,
                                  colors, ctx->stream));
    return POTR_OK;
}

int potr_bin(potr_ctx *ctx, const potr_splats *splats, const potr_camera *cam, int64_t *order,
             int64_t *n_valid, int64_t *tile_offsets, int32_t *tile_splats, int64_t capacity,
             int64_t *n_pairs) {
    if (!ctx || !n_valid || !n_pairs || !order) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    int rc = check_splats(ctx, splats);
    if (rc) return rc;
    if ((rc = check_cam(ctx, cam))) return rc;
    int64_t K = 0;
    if ((rc = compute_scene_bounds(ctx, *splats))) return rc;
    rc = bin_batch(ctx, *splats, cam, 1, false, false, false, &K);
    if (rc) return rc;
    *n_pairs = K;
    if (tile_splats && capacity < K) return fail(ctx, POTR_E_CAPACITY, "tile list capacity");
    ENSURE(ctx->nvalid, sizeof(unsigned long long));
    if (ctx->depth_split)  // sorted full keys for the validity count
        LAUNCH(1, launch_gather_keys(splats->n, P<int32_t>(ctx->sids), P<uint64_t>(ctx->key),
                                     P<uint64_t>(ctx->skey), ctx->stream));
    LAUNCH(3, launch_bin_outputs(splats->n, P<uint64_t>(ctx->skey), ctx->invalid_key0,
                                 P<int32_t>(ctx->sids),
                                 P<unsigned long long>(ctx->nvalid), order, geom(*cam).ntiles,
                                 P<int2>(ctx->ranges), K, tile_offsets, P<int2>(ctx->pair),
                                 tile_splats, spatial_perm(ctx), ctx->stream));
    CK(cudaMemcpyAsync(ctx->pinned, ctx->nvalid.p, sizeof(int64_t), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *n_valid = ctx->pinned[0];
    return POTR_OK;
}

}  // extern "C"

namespace {

int sh_normal_equations(potr_ctx *ctx, const potr_splats *splats, int ncam,
                        const potr_camera *cams, const double *camera_importance,
                        double *normal_eqs, bool add) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    int rc = check_splats_ps(ctx, splats);
    if (rc) return rc;
    if (ncam < 0 || (ncam > 0 && (!cams || !camera_importance)) || !normal_eqs)
        return fail(ctx, POTR_E_ARG, "bad arguments to sh_accumulate");
    if (splats->n == 0) return POTR_OK;
    if (ncam == 0) {
        if (!add)
            CK(cudaMemsetAsync(normal_eqs, 0, sizeof(double) * POTR_NEQ_STRIDE * splats->n,
                               ctx->stream));
        return POTR_OK;
    }
    std::vector<double> eyes(3 * (size_t)ncam);
    for (int s = 0; s < ncam; s++)
        for (int i = 0; i < 3; i++) eyes[3 * s + i] = cams[s].eye[i];
    ENSURE(ctx->eyes, sizeof(double) * eyes.size());
    CK(cudaMemcpyAsync(ctx->eyes.p, eyes.data(), sizeof(double) * eyes.size(),
                       cudaMemcpyHostToDevice, ctx->stream));
    // the pageable source must stay alive until the copy is done
    CK(cudaStreamSynchronize(ctx->stream));
    {
        Stage _st(ctx, POTR_STAGE_SH_ACCUMULATE);
        LAUNCH(1, launch_sh_accumulate(*splats, ncam, P<double>(ctx->eyes), camera_importance,
                                       normal_eqs, add, ctx->stream));
        _st.end();
    }
    return POTR_OK;
}

}  // namespace

extern "C" {

int potr_sh_accumulate(potr_ctx *ctx, const potr_splats *splats, int ncam,
                       const potr_camera *cams, const double *camera_importance,
                       double *normal_eqs) {
    return sh_normal_equations(ctx, splats, ncam, cams, camera_importance, normal_eqs, true);
}

int potr_sh_normal_equations(potr_ctx *ctx, const potr_splats *splats, int ncam,
                             const potr_camera *cams, const double *camera_importance,
                             double *normal_eqs) {
    return sh_normal_equations(ctx, splats, ncam, cams, camera_importance, normal_eqs, false);
}

int potr_sh_solve(potr_ctx *ctx, const potr_splats *splats, const double *normal_eqs,
                  double lambda_y, double parallel_threshold, double zero_threshold, double *rgb,
                  double *ycocg, int8_t *status) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    int rc = check_splats_ps(ctx, splats);
    if (rc) return rc;
    if (!normal_eqs || !rgb || !ycocg || !status)
        return fail(ctx, POTR_E_ARG, "bad arguments to sh_solve");
    if (!(lambda_y >= 0)) return fail(ctx, POTR_E_ARG, "lambda_y must be >= 0");
    if (!(parallel_threshold > 0 && parallel_threshold <= 1))
        return fail(ctx, POTR_E_ARG, "parallel_threshold must be in (0, 1]");
    {
        Stage _st(ctx, POTR_STAGE_SH_SOLVE);
        ENSURE(ctx->sh_scratch, sh_solve_scratch_bytes(splats->n));
        LAUNCH(6, launch_sh_solve(*splats, normal_eqs, lambda_y, parallel_threshold, zero_threshold,
                                  rgb, ycocg, status, ctx->sh_scratch.p, ctx->stream));
        _st.end();
    }
    return POTR_OK;
}

int potr_compact(potr_ctx *ctx, const potr_splats *splats, int ncam, const potr_camera *cams,
                 const double *camera_importance, double lambda_y, double parallel_threshold,
                 double zero_threshold, double *rgb, double *ycocg, int8_t *status) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    int rc = check_splats_ps(ctx, splats);
    if (rc) return rc;
    const int64_t n = splats->n;
    ENSURE(ctx->neq, sizeof(double) * POTR_NEQ_STRIDE * n);
    rc = potr_sh_normal_equations(ctx, splats, ncam, cams, camera_importance,
                                  P<double>(ctx->neq));
    if (rc) return rc;
    return potr_sh_solve(ctx, splats, P<double>(ctx->neq), lambda_y, parallel_threshold,
                         zero_threshold, rgb, ycocg, status);
}

int potr_sort_pairs_u64(potr_ctx *ctx, int64_t n, uint64_t *keys, int64_t *vals, int begin_bit,
                        int end_bit) {
    if (!ctx) return POTR_E_ARG;
    if (n < 0 || (n > 0 && (!keys || !vals)) || begin_bit < 0 || end_bit > 64)
        return fail(ctx, POTR_E_ARG, "sort_pairs: bad arguments");
    if (n == 0 || end_bit <= begin_bit) return POTR_OK;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    ENSURE(ctx->sort_k, sizeof(uint64_t) * n);
    ENSURE(ctx->sort_v, sizeof(int64_t) * n);
    ENSURE(ctx->temp, radix_sort_temp_bytes(n, begin_bit, end_bit));
    bool alt = false;
    CK((radix_sort_pairs<uint64_t, int64_t>(ctx->temp.p, ctx->temp.cap, keys, P<uint64_t>(ctx->sort_k),
                                            vals, P<int64_t>(ctx->sort_v), n, begin_bit, end_bit,
                                            false, &alt, ctx->stream)));
    ctx->launches += sort_launches(begin_bit, end_bit);
    if (alt) {
        CK(cudaMemcpyAsync(keys, ctx->sort_k.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice,
                           ctx->stream));
        CK(cudaMemcpyAsync(vals, ctx->sort_v.p, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice,
                           ctx->stream));
    }
    return POTR_OK;
}

int potr_removal_order(potr_ctx *ctx, int64_t n, const double *delta_mse, const int64_t *idx,
                       double delta_mse_max, double a, int64_t *order) {
    if (!ctx) return POTR_E_ARG;
    if (n < 0 || (n > 0 && (!delta_mse || !order)))
        return fail(ctx, POTR_E_ARG, "removal_order: bad arguments");
    if (!(delta_mse_max > 0) || !(a > 0))
        return fail(ctx, POTR_E_ARG, "removal_order: delta_mse_max and a must be > 0");
    if (n == 0) return POTR_OK;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    ENSURE(ctx->rm_keys, sizeof(uint64_t) * n);
    LAUNCH(1, launch_removal_keys(n, delta_mse, idx, delta_mse_max, a, P<uint64_t>(ctx->rm_keys),
                                  ctx->stream));
    if (idx)
        CK(cudaMemcpyAsync(order, idx, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    else
        LAUNCH(1, launch_iota64(n, order, ctx->stream));
    return potr_sort_pairs_u64(ctx, n, P<uint64_t>(ctx->rm_keys), order, 0, 64);
}

// scipy.ndimage._gaussian_kernel1d(1.5, 0, 5): exp(-0.5 / sigma^2 * x^2) over
// x = -5..5, divided by its numpy sum (pairwise: eight running partials, then
// the tail added in order).
static void ssim_weights(double *w) {
    const double sigma2 = 1.5 * 1.5;
    for (int i = 0; i < 11; i++) {
        const double x = (double)(i - 5);
        w[i] = std::exp(-0.5 / sigma2 * (x * x));
    }
    double s = ((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7]));
    for (int i = 8; i < 11; i++) s += w[i];
    for (int i = 0; i < 11; i++) w[i] = w[i] / s;
}

int potr_image_compare(potr_ctx *ctx, int width, int height, const double *a, const double *b,
                       double *mse, double *ssim) {
    if (!ctx || width <= 0 || height <= 0 || !a || !b)
        return fail(ctx, POTR_E_ARG, "image_compare: bad image arguments");
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    const size_t plane = (size_t)width * height;
    ENSURE(ctx->met_mom, 5 * plane * sizeof(double));
    ENSURE(ctx->met_part, (size_t)image_compare_partials() * sizeof(double));
    ENSURE(ctx->met_w, 11 * sizeof(double));
    ENSURE(ctx->met_out, 4 * sizeof(double));
    double w[11];
    ssim_weights(w);
    CK(cudaMemcpyAsync(ctx->met_w.p, w, sizeof(w), cudaMemcpyHostToDevice, ctx->stream));
    LAUNCH(9, launch_image_compare(width, height, a, b, P<double>(ctx->met_w),
                                   P<double>(ctx->met_mom), P<double>(ctx->met_part),
                                   P<double>(ctx->met_out), ctx->stream));
    double out[4];
    CK(cudaMemcpyAsync(out, ctx->met_out.p, sizeof(out), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (mse) *mse = out[0] / (double)(plane * 3);
    if (ssim) {
        const int64_t cw = width - 10, ch = height - 10;
        const double cnt = cw > 0 && ch > 0 ? (double)(cw * ch) : 0.0;
        // np.mean of an empty crop is NaN, as in the reference
        const double s0 = out[1] / cnt, s1 = out[2] / cnt, s2 = out[3] / cnt;
        *ssim = ((s0 + s1) + s2) / 3.0;
    }
    return POTR_OK;
}

int potr_octree(potr_ctx *ctx, int64_t n, const double *positions, int neyes, const double *eyes,
                double beta, double gamma, const double *center, double half, int max_depth,
                uint8_t *stream, int64_t capacity, int64_t *stream_len, int64_t *order) {
    if (!ctx || !stream_len || !order || !center) return fail(ctx, POTR_E_ARG, "octree: NULL argument");
    if (n < 1 || n > 0x7ffffff0LL || !positions) return fail(ctx, POTR_E_ARG, "need at least one position");
    if (!(gamma > 0.0) || beta < 0.0) return fail(ctx, POTR_E_ARG, "gamma must be > 0 and beta >= 0");
    if (max_depth < 0 || max_depth > 24) return fail(ctx, POTR_E_ARG, "max_depth must be in [0, 24]");
    if (neyes < 0 || (neyes > 0 && !eyes)) return fail(ctx, POTR_E_ARG, "bad camera eyes");
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    ENSURE(ctx->codec_eyes, sizeof(double) * 3 * (neyes > 0 ? neyes : 1));
    if (neyes > 0)
        CK(cudaMemcpyAsync(ctx->codec_eyes.p, eyes, sizeof(double) * 3 * neyes,
                           cudaMemcpyHostToDevice, ctx->stream));
    LAUNCH(9 + 3 * max_depth,
           run_octree(n, positions, neyes, P<double>(ctx->codec_eyes), beta, gamma, center, half,
                      max_depth, stream, capacity, stream_len, order, &ctx->codec_scratch,
                      &ctx->codec_cap, ctx->pinned, ctx->stream));
    if (stream && capacity < *stream_len) return fail(ctx, POTR_E_CAPACITY, "octree stream capacity");
    return POTR_OK;
}

int potr_attribute_streams(potr_ctx *ctx, int64_t n, const int64_t *order, const double *ycocg,
                           const double *opacities, const double *log_scales,
                           const double *rotations, double sf_sh, double sf_opacity,
                           double sf_rotation, double sf_scale, uint8_t *out, int64_t capacity,
                           int64_t *stream_lengths) {
    if (!ctx || !stream_lengths) return fail(ctx, POTR_E_ARG, "attribute_streams: NULL argument");
    if (n < 1 || (int64_t)55 * n > 0x7ffffff0LL || !order || !ycocg || !opacities || !log_scales ||
        !rotations)
        return fail(ctx, POTR_E_ARG, "attribute_streams: bad arrays");
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    LAUNCH(4, run_attr_streams(n, order, ycocg, opacities, log_scales, rotations, sf_sh,
                               sf_opacity, sf_rotation, sf_scale, out, capacity, stream_lengths,
                               &ctx->codec_scratch, &ctx->codec_cap, ctx->pinned, ctx->stream));
    int64_t total = 0;
    for (int s = 0; s < 55; s++) total += stream_lengths[s];
    if (out && capacity < total) return fail(ctx, POTR_E_CAPACITY, "attribute stream capacity");
    return POTR_OK;
}

int potr_octree_decode(potr_ctx *ctx, const uint8_t *stream, int64_t len, const double *center,
                       double half, int max_depth, int64_t capacity, double *positions,
                       int32_t *depths, int64_t *count) {
    if (!ctx || !center || !count || (len > 0 && !stream) ||
        (capacity > 0 && (!positions || !depths)))
        return fail(ctx, POTR_E_ARG, "octree_decode: NULL argument");
    int64_t trailing = 0;
    const int rc = octree_decode_host(stream, len, center, half, max_depth, capacity, positions,
                                      depths, count, &trailing);
    switch (rc) {
        case 0: return POTR_OK;
        case kOctTruncated: return fail(ctx, POTR_E_ARG, "octree: truncated octree stream");
        case kOctZeroLeaf: return fail(ctx, POTR_E_ARG, "octree: leaf with zero splats");
        case kOctDepth:
            return fail(ctx, POTR_E_ARG, "octree: internal node below depth limit " +
                                             std::to_string(max_depth));
        default:
            return fail(ctx, POTR_E_ARG, "octree: " + std::to_string(trailing) +
                                             " trailing bytes after octree");
    }
}

int potr_attribute_decode(potr_ctx *ctx, int64_t n, const uint8_t *streams,
                          const int64_t *stream_lengths, double sf_sh, double sf_opacity,
                          double sf_rotation, double sf_scale, double *sh, double *opacities,
                          double *scales, double *rotations, int64_t *n_clamped) {
    if (!ctx || !stream_lengths || !n_clamped) return fail(ctx, POTR_E_ARG, "attribute_decode: NULL argument");
    if (n < 1 || (int64_t)55 * n > 0x7ffffff0LL || !streams || !sh || !opacities || !scales ||
        !rotations)
        return fail(ctx, POTR_E_ARG, "attribute_decode: bad arrays");
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    int64_t start[56];
    start[0] = 0;
    for (int s = 0; s < 55; s++) {
        if (stream_lengths[s] < 0) return fail(ctx, POTR_E_ARG, "attribute_decode: bad lengths");
        start[s + 1] = start[s] + stream_lengths[s];
    }
    std::string err;
    const int rc = run_attr_decode(n, streams, start, sf_sh, sf_opacity, sf_scale, sf_rotation,
                                   sh, opacities, scales, rotations, n_clamped,
                                   &ctx->codec_scratch, &ctx->codec_cap, ctx->pinned,
                                   ctx->stream, &err);
    ctx->launches += 5 + 3;
    if (rc == 0) return POTR_OK;
    if (rc == kDecCuda) return fail(ctx, POTR_E_CUDA, err);
    if (rc == kDecTrailing) {
        // bitstream.py:163-166: "<what> stream has <k> trailing bytes"
        const int s = std::atoi(err.c_str());  // 1..55
        const char *what = s <= 3 ? "DC" : s <= 48 ? "AC" : s == 49 ? "opacity"
                                                 : s <= 52 ? "scale" : "rotation";
        const uint8_t *b = streams + start[s - 1];
        const int64_t slen = start[s] - start[s - 1];
        int64_t used = 0, vals = 0;
        while (used < slen && vals < n) vals += b[used++] < 0x80;
        return fail(ctx, POTR_E_ARG, std::string("integrity: ") + what + " stream has " +
                                         std::to_string(slen - used) + " trailing bytes");
    }
    return fail(ctx, POTR_E_ARG, "varint: " + err);
}

int potr_set_option(potr_ctx *ctx, int option, int value) {
    if (!ctx) return POTR_E_ARG;
    switch (option) {
        case POTR_OPT_VIEW_BATCH:
            if (value < 1 || value > kMaxViewBatch)
                return fail(ctx, POTR_E_ARG, "view batch must be in [1, 8]");
            ctx->view_batch = value;
            return POTR_OK;
        case POTR_OPT_RAW_DEPTH_KEYS:
            if (value < 0 || value > 2) return fail(ctx, POTR_E_ARG, "depth key mode must be 0..2");
            ctx->depth_keys = value;
            return POTR_OK;
        case POTR_OPT_TILE_CULL:
            ctx->tile_cull = value != 0;
            return POTR_OK;
        case POTR_OPT_SPATIAL_RECORDS:
            ctx->spatial = value != 0;
            return POTR_OK;
        case POTR_OPT_LOOKAHEAD:
            if (value < 1 || value > potr_ctx::kMaxSets)
                return fail(ctx, POTR_E_ARG, "lookahead must be in [1, 8]");
            ctx->lookahead = value;
            return POTR_OK;
    }
    return fail(ctx, POTR_E_ARG, "unknown option");
}

int potr_profile_enable(potr_ctx *ctx, int enable) {
    if (!ctx) return POTR_E_ARG;
    ctx->profile = enable != 0;
    for (int i = 0; i < POTR_STAGE_COUNT; i++) {
        ctx->stage_ms[i] = 0.0;
        ctx->stage_launches[i] = 0;
    }
    return POTR_OK;
}

int potr_profile_read(potr_ctx *ctx, double *stage_ms, int64_t *stage_launches) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    for (auto &ev : ctx->events) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev.second.first, ev.second.second));
        ctx->stage_ms[ev.first] += ms;
        ctx->stage_launches[ev.first] += 1;
        ctx->event_pool.push_back(ev.second.first);
        ctx->event_pool.push_back(ev.second.second);
    }
    ctx->events.clear();
    for (int i = 0; i < POTR_STAGE_COUNT; i++) {
        if (stage_ms) stage_ms[i] = ctx->stage_ms[i];
        if (stage_launches) stage_launches[i] = ctx->stage_launches[i];
    }
    return POTR_OK;
}

int potr_counters_enable(potr_ctx *ctx, int enable) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    ENSURE(ctx->counters, 4 * sizeof(unsigned long long));
    CK(cudaMemsetAsync(ctx->counters.p, 0, 4 * sizeof(unsigned long long), ctx->stream));
    ctx->counting = enable != 0;
    ctx->pairs_total = 0;
    return POTR_OK;
}

int potr_counters_read(potr_ctx *ctx, uint64_t *out) {
    if (!ctx || !out) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    ENSURE(ctx->counters, 4 * sizeof(unsigned long long));
    CK(cudaMemcpyAsync(ctx->pinned, ctx->counters.p, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 3; i++) out[i] = (uint64_t)ctx->pinned[i];
    out[3] = (uint64_t)ctx->pairs_total;
    return POTR_OK;
}

// ---- host-buffer convenience entry points --------------------------------

int potr_copy_to_device(potr_ctx *ctx, void *dst, const void *src, int64_t bytes) {
    if (!ctx || bytes < 0 || (bytes > 0 && (!dst || !src)))
        return fail(ctx, POTR_E_ARG, "copy_to_device: bad arguments");
    if (bytes == 0) return POTR_OK;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    std::string err;
    const int rc = ring_copy(ctx, dst, src, bytes, ctx->stream, ring_threads(0), &err);
    return rc ? fail(ctx, rc, err) : POTR_OK;
}

int potr_upload_async(potr_ctx *ctx, void *dst, const void *src, int64_t bytes) {
    if (!ctx || bytes < 0 || (bytes > 0 && (!dst || !src)))
        return fail(ctx, POTR_E_ARG, "upload_async: bad arguments");
    CK(cudaSetDevice(ctx->device));
    if (bytes == 0) return POTR_OK;
    if (!ctx->copy_stream) {
        CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->upload_after, cudaEventDisableTiming));
    }
    cudaEvent_t ev = nullptr;
    if (!ctx->upload_ev_pool.empty()) {
        ev = ctx->upload_ev_pool.back();
        ctx->upload_ev_pool.pop_back();
    } else {
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    // earlier work on the context stream may still read the destination
    CK(cudaEventRecord(ctx->upload_after, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->upload_after, 0));
    if (!ctx->upload_worker.joinable()) {
        ctx->upload_worker = std::thread([ctx]() {
            cudaSetDevice(ctx->device);
            // one host core stays with the caller, which keeps launching kernels
            const int threads = ring_threads(1);
            std::unique_lock<std::mutex> lk(ctx->upload_mu);
            for (;;) {
                ctx->upload_cv.wait(lk,
                                    [ctx] { return ctx->upload_quit || !ctx->upload_todo.empty(); });
                if (ctx->upload_todo.empty()) return;  // quit
                const potr_ctx::UploadJob job = ctx->upload_todo.front();
                ctx->upload_todo.pop_front();
                const bool skip = ctx->upload_rc != 0;
                lk.unlock();
                int rc = POTR_OK;
                std::string err;
                if (!skip) {
                    cudaPointerAttributes at;
                    cudaError_t e = cudaSuccess;
                    if (cudaPointerGetAttributes(&at, job.src) == cudaSuccess &&
                        at.type == cudaMemoryTypeHost) {  // pinned: the DMA engine alone
                        e = cudaMemcpyAsync(job.dst, job.src, (size_t)job.bytes,
                                            cudaMemcpyHostToDevice, ctx->copy_stream);
                    } else {
                        cudaGetLastError();  // pageable memory is not a CUDA pointer
                        rc = ring_copy(ctx, job.dst, job.src, job.bytes, ctx->copy_stream,
                                       threads, &err);
                    }
                    if (rc == POTR_OK && e == cudaSuccess)
                        e = cudaEventRecord(job.ev, ctx->copy_stream);
                    if (rc == POTR_OK && e != cudaSuccess) {
                        rc = POTR_E_CUDA;
                        err = cudaGetErrorString(e);
                    }
                }
                lk.lock();
                if (rc && !ctx->upload_rc) {
                    ctx->upload_rc = rc;
                    ctx->upload_err = err;
                }
                ctx->upload_done = job.seq;
                ctx->upload_cv.notify_all();
            }
        });
    }
    const potr_ctx::UploadJob job{++ctx->upload_issued, dst, src, bytes, ev};
    ctx->upload_jobs.push_back(job);
    ctx->upload_pending = true;
    {
        std::unique_lock<std::mutex> lk(ctx->upload_mu);
        // a pinned source with nothing queued before it: the DMA engine
        // alone, issued from this thread (FIFO order on copy_stream holds)
        if (ctx->upload_todo.empty() && ctx->upload_done == job.seq - 1 && !ctx->upload_rc) {
            cudaPointerAttributes at;
            if (cudaPointerGetAttributes(&at, src) == cudaSuccess &&
                at.type == cudaMemoryTypeHost) {
                cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice,
                                                ctx->copy_stream);
                if (e == cudaSuccess) e = cudaEventRecord(ev, ctx->copy_stream);
                if (e != cudaSuccess) {
                    ctx->upload_rc = POTR_E_CUDA;
                    ctx->upload_err = cudaGetErrorString(e);
                }
                ctx->upload_done = job.seq;
                return POTR_OK;
            }
            cudaGetLastError();  // pageable memory is not a CUDA pointer
        }
        ctx->upload_todo.push_back(job);
    }
    ctx->upload_cv.notify_all();
    return POTR_OK;
}

int potr_upload_wait(potr_ctx *ctx) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    return upload_join(ctx);
}

namespace {

// Host -> device on the context stream: pinned sources by the DMA engine
// directly, pageable ones through the pinned ring.
int host_to_device(potr_ctx *ctx, void *dst, const void *src, int64_t bytes) {
    if (bytes <= 0) return 0;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost) {
        CK(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, ctx->stream));
        return 0;
    }
    cudaGetLastError();
    std::string err;
    const int rc = ring_copy(ctx, dst, src, bytes, ctx->stream, ring_threads(0), &err);
    return rc ? fail(ctx, rc, err) : 0;
}

// async_sh: the arrays go by potr_upload_async, the SH rows (81% of the
// bytes) last, so that a scoring call bins its first batches while they
// arrive.
int upload_splats(potr_ctx *ctx, int64_t n, const double *pos, const double *sh,
                  const double *op, const double *sc, const double *rot, potr_splats *out,
                  bool async_sh = false) {
    ENSURE(ctx->h_pos, sizeof(double) * 3 * n);
    ENSURE(ctx->h_sh, sizeof(double) * 48 * n);
    ENSURE(ctx->h_op, sizeof(double) * n);
    ENSURE(ctx->h_sc, sizeof(double) * 3 * n);
    ENSURE(ctx->h_rot, sizeof(double) * 4 * n);
    if (n > 0) {
        // async: all five queued on the upload worker, the SH rows last
        auto put = [ctx, async_sh](void *dst, const void *src, int64_t bytes) {
            return async_sh ? potr_upload_async(ctx, dst, src, bytes)
                            : host_to_device(ctx, dst, src, bytes);
        };
        int rc = 0;
        if ((rc = put(ctx->h_pos.p, pos, (int64_t)sizeof(double) * 3 * n))) return rc;
        if (op && (rc = put(ctx->h_op.p, op, (int64_t)sizeof(double) * n))) return rc;
        if (sc && (rc = put(ctx->h_sc.p, sc, (int64_t)sizeof(double) * 3 * n))) return rc;
        if (rot && (rc = put(ctx->h_rot.p, rot, (int64_t)sizeof(double) * 4 * n))) return rc;
        if ((rc = put(ctx->h_sh.p, sh, (int64_t)sizeof(double) * 48 * n))) return rc;
    }
    out->n = n;
    out->positions = P<double>(ctx->h_pos);
    out->sh = P<double>(ctx->h_sh);
    out->opacities = P<double>(ctx->h_op);
    out->scales = P<double>(ctx->h_sc);
    out->rotations = P<double>(ctx->h_rot);
    return 0;
}

}  // namespace

int potr_forward_stats_host(potr_ctx *ctx, int64_t n, const double *positions, const double *sh,
                            const double *opacities, const double *scales,
                            const double *rotations, int ncam, const potr_camera *cams,
                            const double *const *targets, double *importance,
                            double *camera_importance, double *delta_mse, double *mse) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    if (n < 0 || ncam < 0 || (ncam > 0 && !cams) || !importance)
        return fail(ctx, POTR_E_ARG, "bad arguments");
    if (n > 0 && (!positions || !sh || !opacities || !scales || !rotations))
        return fail(ctx, POTR_E_ARG, "splat array pointer is NULL");
    if (targets && (!delta_mse || !mse))
        return fail(ctx, POTR_E_ARG, "targets given without delta_mse/mse outputs");
    std::vector<const double *> dtg;
    if (targets) {
        size_t total = 0;
        for (int s = 0; s < ncam; s++) {
            if (check_cam(ctx, &cams[s])) return POTR_E_ARG;
            if (!targets[s]) return fail(ctx, POTR_E_ARG, "target pointer is NULL");
            total += 3 * (size_t)cams[s].width * cams[s].height;
        }
        ENSURE(ctx->h_tg, sizeof(double) * total);
        size_t off = 0;
        for (int s = 0; s < ncam; s++) {
            size_t cnt = 3 * (size_t)cams[s].width * cams[s].height;
            int trc = host_to_device(ctx, P<double>(ctx->h_tg) + off, targets[s],
                                     (int64_t)(sizeof(double) * cnt));
            if (trc) return trc;
            dtg.push_back(P<double>(ctx->h_tg) + off);
            off += cnt;
        }
    }
    ENSURE(ctx->h_imp, sizeof(double) * n);
    ENSURE(ctx->h_dm, sizeof(double) * n);
    ENSURE(ctx->h_mse, sizeof(double));
    if (camera_importance) ENSURE(ctx->h_ci, sizeof(double) * (size_t)ncam * n);
    // the SH rows upload while the first batches bin (score_views_run); every
    // exit below has joined that upload, so the caller may reuse `sh` at once
    potr_splats sp;
    int rc = upload_splats(ctx, n, positions, sh, opacities, scales, rotations, &sp, true);
    if (rc == 0)
        rc = potr_forward_stats(ctx, &sp, ncam, cams, targets ? dtg.data() : nullptr,
                                P<double>(ctx->h_imp),
                                camera_importance ? P<double>(ctx->h_ci) : nullptr,
                                targets ? P<double>(ctx->h_dm) : nullptr,
                                targets ? P<double>(ctx->h_mse) : nullptr);
    if (ctx->upload_pending) {
        const std::string err = ctx->err;
        const int jrc = upload_join(ctx);
        if (rc) ctx->err = err;
        else rc = jrc;
    }
    if (rc) return rc;
    CK(cudaMemcpyAsync(importance, ctx->h_imp.p, sizeof(double) * n, cudaMemcpyDeviceToHost,
                       ctx->stream));
    if (camera_importance)
        CK(cudaMemcpyAsync(camera_importance, ctx->h_ci.p, sizeof(double) * (size_t)ncam * n,
                           cudaMemcpyDeviceToHost, ctx->stream));
    if (targets) {
        CK(cudaMemcpyAsync(delta_mse, ctx->h_dm.p, sizeof(double) * n, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaMemcpyAsync(mse, ctx->h_mse.p, sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return POTR_OK;
}

int potr_compact_host(potr_ctx *ctx, int64_t n, const double *positions, const double *sh,
                      int ncam, const potr_camera *cams, const double *camera_importance,
                      double lambda_y, double parallel_threshold, double zero_threshold,
                      double *rgb, double *ycocg, int8_t *status) {
    if (!ctx) return POTR_E_ARG;
    CK(cudaSetDevice(ctx->device));
    JOIN_UPLOAD(ctx);
    if (n < 0 || ncam < 0 || !rgb || !ycocg || !status) return fail(ctx, POTR_E_ARG, "bad arguments");
    if (n > 0 && (!positions || !sh || (ncam > 0 && !camera_importance)))
        return fail(ctx, POTR_E_ARG, "input pointer is NULL");
    potr_splats sp;
    int rc = upload_splats(ctx, n, positions, sh, nullptr, nullptr, nullptr, &sp);
    if (rc) return rc;
    ENSURE(ctx->h_ci, sizeof(double) * (size_t)ncam * n);
    if (ncam > 0 && n > 0)
        CK(cudaMemcpyAsync(ctx->h_ci.p, camera_importance, sizeof(double) * (size_t)ncam * n,
                           cudaMemcpyHostToDevice, ctx->stream));
    ENSURE(ctx->h_rgb, sizeof(double) * 48 * n);
    ENSURE(ctx->h_yc, sizeof(double) * 48 * n);
    ENSURE(ctx->h_st, n);
    rc = potr_compact(ctx, &sp, ncam, cams, P<double>(ctx->h_ci), lambda_y, parallel_threshold,
                      zero_threshold, P<double>(ctx->h_rgb), P<double>(ctx->h_yc),
                      P<int8_t>(ctx->h_st));
    if (rc) return rc;
    CK(cudaMemcpyAsync(rgb, ctx->h_rgb.p, sizeof(double) * 48 * n, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaMemcpyAsync(ycocg, ctx->h_yc.p, sizeof(double) * 48 * n, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaMemcpyAsync(status, ctx->h_st.p, (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return POTR_OK;
}

}  // extern "C"
