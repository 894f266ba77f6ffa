// sort.cu -- hand-written radix sort and scans for sm_100a (see sort.cuh).
#include "sort.cuh"

namespace potr {

namespace {

constexpr int kBins = 256;             // 8-bit digits
constexpr int kSortThreads = 256;      // 8 warps; thread t owns digit t in the look-back
constexpr int kSortIpt = 16;           // keys per thread
constexpr int kTileItems = kSortThreads * kSortIpt;
constexpr int kSortWarps = kSortThreads / 32;
static_assert(kSortThreads == kBins, "one thread per digit");

constexpr uint64_t kFlagAgg = 1ull << 62;  // tile count published
constexpr uint64_t kFlagInc = 2ull << 62;  // inclusive prefix published
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_relaxed(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
    return (uint32_t)(((uint64_t)k >> shift) & (kBins - 1));
}

__device__ __forceinline__ int64_t cnt_gather(const int32_t *ids, const int32_t *cnt, int64_t i) {
    return (int64_t)cnt[ids[i]];
}

template <typename V>
__global__ void k_iota_vals(int64_t n, V *v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (V)i;
}

int passes_for(int begin_bit, int end_bit) {
    return end_bit > begin_bit ? (end_bit - begin_bit + 7) / 8 : 0;
}

int64_t tiles_for(int64_t n) { return (n + kTileItems - 1) / kTileItems; }

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Exclusive scan of one value per thread over the CTA (256 threads).
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *warp_tot) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    uint32_t before = 0;
    for (int i = 0; i < w; i++) before += warp_tot[i];
    __syncthreads();
    return before + x - v;
}

// All passes' digit histograms in one read of the keys.  Lanes holding the
// same digit add together (__match_any_sync), so a constant digit costs one
// shared atomic per warp instead of 32 colliding ones.
template <typename K>
__global__ void __launch_bounds__(256) k_radix_hist(const K *__restrict__ keys, int64_t n,
                                                   int begin_bit, int passes,
                                                   uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[8 * kBins];
    for (int i = threadIdx.x; i < passes * kBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const bool v = i < n;
        const K k = v ? keys[i] : (K)0;
        for (int p = 0; p < passes; p++) {
            const uint32_t d = v ? digit_of(k, begin_bit + 8 * p) : kBins;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (v && lane == __ffs(peers) - 1) atomicAdd(&h[p * kBins + d], __popc(peers));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kBins; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

// One LSD pass over digit (key >> shift) & 255.
template <typename K, typename V, bool IOTA>
__global__ void __launch_bounds__(kSortThreads) k_onesweep(const K *__restrict__ kin,
                                                           K *__restrict__ kout,
                                                           const V *__restrict__ vin,
                                                           V *__restrict__ vout, int64_t n,
                                                           int shift,
                                                           const uint32_t *__restrict__ hist,
                                                           uint64_t *status, uint32_t *tile_ctr) {
    constexpr int kStageBytes = kTileItems * (sizeof(K) > sizeof(V) ? sizeof(K) : sizeof(V));
    __shared__ uint32_t whist[kSortWarps][kBins];  // per-warp digit counts -> offsets
    __shared__ uint32_t boff[kBins];               // tile-local start of each digit
    __shared__ int64_t gbase[kBins];               // global start of the digit minus boff
    __shared__ uint32_t warp_tot[kSortWarps];
    __shared__ uint32_t tile_s;
    __shared__ __align__(16) unsigned char stage_raw[kStageBytes];
    K *stage_k = reinterpret_cast<K *>(stage_raw);
    V *stage_v = reinterpret_cast<V *>(stage_raw);

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, t = threadIdx.x;
    const unsigned FULL = 0xffffffffu;
    if (t == 0) tile_s = atomicAdd(tile_ctr, 1u);
    for (int i = lane; i < kBins; i += 32) whist[w][i] = 0;
    __syncthreads();
    const int64_t tile = tile_s;
    const int64_t base = tile * kTileItems;
    const int tile_n = (int)(n - base < kTileItems ? n - base : kTileItems);

    // warp-striped: warp w holds tile items [w*32*IPT, (w+1)*32*IPT), round i
    // item w*32*IPT + i*32 + lane -- rounds in order keep the ranking stable
    K k[kSortIpt];
    uint32_t rank[kSortIpt];
    const int wbase = w * 32 * kSortIpt;
#pragma unroll
    for (int i = 0; i < kSortIpt; i++) {
        const int j = wbase + i * 32 + lane;
        k[i] = j < tile_n ? kin[base + j] : (K)0;
    }
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kSortIpt; i++) {
        const int j = wbase + i * 32 + lane;
        const bool v = j < tile_n;
        const uint32_t d = v ? digit_of(k[i], shift) : kBins;
        const unsigned peers = __match_any_sync(FULL, d);
        const int leader = __ffs(peers) - 1;
        uint32_t b = 0;
        if (v && lane == leader) {
            b = whist[w][d];
            whist[w][d] = b + __popc(peers);
        }
        b = __shfl_sync(FULL, b, leader);
        rank[i] = b + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();

    // thread t: digit t.  Offsets of the warps inside the tile, the tile count,
    // its publication, the digit's start in the tile and in the output.
    uint32_t cnt = 0;
#pragma unroll
    for (int q = 0; q < kSortWarps; q++) {
        const uint32_t c = whist[q][t];
        whist[q][t] = cnt;
        cnt += c;
    }
    uint64_t *my_status = status + tile * kBins + t;
    st_relaxed(my_status, (tile == 0 ? kFlagInc : kFlagAgg) | (uint64_t)cnt);
    const uint32_t hcount = hist[t];
    const uint32_t local_start = block_exclusive_scan(cnt, warp_tot);
    const uint32_t global_start = block_exclusive_scan(hcount, warp_tot);
    uint64_t prefix = 0;
    if (tile > 0) {
        for (int64_t j = tile - 1;;) {
            const uint64_t s = ld_relaxed(status + j * kBins + t);
            const uint64_t flag = s & ~kValMask;
            if (flag == 0) continue;  // predecessor not published yet
            prefix += s & kValMask;
            if (flag == kFlagInc) break;
            j--;
        }
        st_relaxed(my_status, kFlagInc | (prefix + cnt));
    }
    boff[t] = local_start;
    gbase[t] = (int64_t)global_start + (int64_t)prefix - (int64_t)local_start;
    __syncthreads();

    // keys: into tile order through shared memory, then out in digit runs
    int pos[kSortIpt];
#pragma unroll
    for (int i = 0; i < kSortIpt; i++) {
        const int j = wbase + i * 32 + lane;
        pos[i] = -1;
        if (j < tile_n) {
            const uint32_t d = digit_of(k[i], shift);
            pos[i] = (int)(boff[d] + whist[w][d] + rank[i]);
            stage_k[pos[i]] = k[i];
        }
    }
    __syncthreads();
    int64_t dst[kSortIpt];
#pragma unroll
    for (int i = 0; i < kSortIpt; i++) {
        const int j = t + i * kSortThreads;
        dst[i] = -1;
        if (j < tile_n) {
            const K kk = stage_k[j];
            dst[i] = gbase[digit_of(kk, shift)] + j;
            kout[dst[i]] = kk;
        }
    }
    __syncthreads();
    // values: the same permutation
#pragma unroll
    for (int i = 0; i < kSortIpt; i++) {
        const int j = wbase + i * 32 + lane;
        if (pos[i] >= 0) stage_v[pos[i]] = IOTA ? (V)(base + j) : vin[base + j];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSortIpt; i++) {
        const int j = t + i * kSortThreads;
        if (dst[i] >= 0) vout[dst[i]] = stage_v[j];
    }
}

struct SortLayout {
    uint32_t *hist;      // passes x 256
    uint32_t *ctr;       // passes tile counters
    uint64_t *status;    // passes x tiles x 256
    size_t bytes;
};

SortLayout sort_layout(void *temp, int64_t n, int passes) {
    SortLayout L;
    char *p = reinterpret_cast<char *>(temp);
    size_t off = 0;
    L.hist = reinterpret_cast<uint32_t *>(p + off);
    off += align256(sizeof(uint32_t) * kBins * (passes > 0 ? passes : 1));
    L.ctr = reinterpret_cast<uint32_t *>(p + off);
    off += align256(sizeof(uint32_t) * 8);
    L.status = reinterpret_cast<uint64_t *>(p + off);
    off += align256(sizeof(uint64_t) * kBins * (size_t)tiles_for(n) * (passes > 0 ? passes : 1));
    L.bytes = off;
    return L;
}

// ---------------------------------------------------------------------------
// scans: one tile of kScanThreads x kScanIpt items per CTA (blocked: thread t
// holds items t*IPT .. t*IPT+IPT-1 of the tile), look-back on per-tile
// (flag, aggregate, inclusive) published with release / acquire.

constexpr int kScanThreads = 256;
constexpr int kScanIpt = 16;
constexpr int kScanTile = kScanThreads * kScanIpt;

template <typename T>
struct SumOp {
    static __device__ __forceinline__ T identity() { return (T)0; }
    __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
template <typename T>
struct MaxOp {
    static __device__ __forceinline__ T identity() { return (T)INT32_MIN; }
    __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
};

// Exclusive scan of one value per thread over the CTA; *total = the reduction.
template <typename T, typename Op>
__device__ __forceinline__ T block_exclusive(T v, Op op, T *warp_tot, T *total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = op(y, x);
    }
    T ex = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) ex = Op::identity();
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        T acc = Op::identity();
        for (int i = 0; i < kScanThreads / 32; i++) {
            const T c = warp_tot[i];
            warp_tot[i] = acc;  // exclusive warp offsets
            acc = op(acc, c);
        }
        *total = acc;
    }
    __syncthreads();
    const T r = op(warp_tot[w], ex);
    __syncthreads();
    return r;
}

// Thread 0: publish the tile aggregate, look back for the exclusive prefix of
// all earlier tiles, publish the inclusive value.  vals[2j] / vals[2j+1] hold
// tile j's aggregate / inclusive value (as int64), flags[j] = 1 / 2 once
// they are written.  The values are read with L1-bypassing loads: another
// CTA on this SM may have cached the line when only the aggregate was there.
template <typename T, typename Op>
__device__ T tile_lookback(int64_t tile, T aggregate, Op op, uint32_t *flags, int64_t *vals) {
    if (tile == 0) {
        st_relaxed(reinterpret_cast<uint64_t *>(&vals[1]), (uint64_t)(int64_t)aggregate);
        __threadfence();
        st_release(&flags[0], 2u);
        return Op::identity();
    }
    st_relaxed(reinterpret_cast<uint64_t *>(&vals[2 * tile]), (uint64_t)(int64_t)aggregate);
    __threadfence();
    st_release(&flags[tile], 1u);
    T prefix = Op::identity();
    for (int64_t j = tile - 1;;) {
        const uint32_t f = ld_acquire(&flags[j]);
        if (f == 0) continue;
        const int64_t x = (int64_t)ld_relaxed(
            reinterpret_cast<const uint64_t *>(&vals[f == 2u ? 2 * j + 1 : 2 * j]));
        prefix = op((T)x, prefix);
        if (f == 2u) break;
        j--;
    }
    st_relaxed(reinterpret_cast<uint64_t *>(&vals[2 * tile + 1]),
               (uint64_t)(int64_t)op(prefix, aggregate));
    __threadfence();
    st_release(&flags[tile], 2u);
    return prefix;
}

// MODE 0: out[i] = inclusive sum of cnt[ids[i]]       (T = int64_t)
// MODE 1: out[i] = exclusive sum of in64[i]           (T = int64_t)
// MODE 2: out[i] = inclusive max of in32[i]           (T = int32_t)
// MODE 3: out32[k] = in32[i], i the k-th flagged item (T = int64_t); *count
template <int MODE, typename T, typename Op>
__global__ void __launch_bounds__(kScanThreads) k_scan(const int32_t *__restrict__ ids,
                                                       const int32_t *__restrict__ in32,
                                                       const int64_t *__restrict__ in64,
                                                       const uint8_t *__restrict__ flg,
                                                       T *__restrict__ out,
                                                       int32_t *__restrict__ out32,
                                                       int32_t *count, int64_t n,
                                                       uint32_t *tile_ctr, uint32_t *flags,
                                                       int64_t *vals) {
    __shared__ T warp_tot[kScanThreads / 32];
    __shared__ T s_total, s_prefix;
    __shared__ uint32_t tile_s;
    const Op op;
    if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = tile_s;
    const int64_t i0 = tile * kScanTile + (int64_t)threadIdx.x * kScanIpt;
    T x[kScanIpt];
    T acc = Op::identity();
#pragma unroll
    for (int q = 0; q < kScanIpt; q++) {
        const int64_t i = i0 + q;
        T v = Op::identity();
        if (i < n) {
            if (MODE == 0) v = (T)cnt_gather(ids, in32, i);
            if (MODE == 1) v = (T)in64[i];
            if (MODE == 2) v = (T)in32[i];
            if (MODE == 3) v = (T)(flg[i] != 0);
        }
        x[q] = v;
        acc = op(acc, v);
    }
    const T excl = block_exclusive(acc, op, warp_tot, &s_total);
    if (threadIdx.x == 0) s_prefix = tile_lookback(tile, s_total, op, flags, vals);
    __syncthreads();
    T run = op(s_prefix, excl);
#pragma unroll
    for (int q = 0; q < kScanIpt; q++) {
        const int64_t i = i0 + q;
        if (i >= n) break;
        if (MODE == 0 || MODE == 2) {
            run = op(run, x[q]);
            out[i] = run;
        } else if (MODE == 1) {
            out[i] = run;
            run = op(run, x[q]);
        } else {
            if (x[q]) out32[run] = in32[i];
            run = op(run, x[q]);
        }
    }
    if (MODE == 3 && i0 < n && i0 + kScanIpt >= n) *count = (int32_t)run;
}

struct ScanLayout {
    uint32_t *ctr, *flags;
    void *vals;
    size_t bytes;
};

ScanLayout scan_layout(void *temp, int64_t n) {
    ScanLayout L;
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    char *p = reinterpret_cast<char *>(temp);
    size_t off = 0;
    L.ctr = reinterpret_cast<uint32_t *>(p + off);
    off += 256;
    L.flags = reinterpret_cast<uint32_t *>(p + off);
    off += align256(sizeof(uint32_t) * (size_t)(tiles > 0 ? tiles : 1));
    L.vals = p + off;
    off += align256(2 * sizeof(int64_t) * (size_t)(tiles > 0 ? tiles : 1));
    L.bytes = off;
    return L;
}

template <int MODE, typename T, typename Op>
cudaError_t run_scan(void *temp, size_t temp_bytes, const int32_t *ids, const int32_t *in32,
                     const int64_t *in64, const uint8_t *flg, T *out, int32_t *out32,
                     int32_t *count, int64_t n, cudaStream_t st) {
    if (n <= 0) {
        if (MODE == 3 && count) return cudaMemsetAsync(count, 0, sizeof(int32_t), st);
        return cudaSuccess;
    }
    ScanLayout L = scan_layout(temp, n);
    if (L.bytes > temp_bytes) return cudaErrorInvalidValue;
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    cudaError_t e = cudaMemsetAsync(temp, 0, L.bytes - align256(2 * sizeof(int64_t) * tiles), st);
    if (e != cudaSuccess) return e;
    k_scan<MODE, T, Op><<<(unsigned)tiles, kScanThreads, 0, st>>>(
        ids, in32, in64, flg, out, out32, count, n, L.ctr, L.flags,
        reinterpret_cast<int64_t *>(L.vals));
    return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------------------
// host entry points

size_t radix_sort_temp_bytes(int64_t n, int begin_bit, int end_bit) {
    return sort_layout(nullptr, n, passes_for(begin_bit, end_bit)).bytes;
}

template <typename K, typename V>
cudaError_t radix_sort_pairs(void *temp, size_t temp_bytes, K *keys, K *keys_alt, V *vals,
                             V *vals_alt, int64_t n, int begin_bit, int end_bit, bool iota_vals,
                             bool *in_alt, cudaStream_t st) {
    *in_alt = false;
    if (n <= 0) return cudaSuccess;
    const int kbits = 8 * (int)sizeof(K);
    if (end_bit > kbits) end_bit = kbits;
    const int passes = passes_for(begin_bit, end_bit);
    if (passes == 0) {
        if (!iota_vals) return cudaSuccess;
        // no key bits: the order is the input order
        k_iota_vals<V><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, vals);
        return cudaGetLastError();
    }
    SortLayout L = sort_layout(temp, n, passes);
    if (L.bytes > temp_bytes) return cudaErrorInvalidValue;
    // counters, histograms and the look-back status of every pass
    cudaError_t e = cudaMemsetAsync(temp, 0, L.bytes, st);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (n + 255) / 256;
    k_radix_hist<K><<<(unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, st>>>(
        keys, n, begin_bit, passes, L.hist);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t tiles = tiles_for(n);
    K *ka = keys, *kb = keys_alt;
    V *va = vals, *vb = vals_alt;
    for (int p = 0; p < passes; p++) {
        const int shift = begin_bit + 8 * p;
        uint64_t *status = L.status + (size_t)p * kBins * tiles;
        if (p == 0 && iota_vals)
            k_onesweep<K, V, true><<<(unsigned)tiles, kSortThreads, 0, st>>>(
                ka, kb, nullptr, vb, n, shift, L.hist + p * kBins, status, L.ctr + p);
        else
            k_onesweep<K, V, false><<<(unsigned)tiles, kSortThreads, 0, st>>>(
                ka, kb, va, vb, n, shift, L.hist + p * kBins, status, L.ctr + p);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        K *tk = ka;
        ka = kb;
        kb = tk;
        V *tv = va;
        va = vb;
        vb = tv;
    }
    *in_alt = (passes & 1) != 0;
    return cudaSuccess;
}

template cudaError_t radix_sort_pairs<uint16_t, int32_t>(void *, size_t, uint16_t *, uint16_t *,
                                                         int32_t *, int32_t *, int64_t, int, int,
                                                         bool, bool *, cudaStream_t);
template cudaError_t radix_sort_pairs<uint32_t, int32_t>(void *, size_t, uint32_t *, uint32_t *,
                                                         int32_t *, int32_t *, int64_t, int, int,
                                                         bool, bool *, cudaStream_t);
template cudaError_t radix_sort_pairs<uint64_t, int32_t>(void *, size_t, uint64_t *, uint64_t *,
                                                         int32_t *, int32_t *, int64_t, int, int,
                                                         bool, bool *, cudaStream_t);
template cudaError_t radix_sort_pairs<uint64_t, int64_t>(void *, size_t, uint64_t *, uint64_t *,
                                                         int64_t *, int64_t *, int64_t, int, int,
                                                         bool, bool *, cudaStream_t);

size_t scan_temp_bytes(int64_t n) { return scan_layout(nullptr, n).bytes; }

cudaError_t inclusive_sum_gather(void *temp, size_t temp_bytes, const int32_t *ids,
                                 const int32_t *cnt, int64_t *out, int64_t n, cudaStream_t st) {
    return run_scan<0, int64_t, SumOp<int64_t>>(temp, temp_bytes, ids, cnt, nullptr, nullptr, out,
                                                nullptr, nullptr, n, st);
}

cudaError_t exclusive_sum_i64(void *temp, size_t temp_bytes, const int64_t *in, int64_t *out,
                              int64_t n, cudaStream_t st) {
    return run_scan<1, int64_t, SumOp<int64_t>>(temp, temp_bytes, nullptr, nullptr, in, nullptr,
                                                out, nullptr, nullptr, n, st);
}

cudaError_t inclusive_max_i32(void *temp, size_t temp_bytes, const int32_t *in, int32_t *out,
                              int64_t n, cudaStream_t st) {
    return run_scan<2, int32_t, MaxOp<int32_t>>(temp, temp_bytes, nullptr, in, nullptr, nullptr,
                                                out, nullptr, nullptr, n, st);
}

cudaError_t select_flagged_i32(void *temp, size_t temp_bytes, const int32_t *in,
                               const uint8_t *flags, int32_t *out, int32_t *count, int64_t n,
                               cudaStream_t st) {
    return run_scan<3, int64_t, SumOp<int64_t>>(temp, temp_bytes, nullptr, in, nullptr, flags,
                                                nullptr, out, count, n, st);
}

}  // namespace potr
