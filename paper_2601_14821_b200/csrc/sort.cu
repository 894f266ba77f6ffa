// sort.cu -- hand-written radix sort and scans for sm_100a (see sort.cuh).
#include "common.cuh"
#include "sort.cuh"

namespace potr {

namespace {

constexpr int kBins = 256;             // 8-bit digits
constexpr int kSortThreads = 256;      // 8 warps; thread t owns digit t in the look-back
#ifndef POTR_SORT_IPT
#define POTR_SORT_IPT 20
#endif
constexpr int kSortIpt = POTR_SORT_IPT;  // keys per thread
// Keys per thread by (key, value) type: the packed tile sort (16-bit keys,
// 64-bit (slot, record) values) takes fewer so it fits 64 registers.
#ifndef POTR_SORT_PACKED_IPT
#define POTR_SORT_PACKED_IPT 16  // 16 at 64 registers: 29.2 -> 28.4 ms per C3 step
#endif
#ifndef POTR_SORT32_IPT
#define POTR_SORT32_IPT kSortIpt
#endif
template <typename K, typename V>
struct SortIpt {
    static constexpr int value = kSortIpt;
};
template <>
struct SortIpt<uint16_t, int64_t> {
    static constexpr int value = POTR_SORT_PACKED_IPT;
};
template <>
struct SortIpt<uint32_t, int32_t> {
    static constexpr int value = POTR_SORT32_IPT;
};
constexpr int kMinSortIpt0 = POTR_SORT_PACKED_IPT < kSortIpt ? POTR_SORT_PACKED_IPT : kSortIpt;
constexpr int kMinSortIpt = POTR_SORT32_IPT < kMinSortIpt0 ? POTR_SORT32_IPT : kMinSortIpt0;
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

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
    return (uint32_t)(((uint64_t)k >> shift) & (kBins - 1));
}

// Lanes holding the same 8-bit digit (d < 256), or the same invalid marker
// (d = 256): eight ballots on the digit bits -- full-rate VOTE/LOP instead of
// MATCH, whose address-divergence-unit pipe saturated in the first version.
__device__ __forceinline__ unsigned digit_peers(uint32_t d) {
    const unsigned FULL = 0xffffffffu;
    unsigned peers = __ballot_sync(FULL, d >> 8) ;
    peers = (d >> 8) ? peers : ~peers;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        const unsigned x = __ballot_sync(FULL, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? x : ~x;
    }
    return peers;
}

int passes_for(int begin_bit, int end_bit) {
    return end_bit > begin_bit ? (end_bit - begin_bit + 7) / 8 : 0;
}

template <typename K, typename V>
int64_t tiles_for(int64_t n) {
    constexpr int64_t items = (int64_t)kSortThreads * SortIpt<K, V>::value;
    return (n + items - 1) / items;
}
// the most tiles any (key, value) type cuts n items into (look-back sizing)
int64_t max_tiles_for(int64_t n) {
    const int64_t items = (int64_t)kSortThreads * kMinSortIpt;
    return (n + items - 1) / items;
}

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

// All passes' digit histograms in one read of the keys: plain shared atomics
// into two sub-histograms per CTA (even / odd warps).
template <typename K, int PASSES>
__global__ void __launch_bounds__(256) k_radix_hist(const K *__restrict__ keys, int64_t n,
                                                   int begin_bit, uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[2][PASSES * kBins];
    for (int i = threadIdx.x; i < 2 * PASSES * kBins; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t *hw = h[(threadIdx.x >> 5) & 1];
    constexpr int kQ = 8;  // keys per thread per sweep (independent loads)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kQ;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * kQ; base < n; base += stride) {
        K k[kQ];
        bool v[kQ];
#pragma unroll
        for (int q = 0; q < kQ; q++) {
            const int64_t i = base + q * blockDim.x + threadIdx.x;
            v[q] = i < n;
            k[q] = v[q] ? keys[i] : (K)0;
        }
#pragma unroll
        for (int q = 0; q < kQ; q++) {
            if (!v[q]) continue;
#pragma unroll
            for (int p = 0; p < PASSES; p++)
                atomicAdd(&hw[p * kBins + digit_of(k[q], begin_bit + 8 * p)], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < PASSES * kBins; i += blockDim.x) {
        const uint32_t c = h[0][i] + h[1][i];
        if (c) atomicAdd(&hist[i], c);
    }
}

template <typename K>
void launch_radix_hist(unsigned grid, const K *keys, int64_t n, int begin_bit, int passes,
                       uint32_t *hist, cudaStream_t st) {
    switch (passes) {
        case 1: k_radix_hist<K, 1><<<grid, 256, 0, st>>>(keys, n, begin_bit, hist); break;
        case 2: k_radix_hist<K, 2><<<grid, 256, 0, st>>>(keys, n, begin_bit, hist); break;
        case 3: k_radix_hist<K, 3><<<grid, 256, 0, st>>>(keys, n, begin_bit, hist); break;
        case 4: k_radix_hist<K, 4><<<grid, 256, 0, st>>>(keys, n, begin_bit, hist); break;
        case 5: k_radix_hist<K, 5><<<grid, 256, 0, st>>>(keys, n, begin_bit, hist); break;
        case 6: k_radix_hist<K, 6><<<grid, 256, 0, st>>>(keys, n, begin_bit, hist); break;
        case 7: k_radix_hist<K, 7><<<grid, 256, 0, st>>>(keys, n, begin_bit, hist); break;
        default: k_radix_hist<K, 8><<<grid, 256, 0, st>>>(keys, n, begin_bit, hist); break;
    }
}

// Where a pass's input values come from.
enum ValMode : int {
    kValRead = 0,  // vin[i]
    kValIota = 1,  // vbase + i (vin not read)
    kValPack = 2,  // int64 = (hi[i] << 32) | (uint32)(vbase + i): an int2 {vbase + i, hi[i]}
};

template <typename V, int VM>
__device__ __forceinline__ V input_value(const V *__restrict__ vin, const int32_t *__restrict__ hi,
                                         int64_t vbase, int64_t i) {
    if constexpr (VM == kValIota) {
        return (V)(vbase + i);
    } else if constexpr (VM == kValPack) {
        static_assert(sizeof(V) == 8, "packed values are 64-bit");
        return (V)(((uint64_t)(uint32_t)hi[i] << 32) | (uint64_t)(uint32_t)(vbase + i));
    } else {
        return vin[i];
    }
}

// One LSD pass over digit (key >> shift) & 255.  Dynamic shared memory: the
// tile's keys and values staged in digit order (kSortThreads x IPT each).
// CTAs per SM the register allocation must allow (0: ptxas's choice).  The
// depth sort's 32-bit keys with 32-bit values run faster at 4 CTAs (64
// registers: 22.1 -> 20.8 ms per C3 step); so do the packed tile-sort passes
// with 16 keys per thread (at 20 they spill).
#ifndef POTR_SORT32_MIN_BLOCKS
#define POTR_SORT32_MIN_BLOCKS 4
#endif
template <typename K, typename V>
struct OnesweepMinBlocks {
    static constexpr int value = 0;
};
template <>
struct OnesweepMinBlocks<uint32_t, int32_t> {
    static constexpr int value = POTR_SORT32_MIN_BLOCKS;
};
#ifndef POTR_SORT_PACKED_MIN_BLOCKS
#define POTR_SORT_PACKED_MIN_BLOCKS 4
#endif
template <>
struct OnesweepMinBlocks<uint16_t, int64_t> {
    static constexpr int value = POTR_SORT_PACKED_MIN_BLOCKS;
};

template <typename K, typename V, int VM>
__global__ void __launch_bounds__(kSortThreads, (OnesweepMinBlocks<K, V>::value)) k_onesweep(const K *__restrict__ kin,
                                                           K *__restrict__ kout,
                                                           const V *__restrict__ vin,
                                                           const int32_t *__restrict__ hi,
                                                           int64_t vbase,
                                                           V *__restrict__ vout, int64_t n,
                                                           int shift,
                                                           const uint32_t *__restrict__ hist,
                                                           uint64_t *status, uint32_t *tile_ctr) {
    constexpr int IPT = SortIpt<K, V>::value;
    constexpr int TILE = kSortThreads * IPT;
    __shared__ uint32_t whist[kSortWarps][kBins];  // per-warp digit counts -> offsets
    __shared__ uint32_t boff[kBins];               // tile-local start of each digit
    __shared__ int64_t gbase[kBins];               // global start of the digit minus boff
    __shared__ uint32_t warp_tot[kSortWarps];
    __shared__ uint32_t tile_s;
    extern __shared__ __align__(16) unsigned char stage_raw[];
    V *stage_v = reinterpret_cast<V *>(stage_raw);
    K *stage_k = reinterpret_cast<K *>(stage_raw + sizeof(V) * TILE);

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, t = threadIdx.x;
    const unsigned FULL = 0xffffffffu;
    if (t == 0) tile_s = atomicAdd(tile_ctr, 1u);
    for (int i = lane; i < kBins; i += 32) whist[w][i] = 0;
    __syncthreads();
    const int64_t tile = tile_s;
    const int64_t base = tile * TILE;
    const int tile_n = (int)(n - base < TILE ? n - base : TILE);

    // warp-striped: warp w holds tile items [w*32*IPT, (w+1)*32*IPT), round i
    // item w*32*IPT + i*32 + lane -- rounds in order keep the ranking stable
    K k[IPT];
    uint32_t rank[IPT];
    const int wbase = w * 32 * IPT;
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        const int j = wbase + i * 32 + lane;
        k[i] = j < tile_n ? kin[base + j] : (K)0;
    }
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        const int j = wbase + i * 32 + lane;
        const bool v = j < tile_n;
        const uint32_t d = v ? digit_of(k[i], shift) : kBins;
        // alternate the two ways of finding equal digits so that neither the
        // ADU (MATCH) nor the ALU (VOTE/LOP) pipe limits the ranking alone
        const unsigned peers = (i & 1) ? __match_any_sync(FULL, d) : digit_peers(d);
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
        // four predecessors per step (independent loads): the look-back walks
        // over tiles that have only published their own count
        for (int64_t j = tile - 1;;) {
            uint64_t s4[4];
#pragma unroll
            for (int q = 0; q < 4; q++)
                s4[q] = j - q >= 0 ? ld_relaxed(status + (j - q) * kBins + t) : kFlagInc;
            int q = 0;
            bool done = false;
            for (; q < 4; q++) {
                const uint64_t flag = s4[q] & ~kValMask;
                if (flag == 0) break;  // not published yet: reload from here
                prefix += s4[q] & kValMask;
                if (flag == kFlagInc) {
                    done = true;
                    break;
                }
            }
            if (done) break;
            j -= q;
        }
        st_relaxed(my_status, kFlagInc | (prefix + cnt));
    }
    boff[t] = local_start;
    gbase[t] = (int64_t)global_start + (int64_t)prefix - (int64_t)local_start;
    __syncthreads();

    // keys and values into digit order through shared memory ...
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        const int j = wbase + i * 32 + lane;
        if (j < tile_n) {
            const uint32_t d = digit_of(k[i], shift);
            const int pos = (int)(boff[d] + whist[w][d] + rank[i]);
            POTR_CHECK(pos >= 0 && pos < tile_n);
            stage_k[pos] = k[i];
            stage_v[pos] = input_value<V, VM>(vin, hi, vbase, base + j);
        }
    }
    __syncthreads();
    // ... then out in digit runs (consecutive addresses per digit)
#pragma unroll 4
    for (int j = t; j < tile_n; j += kSortThreads) {
        const K kk = stage_k[j];
        const int64_t dst = gbase[digit_of(kk, shift)] + j;
        POTR_CHECK(dst >= 0 && dst < n);
        kout[dst] = kk;
        vout[dst] = stage_v[j];
    }
}

template <typename K, typename V>
constexpr size_t onesweep_smem() {
    return (sizeof(K) + sizeof(V)) * (size_t)kSortThreads * SortIpt<K, V>::value;
}

template <typename K, typename V, int VM>
void set_smem_attr() {
    static bool done = false;
    if (!done) {
        cudaFuncSetAttribute(k_onesweep<K, V, VM>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)onesweep_smem<K, V>());
        done = true;
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
    off += align256(sizeof(uint64_t) * kBins * (size_t)max_tiles_for(n) * (passes > 0 ? passes : 1));
    L.bytes = off;
    return L;
}

// ---------------------------------------------------------------------------
// scans: one tile of kScanThreads x kScanIpt items per CTA (blocked: thread t
// holds items t*IPT .. t*IPT+IPT-1 of the tile), look-back on per-tile
// (flag | value) words packed in 64 bits, published and read relaxed (one
// word carries both, so no acquire / L1 invalidation is needed).

constexpr int kScanThreads = 256;
#ifndef POTR_SCAN_IPT
#define POTR_SCAN_IPT 16
#endif
constexpr int kScanIpt = POTR_SCAN_IPT;
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

// Warp 0: publish the tile aggregate, look back for the exclusive prefix of
// all earlier tiles (32 predecessors per step, one per lane), publish the
// inclusive value.  status[j] packs tile j's flag (kFlagAgg / kFlagInc, top
// two bits) with its value (biased by 2^31 so int32 maxima stay
// non-negative) in one 64-bit word: a single relaxed load sees a consistent
// pair, so no acquire (which invalidates L1) and no fence are needed.
constexpr int64_t kScanBias = (int64_t)1 << 31;

template <typename T, typename Op>
__device__ T tile_lookback(int64_t tile, T aggregate, Op op, uint64_t *status) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const auto pack = [](uint64_t flag, T x) {
        return flag | ((uint64_t)((int64_t)x + kScanBias) & kValMask);
    };
    if (tile == 0) {
        if (lane == 0) st_relaxed(&status[0], pack(kFlagInc, aggregate));
        return Op::identity();
    }
    if (lane == 0) st_relaxed(&status[tile], pack(kFlagAgg, aggregate));
    T prefix = Op::identity();
    for (int64_t j = tile - 1;;) {
        const int64_t idx = j - lane;
        const uint64_t sw = idx >= 0 ? ld_relaxed(&status[idx]) : pack(kFlagInc, Op::identity());
        const uint64_t f = sw & ~kValMask;
        const unsigned inc = __ballot_sync(FULL, f == kFlagInc);
        const unsigned zero = __ballot_sync(FULL, f == 0);
        const int k = inc ? __ffs(inc) - 1 : 31;
        const unsigned need = (2u << k) - 1u;  // lanes 0..k (k = 31: all)
        if (zero & need) continue;              // a needed predecessor is not published yet
        T x = ((need >> lane) & 1u) ? (T)((int64_t)(sw & kValMask) - kScanBias)
                                     : Op::identity();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x = op(x, __shfl_xor_sync(FULL, x, o));
        prefix = op(prefix, x);
        if (inc) break;
        j -= 32;
    }
    if (lane == 0) st_relaxed(&status[tile], pack(kFlagInc, op(prefix, aggregate)));
    return prefix;
}

// MODE 0: out[i] = inclusive sum of cnt[ids[i]]       (T = int64_t)
// MODE 1: out[i] = exclusive sum of in64[i]           (T = int64_t)
// MODE 2: out[i] = inclusive max of in32[i]           (T = int32_t)
// MODE 3: out32[k] = in32[i], i the k-th flagged item (T = int64_t); *count
// Warp-striped: warp w of the tile owns items w*32*IPT + r*32 + lane, so
// every load and store is coalesced; each warp scans its rounds in order with
// shuffles, the warps' totals are combined in shared memory, and the tile's
// prefix comes from the look-back.
template <int MODE, typename T, typename Op>
// MODE 0 (the pair-count scan of every batch) at 4 CTAs per SM (64
// registers); the other modes keep ptxas's allocation
#ifndef POTR_SCAN0_MIN_BLOCKS
#define POTR_SCAN0_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kScanThreads, (MODE == 0 ? POTR_SCAN0_MIN_BLOCKS : 0)) k_scan(const int32_t *__restrict__ ids,
                                                       const int32_t *__restrict__ in32,
                                                       const int64_t *__restrict__ in64,
                                                       const uint8_t *__restrict__ flg,
                                                       T *__restrict__ out,
                                                       int32_t *__restrict__ out32,
                                                       int32_t *count, int64_t n,
                                                       uint32_t *tile_ctr, uint64_t *status) {
    constexpr int W = kScanThreads / 32;
    __shared__ T warp_sum[W];
    __shared__ T warp_pre[W];
    __shared__ T s_prefix;
    __shared__ uint32_t tile_s;
    const unsigned FULL = 0xffffffffu;
    const Op op;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = tile_s;
    const int64_t wbase = tile * kScanTile + (int64_t)w * 32 * kScanIpt;
    T v[kScanIpt];
    int32_t idv[kScanIpt];
    if (MODE == 0) {
#pragma unroll
        for (int r = 0; r < kScanIpt; r++) {
            const int64_t i = wbase + r * 32 + lane;
            idv[r] = i < n ? ids[i] : -1;
        }
    }
#pragma unroll
    for (int r = 0; r < kScanIpt; r++) {
        const int64_t i = wbase + r * 32 + lane;
        T x = Op::identity();
        if (i < n) {
            if (MODE == 0) x = (T)in32[idv[r]];
            if (MODE == 1) x = (T)in64[i];
            if (MODE == 2) x = (T)in32[i];
            if (MODE == 3) x = (T)(flg[i] != 0);
        }
        v[r] = x;
    }
    // warp-inclusive values over the rounds; own values kept for the
    // exclusive modes (sums: excl = incl - own)
    T carry = Op::identity();
    T own[kScanIpt];
#pragma unroll
    for (int r = 0; r < kScanIpt; r++) {
        own[r] = v[r];
        T x = v[r];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x = op(y, x);
        }
        x = op(carry, x);
        v[r] = x;
        carry = __shfl_sync(FULL, x, 31);
    }
    if (lane == 0) warp_sum[w] = carry;
    __syncthreads();
    if (threadIdx.x < 32) {
        T acc = Op::identity();
        if (lane == 0) {
            for (int q = 0; q < W; q++) {
                warp_pre[q] = acc;
                acc = op(acc, warp_sum[q]);
            }
        }
        acc = __shfl_sync(FULL, acc, 0);
        const T p = tile_lookback(tile, acc, op, status);
        if (lane == 0) s_prefix = p;
    }
    __syncthreads();
    const T base = op(s_prefix, warp_pre[w]);
    T last = Op::identity();
#pragma unroll
    for (int r = 0; r < kScanIpt; r++) {
        const int64_t i = wbase + r * 32 + lane;
        const T incl = op(base, v[r]);
        if (i < n) {
            if (MODE == 0 || MODE == 2) out[i] = incl;
            if (MODE == 1) out[i] = incl - own[r];
            if (MODE == 3 && own[r]) out32[incl - 1] = in32[i];
            if (i == n - 1) last = incl;
        }
    }
    if (MODE == 3 && wbase <= n - 1 && n - 1 < wbase + 32 * kScanIpt && ((n - 1 - wbase) & 31) == lane)
        *count = (int32_t)last;
}

struct ScanLayout {
    uint32_t *ctr;
    uint64_t *status;
    size_t bytes;
};

ScanLayout scan_layout(void *temp, int64_t n) {
    ScanLayout L;
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    char *p = reinterpret_cast<char *>(temp);
    L.ctr = reinterpret_cast<uint32_t *>(p);
    L.status = reinterpret_cast<uint64_t *>(p + 256);
    L.bytes = 256 + align256(sizeof(uint64_t) * (size_t)(tiles > 0 ? tiles : 1));
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
    cudaError_t e = cudaMemsetAsync(temp, 0, L.bytes, st);
    if (e != cudaSuccess) return e;
    k_scan<MODE, T, Op><<<(unsigned)tiles, kScanThreads, 0, st>>>(
        ids, in32, in64, flg, out, out32, count, n, L.ctr, L.status);
    return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------------------
// host entry points

size_t radix_sort_temp_bytes(int64_t n, int begin_bit, int end_bit) {
    return sort_layout(nullptr, n, passes_for(begin_bit, end_bit)).bytes;
}

namespace {

template <typename V, int VM>
__global__ void k_init_vals(int64_t n, const int32_t *__restrict__ hi, int64_t vbase, V *v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = input_value<V, VM>(nullptr, hi, vbase, i);
}

template <typename K, typename V, int VM>
void launch_onesweep(int64_t tiles, const K *kin, K *kout, const V *vin, const int32_t *hi,
                     int64_t vbase, V *vout, int64_t n, int shift, const uint32_t *hist,
                     uint64_t *status, uint32_t *ctr, cudaStream_t st) {
    constexpr size_t smem = onesweep_smem<K, V>();
    set_smem_attr<K, V, VM>();
    k_onesweep<K, V, VM><<<(unsigned)tiles, kSortThreads, smem, st>>>(
        kin, kout, vin, hi, vbase, vout, n, shift, hist, status, ctr);
}

// The LSD passes; the first pass takes its values per vm0, later ones read
// the previous pass's output.
template <typename K, typename V, int VM0>
cudaError_t sort_impl(void *temp, size_t temp_bytes, K *keys, K *keys_alt, V *vals, V *vals_alt,
                      const int32_t *hi, int64_t vbase, int64_t n, int begin_bit, int end_bit,
                      bool *in_alt, cudaStream_t st) {
    *in_alt = false;
    if (n <= 0) return cudaSuccess;
    const int kbits = 8 * (int)sizeof(K);
    if (end_bit > kbits) end_bit = kbits;
    const int passes = passes_for(begin_bit, end_bit);
    if (passes == 0) {
        if constexpr (VM0 == kValRead) {
            return cudaSuccess;
        } else {
            // no key bits: the order is the input order
            k_init_vals<V, VM0><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, hi, vbase, vals);
            return cudaGetLastError();
        }
    }
    SortLayout L = sort_layout(temp, n, passes);
    if (L.bytes > temp_bytes) return cudaErrorInvalidValue;
    // counters, histograms and the look-back status of every pass
    cudaError_t e = cudaMemsetAsync(temp, 0, L.bytes, st);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (n + 255) / 256;
    launch_radix_hist<K>((unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), keys, n, begin_bit,
                         passes, L.hist, st);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t tiles = tiles_for<K, V>(n);
    K *ka = keys, *kb = keys_alt;
    V *va = vals, *vb = vals_alt;
    for (int p = 0; p < passes; p++) {
        const int shift = begin_bit + 8 * p;
        uint64_t *status = L.status + (size_t)p * kBins * tiles;
        if (p == 0)
            launch_onesweep<K, V, VM0>(tiles, ka, kb, va, hi, vbase, vb, n, shift,
                                       L.hist + p * kBins, status, L.ctr + p, st);
        else
            launch_onesweep<K, V, kValRead>(tiles, ka, kb, va, nullptr, 0, vb, n, shift,
                                            L.hist + p * kBins, status, L.ctr + p, st);
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

}  // namespace

template <typename K, typename V>
cudaError_t radix_sort_pairs(void *temp, size_t temp_bytes, K *keys, K *keys_alt, V *vals,
                             V *vals_alt, int64_t n, int begin_bit, int end_bit, bool iota_vals,
                             bool *in_alt, cudaStream_t st, int64_t iota_base) {
    if (iota_vals)
        return sort_impl<K, V, kValIota>(temp, temp_bytes, keys, keys_alt, vals, vals_alt,
                                         nullptr, iota_base, n, begin_bit, end_bit, in_alt, st);
    return sort_impl<K, V, kValRead>(temp, temp_bytes, keys, keys_alt, vals, vals_alt, nullptr,
                                     0, n, begin_bit, end_bit, in_alt, st);
}

template <typename K>
cudaError_t radix_sort_packed(void *temp, size_t temp_bytes, K *keys, K *keys_alt,
                              const int32_t *hi, int64_t vbase, int2 *vals, int2 *vals_alt,
                              int64_t n, int begin_bit, int end_bit, bool *in_alt,
                              cudaStream_t st) {
    static_assert(sizeof(int2) == sizeof(int64_t), "int2 is one 64-bit word");
    return sort_impl<K, int64_t, kValPack>(temp, temp_bytes, keys, keys_alt,
                                           reinterpret_cast<int64_t *>(vals),
                                           reinterpret_cast<int64_t *>(vals_alt), hi, vbase, n,
                                           begin_bit, end_bit, in_alt, st);
}

template cudaError_t radix_sort_packed<uint16_t>(void *, size_t, uint16_t *, uint16_t *,
                                                 const int32_t *, int64_t, int2 *, int2 *,
                                                 int64_t, int, int, bool *, cudaStream_t);
template cudaError_t radix_sort_packed<uint32_t>(void *, size_t, uint32_t *, uint32_t *,
                                                 const int32_t *, int64_t, int2 *, int2 *,
                                                 int64_t, int, int, bool *, cudaStream_t);

template cudaError_t radix_sort_pairs<uint16_t, int32_t>(void *, size_t, uint16_t *, uint16_t *,
                                                         int32_t *, int32_t *, int64_t, int, int,
                                                         bool, bool *, cudaStream_t, int64_t);
template cudaError_t radix_sort_pairs<uint32_t, int32_t>(void *, size_t, uint32_t *, uint32_t *,
                                                         int32_t *, int32_t *, int64_t, int, int,
                                                         bool, bool *, cudaStream_t, int64_t);
template cudaError_t radix_sort_pairs<uint64_t, int32_t>(void *, size_t, uint64_t *, uint64_t *,
                                                         int32_t *, int32_t *, int64_t, int, int,
                                                         bool, bool *, cudaStream_t, int64_t);
template cudaError_t radix_sort_pairs<uint64_t, int64_t>(void *, size_t, uint64_t *, uint64_t *,
                                                         int64_t *, int64_t *, int64_t, int, int,
                                                         bool, bool *, cudaStream_t, int64_t);

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
