// codec.cu -- the data-parallel parts of the codec back end (SURVEY.md 8f
// row 4): the camera-adaptive position octree (quantize.py:92-170) built and
// serialised on the GPU, and the quantised, zigzag/LEB128-coded attribute
// streams (bitstream.py:116-155, varint.py).  zstd stays libzstd on the host
// (byte identity).  Every output byte equals the reference's
// (tests/test_gpu_parity.py::test_codec_*).
//
// Octree.  The reference recurses: a node with one splat whose half-diagonal
// sqrt(3) h is below the splat's tolerance, or any node at the depth limit,
// is a leaf; otherwise the splats are split by octant (4 (x >= cx) + 2 (y >=
// cy) + (z >= cz)) and the children visited in ascending octant order.  Here
// every splat descends alone to the depth limit with the same arithmetic
// (centre +- h/2, h/2 per level), giving its 3-bit octant path; a stable sort
// of the paths is the DFS order (equal paths keep ascending index, as
// `idx[octant == o]` does).  With lcp(t) the common path length of sorted
// neighbours, a splat is alone from depth D = 1 + max(lcp(t), lcp(t+1)) and
// its leaf depth is min(max_depth, max(D, first depth whose half-diagonal
// meets its tolerance)); identical paths share one leaf at the limit.  In DFS
// order, the leading splat of each leaf emits the internal nodes deeper than
// lcp(t) on its path (their occupancy bytes) and then its leaf (0x00 +
// LEB128 count).  A node's occupancy collects its own first splat's child
// octant and, by atomicOr, the octant of every later leaf that branches off
// exactly at its depth.

#include <cstring>
#include <string>

#include "common.cuh"
#include "raster.cuh"
#include "sort.cuh"

namespace potr {

constexpr double kSqrt3 = 1.7320508075688772;  // np.sqrt(3.0)

static inline unsigned blocks_for(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// quantize.py:92-96 + :120-123: tol = max(gamma, beta * min over eyes of |p - eye|)
__global__ void k_oct_tol(int64_t n, const double *__restrict__ pos, int neyes,
                          const double *__restrict__ eyes, double beta, double gamma,
                          double *__restrict__ tol) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double t = gamma;
    if (beta > 0.0 && neyes > 0) {
        double dmin = 0.0;
        for (int e = 0; e < neyes; e++) {
            const double d0 = pos[3 * k] - eyes[3 * e], d1 = pos[3 * k + 1] - eyes[3 * e + 1];
            const double d2 = pos[3 * k + 2] - eyes[3 * e + 2];
            const double d = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
            dmin = (e == 0 || d < dmin) ? d : dmin;
        }
        const double bt = beta * dmin;
        t = bt > gamma ? bt : gamma;  // np.maximum(gamma, .)
    }
    tol[k] = t;
}

// The octant path to the depth limit (hi: levels 0-11, lo: 12-23, 3 bits
// each, level 0 most significant) and the first depth whose half-diagonal
// meets the tolerance.
__global__ void k_oct_path(int64_t n, const double *__restrict__ pos,
                           const double *__restrict__ tol, double cx, double cy, double cz,
                           double half, int max_depth, uint64_t *__restrict__ khi,
                           uint64_t *__restrict__ klo, int8_t *__restrict__ dtol,
                           int32_t *__restrict__ idx) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double p0 = pos[3 * k], p1 = pos[3 * k + 1], p2 = pos[3 * k + 2], t = tol[k];
    double c0 = cx, c1 = cy, c2 = cz, h = half;
    uint64_t hi = 0, lo = 0;
    int dt = max_depth;
    for (int d = 0; d < max_depth; d++) {
        if (dt == max_depth && kSqrt3 * h < t) dt = d;
        const int o = 4 * (p0 >= c0) + 2 * (p1 >= c1) + (p2 >= c2);
        if (d < 12) hi |= (uint64_t)o << (3 * (11 - d));
        else lo |= (uint64_t)o << (3 * (23 - d));
        const double off = h * 0.5;  // _child_center (quantize.py:66-73)
        c0 = c0 + ((o & 4) ? off : -off);
        c1 = c1 + ((o & 2) ? off : -off);
        c2 = c2 + ((o & 1) ? off : -off);
        h = h * 0.5;
    }
    khi[k] = hi;
    klo[k] = lo;
    dtol[k] = (int8_t)dt;
    idx[k] = (int32_t)k;
}

__global__ void k_gather_u64(int64_t n, const int32_t *__restrict__ idx,
                             const uint64_t *__restrict__ src, uint64_t *__restrict__ dst) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) dst[t] = src[idx[t]];
}

__device__ __forceinline__ int digit_at(uint64_t hi, uint64_t lo, int d) {
    return d < 12 ? (int)((hi >> (3 * (11 - d))) & 7) : (int)((lo >> (3 * (23 - d))) & 7);
}

__device__ __forceinline__ int path_lcp(uint64_t ha, uint64_t la, uint64_t hb, uint64_t lb,
                                        int max_depth) {
    int l;
    if (ha != hb) l = (__clzll((long long)(ha ^ hb)) - 28) / 3;
    else if (la != lb) l = 12 + (__clzll((long long)(la ^ lb)) - 28) / 3;
    else l = 24;
    return l < max_depth ? l : max_depth;
}

// Per sorted position: lcp with the previous splat (-1 at 0), group-start flag.
__global__ void k_oct_lcp(int64_t n, const int32_t *__restrict__ order,
                          const uint64_t *__restrict__ khi, const uint64_t *__restrict__ klo,
                          int max_depth, int32_t *__restrict__ lcp, uint8_t *__restrict__ start) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    int l = -1;
    if (t > 0) {
        const int a = order[t - 1], b = order[t];
        l = path_lcp(khi[a], klo[a], khi[b], klo[b], max_depth);
    }
    lcp[t] = l;
    start[t] = (uint8_t)(l < max_depth);
}

__device__ __forceinline__ int uleb_len(uint64_t v) {
    int c = 1;
    while (v > 0x7F) {
        v >>= 7;
        c++;
    }
    return c;
}

// Per leaf (group of equal paths, led by sorted position t = gstart[j]):
// depth range [a, L) of the internal nodes it emits, leaf depth L, count,
// byte count; and the child octant of its own new internal nodes.
__global__ void k_oct_leaf(int64_t ng, int64_t n, const int32_t *__restrict__ gstart,
                           const int32_t *__restrict__ lcp, const int32_t *__restrict__ order,
                           const uint64_t *__restrict__ khi, const uint64_t *__restrict__ klo,
                           const int8_t *__restrict__ dtol, int max_depth,
                           int32_t *__restrict__ glcp, int8_t *__restrict__ gleaf,
                           int32_t *__restrict__ gcount, int64_t *__restrict__ gbytes,
                           uint32_t *__restrict__ occ) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ng) return;
    const int64_t t = gstart[j];
    const int64_t e = j + 1 < ng ? gstart[j + 1] : n;
    const int count = (int)(e - t);
    const int l0 = lcp[t];
    int L = max_depth;
    if (count == 1) {
        const int l1 = t + 1 < n ? lcp[t + 1] : -1;
        const int D = 1 + (l0 > l1 ? l0 : l1);
        const int dt = dtol[order[t]];
        const int m = D > dt ? D : dt;
        L = m < max_depth ? m : max_depth;
    }
    const int a = l0 + 1;
    glcp[j] = l0;
    gleaf[j] = (int8_t)L;
    gcount[j] = count;
    gbytes[j] = (int64_t)(L - a) + 1 + uleb_len((uint64_t)count);
    const int s = order[t];
    const uint64_t hi = khi[s], lo = klo[s];
    for (int d = a; d < L; d++) occ[j * max_depth + d] = 1u << digit_at(hi, lo, d);
}

// Level d of the "node start" scan: the latest group at or before j whose
// lcp is below d starts the depth-d node containing j.
__global__ void k_oct_mark(int64_t ng, const int32_t *__restrict__ glcp, int d,
                           int32_t *__restrict__ mark) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < ng) mark[j] = glcp[j] < d ? (int32_t)j : -1;
}

// Groups branching at depth d add their child octant to that node.
__global__ void k_oct_branch(int64_t ng, const int32_t *__restrict__ glcp,
                             const int32_t *__restrict__ seg, int d,
                             const int32_t *__restrict__ gstart, const int32_t *__restrict__ order,
                             const uint64_t *__restrict__ khi, const uint64_t *__restrict__ klo,
                             int max_depth, uint32_t *__restrict__ occ) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ng || j == 0 || glcp[j] != d) return;
    const int S = seg[j - 1];
    const int s = order[gstart[j]];
    atomicOr(&occ[(int64_t)S * max_depth + d], 1u << digit_at(khi[s], klo[s], d));
}

__global__ void k_oct_emit(int64_t ng, const int32_t *__restrict__ glcp,
                           const int8_t *__restrict__ gleaf, const int32_t *__restrict__ gcount,
                           const int64_t *__restrict__ goff, const uint32_t *__restrict__ occ,
                           int max_depth, uint8_t *__restrict__ out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ng) return;
    int64_t o = goff[j];
    const int a = glcp[j] + 1, L = gleaf[j];
    for (int d = a; d < L; d++) out[o++] = (uint8_t)occ[j * max_depth + d];
    out[o++] = 0x00;
    uint64_t v = (uint64_t)gcount[j];
    while (v > 0x7F) {
        out[o++] = (uint8_t)((v & 0x7F) | 0x80);
        v >>= 7;
    }
    out[o] = (uint8_t)v;
}

__global__ void k_iota32(int64_t n, int32_t *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[t] = (int32_t)t;
}

__global__ void k_order_i64(int64_t n, const int32_t *__restrict__ src, int64_t *__restrict__ dst) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) dst[t] = src[t];
}

// ---------------------------------------------------------------------------
// attribute streams (bitstream.py:116-155): 55 streams x n values, stream s
// of value i at s * n + i, each coded as a LEB128 varint (zigzag first for
// the signed ones), concatenated in stream order.

__device__ __forceinline__ int64_t quant(double x, double sf) {
    return (int64_t)floor(0.5 + x * sf);  // quantize_uniform: floor(0.5 + x * sf)
}
__device__ __forceinline__ uint64_t zigzag(int64_t x) {
    return ((uint64_t)x << 1) ^ (uint64_t)(x >> 63);
}

constexpr int kStreams = 55;  // streams 1..55 of the container (0 is the octree)

__global__ void k_attr_values(int64_t n, const int64_t *__restrict__ order,
                              const double *__restrict__ ycocg, const double *__restrict__ opac,
                              const double *__restrict__ log_scales,
                              const double *__restrict__ rot, double sf_sh, double sf_op,
                              double sf_rot, double sf_sc, uint64_t *__restrict__ val,
                              uint8_t *__restrict__ len) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t k = order[i];
    const int64_t kp = i > 0 ? order[i - 1] : -1;
    auto put = [&](int s, uint64_t v) {  // s: 0-based index among the 55
        val[(int64_t)s * n + i] = v;
        len[(int64_t)s * n + i] = (uint8_t)uleb_len(v);
    };
    // DC per channel: differences along the DFS order, first value raw
    for (int ch = 0; ch < 3; ch++) {
        const int64_t v = quant(ycocg[48 * k + 16 * ch], sf_sh);
        const int64_t p = kp >= 0 ? quant(ycocg[48 * kp + 16 * ch], sf_sh) : 0;
        put(ch, zigzag(v - p));
    }
    // AC: stream 3 + coef * 3 + ch holds coefficient coef + 1 of channel ch
    for (int coef = 0; coef < 15; coef++)
        for (int ch = 0; ch < 3; ch++)
            put(3 + coef * 3 + ch, zigzag(quant(ycocg[48 * k + 16 * ch + coef + 1], sf_sh)));
    put(48, (uint64_t)quant(opac[k], sf_op));  // astype(uint64), no zigzag
    for (int ax = 0; ax < 3; ax++) put(49 + ax, zigzag(quant(log_scales[3 * k + ax], sf_sc)));
    const double sgn = rot[4 * k] < 0.0 ? -1.0 : 1.0;  // _ensure_w_nonneg
    for (int ax = 0; ax < 3; ax++) put(52 + ax, zigzag(quant(rot[4 * k + 1 + ax] * sgn, sf_rot)));
}

__global__ void k_attr_len64(int64_t m, const uint8_t *__restrict__ len, int64_t *__restrict__ l64) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) l64[i] = len[i];
}

__global__ void k_attr_emit(int64_t m, const uint64_t *__restrict__ val,
                            const int64_t *__restrict__ off, uint8_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    int64_t o = off[i];
    uint64_t v = val[i];
    while (v > 0x7F) {
        out[o++] = (uint8_t)((v & 0x7F) | 0x80);
        v >>= 7;
    }
    out[o] = (uint8_t)v;
}

// ---------------------------------------------------------------------------

#define CODEC_CK(x)                          \
    do {                                     \
        cudaError_t _e = (x);                \
        if (_e != cudaSuccess) return _e;    \
    } while (0)

// Carves typed arrays out of one allocation.
struct Carver {
    char *base;
    size_t off = 0;
    template <typename T>
    T *take(int64_t count) {
        off = (off + 255) & ~(size_t)255;
        T *p = reinterpret_cast<T *>(base + off);
        off += sizeof(T) * (size_t)(count > 0 ? count : 1);
        return p;
    }
};

static size_t octree_scratch_bytes(int64_t n, int max_depth, size_t temp) {
    // khi klo (x2 for the sorts) idx x3 dtol tol lcp start gstart glcp gleaf gcount gbytes
    // goff mark seg occ, temp
    size_t b = 0;
    auto add = [&](size_t s) { b += ((s + 255) & ~(size_t)255) + 256; };
    add(8 * n), add(8 * n), add(8 * n), add(8 * n), add(8 * n);
    add(4 * n), add(4 * n), add(4 * n);
    add(n), add(8 * n), add(4 * n), add(n), add(4 * n), add(4 * n), add(n), add(4 * n);
    add(8 * n), add(8 * (n + 1)), add(4 * n), add(4 * n), add(4 * n * (size_t)max_depth), add(8);
    add(temp);
    return b;
}

cudaError_t run_octree(int64_t n, const double *pos, int neyes, const double *eyes_dev,
                       double beta, double gamma, const double *center, double half,
                       int max_depth, uint8_t *out, int64_t capacity, int64_t *out_len,
                       int64_t *order_out, void **scratch, size_t *scratch_cap,
                       int64_t *pinned, cudaStream_t st) {
    // scratch of the sorts and scans (sort.cu)
    size_t t1 = radix_sort_temp_bytes(n, 0, 36);
    const size_t t3 = scan_temp_bytes(n + 1);
    t1 = t1 > t3 ? t1 : t3;
    const size_t need = octree_scratch_bytes(n, max_depth, t1);
    if (*scratch_cap < need) {
        if (*scratch) cudaFree(*scratch);
        *scratch = nullptr;
        *scratch_cap = 0;
        CODEC_CK(cudaMalloc(scratch, need));
        *scratch_cap = need;
    }
    Carver cv{reinterpret_cast<char *>(*scratch)};
    uint64_t *khi = cv.take<uint64_t>(n), *klo = cv.take<uint64_t>(n);
    uint64_t *ka = cv.take<uint64_t>(n), *kb = cv.take<uint64_t>(n), *kc = cv.take<uint64_t>(n);
    int32_t *ia = cv.take<int32_t>(n), *ib = cv.take<int32_t>(n), *ic = cv.take<int32_t>(n);
    int8_t *dtol = cv.take<int8_t>(n);
    double *tol = cv.take<double>(n);
    int32_t *lcp = cv.take<int32_t>(n);
    uint8_t *start = cv.take<uint8_t>(n);
    int32_t *gstart = cv.take<int32_t>(n), *glcp = cv.take<int32_t>(n);
    int8_t *gleaf = cv.take<int8_t>(n);
    int32_t *gcount = cv.take<int32_t>(n);
    int64_t *gbytes = cv.take<int64_t>(n + 1), *goff = cv.take<int64_t>(n + 1);
    int32_t *mark = cv.take<int32_t>(n), *seg = cv.take<int32_t>(n);
    uint32_t *occ = cv.take<uint32_t>(n * (int64_t)max_depth);
    int32_t *ng_dev = cv.take<int32_t>(2);
    void *temp = cv.take<char>((int64_t)t1);

    k_oct_tol<<<blocks_for(n, 256), 256, 0, st>>>(n, pos, neyes, eyes_dev, beta, gamma, tol);
    k_oct_path<<<blocks_for(n, 256), 256, 0, st>>>(n, pos, tol, center[0], center[1], center[2],
                                                   half, max_depth, khi, klo, dtol, ia);
    CODEC_CK(cudaGetLastError());
    // stable sort by (hi, lo): by lo first, then stably by hi
    {
        CODEC_CK(cudaMemcpyAsync(ka, klo, 8 * n, cudaMemcpyDeviceToDevice, st));
        bool alt = false;
        CODEC_CK((radix_sort_pairs<uint64_t, int32_t>(temp, t1, ka, kb, ia, ib, n, 0, 36, false,
                                                      &alt, st)));
        int32_t *idx1 = alt ? ib : ia, *idx_free = alt ? ia : ib;
        k_gather_u64<<<blocks_for(n, 256), 256, 0, st>>>(n, idx1, khi, kc);
        CODEC_CK((radix_sort_pairs<uint64_t, int32_t>(temp, t1, kc, alt ? ka : kb, idx1,
                                                      idx_free, n, 0, 36, false, &alt, st)));
        int32_t *ord = alt ? idx_free : idx1;
        if (ord != ic) CODEC_CK(cudaMemcpyAsync(ic, ord, 4 * n, cudaMemcpyDeviceToDevice, st));
    }
    int32_t *order = ic;
    k_oct_lcp<<<blocks_for(n, 256), 256, 0, st>>>(n, order, khi, klo, max_depth, lcp, start);
    {
        k_iota32<<<blocks_for(n, 256), 256, 0, st>>>(n, mark);
        CODEC_CK(select_flagged_i32(temp, t1, mark, start, gstart, ng_dev, n, st));
    }
    int32_t ngh = 0;
    CODEC_CK(cudaMemcpyAsync(pinned, ng_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CODEC_CK(cudaStreamSynchronize(st));
    std::memcpy(&ngh, pinned, sizeof(int32_t));
    const int64_t ng = ngh;
    k_oct_leaf<<<blocks_for(ng, 256), 256, 0, st>>>(ng, n, gstart, lcp, order, khi, klo, dtol,
                                                    max_depth, glcp, gleaf, gcount, gbytes, occ);
    CODEC_CK(cudaGetLastError());
    for (int d = 0; d < max_depth; d++) {
        k_oct_mark<<<blocks_for(ng, 256), 256, 0, st>>>(ng, glcp, d, mark);
        CODEC_CK(inclusive_max_i32(temp, t1, mark, seg, ng, st));
        k_oct_branch<<<blocks_for(ng, 256), 256, 0, st>>>(ng, glcp, seg, d, gstart, order, khi,
                                                          klo, max_depth, occ);
    }
    {
        CODEC_CK(cudaMemsetAsync(gbytes + ng, 0, sizeof(int64_t), st));
        CODEC_CK(exclusive_sum_i64(temp, t1, gbytes, goff, ng + 1, st));
    }
    CODEC_CK(cudaMemcpyAsync(pinned, goff + ng, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CODEC_CK(cudaStreamSynchronize(st));
    *out_len = pinned[0];
    k_order_i64<<<blocks_for(n, 256), 256, 0, st>>>(n, order, order_out);
    if (out && capacity >= *out_len)
        k_oct_emit<<<blocks_for(ng, 256), 256, 0, st>>>(ng, glcp, gleaf, gcount, goff, occ,
                                                        max_depth, out);
    return cudaGetLastError();
}

cudaError_t run_attr_streams(int64_t n, const int64_t *order, const double *ycocg,
                             const double *opac, const double *log_scales, const double *rot,
                             double sf_sh, double sf_op, double sf_rot, double sf_sc, uint8_t *out,
                             int64_t capacity, int64_t *stream_lengths, void **scratch,
                             size_t *scratch_cap, int64_t *pinned, cudaStream_t st) {
    const int64_t m = (int64_t)kStreams * n;
    const size_t tb = scan_temp_bytes(m + 1);
    const size_t need = 8 * (size_t)m + (size_t)m + 8 * (size_t)(m + 1) * 2 + tb + 4096;
    if (*scratch_cap < need) {
        if (*scratch) cudaFree(*scratch);
        *scratch = nullptr;
        *scratch_cap = 0;
        CODEC_CK(cudaMalloc(scratch, need));
        *scratch_cap = need;
    }
    Carver cv{reinterpret_cast<char *>(*scratch)};
    uint64_t *val = cv.take<uint64_t>(m);
    uint8_t *len = cv.take<uint8_t>(m);
    int64_t *l64 = cv.take<int64_t>(m + 1);
    int64_t *off = cv.take<int64_t>(m + 1);
    void *temp = cv.take<char>((int64_t)tb);
    k_attr_values<<<blocks_for(n, 128), 128, 0, st>>>(n, order, ycocg, opac, log_scales, rot,
                                                      sf_sh, sf_op, sf_rot, sf_sc, val, len);
    k_attr_len64<<<blocks_for(m, 256), 256, 0, st>>>(m, len, l64);
    CODEC_CK(cudaMemsetAsync(l64 + m, 0, sizeof(int64_t), st));
    CODEC_CK(exclusive_sum_i64(temp, tb, l64, off, m + 1, st));
    // stream boundaries: off[s * n] for s = 0..55
    for (int s = 0; s <= kStreams; s++)
        CODEC_CK(cudaMemcpyAsync(pinned + s, off + (int64_t)s * n, sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, st));
    CODEC_CK(cudaStreamSynchronize(st));
    for (int s = 0; s < kStreams; s++) stream_lengths[s] = pinned[s + 1] - pinned[s];
    if (out && capacity >= pinned[kStreams])
        k_attr_emit<<<blocks_for(m, 256), 256, 0, st>>>(m, val, off, out);
    return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// Decode side (bitstream.py:169-220, :278; quantize.py:180-226).
//
// The octree stream is a preorder walk whose node boundaries are only known
// by parsing it (a node's size depends on its whole subtree), so it is
// decoded by a host loop in this library (one pass over a few MB).  The 55
// attribute streams are the data-parallel part: a byte ends a LEB128 value
// iff its top bit is clear, so an exclusive scan of those flags numbers every
// value, each terminating byte decodes its value from at most ten bytes back,
// the DC columns are prefix-summed (their delta coding), and one thread per
// splat dequantises, clamps the quaternions and converts YCoCg to RGB.

// quantize.py:69-76
static inline void child_center(const double *c, double h, int o, double *out) {
    const double off = h * 0.5;
    out[0] = c[0] + ((o & 4) ? off : -off);
    out[1] = c[1] + ((o & 2) ? off : -off);
    out[2] = c[2] + ((o & 1) ? off : -off);
}

namespace {
struct OctDecoder {
    const uint8_t *buf;
    int64_t len, pos = 0, count = 0, capacity;
    int max_depth;
    double *positions;
    int32_t *depths;
    int err = 0;  // OctDecodeError

    void read(const double *c, double h, int depth) {
        if (err) return;
        if (pos >= len) {
            err = kOctTruncated;
            return;
        }
        const uint8_t byte = buf[pos++];
        if (byte == 0x00) {
            // leaf: LEB128 count (varint.py _uleb_decode)
            uint64_t v = 0;
            int shift = 0;
            for (;;) {
                if (pos >= len) {
                    err = kOctTruncated;
                    return;
                }
                const uint8_t b = buf[pos++];
                if (shift < 64) v |= (uint64_t)(b & 0x7f) << shift;
                if (b < 0x80) break;
                shift += 7;
                if (shift > 63) {
                    err = kOctTruncated;  // overlong count (reported as truncated)
                    return;
                }
            }
            if ((int64_t)v < 1) {
                err = kOctZeroLeaf;
                return;
            }
            for (uint64_t i = 0; i < v; i++, count++) {
                if (count < capacity) {
                    positions[3 * count] = c[0];
                    positions[3 * count + 1] = c[1];
                    positions[3 * count + 2] = c[2];
                    depths[count] = depth;
                }
            }
            return;
        }
        if (depth >= max_depth) {
            err = kOctDepth;
            return;
        }
        for (int o = 0; o < 8; o++) {
            if (!(byte & (1 << o))) continue;
            double cc[3];
            child_center(c, h, o, cc);
            read(cc, h * 0.5, depth + 1);
            if (err) return;
        }
    }
};
}  // namespace

int octree_decode_host(const uint8_t *buf, int64_t len, const double *center, double half,
                       int max_depth, int64_t capacity, double *positions, int32_t *depths,
                       int64_t *count, int64_t *trailing) {
    OctDecoder d;
    d.buf = buf;
    d.len = len;
    d.capacity = capacity;
    d.max_depth = max_depth;
    d.positions = positions;
    d.depths = depths;
    d.read(center, half, 0);
    *count = d.count;
    *trailing = d.len - d.pos;
    if (d.err) return d.err;
    if (d.pos != d.len) return kOctTrailing;
    return 0;
}

__global__ void k_vflags(int64_t L, const uint8_t *__restrict__ b, int64_t *__restrict__ f) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < L) f[p] = b[p] < 0x80 ? 1 : 0;
}

// Every terminating byte decodes its value; the value's global index is the
// scan of terminators before it (stream s holds values s*n .. s*n + n-1 once
// every stream was checked to hold exactly n).
__global__ void k_vdecode(int64_t L, const uint8_t *__restrict__ b, const int64_t *__restrict__ ex,
                          const int64_t *__restrict__ sstart, int64_t n,
                          uint64_t *__restrict__ vals, int *__restrict__ overlong) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= L || b[p] >= 0x80) return;
    const int64_t g = ex[p];
    const int64_t s = g / n;
    const int64_t lo = sstart[s];
    int64_t q = p;
    while (q > lo && b[q - 1] >= 0x80 && p - q < 10) q--;
    if (p - q + 1 > 10 || (q > lo && b[q - 1] >= 0x80)) {
        atomicOr(overlong, 1);
        return;
    }
    uint64_t v = 0;
    for (int64_t j = q; j <= p; j++) v |= (uint64_t)(b[j] & 0x7f) << (7 * (j - q));
    vals[g] = v;
}

__device__ __forceinline__ int64_t zigzag_dec(uint64_t z) {
    return (int64_t)((z >> 1) ^ (0ull - (z & 1ull)));
}

__global__ void k_dc_zz(int64_t n, const uint64_t *__restrict__ vals, int64_t *__restrict__ dz) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * n) return;
    dz[i] = zigzag_dec(vals[i]);  // streams 1..3 are the first 3n values
}

// bitstream.py:169-220 for splat i.  Value v of attribute stream s (1..55)
// sits at vals[(s - 1) * n + i]; dc holds the DC columns' exclusive sums.
__global__ void k_attr_assemble(int64_t n, const uint64_t *__restrict__ vals,
                                const int64_t *__restrict__ dz, const int64_t *__restrict__ dcx,
                                double sf_sh, double sf_op, double sf_sc, double sf_rot,
                                double *__restrict__ sh, double *__restrict__ opac,
                                double *__restrict__ scales, double *__restrict__ rot,
                                unsigned long long *__restrict__ n_over) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const auto V = [&](int s) { return vals[(int64_t)(s - 1) * n + i]; };
    double yc[48];
    for (int ch = 0; ch < 3; ch++) {
        const int64_t cum = dcx[(int64_t)ch * n + i] + dz[(int64_t)ch * n + i];  // np.cumsum
        yc[ch * 16] = ((double)cum + 0.0) / sf_sh;
    }
    for (int coef = 0; coef < 15; coef++)
        for (int ch = 0; ch < 3; ch++)
            yc[ch * 16 + coef + 1] = ((double)zigzag_dec(V(4 + coef * 3 + ch)) + 0.0) / sf_sh;
    double o = ((double)(int64_t)V(49) + 0.25) / sf_op;
    o = o < 1e-9 ? 1e-9 : o;  // np.clip(opacities, 1e-9, 1 - 1e-9)
    o = o > 1.0 - 1e-9 ? 1.0 - 1e-9 : o;
    opac[i] = o;
    for (int a = 0; a < 3; a++)
        scales[3 * i + a] = exp(((double)zigzag_dec(V(50 + a)) + 0.0) / sf_sc);
    double x = ((double)zigzag_dec(V(53)) + 0.0) / sf_rot;
    double y = ((double)zigzag_dec(V(54)) + 0.0) / sf_rot;
    double z = ((double)zigzag_dec(V(55)) + 0.0) / sf_rot;
    double norm2 = (x * x + y * y) + z * z;
    if (norm2 > 1.0) {
        atomicAdd(n_over, 1ull);
        const double r = sqrt(norm2);
        x /= r, y /= r, z /= r;
        norm2 = 1.0;
    }
    const double w1 = 1.0 - norm2;
    rot[4 * i] = sqrt(w1 > 0.0 ? w1 : 0.0);
    rot[4 * i + 1] = x, rot[4 * i + 2] = y, rot[4 * i + 3] = z;
    // coeffs_ycocg_to_rgb (compaction.py:85-86): rgb_ic = sum_j M_ij yc_jc
    constexpr double M[9] = {1.0, 1.0, -1.0, 1.0, 0.0, 1.0, 1.0, -1.0, -1.0};
    for (int r = 0; r < 3; r++)
        for (int c = 0; c < 16; c++) {
            double acc = 0.0;
            for (int j = 0; j < 3; j++) acc += M[r * 3 + j] * yc[j * 16 + c];
            sh[48 * i + r * 16 + c] = acc;
        }
}

int run_attr_decode(int64_t n, const uint8_t *host_bytes, const int64_t *sstart_host,
                    double sf_sh, double sf_op, double sf_sc, double sf_rot, double *sh,
                    double *opac, double *scales, double *rot, int64_t *n_over, void **scratch,
                    size_t *scratch_cap, int64_t *pinned, cudaStream_t st, std::string *err) {
#define DEC_CK(x)                                                          \
    do {                                                                   \
        cudaError_t _e = (x);                                              \
        if (_e != cudaSuccess) {                                           \
            *err = std::string(#x) + ": " + cudaGetErrorString(_e);        \
            return kDecCuda;                                               \
        }                                                                  \
    } while (0)
    const int64_t L = sstart_host[kStreams];
    const int64_t m = (int64_t)kStreams * n;
    const size_t tb = scan_temp_bytes((L + 1) > 3 * n ? L + 1 : 3 * n);
    const size_t need = (size_t)L + 8 * (size_t)(L + 1) * 2 + 8 * (size_t)m +
                        8 * (size_t)(3 * n) * 2 + 8 * (kStreams + 1) + 16 + tb + 8 * 256;
    if (*scratch_cap < need) {
        if (*scratch) cudaFree(*scratch);
        *scratch = nullptr;
        *scratch_cap = 0;
        DEC_CK(cudaMalloc(scratch, need));
        *scratch_cap = need;
    }
    Carver cv{reinterpret_cast<char *>(*scratch)};
    uint8_t *bytes = cv.take<uint8_t>(L);
    int64_t *flag = cv.take<int64_t>(L + 1);
    int64_t *ex = cv.take<int64_t>(L + 1);
    uint64_t *vals = cv.take<uint64_t>(m);
    int64_t *dz = cv.take<int64_t>(3 * n);
    int64_t *dcx = cv.take<int64_t>(3 * n);
    int64_t *sstart = cv.take<int64_t>(kStreams + 1);
    int *flags = cv.take<int>(4);
    unsigned long long *over = reinterpret_cast<unsigned long long *>(cv.take<int64_t>(1));
    void *temp = cv.take<char>((int64_t)tb);
    DEC_CK(cudaMemcpyAsync(bytes, host_bytes, (size_t)L, cudaMemcpyHostToDevice, st));
    DEC_CK(cudaMemcpyAsync(sstart, sstart_host, sizeof(int64_t) * (kStreams + 1),
                           cudaMemcpyHostToDevice, st));
    DEC_CK(cudaMemsetAsync(flags, 0, 4 * sizeof(int), st));
    DEC_CK(cudaMemsetAsync(over, 0, sizeof(unsigned long long), st));
    k_vflags<<<blocks_for(L, 256), 256, 0, st>>>(L, bytes, flag);
    DEC_CK(cudaMemsetAsync(flag + L, 0, sizeof(int64_t), st));
    DEC_CK(exclusive_sum_i64(temp, tb, flag, ex, L + 1, st));
    // values per stream: the scan at the stream boundaries
    for (int s = 0; s <= kStreams; s++)
        DEC_CK(cudaMemcpyAsync(pinned + s, ex + sstart_host[s], sizeof(int64_t),
                               cudaMemcpyDeviceToHost, st));
    DEC_CK(cudaStreamSynchronize(st));
    for (int s = 0; s < kStreams; s++) {
        const int64_t cnt = pinned[s + 1] - pinned[s];
        const int64_t slen = sstart_host[s + 1] - sstart_host[s];
        const bool ends = slen > 0 && host_bytes[sstart_host[s + 1] - 1] < 0x80;
        if (cnt < n || (cnt == n && !ends)) {  // fewer than n complete values
            *err = "truncated varint stream (attribute stream " + std::to_string(s + 1) + ")";
            return kDecTruncated;
        }
        if (cnt > n || !ends) {
            *err = std::to_string(s + 1);  // the stream id; the caller names it
            return kDecTrailing;
        }
    }
    k_vdecode<<<blocks_for(L, 256), 256, 0, st>>>(L, bytes, ex, sstart, n, vals, flags);
    k_dc_zz<<<blocks_for(3 * n, 256), 256, 0, st>>>(n, vals, dz);
    for (int ch = 0; ch < 3; ch++)
        DEC_CK(exclusive_sum_i64(temp, tb, dz + (int64_t)ch * n, dcx + (int64_t)ch * n, n, st));
    k_attr_assemble<<<blocks_for(n, 128), 128, 0, st>>>(n, vals, dz, dcx, sf_sh, sf_op, sf_sc,
                                                        sf_rot, sh, opac, scales, rot, over);
    DEC_CK(cudaGetLastError());
    DEC_CK(cudaMemcpyAsync(pinned, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    DEC_CK(cudaMemcpyAsync(pinned + 1, over, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           st));
    DEC_CK(cudaStreamSynchronize(st));
    int ov = 0;
    std::memcpy(&ov, pinned, sizeof(int));
    if (ov) {
        *err = "overlong varint";
        return kDecOverlong;
    }
    *n_over = pinned[1];
    return 0;
#undef DEC_CK
}


}  // namespace potr
