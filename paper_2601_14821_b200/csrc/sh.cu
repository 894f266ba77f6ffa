// sh.cu -- kernel (e): training-free SH recompute (compaction.py:89-243).
//
// The reference builds, per splat, Y = basis * w and C = YCoCg(basis . sh^T) * w
// over the cameras that see it (compaction.py:89-107) and then only ever uses
// Y^T Y and Y^T C (sparsify :110-124, ridge :127-148).  So the GPU never
// materialises Y: k_sh_accumulate streams the (S, N) per-camera importances
// once and accumulates, per splat, the 16x16 Gram matrix G (136 unique
// entries) and the 16x3 right-hand sides B in fp64 registers (a warp per
// splat, each lane owning ~6 of the 184 entries) in camera order with fused
// multiply-adds -- the oracle restates the same order, so the two agree bit
// for bit; the reference's BLAS dgemm differs by rounding (tests: 1e-9).  k_sh_solve then does the
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

// Normal equations of kShSplatsPerBlock consecutive splats per CTA (each warp
// takes its splats one at a time).  Views are taken 32 at a time: the (view,
// splat) tile of camera_importance is staged in shared memory with coalesced
// loads; then for one splat each lane evaluates one view
// (direction, SH basis, raw colour, YCoCg -- compaction.py:100-107) and
// publishes the rows a = (w*y (16), 0, 0, w*YCoCg(colour) (3), 0...) to shared
// memory.  The wanted entries of sum_v a a^T -- G_ij (i <= j < 16) and B_ic =
// sum a_i a_18+c -- come from the fp64 tensor cores: per splat and per four
// of its seen views (ascending), five mma.m8n8k4 (G rows 0-7 x cols 0-7, 0-7
// x 8-15, 8-15 x 8-15; B rows 0-7 and 8-15 x row entries 16-23), whose A and
// B fragments are the same three shared loads per lane.  The fp64 MMA rounds
// exactly as a chain of fused multiply-adds in k order (tools/dmma_check.cu:
// 4.2M of 4.2M entries equal), so every entry is the same fma chain over the
// splat's seen views, in ascending view order, as the oracle's -- bit for bit.
// A step short of four views pads with the zero row: fma(0, 0, acc) == acc
// exactly (acc is never -0).  Views a splat is not seen from (w = 0) are
// skipped: they would add exact zeros, so the sums equal the reference's
// sums over its `seen` rows (compaction.py:97-107, :114, :133-137).
// 4 splats per 4-warp CTA, 6 CTAs per SM (<= 85 registers, no spills):
// 25.8 ms at C4 (16 per CTA at 3 per SM: 32.9; 8 at 4: 28.8; a spill of even
// 20 bytes at 7 per SM: 36.1)
#ifndef POTR_SH_MIN_BLOCKS
#define POTR_SH_MIN_BLOCKS 6
#endif
#ifndef POTR_SH_SPLATS
#define POTR_SH_SPLATS 4
#endif
constexpr int kShSplatsPerBlock = POTR_SH_SPLATS;
#ifndef POTR_SH_WARPS
#define POTR_SH_WARPS 4
#endif
constexpr int kShWarps = POTR_SH_WARPS;
// Row layout: w*y at 0..15, w*YCoCg at 18..20, zeros at 16, 17, 21..24.  The
// odd stride keeps the 16 rows a half-warp stores per instruction on distinct
// banks; 25 >= 24 so the B fragments' entries 16..23 stay inside the row.
constexpr int kShRow = 25;
constexpr int kShYc = 18;

// Entry index of (i, j), j >= i, in the (185, N) layout: G upper triangle
// then B (136 + 3 i + c, row entry j = 18 + c); -1 outside the wanted region.
__device__ __forceinline__ int sh_entry(int i, int j) {
    if (j < i) return -1;
    if (j < 16) return i * 16 - (i * (i - 1)) / 2 + (j - i);
    if (j >= kShYc && j < kShYc + 3) return 136 + 3 * i + (j - kShYc);
    return -1;
}

// D += A B on the fp64 tensor cores, one m8n8k4 tile: A fragment a (row
// lane/4, col lane%4), B fragment b (row lane%4, col lane/4), C/D (row lane/4,
// cols 2 (lane%4) + {0, 1}).
__device__ __forceinline__ void dmma_acc(double (&d)[2], double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

// kAdd: add into normal_eqs (potr_sh_accumulate); else overwrite it
// (potr_sh_normal_equations: no read of the old values, no zeroing pass).
//
// Views are taken kShWin at a time: the window's (view, splat) tile of
// camera_importance is staged in shared memory, then each warp lists its
// splat's SEEN views of the window (ascending) and evaluates them 32 at a
// time, lane j the j-th seen view -- every lane busy, where a lane per view
// idled on the ~26% of (splat, view) pairs with w = 0 -- and the MMAs take
// the rows in list order, which is ascending view order: the same fma chain
// per entry as before.
#ifndef POTR_SH_WIN
#define POTR_SH_WIN 128
#endif
constexpr int kShWin = POTR_SH_WIN;

template <bool kAdd>
__global__ void __launch_bounds__(32 * kShWarps, POTR_SH_MIN_BLOCKS)
    k_sh_accumulate(potr_splats sp, int ncam, const double *__restrict__ eyes,
                    const double *__restrict__ cam_imp, double *__restrict__ neq) {
    __shared__ double wwin[kShWin][kShSplatsPerBlock + 1];
    __shared__ uint8_t seen_v[kShWarps][kShWin];  // a warp's seen views of the window
    // per warp: 32 rows + a zero row (a step short of four views pads with
    // it: fma(0, 0, acc) == acc exactly, acc is never -0)
    extern __shared__ __align__(16) double sh_dyn[];
    double(*A)[33][kShRow] = reinterpret_cast<double(*)[33][kShRow]>(sh_dyn);
    __shared__ double shs[kShSplatsPerBlock][48];
    __shared__ double pos[kShSplatsPerBlock][3];
    static_assert(kShWin <= 256, "window views index as bytes");
    const int64_t n = sp.n;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t k0 = (int64_t)blockIdx.x * kShSplatsPerBlock;
    const int nk = (int)(n - k0 < kShSplatsPerBlock ? n - k0 : kShSplatsPerBlock);
    for (int i = threadIdx.x; i < nk * 48; i += blockDim.x)
        shs[i / 48][i % 48] = sp.sh[(k0 + i / 48) * 48 + i % 48];
    for (int i = threadIdx.x; i < nk * 3; i += blockDim.x)
        pos[i / 3][i % 3] = sp.positions[(k0 + i / 3) * 3 + i % 3];
    for (int i = threadIdx.x; i < kShWarps * 33 * kShRow; i += blockDim.x)
        (&A[0][0][0])[i] = 0.0;  // the pad columns and the zero row stay zero

    constexpr int kPerWarp = kShSplatsPerBlock / kShWarps;  // splats of this warp
    // per splat: five 8x8 fp64 MMA accumulators (G00, G01, G11, B0, B1), two
    // doubles per lane each
    double acc[kPerWarp][5][2];
    int seen[kPerWarp];
#pragma unroll
    for (int q = 0; q < kPerWarp; q++) {
        seen[q] = 0;
#pragma unroll
        for (int t = 0; t < 5; t++) acc[q][t][0] = acc[q][t][1] = 0.0;
    }
    const double(*rows)[kShRow] = A[w];
    const unsigned lt = (1u << lane) - 1u;
    for (int s0 = 0; s0 < ncam; s0 += kShWin) {
        const int nv = ncam - s0 < kShWin ? ncam - s0 : kShWin;
        __syncthreads();  // previous window done with wwin; first: sh / pos staged
        for (int i = threadIdx.x; i < nv * kShSplatsPerBlock; i += blockDim.x) {
            const int v = i / kShSplatsPerBlock, kk = i % kShSplatsPerBlock;
            wwin[v][kk] = kk < nk ? cam_imp[(int64_t)(s0 + v) * n + k0 + kk] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kPerWarp; q++) {
            const int kk = w * kPerWarp + q;
            if (kk >= nk) break;  // warp-uniform
            // the splat's seen views of the window, ascending
            int cnt = 0;
            for (int vb = 0; vb < nv; vb += 32) {
                const int v = vb + lane;
                const bool sv = v < nv && wwin[v][kk] > 0.0;
                const unsigned b = __ballot_sync(0xffffffffu, sv);
                if (sv) seen_v[w][cnt + __popc(b & lt)] = (uint8_t)v;
                cnt += __popc(b);
            }
            seen[q] += cnt;
            __syncwarp();
            for (int r0 = 0; r0 < cnt; r0 += 32) {  // warp-uniform
                const int nr = cnt - r0 < 32 ? cnt - r0 : 32;
                if (lane < nr) {
                    const int v = seen_v[w][r0 + lane];
                    const double wv = wwin[v][kk];
                    const double *eye = eyes + 3 * (s0 + v);
                    double *row = A[w][lane];
                    const double d0 = pos[kk][0] - __ldg(eye), d1 = pos[kk][1] - __ldg(eye + 1),
                                 d2 = pos[kk][2] - __ldg(eye + 2);
                    const double nrm = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
                    double y[16];
                    sh_basis16(d0 / nrm, d1 / nrm, d2 / nrm, y);
                    // colors = basis @ sh^T (compaction.py:104): fused
                    // multiply-adds in two interleaved partial sums (the
                    // oracle's order; a 16-deep add chain was the largest stall)
                    double col[3];
#pragma unroll
                    for (int c = 0; c < 3; c++) {
                        double a0 = 0.0, a1 = 0.0;
#pragma unroll
                        for (int i = 0; i < 16; i += 2) {
                            a0 = fma(y[i], shs[kk][c * 16 + i], a0);
                            a1 = fma(y[i + 1], shs[kk][c * 16 + i + 1], a1);
                        }
                        col[c] = a0 + a1;
                    }
#pragma unroll
                    for (int i = 0; i < 16; i++) row[i] = y[i] * wv;
#pragma unroll
                    for (int c = 0; c < 3; c++) {
                        const double yc = col[0] * kRgbToYcocg[c * 3] +
                                          col[1] * kRgbToYcocg[c * 3 + 1] +
                                          col[2] * kRgbToYcocg[c * 3 + 2];
                        row[kShYc + c] = yc * wv;
                    }
                }
                __syncwarp();
                // rows 0..nr-1 four at a time (ascending views); lane l loads
                // entries l/4, 8 + l/4, 16 + l/4 of row 4u + l%4 (the zero row
                // past nr)
                for (int u = 0; u < nr; u += 4) {
                    const int rr = u + (lane & 3);
                    const double *row = rows[rr < nr ? rr : 32];
                    const int r = lane >> 2;
                    const double x0 = row[r], x1 = row[8 + r], x2 = row[16 + r];
                    dmma_acc(acc[q][0], x0, x0);
                    dmma_acc(acc[q][1], x0, x1);
                    dmma_acc(acc[q][2], x1, x1);
                    dmma_acc(acc[q][3], x0, x2);
                    dmma_acc(acc[q][4], x1, x2);
                }
                __syncwarp();
            }
        }
    }
    // tile t's block of rows / columns: G00 (0, 0), G01 (0, 8), G11 (8, 8),
    // B0 (0, 16), B1 (8, 16); lane l holds row l/4, columns 2 (l%4) + {0, 1}
    constexpr int kTileRow[5] = {0, 0, 8, 0, 8}, kTileCol[5] = {0, 8, 8, 16, 16};
#pragma unroll
    for (int q = 0; q < kPerWarp; q++) {
        const int kk = w * kPerWarp + q;
        if (kk >= nk) continue;  // warp-uniform
        const int64_t k = k0 + kk;
        // all reads issue before the first write (one latency, not ten)
        int e[5][2];
        double old[5][2];
#pragma unroll
        for (int t = 0; t < 5; t++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
                e[t][h] = sh_entry(kTileRow[t] + (lane >> 2), kTileCol[t] + 2 * (lane & 3) + h);
                old[t][h] = kAdd && e[t][h] >= 0 ? neq[(int64_t)e[t][h] * n + k] : 0.0;
            }
#pragma unroll
        for (int t = 0; t < 5; t++)
#pragma unroll
            for (int h = 0; h < 2; h++)
                if (e[t][h] >= 0)
                    neq[(int64_t)e[t][h] * n + k] = kAdd ? old[t][h] + acc[q][t][h] : acc[q][t][h];
        if (lane == 0) {
            if (kAdd) neq[(int64_t)184 * n + k] += (double)seen[q];
            else neq[(int64_t)184 * n + k] = (double)seen[q];
        }
    }
}

// Upper Cholesky of the m x m principal block, packed with tri() (LAPACK
// dpotrf 'U' semantics: a pivot <= 0 or NaN fails).  S: the stride between
// packed entries (1 in local memory; the block size for a thread's slice of a
// shared-memory array, [entry][thread], so a warp's accesses hit 32 banks).
template <int S = 1>
__device__ int chol_upper(double *A, int m) {
    for (int j = 0; j < m; j++) {
        double ajj = A[tri(j, j) * S];
        for (int k = 0; k < j; k++) ajj -= A[tri(k, j) * S] * A[tri(k, j) * S];
        if (!(ajj > 0.0)) return j + 1;
        ajj = sqrt(ajj);
        A[tri(j, j) * S] = ajj;
        for (int c = j + 1; c < m; c++) {
            double v = A[tri(j, c) * S];
            for (int k = 0; k < j; k++) v -= A[tri(k, j) * S] * A[tri(k, c) * S];
            A[tri(j, c) * S] = v / ajj;
        }
    }
    return 0;
}

// dpotrs: U^T y = b, U x = y
template <int S = 1>
__device__ void chol_solve(const double *U, int m, double *b) {
    for (int i = 0; i < m; i++) {
        double v = b[i];
        for (int k = 0; k < i; k++) v -= U[tri(k, i) * S] * b[k];
        b[i] = v / U[tri(i, i) * S];
    }
    for (int i = m - 1; i >= 0; i--) {
        double v = b[i];
        for (int k = i + 1; k < m; k++) v -= U[tri(i, k) * S] * b[k];
        b[i] = v / U[tri(i, i) * S];
    }
}

// _solve_channel (compaction.py:127-148) on the normal equations, split into
// the factorisation of A = G[c, c] + lam I (no lam on DC) and the solve for one
// channel's right-hand side, so channels that share (mask, lam) share the
// factor.  factor_channel returns 0 ok, 1 ok after the 1e-10 jitter, -1
// RidgeError; the retry rebuilds A from G (the same values the reference's
// retry starts from).
template <int S = 1>
__device__ int factor_channel(const double *__restrict__ G, int64_t gs, unsigned mask, double lam,
                              double *A, int *cols, int *mout) {
    int m = 0;
    for (int i = 0; i < 16; i++)
        if (mask >> i & 1u) cols[m++] = i;
    *mout = m;
    for (int attempt = 0; attempt < 2; attempt++) {
        for (int i = 0; i < m; i++) {
            for (int j = i; j < m; j++) A[tri(i, j) * S] = __ldg(G + tri(cols[i], cols[j]) * gs);
            A[tri(i, i) * S] += (cols[i] == 0) ? 0.0 : lam;
            if (attempt) A[tri(i, i) * S] += 1e-10;
        }
        if (!chol_upper<S>(A, m)) return attempt;
    }
    return -1;
}

template <int S = 1>
__device__ void solve_factored(const double *A, int m, const int *cols,
                               const double *__restrict__ B, int64_t gs, int ch, double *out) {
    double b[16];
    for (int i = 0; i < m; i++) b[i] = __ldg(B + (cols[i] * 3 + ch) * gs);
    chol_solve<S>(A, m, b);
    for (int i = 0; i < 16; i++) out[i] = 0.0;
    for (int i = 0; i < m; i++) out[cols[i]] = b[i];
}

// pass-2 mask: drop AC columns whose pass-1 coefficient is below the threshold
__device__ unsigned pass2_mask(unsigned mask, const double *first, double zero_thr) {
    unsigned m2 = mask;
    for (int i = 1; i < 16; i++)
        if (fabs(first[i]) < zero_thr) m2 &= ~(1u << i);
    return m2;
}

__device__ void coeffs_convert(const double *M, const double *in, double *out) {
    for (int i = 0; i < 3; i++)
        for (int c = 0; c < 16; c++) {
            double acc = 0.0;
            for (int j = 0; j < 3; j++) acc += M[i * 3 + j] * in[j * 16 + c];
            out[i * 16 + c] = acc;
        }
}

// ---------------------------------------------------------------------------
// The solves.  k_sh_mask first runs the parallel-column sparsification of
// every splat (compaction.py:110-124) and files the splat under the size of
// its kept set: the factor of every later system of the splat (pass 1 and
// pass 2 of the three channels, masks that are subsets of the kept set) has
// at most that many columns.  Each size class is then solved by a kernel
// whose factor lives in registers, fully unrolled for its capacity
// (k_sh_solve_reg<8>: 74% of the C3 splats, <12>: 23%); the rare larger
// systems run k_sh_solve_smem (each thread's factor in shared memory) and the
// unseen splats' DC fallback the generic kernel.  Results do not depend on the class order: every
// splat is solved independently, with the oracle's operation order
// (potr_oracle.c chol_upper / chol_solve_upper / compact_one).

// The kept set of one splat (G entries read in place from the (185, N) layout).
__device__ unsigned sparsify_mask(const double *__restrict__ G, int64_t gs, double par_thr) {
    double norms[16];
#pragma unroll
    for (int i = 0; i < 16; i++) norms[i] = sqrt(__ldg(G + tri(i, i) * gs));
    unsigned mask = 1u;
#pragma unroll
    for (int i = 1; i < 16; i++) {
        // column i's entries against the earlier columns, loaded together
        // (independent loads; the kept-set test below picks what it needs)
        double g[15];
#pragma unroll
        for (int j = 0; j < i; j++) g[j] = __ldg(G + tri(j, i) * gs);  // j < i
        if (norms[i] == 0.0) continue;
        bool par = false;
#pragma unroll
        for (int j = 0; j < i; j++) {
            if (!(mask >> j & 1u)) continue;
            const double cs = fabs(g[j]) / (norms[i] * norms[j]);
            if (cs > par_thr) par = true;
        }
        if (!par) mask |= 1u << i;
    }
    return mask;
}

// 0: unseen, 1: <= 8 columns, 2: <= 12, 3: <= 16, 4: <= 10
constexpr int kSolveClasses = 5;
__device__ __forceinline__ int solve_class(unsigned mask) {
    const int m = __popc(mask);
    return m <= 8 ? 1 : m <= 10 ? 4 : m <= 12 ? 2 : 3;
}

__global__ void __launch_bounds__(128) k_sh_mask(int64_t n, const double *__restrict__ neq,
                                                 double par_thr, uint16_t *__restrict__ masks,
                                                 int *__restrict__ counts,
                                                 int32_t *__restrict__ lists) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int cls = -1;
    if (k < n) {
        unsigned mask = 0u;
        if (neq[(int64_t)184 * n + k] == 0.0) {
            cls = 0;
        } else {
            mask = sparsify_mask(neq + k, n, par_thr);
            cls = solve_class(mask);
        }
        masks[k] = (uint16_t)mask;
    }
    // warp-aggregated append to the class lists (order is irrelevant: the
    // splats are solved independently)
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < kSolveClasses; c++) {
        const unsigned peers = __ballot_sync(0xffffffffu, cls == c);
        if (!peers) continue;
        int base = 0;
        if (lane == __ffs(peers) - 1) base = atomicAdd(&counts[c], __popc(peers));
        base = __shfl_sync(0xffffffffu, base, __ffs(peers) - 1);
        if (cls == c) lists[(int64_t)c * n + base + __popc(peers & ((1u << lane) - 1u))] = (int32_t)k;
    }
}

// Final (YCoCg -> RGB) or failed (original coefficients) outputs.
__device__ void finish_splat(int status, const double *sh, double *rgb, double *yc) {
    if (status == 2) {
        for (int i = 0; i < 48; i++) rgb[i] = sh[i];
        coeffs_convert(kRgbToYcocg, rgb, yc);
    } else {
        coeffs_convert(kYcocgToRgb, yc, rgb);
    }
}

// --- register-resident solves, capacity MC columns ---------------------------

template <int MC>
__device__ __forceinline__ constexpr int trm(int i, int j) {  // packed upper, row-major
    return i * MC - (i * (i - 1)) / 2 + (j - i);
}

// Register-resident factor / solve of the kept m x m system, capacity MC.
// kPadMC: for MC > 8 the system is padded to MC with identity rows / columns
// and the factorisation runs branch free over all MC columns (the factor is
// blockdiag(chol(A_m), I): its leading block gets exactly the operations, in
// the same order, of an m x m factorisation -- the padded terms add or
// subtract exact zeros after the real ones).  No index then depends on m and
// the 12-column factor stays in registers; with the m-guarded loops it went
// to local memory.  For MC <= 8 the guarded loops already stay in registers
// and do less work.
template <int MC>
constexpr bool kPadMC = MC > 8;

// Upper Cholesky (dpotrf 'U' semantics), fully unrolled.  Returns false when a
// real pivot is <= 0 or NaN (padded pivots are 1).
template <int MC>
__device__ __forceinline__ bool chol_reg(double (&U)[MC * (MC + 1) / 2], int m) {
    bool ok = true;
#pragma unroll
    for (int j = 0; j < MC; j++) {
        if (kPadMC<MC> || j < m) {
            double ajj = U[trm<MC>(j, j)];
#pragma unroll
            for (int k = 0; k < j; k++) ajj -= U[trm<MC>(k, j)] * U[trm<MC>(k, j)];
            ok = ok && ajj > 0.0;
            ajj = sqrt(ajj);
            U[trm<MC>(j, j)] = ajj;
#pragma unroll
            for (int c = j + 1; c < MC; c++) {
                if (kPadMC<MC> || c < m) {
                    double v = U[trm<MC>(j, c)];
#pragma unroll
                    for (int k = 0; k < j; k++) v -= U[trm<MC>(k, j)] * U[trm<MC>(k, c)];
                    U[trm<MC>(j, c)] = v / ajj;
                }
            }
        }
    }
    return ok;
}

// dpotrs on the register factor: U^T y = b, U x = y (padded entries of b are
// zero and stay zero).
template <int MC>
__device__ __forceinline__ void chol_solve_reg(const double (&U)[MC * (MC + 1) / 2], int m,
                                               double (&b)[MC]) {
#pragma unroll
    for (int i = 0; i < MC; i++) {
        if (kPadMC<MC> || i < m) {
            double v = b[i];
#pragma unroll
            for (int k = 0; k < i; k++) v -= U[trm<MC>(k, i)] * b[k];
            b[i] = v / U[trm<MC>(i, i)];
        }
    }
#pragma unroll
    for (int i = MC - 1; i >= 0; i--) {
        if (kPadMC<MC> || i < m) {
            double v = b[i];
#pragma unroll
            for (int k = i + 1; k < MC; k++)
                if (kPadMC<MC> || k < m) v -= U[trm<MC>(i, k)] * b[k];
            b[i] = v / U[trm<MC>(i, i)];
        }
    }
}

template <int MC>
__global__ void __launch_bounds__(128, MC <= 8 ? 4 : 2)
    k_sh_solve_reg(potr_splats sp, const double *__restrict__ neq,
                   const uint16_t *__restrict__ masks, const int32_t *__restrict__ list,
                   const int *__restrict__ count, double lambda_y, double zero_thr,
                   double *rgb_out, double *ycocg_out, int8_t *__restrict__ status_out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= *count) return;
    const int64_t n = sp.n;
    const int64_t k = list[t];
    POTR_CHECK(k >= 0 && k < n);
    const double *G = neq + k, *B = neq + (int64_t)136 * n + k;
    const unsigned mask1 = masks[k];
    POTR_CHECK(__popc(mask1) <= MC);
    double *yc = ycocg_out + 48 * k;
    double U[MC * (MC + 1) / 2];
    double b[MC];
    int cols[MC];
    // compact_splat (:169-192) as five factor/solve tasks: Y pass 1 (lambda),
    // Y pass 2, Co+Cg pass 1 (3 lambda, one factor, two right-hand sides),
    // Co pass 2, Cg pass 2.  A RidgeError anywhere keeps the original
    // coefficients, so Cg's pass 1 before Co's pass 2 changes no output.
    unsigned drop0 = 0u, drop1 = 0u, drop2 = 0u;
    int status = 0;
#pragma unroll 1
    for (int task = 0; task < 5; task++) {
        const unsigned mask = task == 0 || task == 2 ? mask1
                              : mask1 & ~(task == 1 ? drop0 : task == 3 ? drop1 : drop2);
        const double lam = task < 2 ? lambda_y : 3.0 * lambda_y;
        const int m = __popc(mask);
        unsigned mm = mask;
#pragma unroll
        for (int i = 0; i < MC; i++) {
            cols[i] = mm ? __ffs(mm) - 1 : 0;
            mm &= mm - 1u;
        }
        // the m x m system (padded to MC with identity rows / columns when
        // kPadMC); the 1e-10 jitter retry (compaction.py:138-145) is the rare
        // second call
        auto factor = [&](bool jitter) {
#pragma unroll
            for (int i = 0; i < MC; i++)
#pragma unroll
                for (int j = i; j < MC; j++) {
                    if (j < m)
                        U[trm<MC>(i, j)] = __ldg(G + tri(cols[i], cols[j]) * n);
                    else if (kPadMC<MC>)
                        U[trm<MC>(i, j)] = i == j ? 1.0 : 0.0;
                }
#pragma unroll
            for (int i = 0; i < MC; i++) {
                if (i < m) {
                    U[trm<MC>(i, i)] += (cols[i] == 0) ? 0.0 : lam;
                    if (jitter) U[trm<MC>(i, i)] += 1e-10;
                }
            }
            return chol_reg<MC>(U, m);
        };
        int rc = 0;
        if (!factor(false)) rc = factor(true) ? 1 : -1;
        if (rc < 0) {
            status = 2;
            break;
        }
        status |= rc;
#pragma unroll 1
        for (int r = 0; r < (task == 2 ? 2 : 1); r++) {
            const int ch = task < 2 ? 0 : task == 2 ? 1 + r : task - 2;
#pragma unroll
            for (int i = 0; i < MC; i++) b[i] = i < m ? __ldg(B + (cols[i] * 3 + ch) * n) : 0.0;
            chol_solve_reg<MC>(U, m, b);
            if (task == 1 || task >= 3) {
                for (int i = 0; i < 16; i++) yc[ch * 16 + i] = 0.0;
#pragma unroll
                for (int i = 0; i < MC; i++)
                    if (i < m) yc[ch * 16 + cols[i]] = b[i];
            } else {
                unsigned d = 0u;
#pragma unroll
                for (int i = 0; i < MC; i++)
                    if (i < m && cols[i] > 0 && fabs(b[i]) < zero_thr) d |= 1u << cols[i];
                if (task == 0) drop0 = d;
                else if (r == 0) drop1 = d;
                else drop2 = d;
            }
        }
    }
    finish_splat(status, sp.sh + 48 * k, rgb_out + 48 * k, yc);
    status_out[k] = (int8_t)status;
}

// The three channels of a seen splat (compact_splat, compaction.py:169-192)
// with the packed factor at A (stride S); writes yc, returns the status.
template <int S>
__device__ int solve_seen(const double *__restrict__ neq, int64_t n, int64_t k, unsigned mask,
                          double lambda_y, double zero_thr, double *A, double *yc) {
    const double *G = neq + k, *B = neq + (int64_t)136 * n + k;
    double first[16], first2[16];
    int cols[16], m, rc;
    int status = 0;
    for (int ch = 0; ch < 3 && status != 2; ch++) {
        if (ch < 2) {
            rc = factor_channel<S>(G, n, mask, ch == 0 ? lambda_y : 3.0 * lambda_y, A, cols, &m);
            if (rc < 0) {
                status = 2;
                break;
            }
            if (rc > 0) status = 1;
            solve_factored<S>(A, m, cols, B, n, ch, first);
            if (ch == 1) solve_factored<S>(A, m, cols, B, n, 2, first2);
        } else {
            for (int i = 0; i < 16; i++) first[i] = first2[i];
        }
        rc = factor_channel<S>(G, n, pass2_mask(mask, first, zero_thr),
                               ch == 0 ? lambda_y : 3.0 * lambda_y, A, cols, &m);
        if (rc < 0) {
            status = 2;
            break;
        }
        if (rc > 0) status = 1;
        solve_factored<S>(A, m, cols, B, n, ch, yc + ch * 16);
    }
    return status;
}

// --- the generic solve (any size; unseen splats' DC fallback) ----------------

__global__ void __launch_bounds__(128) k_sh_solve(potr_splats sp, const double *__restrict__ neq,
                                                  const uint16_t *__restrict__ masks,
                                                  const int32_t *__restrict__ list,
                                                  const int *__restrict__ count,
                                                  double lambda_y, double zero_thr,
                                                  double *rgb_out, double *ycocg_out,
                                                  int8_t *__restrict__ status_out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= *count) return;
    const int64_t n = sp.n;
    const int64_t k = list[t];
    const double *sh = sp.sh + 48 * k;
    double *rgb = rgb_out + 48 * k, *yc = ycocg_out + 48 * k;
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
                        for (int t2 = 0; t2 < 16; t2++) col += basis[t2] * sh[c * 16 + t2];
                        acc[c] += col;
                    }
                }
        for (int i = 0; i < 48; i++) rgb[i] = 0.0;
        for (int c = 0; c < 3; c++) rgb[c * 16] = acc[c] / 26.0 / kShDC;
        coeffs_convert(kRgbToYcocg, rgb, yc);
        status = 3;
    } else {
        double Af[136];
        status = solve_seen<1>(neq, n, k, masks[k], lambda_y, zero_thr, Af, yc);
        finish_splat(status, sh, rgb, yc);
    }
    status_out[k] = (int8_t)status;
}

// The large kept sets (> 12 columns, ~3% of the C3 splats): the generic solve
// with each thread's packed factor in shared memory ([entry][thread]) instead
// of local memory, persistent over the class list.
constexpr int kShSmemThreads = 64;
__global__ void __launch_bounds__(kShSmemThreads) k_sh_solve_smem(
    potr_splats sp, const double *__restrict__ neq, const uint16_t *__restrict__ masks,
    const int32_t *__restrict__ list, const int *__restrict__ count, double lambda_y,
    double zero_thr, double *rgb_out, double *ycocg_out, int8_t *__restrict__ status_out) {
    extern __shared__ double af_s[];  // [136][kShSmemThreads]
    const int64_t n = sp.n;
    const int cnt = *count;
    for (int t = blockIdx.x * kShSmemThreads + threadIdx.x; t < cnt;
         t += gridDim.x * kShSmemThreads) {
        const int64_t k = list[t];
        POTR_CHECK(k >= 0 && k < n);
        double *yc = ycocg_out + 48 * k;
        const int status = solve_seen<kShSmemThreads>(neq, n, k, masks[k], lambda_y, zero_thr,
                                                      af_s + threadIdx.x, yc);
        finish_splat(status, sp.sh + 48 * k, rgb_out + 48 * k, yc);
        status_out[k] = (int8_t)status;
    }
}

cudaError_t launch_sh_accumulate(const potr_splats &sp, int ncam, const double *eyes_dev,
                                 const double *cam_imp, double *neq, bool add, cudaStream_t st) {
    if (sp.n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((sp.n + kShSplatsPerBlock - 1) / kShSplatsPerBlock);
    constexpr size_t smem = sizeof(double) * kShWarps * 33 * kShRow;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_sh_accumulate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(k_sh_accumulate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    if (add)
        k_sh_accumulate<true><<<blocks, 32 * kShWarps, smem, st>>>(sp, ncam, eyes_dev, cam_imp,
                                                                   neq);
    else
        k_sh_accumulate<false><<<blocks, 32 * kShWarps, smem, st>>>(sp, ncam, eyes_dev, cam_imp,
                                                                    neq);
    return cudaGetLastError();
}

size_t sh_solve_scratch_bytes(int64_t n) {
    // masks (u16), class counts, class lists (int32 x n each)
    return ((sizeof(uint16_t) * (size_t)n + 255) & ~(size_t)255) + 256 +
           sizeof(int32_t) * (size_t)kSolveClasses * (size_t)n;
}

cudaError_t launch_sh_solve(const potr_splats &sp, const double *neq, double lambda_y,
                            double par_thr, double zero_thr, double *rgb, double *ycocg,
                            int8_t *status, void *scratch, cudaStream_t st) {
    const int64_t n = sp.n;
    if (n == 0) return cudaSuccess;
    char *p = reinterpret_cast<char *>(scratch);
    uint16_t *masks = reinterpret_cast<uint16_t *>(p);
    p += (sizeof(uint16_t) * (size_t)n + 255) & ~(size_t)255;
    int *counts = reinterpret_cast<int *>(p);
    p += 256;
    int32_t *lists = reinterpret_cast<int32_t *>(p);
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int) * kSolveClasses, st);
    if (e != cudaSuccess) return e;
    const unsigned g = (unsigned)((n + 127) / 128);
    k_sh_mask<<<g, 128, 0, st>>>(n, neq, par_thr, masks, counts, lists);
    k_sh_solve_reg<8><<<g, 128, 0, st>>>(sp, neq, masks, lists + n, counts + 1, lambda_y,
                                         zero_thr, rgb, ycocg, status);
    k_sh_solve_reg<10><<<g, 128, 0, st>>>(sp, neq, masks, lists + 4 * n, counts + 4, lambda_y,
                                          zero_thr, rgb, ycocg, status);
    k_sh_solve_reg<12><<<g, 128, 0, st>>>(sp, neq, masks, lists + 2 * n, counts + 2, lambda_y,
                                          zero_thr, rgb, ycocg, status);
    {
        constexpr size_t smem = sizeof(double) * 136 * kShSmemThreads;
        static int grid = 0;
        if (!grid) {
            cudaFuncSetAttribute(k_sh_solve_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
            int per_sm = 0, sms = 0, dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sh_solve_smem,
                                                          kShSmemThreads, smem);
            grid = sms * (per_sm > 0 ? per_sm : 1);
        }
        k_sh_solve_smem<<<grid, kShSmemThreads, smem, st>>>(sp, neq, masks, lists + 3 * n,
                                                            counts + 3, lambda_y, zero_thr, rgb,
                                                            ycocg, status);
    }
    k_sh_solve<<<g, 128, 0, st>>>(sp, neq, masks, lists, counts, lambda_y, zero_thr, rgb, ycocg,
                                  status);
    return cudaGetLastError();
}

}  // namespace potr
