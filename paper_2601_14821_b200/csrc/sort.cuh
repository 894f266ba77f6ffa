// sort.cuh -- hand-written device primitives for sm_100a (sort.cu): the LSD
// radix sort behind the depth order (rasterizer.py:248-250, np.argsort
// kind="stable"), the tile binning (:135-148), the spatial slot order, the
// records order and the codec's DFS order; and the single-pass scans behind
// the pair offsets and the codec.
//
// Radix sort: 8-bit digits, one histogram kernel for all passes, then one
// "one-sweep" kernel per pass: a CTA takes the next tile of kTileItems keys
// (dynamic tile index, so tiles are claimed in order), ranks them stably
// inside the tile (warp-striped loads; equal digits found by ballots on the
// digit bits and by __match_any_sync in alternate rounds), publishes
// its per-digit counts, looks back over the preceding tiles' published counts
// (decoupled look-back, one thread per digit) for its global digit offsets,
// and scatters through shared memory so that each digit's run leaves in
// consecutive addresses.  Stable: equal digits keep input order, so equal keys
// keep input order across all passes.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace potr {

// Scratch for radix_sort_pairs of n items over [begin_bit, end_bit).
size_t radix_sort_temp_bytes(int64_t n, int begin_bit, int end_bit);

// Stable sort of (keys, vals) by keys' bits [begin_bit, end_bit), double-
// buffered: the result ends in (keys, vals) or, when *in_alt is set, in
// (keys_alt, vals_alt).  iota_vals: the input values are iota_base + 0..n-1
// (vals is not read, only written).  K: uint16_t, uint32_t, uint64_t; V:
// int32_t, int64_t.
template <typename K, typename V>
cudaError_t radix_sort_pairs(void *temp, size_t temp_bytes, K *keys, K *keys_alt, V *vals,
                             V *vals_alt, int64_t n, int begin_bit, int end_bit, bool iota_vals,
                             bool *in_alt, cudaStream_t st, int64_t iota_base = 0);

// Stable sort of keys with packed int2 values: item i enters as
// {vbase + i, hi[i]} (hi read once, in order, by the first pass), so the
// sorted values carry both the item's index and its payload -- no gather after
// the sort.  Result in (keys, vals) or, with *in_alt, (keys_alt, vals_alt).
// K: uint16_t, uint32_t.
template <typename K>
cudaError_t radix_sort_packed(void *temp, size_t temp_bytes, K *keys, K *keys_alt,
                              const int32_t *hi, int64_t vbase, int2 *vals, int2 *vals_alt,
                              int64_t n, int begin_bit, int end_bit, bool *in_alt,
                              cudaStream_t st);

// Kernel launches of one radix_sort_pairs call (histogram + one per pass).
inline int sort_launches(int begin_bit, int end_bit) {
    return end_bit > begin_bit ? 1 + (end_bit - begin_bit + 7) / 8 : 0;
}

// Single-pass scans (decoupled look-back).
size_t scan_temp_bytes(int64_t n);
// out[i] = sum_{j <= i} cnt[ids[i]]  (the pair-offset scan over counts in
// depth order: out points at offs + 1)
cudaError_t inclusive_sum_gather(void *temp, size_t temp_bytes, const int32_t *ids,
                                 const int32_t *cnt, int64_t *out, int64_t n, cudaStream_t st);
// out[i] = sum_{j < i} in[j]
cudaError_t exclusive_sum_i64(void *temp, size_t temp_bytes, const int64_t *in, int64_t *out,
                              int64_t n, cudaStream_t st);
// out[i] = max_{j <= i} in[j]
cudaError_t inclusive_max_i32(void *temp, size_t temp_bytes, const int32_t *in, int32_t *out,
                              int64_t n, cudaStream_t st);
// out[k] = in[i] for the k-th i with flags[i] != 0, in order; *count = k total
// (device pointer)
cudaError_t select_flagged_i32(void *temp, size_t temp_bytes, const int32_t *in,
                               const uint8_t *flags, int32_t *out, int32_t *count, int64_t n,
                               cudaStream_t st);

}  // namespace potr
