// kernels.h -- internal launcher interface between api.cu and the kernel files.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

#ifndef LIRANK_TMA_UPDATE
#define LIRANK_TMA_UPDATE 1
#endif

namespace lirank {

// Fused exchange (EMB_F_P2P): a pooling kernel stores the pooled row of the bag with
// block-order index (s * B + b) * Fb + j (source block s, owner-local feature j, sample b)
// straight into rank s's receive buffer over NVLink peer memory:
//   base[s] + ((slot * B + b) * F_out + fcol[j]) * D.
// Table-wise: F_out = F, slot 0, fcol[j] = the global feature (the row lands in its final
// [B][F][D] place).  Row-wise: one [B][F][D] slot per owner (slot = this rank) that the
// destination sums in rank order.  base[0] == NULL: off (rows go to `out` in block order).
constexpr int kPeerMax = 16;
struct PeerOut {
  float* base[kPeerMax];
  const int32_t* fcol;  // device [Fb]
  int32_t F_out;
  int32_t slot;
  int32_t skip_empty;   // row-wise: bags with no id on this owner are not stored (the
                        // destination's slot sum skips them by its a1 lengths)
};

struct FwdArgs {
  const float* W;
  int pitch;
  const int* ids;
  const int* offsets;
  int B, F, D;
  int Fb;              // features per source block (0: F, unsharded)
  const FeatMeta* meta;
  float* out;
  uint2* kv_out;       // NULL: do not record occurrences ({row key, bag} per id)
  uint32_t sentinel;
  uint32_t* status;
  bool mean;
  uint32_t* order_ws;  // NULL: bags in index order; else [kOrderWsWords(F*B)] scratch
  PeerOut peer;        // fused exchange destination (base[0] NULL: off)
};
cudaError_t launch_pool_fwd_f32(const FwdArgs& a, cudaStream_t s);

// Bags visited longest first: a permutation of the F*B bags by length (256 bins), so the
// lane groups of a warp walk bags of about the same length (the id loop runs to the warp's
// longest bag).  Scratch: the permutation + 2 x 256 bin counters.
constexpr int kLenBins = 256;
inline int64_t kOrderWsWords(int64_t bags) { return bags + 2 * kLenBins; }
// the longest-first bag permutation of F*B bags into ws (2 kernels); NULL if bags < 2
const uint32_t* launch_bag_order(const int* offsets, long long bags, uint32_t* ws, cudaStream_t s);
// kernels one forward launch issues: the pooling kernel, plus the 2 ordering kernels and,
// for a2 (fp32), the short-bag kernel
inline int fwd_launches(int64_t bags, bool ordered, bool fp32) {
  return bags <= 0 ? 0 : (ordered && bags >= 2 ? (fp32 ? 4 : 3) : 1);
}

struct FwdQ8Args {
  const uint8_t* codes;   // q8 rows: [codes][pad][middle, scale][pad], qpitch bytes
  int qpitch;
  int meta_off;           // byte offset of {middle, scale} in a q8 row
  const int* ids;
  const int* offsets;
  int B, F, D;
  int Fb;
  const FeatMeta* meta;
  float* out;
  uint32_t* status;
  bool mean;
  uint32_t* order_ws;  // as FwdArgs::order_ws
  bool order_ready;    // order_ws already holds an order of these F*B bags: reuse it
  bool minmax;         // min-max store (uint8 codes, meta {min, scale})
  PeerOut peer;        // as FwdArgs::peer
};
cudaError_t launch_pool_fwd_q8(const FwdQ8Args& a, cudaStream_t s);

// ---- a5 dedup: LSD radix sort (onesweep) + run-length encode -------------------------
// Occurrences are packed {key = stored row (sentinel if invalid), bag index} pairs.
constexpr int kRadixBinsMax = 512;      // 8- or 9-bit digits
constexpr int kSortThreads = 256;
constexpr int kSortTileMin = kSortThreads * 8;  // smallest onesweep tile (capacity sizing)
constexpr int kMaxPasses = 4;           // keys < 2^32
constexpr int kHistWords = kMaxPasses * kRadixBinsMax;

struct SortWs {
  uint32_t* hist;         // [kHistWords] digit histograms, then [kMaxPasses + 2] tile
  uint32_t* counters;     // counters (both zeroed by the sort)
  unsigned long long* status;  // [max_tiles][kRadixBinsMax] look-back words (epoch tagged)
  int64_t max_tiles;
};

// Sorts n pairs by the low `bits` bits of .x, stably.  n is the launch capacity; with n_dev
// (device scalar, optional) the kernels sort min(n, *n_dev) pairs -- the sharded path's
// received count, never read by the host.  Ping-pongs between kv0 and kv1;
// *result_in_1 tells whether the result is in kv1.  Uses epochs [*epoch, *epoch+passes): the
// epoch is read from device memory by the kernels (graph-replayable), advanced by the caller.
cudaError_t radix_sort_pairs(uint2* kv0, uint2* kv1, int64_t n, const uint32_t* n_dev, int bits, const SortWs& ws,
                             const uint32_t* epoch, int* passes_out, bool* result_in_1, int64_t* launches,
                             cudaStream_t s);

// Run-length encode sorted pairs (sentinel = invalid, sorts last): unique[U], seg[U+1],
// *U_out, and chunk_u0[c] = segment containing occurrence c << chunk_log2.  For n == 0 the
// caller writes U = 0, seg[0] = 0; a device count *n_dev == 0 makes the kernel write them.
cudaError_t launch_rle(const uint2* kv, int64_t n, const uint32_t* n_dev, uint32_t sentinel, uint32_t* unique,
                       uint32_t* seg, uint32_t* U_out, uint32_t* chunk_u0, int chunk_log2, uint32_t* counter,
                       unsigned long long* status, const uint32_t* epoch, uint32_t epoch_off,
                       cudaStream_t s);
// *epoch += n, in stream order after the kernels that used epochs [*epoch, *epoch + n)
cudaError_t launch_epoch_advance(uint32_t* epoch, uint32_t n, cudaStream_t s);

// ---- a6-a8 ----------------------------------------------------------------------------
// Occurrences per lane group in the segment-reduce: 2^chunk_log2, 32..128.  128 once the
// batch fills every SM twice over (Feed-1: 13.2M ids -> 103k chunks); smaller for small
// batches so that ~kSegGroups groups still run (a 5k-id batch: 163 chunks of 32, not 41 of 128).
// (max 128, round 2: Feed-1 a6 0.563 -> 0.548 ms, Ads 1.955 -> 1.838, alpha = 0 0.838 -> 0.827 vs
// 256 -- twice the lane-group "waves", so the last one idles less; 64 0.578 / 1.866 / 0.814; a
// persistent grid claiming blocks dynamically instead: 0.583)
constexpr int kChunkLog2Min = 5, kChunkLog2Max = 7;
constexpr int64_t kSegGroups = 148 * 4 * 32;  // resident lane groups (148 SMs x 4 CTAs x 32)
inline int chunk_log2_for(int64_t n) {
  int l = kChunkLog2Min;
  while (l < kChunkLog2Max && (n >> (l + 1)) >= kSegGroups) ++l;
  return l;
}
// chunks a workspace must hold for any call of up to n occurrences (chunk_log2_for(m) for
// every m <= n)
inline int64_t chunks_cap_for(int64_t n) {
  int64_t m = 0;
  for (int l = kChunkLog2Min; l <= kChunkLog2Max; ++l) {
    const int64_t lo = l == kChunkLog2Min ? 0 : (kSegGroups << l);  // smallest n using l
    if (lo > n) break;
    int64_t hi = n;
    if (l < kChunkLog2Max && hi > (kSegGroups << (l + 1)) - 1) hi = (kSegGroups << (l + 1)) - 1;
    const int64_t c = (hi + (int64_t(1) << l) - 1) >> l;
    m = c > m ? c : m;
  }
  return m + 1;
}

struct BwdArgs {
  // dedup results
  const uint32_t* unique;   // [U]
  const uint32_t* seg;      // [U+1]
  const uint32_t* U;        // device scalar
  const uint2* kv;          // sorted {key, bag} per occurrence
  const uint32_t* chunk_u0; // [chunks] segment containing the chunk's first occurrence
  int64_t nnz;              // upper bound of valid occurrences
  int chunk_log2;           // segment-reduce chunk = 2^chunk_log2 occurrences (as the RLE's)
  // gradient input
  const float* grad;        // [B][F][D]
  const int* offsets;       // [F*B+1] (MEAN only)
  int B, F, D, pitch;
  bool mean;
  // workspace
  float* G;                 // [max_unique][pitch]
  double* part_first;       // [chunks][pitch]
  double* part_last;        // [chunks][pitch]
  double* norm_main;        // [chunks]
  double* norm_fix;         // [chunks]
  uint32_t* owner_list;     // [chunks]
  uint32_t* owner_count;    // device scalar (zeroed by launch_segreduce)
  int64_t chunks;
  // norm / clip
  double* S_local;
  double* norm_parts;   // [kNormParts] CTA partials of the norm (k_norm_partial)
  uint32_t* norm_done;  // CTA arrival counter (0 between launches)          // device scalar: this rank's sum of squares
  double* S_global;         // device scalar
  float* clip;              // device scalar
  uint32_t* status;
  double extra_sq_norm;
  const double* extra_dev;  // optional device fp64 added to S (the caller's dense term)
  float* clip_out;          // optional device copy of the clip factor c
  float max_norm;
  // update
  float* Wt;                // tables
  float* A;                 // accumulators
  bool rowwise;
  float lr, eps;
  uint8_t* q8_codes;        // requantize touched rows (NULL: no)
  int q8_meta_off;
  bool q8_minmax;           // re-quantize min-max (else middle-max)
  bool tma;                 // D = 64 row-wise: the TMA-pipelined update kernel
  int qpitch;
};
cudaError_t launch_segreduce(const BwdArgs& a, int64_t* launches, cudaStream_t s);
// reduces norm partials -> S_local (deterministic fixed order)
// ---- NEXT-3: incremental training (incremental.cu) ----------------------------------
struct FimArgs {
  const float *w0, *H0, *w1, *H1;  // [local_rows][pitch] anchors (a NULL pair drops its term)
  float lambda, alpha;
};
cudaError_t launch_cold_init(const float* w0, const float* w1, int64_t n, float alpha, float* w,
                             cudaStream_t s);
// adds the penalty gradient to G of the touched rows and rewrites the norm partials
// (norm_main[0..ngroups), norm_fix zeroed); returns ngroups (-1: launch error)
int64_t launch_fim_penalty(const BwdArgs& a, const FimArgs& f, cudaStream_t s);

cudaError_t launch_norm_partial(const BwdArgs& a, cudaStream_t s);
// S_global = sum of `nparts` rank partials (rank order) + extra -> clip factor, status
cudaError_t launch_norm_finalize(const double* parts, int nparts, const BwdArgs& a,
                                 cudaStream_t s);
cudaError_t launch_adagrad(const BwdArgs& a, cudaStream_t s);

// ---- a9 ----------------------------------------------------------------------------
cudaError_t launch_quantize(const float* W, int pitch, int64_t rows, int D, uint8_t* codes,
                            int qpitch, int meta_off, bool minmax, uint32_t* status, cudaStream_t s);

// ---- misc --------------------------------------------------------------------------
cudaError_t launch_fill(float* p, int64_t n, float v, cudaStream_t s);
cudaError_t launch_gather_rows(const float* src, int pitch, const int64_t* rows, int64_t n,
                               int D, float* dst, cudaStream_t s);

}  // namespace lirank
