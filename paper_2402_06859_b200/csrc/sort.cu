// sort.cu -- a5 dedup: stable LSD radix sort of (row key, bag) pairs + run-length encode.
//
// The dedup gives, for every touched row, the CSR list of its occurrences in ascending
// occurrence order (the tie order is reading 16).  Keys are the
// stored-row index (< 2^31); invalid occurrences carry a sentinel key (= local rows) that
// sorts after every valid key and is cut off by the run-length encode.
//
// Design (B200): "onesweep" LSD radix sort over packed 8-byte {key, bag} pairs.
// * One upfront histogram kernel computes the digit histograms of every pass in a single
//   read of the keys (per-warp private shared-memory histograms).
// * ONE kernel per digit pass (8- or 9-bit digits: 27-bit Feed-1 keys take 3 passes):
//   a 7680-pair tile (512 threads x 15) is loaded with coalesced 8-B loads and ranked in registers (warp
//   multisplit by ballots, stable in index order), the tile's digit counts are published
//   and the global offsets found by a decoupled look-back over earlier tiles (64-bit
//   epoch-tagged status words, so no per-step memset), overlapped with staging the tile
//   in shared memory in sorted order; the tile is then written out in digit runs
//   (coalesced).  Each pass moves 16 B per pair.  Tiles are claimed in launch order
//   through an atomic counter, so a look-back only waits on tiles already resident.

#include "common.cuh"
#include "kernels.h"
#include "lookback.cuh"

namespace lirank {

namespace {

constexpr int NW = kSortThreads / 32;

// Lanes of the warp whose digit equals mine (warp multisplit by ballots), among `valid`:
// AND over the bits b of (my bit b set ? ballot(bit b) : ~ballot(bit b)).  Written so that
// ptxas moves the digit's low bits into predicate registers with one R2P and then spends
// VOTE + a predicated NOT + an AND per bit (3 instructions; the shift/compare/sign form cost 5).
template <int BITS>
__device__ __forceinline__ unsigned peers_of(uint32_t d, unsigned valid) {
  unsigned m = valid;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    unsigned bb, sel;
    asm("{ .reg .pred p; .reg .b32 t; and.b32 t, %1, %2; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 %0, p, 0xffffffff; }"
        : "=r"(bb) : "r"(d), "r"(1u << b));
    asm("{ .reg .pred p; .reg .b32 t; and.b32 t, %1, %2; setp.ne.u32 p, t, 0; selp.b32 %0, %3, %4, p; }"
        : "=r"(sel) : "r"(d), "r"(1u << b), "r"(bb), "r"(~bb));
    m &= sel;
  }
  return m;
}

// Exclusive block scan of one value per thread (NWARPS warps); returns the exclusive
// prefix, *total gets the block sum.
template <int NWARPS = NW>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NWARPS; ++w) {
    const uint32_t s = s_warp[w];
    if (w < warp) wpre += s;
    tot += s;
  }
  __syncthreads();
  *total = tot;
  return wpre + x - v;
}

}  // namespace

// ---------------------------------------------------------------------------
// Upfront histogram of every digit pass.  128-thread CTAs, per-warp private shared
// histograms (shared atomics; a private copy per warp keeps Zipf-hot digits from
// serialising a whole CTA), 8 keys per lane in flight.
// ---------------------------------------------------------------------------
template <int BITS>
__global__ void __launch_bounds__(128)
k_radix_hist(const uint2* __restrict__ kv, int64_t n, const uint32_t* n_dev, int passes, uint32_t* hist) {
  pdl_wait();
  if (n_dev) n = min(n, (int64_t)*n_dev);  // device-resident count (sharded: no host sync)
  constexpr int BINS = 1 << BITS;
  extern __shared__ uint32_t sh[];  // [4 warps][passes][BINS]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per_warp = passes * BINS;
  for (int i = threadIdx.x; i < 4 * per_warp; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t* wh = sh + warp * per_warp;
  constexpr int KU = 8;  // keys per lane in flight
  const int64_t wstride = (int64_t)gridDim.x * 4 * 32 * KU;
  for (int64_t base = ((int64_t)blockIdx.x * 4 + warp) * 32 * KU; base < n; base += wstride) {
    uint32_t k[KU];
#pragma unroll
    for (int q = 0; q < KU; ++q) {
      const int64_t i = base + q * 32 + lane;
      k[q] = i < n ? __ldg(&kv[i].x) : 0u;
    }
#pragma unroll
    for (int q = 0; q < KU; ++q) {
      if (base + q * 32 + lane < n)
        for (int p = 0; p < passes; ++p)
          atomicAdd(&wh[p * BINS + ((k[q] >> (p * BITS)) & (BINS - 1))], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < per_warp; i += blockDim.x) {
    const uint32_t s = sh[i] + sh[per_warp + i] + sh[2 * per_warp + i] + sh[3 * per_warp + i];
    if (s) atomicAdd(hist + i, s);
  }
}

// Digit histograms -> exclusive prefix sums in place (one CTA per pass), so the onesweep
// tiles read each digit's global start instead of scanning the histogram themselves.
__global__ void __launch_bounds__(512)
k_hist_excl(uint32_t* hist, int bins) {
  pdl_wait();
  __shared__ uint32_t s_warp[16];
  uint32_t* h = hist + (size_t)blockIdx.x * bins;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t v = t < bins ? h[t] : 0u;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (t == 0) {
    uint32_t c = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { const uint32_t q = s_warp[w]; s_warp[w] = c; c += q; }
  }
  __syncthreads();
  if (t < bins) h[t] = s_warp[warp] + x - v;
}

// ---------------------------------------------------------------------------
// One digit pass.  ITEMS pairs per thread (tile = 256 * ITEMS); RANK selects the warp
// ranking primitive (match.any vs a BITS-ballot multisplit).
// ---------------------------------------------------------------------------
// Load the warp's ITEMS x 32 pairs and rank each within the warp (stable: by item, then
// lane) against the warp's running digit counters wh[].  FULL: every index is < n.
// RANK selects how a lane finds the lanes holding the same digit ("peers"): 0: BITS ballots
// (warp multisplit), 1: match.any.  (Measured on Feed-1, 3 passes alone: ballots 0.347 ms;
// match.any slower; a shared-memory atomic-OR match -- each lane ORs its bit into a per-warp
// word of its digit and reads it back -- 0.41-0.44 ms at 3-4 CTAs/SM.)
template <int BITS, int ITEMS, int RANK, bool FULL>
__device__ __forceinline__ void load_rank(const uint2* __restrict__ in, uint2 (&kv)[ITEMS],
                                          uint32_t (&r)[ITEMS], int64_t base, int64_t n, int shift,
                                          uint32_t* wh, int lane, unsigned lt) {
  constexpr int BINS = 1 << BITS;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = base + i * 32 + lane;
    kv[i] = (FULL || idx < n) ? in[idx] : make_uint2(0u, 0u);
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = base + i * 32 + lane;
    const bool ok = FULL || idx < n;
    const uint32_t d = ok ? (kv[i].x >> shift) & (BINS - 1) : (uint32_t)BINS;
    unsigned peers;
    if (RANK == 1) {
      peers = __match_any_sync(0xffffffffu, d);
    } else {
      peers = FULL ? peers_of<BITS>(d, 0xffffffffu)
                   : peers_of<BITS + 1>(d, 0xffffffffu);  // bit BITS separates out-of-range lanes
    }
    const uint32_t cur = ok ? wh[d] : 0u;
    r[i] = cur + __popc(peers & lt);
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) wh[d] = cur + __popc(peers);
    __syncwarp();
  }
}

// The tile after its claim: rank, publish / scan the digit counts, stage in sorted order,
// look back, write out.  FULL (every tile but the last): no bounds checks anywhere.
template <int BITS, int ITEMS, int RANK, bool FULL, int LB, int SLEEP, int THREADS>
__device__ __forceinline__ void onesweep_tile(const uint2* __restrict__ in, uint2* __restrict__ out, int64_t n,
                                              int shift, const uint32_t* __restrict__ hist,
                                              unsigned long long* status, uint32_t epoch, int64_t tile,
                                              uint8_t* smem_raw) {
  constexpr int BINS = 1 << BITS;
  constexpr int NWT = THREADS / 32;
  constexpr int DPT = (BINS + THREADS - 1) / THREADS;  // digits per thread (digit tid + q * THREADS)
  constexpr int TILE = THREADS * ITEMS;
  uint2* stage = reinterpret_cast<uint2*>(smem_raw);                           // [TILE]
  uint32_t* warp_hist = reinterpret_cast<uint32_t*>(stage + TILE);            // [NWT][BINS]
  uint32_t* digit_off = warp_hist + NWT * BINS;                                  // [BINS]
  uint32_t* s_misc = digit_off + BINS;                                          // [NWT + 2]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tile0 = tile * TILE;
  const int64_t base = tile0 + (int64_t)warp * (ITEMS * 32);

  uint2 kv[ITEMS];
  uint32_t r[ITEMS];
  const unsigned lt = lanemask_lt();
  uint32_t* wh = warp_hist + warp * BINS;
  load_rank<BITS, ITEMS, RANK, FULL>(in, kv, r, base, n, shift, wh, lane, lt);
  __syncthreads();

  // per digit: exclusive prefix over warps, tile total, and the tile's exclusive prefix over
  // digits (its sorted-order layout); warp_hist[w][d] becomes the stage slot of warp w's
  // first item with digit d (tile prefix + warp prefix: one lookup per item below)
  uint32_t total[DPT], tile_excl[DPT];
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const int dg = tid + q * THREADS;
    uint32_t t = 0;
    if (dg < BINS) {
#pragma unroll
      for (int w = 0; w < NWT; ++w) {
        const uint32_t c = warp_hist[w * BINS + dg];
        warp_hist[w * BINS + dg] = t;
        t += c;
      }
      lb_publish(status, tile, BINS, dg, epoch, t);
    }
    total[q] = t;
  }
  {
    uint32_t carry = 0;
#pragma unroll
    for (int q = 0; q < DPT; ++q) {
      uint32_t blk_total;
      tile_excl[q] = carry + block_excl_scan<NWT>(total[q], s_misc, &blk_total);
      carry += blk_total;
    }
  }
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const int dg = tid + q * THREADS;
    if (dg < BINS)
#pragma unroll
      for (int w = 0; w < NWT; ++w) warp_hist[w * BINS + dg] += tile_excl[q];
  }
  __syncthreads();
  // stage the tile in sorted order (overlaps the look-back of earlier tiles); item i of this
  // lane is valid iff i < nv
  const int nv = FULL ? ITEMS : (int)max((int64_t)0, min((int64_t)ITEMS, (n - base - lane + 31) / 32));
#pragma unroll
  for (int i = 0; i < ITEMS; ++i)
    if (FULL || i < nv) stage[wh[(kv[i].x >> shift) & (BINS - 1)] + r[i]] = kv[i];
  // global position of sorted-tile slot j with digit d: hist_excl[d] + prev[d] + (j - tile_excl[d])
  // (`hist` holds the exclusive prefix of the pass's digit counts, k_hist_excl)
  uint32_t hist_excl[DPT];
#pragma unroll
  for (int q = 0; q < DPT; ++q) hist_excl[q] = tid + q * THREADS < BINS ? __ldg(hist + tid + q * THREADS) : 0u;
  uint32_t prev[DPT];
#pragma unroll
  for (int q = 0; q < DPT; ++q)
    prev[q] = tid + q * THREADS < BINS ? lb_wait<LB, SLEEP>(status, tile, BINS, tid + q * THREADS, epoch, total[q]) : 0u;
#pragma unroll
  for (int q = 0; q < DPT; ++q)
    if (tid + q * THREADS < BINS) digit_off[tid + q * THREADS] = hist_excl[q] + prev[q] - tile_excl[q];
  __syncthreads();  // stage and digit_off complete
  const int64_t cnt = FULL ? TILE : (n - tile0 < TILE ? n - tile0 : TILE);
#pragma unroll 4
  for (int j = tid; j < cnt; j += THREADS) {
    const uint2 x = stage[j];
    const uint32_t d = (x.x >> shift) & (BINS - 1);
    out[digit_off[d] + j] = x;
  }
}

template <int BITS, int ITEMS, int RANK, int MINB = 4, int LB = 8, int SLEEP = 64, int THREADS = kSortThreads>
__global__ void __launch_bounds__(THREADS, MINB)
k_onesweep(const uint2* __restrict__ in, uint2* __restrict__ out, int64_t n, const uint32_t* n_dev,
           int shift, const uint32_t* __restrict__ hist, uint32_t* tile_counter,
           unsigned long long* status, const uint32_t* epoch_p, uint32_t epoch_off) {
  pdl_wait();
  if (n_dev) n = min(n, (int64_t)*n_dev);
  constexpr int BINS = 1 << BITS;
  const uint32_t epoch = *epoch_p + epoch_off;  // device-resident: graph replays advance it
  constexpr int TILE = THREADS * ITEMS;
  constexpr int NWT = THREADS / 32;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint32_t* warp_hist = reinterpret_cast<uint32_t*>(smem_raw + sizeof(uint2) * TILE);  // [NWT][BINS]
  uint32_t* s_misc = warp_hist + NWT * BINS + BINS;                                       // [NWT + 2]
  const int tid = threadIdx.x;
  if (tid == 0) s_misc[NWT] = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < NWT * BINS / 4; i += THREADS)  // 16-B stores: (NWT * BINS) % 4 == 0
    reinterpret_cast<uint4*>(warp_hist)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  const int64_t tile = s_misc[NWT];
  const int64_t tile0 = tile * TILE;
  // grid sized for a capacity: tiles past the device count have nothing to do (no later
  // tile looks back at them -- every later tile is past it too)
  if (tile0 >= n) return;
  // every tile but the last is full: no bounds checks, and its ranking needs BITS ballots
  // (the last one separates out-of-range lanes with one more bit)
  if (tile0 + TILE <= n)
    onesweep_tile<BITS, ITEMS, RANK, true, LB, SLEEP, THREADS>(in, out, n, shift, hist, status, epoch, tile, smem_raw);
  else
    onesweep_tile<BITS, ITEMS, RANK, false, LB, SLEEP, THREADS>(in, out, n, shift, hist, status, epoch, tile, smem_raw);
}

template <int BITS, int ITEMS, int RANK, int MINB, int LB = 8, int SLEEP = 64, int THREADS = kSortThreads>
static cudaError_t onesweep_pass(const uint2* a, uint2* b, int64_t n, const uint32_t* n_dev, int shift,
                                 const uint32_t* hist,
                                 uint32_t* counter, unsigned long long* status, const uint32_t* epoch,
                                 uint32_t epoch_off, cudaStream_t s) {
  constexpr int TILE = THREADS * ITEMS;
  constexpr int NWT = THREADS / 32;
  const size_t sm = sizeof(uint2) * TILE + sizeof(uint32_t) * (NWT * (1 << BITS) + (1 << BITS) + NWT + 2);
  // the attribute is per device: set once per device (before any graph capture of a step)
  static bool attr[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices || !attr[dev]) {
    cudaFuncSetAttribute(k_onesweep<BITS, ITEMS, RANK, MINB, LB, SLEEP, THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (dev >= 0 && dev < kMaxDevices) attr[dev] = true;
  }
  const int64_t tiles = (n + TILE - 1) / TILE;
  launch_pdl(k_onesweep<BITS, ITEMS, RANK, MINB, LB, SLEEP, THREADS>, (unsigned)tiles, THREADS, sm, s, a, b, n, n_dev, shift, hist,
                                                                                counter, status, epoch,
                                                                                epoch_off);
  return cudaGetLastError();
}

cudaError_t radix_sort_pairs(uint2* kv0, uint2* kv1, int64_t n, const uint32_t* n_dev, int bits, const SortWs& ws,
                             const uint32_t* epoch, int* passes_out, bool* result_in_1, int64_t* launches,
                             cudaStream_t s) {
  // digit width: 9 bits when it saves a pass (e.g. 27-bit Feed-1 keys: 3 passes, not 4)
  const int dbits = (bits > 24 && bits <= 27) || (bits > 16 && bits <= 18) ? 9 : 8;
  const int passes = (bits + dbits - 1) / dbits;
  *passes_out = passes;
  *result_in_1 = false;
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(ws.hist, 0, sizeof(uint32_t) * (kHistWords + kMaxPasses + 2), s);
  if (e != cudaSuccess) return e;
  if (passes == 0) return cudaSuccess;
  if ((n + kSortTileMin - 1) / kSortTileMin > ws.max_tiles) return cudaErrorInvalidValue;
  const int bins = 1 << dbits;
  {
    const int64_t want = (n + 128 * 8 - 1) / (128 * 8);
    const unsigned grid = (unsigned)(want < 148 * 8 ? want : 148 * 8);
    const size_t sm = sizeof(uint32_t) * 4 * passes * bins;
    if (dbits == 9) launch_pdl(k_radix_hist<9>, grid, 128, sm, s, (const uint2*)kv0, n, n_dev, passes, ws.hist);
    else launch_pdl(k_radix_hist<8>, grid, 128, sm, s, (const uint2*)kv0, n, n_dev, passes, ws.hist);
    launch_pdl(k_hist_excl, passes, 512, 0, s, ws.hist, bins);
    *launches += 2;
  }
  uint2 *a = kv0, *b = kv1;
  for (int p = 0; p < passes; ++p) {
    const int shift = p * dbits;
    const uint32_t* hp = ws.hist + p * bins;
    uint32_t* ctr = ws.counters + p;
    // tile geometry, measured on Feed-1 alone (tools/sort_probe.py, 3 passes), 256-thread CTAs
    // first: 16 items x 4 CTAs 0.334 ms, 18 x 3 0.313, 20 x 3
    // 0.308, 22 x 3 0.301, 24 x 2 0.317, 28 x 2 0.314, 32 x 2 0.317, 12 x 4 0.352 -- larger
    // tiles mean fewer tiles in each digit's look-back walk; a look-back window of 4 or 8 is
    // the same, 16 (more registers) 0.51; exponential back-off of the poll changes nothing
    // (CTA width, round 2: 512 threads x 16 items at 2 CTAs/SM 0.297 ms vs 256 x 22 at 3 CTAs
    // 0.31 in the same run, 384 x 22 x 2 0.315, 384 x 20 x 2 0.310, 512 x 12 x 2 0.303; Ads
    // 0.964 vs 0.998 ms: the wider tile halves the look-back walks per item at equal occupancy;
    // then 512 x 15: 0.297 -> 0.286 ms, Ads 0.965 -> 0.931, alpha 0 0.306 -> 0.297 (14: 0.287 /
    // 0.953, 17: 0.295 / 0.963) -- fewer spilled registers at the 64-register cap, and Feed-1's
    // 1724 tiles fill the 296 resident CTAs in 5.8 rounds instead of 5.5; at 512 x 15 the
    // look-back window 4 / 8 / 16: 0.286 / 0.286 / 0.469 ms, poll sleep 32 / 64 / 256 ns: same)
#define OS(BITS) e = onesweep_pass<BITS, 15, 0, 2, 8, 64, 512>(a, b, n, n_dev, shift, hp, ctr, ws.status, epoch, (uint32_t)p, s);
    if (dbits == 9) { OS(9) } else { OS(8) }
#undef OS
    if (e != cudaSuccess) return e;
    ++*launches;
    uint2* t = a; a = b; b = t;
  }
  *result_in_1 = (passes & 1) != 0;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Run-length encode of the sorted keys (single pass, decoupled look-back over tiles).
// A "head" is the first occurrence of a key; the first sentinel (invalid) key is also a
// head, so its position is U and seg[U] = n_valid.  Without sentinels the tile holding
// item n-1 writes seg[U] = n.  Also records, for every segment-reduce chunk c, the
// segment that contains occurrence c << chunk_log2 (chunk_u0[c]).  n: capacity (grid
// size); n_dev (optional): the device-resident count, read by the kernel.
// ---------------------------------------------------------------------------
template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads)
k_rle(const uint2* __restrict__ kv, int64_t n, const uint32_t* n_dev, uint32_t sentinel, uint32_t* unique,
      uint32_t* seg, uint32_t* U_out, uint32_t* chunk_u0, int chunk_log2, uint32_t* tile_counter,
      unsigned long long* status, const uint32_t* epoch_p, uint32_t epoch_off) {
  pdl_wait();
  if (n_dev) n = min(n, (int64_t)*n_dev);
  const uint32_t epoch = *epoch_p + epoch_off;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[NW];
  __shared__ uint32_t s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  if (n == 0) {  // (device count 0) no occurrence: U = 0
    if (tile == 0 && tid == 0) { *U_out = 0u; seg[0] = 0u; }
    return;
  }
  constexpr int TILE = kSortThreads * ITEMS;
  if (tile * TILE >= n) return;  // past the device count
  const int64_t base = tile * TILE + (int64_t)warp * (ITEMS * 32);
  unsigned ball[ITEMS];
  uint32_t kk[ITEMS];
  uint32_t wcount = 0;
  const unsigned lt = lanemask_lt();
  // (each item also loads its predecessor's key -- an L1 hit; taking it from the previous
  // lane by a shuffle instead measured slower: 0.059 -> 0.061 ms on Feed-1)
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = base + i * 32 + lane;
    bool head = false;
    uint32_t k = 0;
    if (idx < n) {
      k = __ldg(&kv[idx].x);
      head = (idx == 0) || (__ldg(&kv[idx - 1].x) != k);
    }
    kk[i] = k;
    ball[i] = __ballot_sync(0xffffffffu, head);
    wcount += __popc(ball[i]);
  }
  if (lane == 0) s_warp[warp] = wcount;
  __syncthreads();
  if (warp == 0) {  // the warps' prefix and the tile total, then a warp-wide look-back
    const uint32_t c = lane < NW ? s_warp[lane] : 0u;
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const uint32_t t = __shfl_sync(0xffffffffu, x, NW - 1);
    if (lane < NW) s_warp[lane] = x - c;
    if (lane == 0) lb_publish(status, tile, kRadixBinsMax, 0, epoch, t);
    const uint32_t ex = lb_wait_warp(status, tile, kRadixBinsMax, 0, epoch, t, lane);
    if (lane == 0) s_excl = ex;
  }
  __syncthreads();
  uint32_t pos = s_excl + s_warp[warp];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = base + i * 32 + lane;
    const bool head = (ball[i] >> lane) & 1u;
    const uint32_t p = pos + __popc(ball[i] & lt);  // heads before idx
    if (head) {
      if (kk[i] != sentinel) unique[p] = kk[i];
      seg[p] = (uint32_t)idx;
    }
    if (idx < n && (idx & ((1 << chunk_log2) - 1)) == 0) chunk_u0[idx >> chunk_log2] = p + (head ? 1u : 0u) - 1u;
    pos += __popc(ball[i]);
    if (idx == n - 1) {
      // pos now = number of heads in [0, n) (incl. the sentinel head if any)
      const bool has_sentinel = kk[i] == sentinel;
      const uint32_t U = pos - (has_sentinel ? 1u : 0u);
      *U_out = U;
      if (!has_sentinel) seg[U] = (uint32_t)n;
    }
  }
}

cudaError_t launch_rle(const uint2* kv, int64_t n, const uint32_t* n_dev, uint32_t sentinel, uint32_t* unique,
                       uint32_t* seg, uint32_t* U_out, uint32_t* chunk_u0, int chunk_log2, uint32_t* counter,
                       unsigned long long* status, const uint32_t* epoch, uint32_t epoch_off,
                       cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  // 16 items per thread measured best (Feed-1: 8 -> 0.082 ms, 16 -> 0.059, 24 -> 0.065, 32 -> 0.073);
  // with the warp-wide look-back, round 2: 12 0.0569, 14 0.0548, 16 0.0548, 18 0.0544, 20 0.066 ms
  // (Ads: 0.171 / 0.158 / 0.155 / 0.148 / 0.207) -> 18;
  // CTA width, round 2 (16 items): 256 threads 0.059 ms, 512 0.063, 1024 0.066, 128 0.068;
  // 8 x 512 0.068, 8 x 256 0.083, 32 x 128 0.091 -- fewer look-backs do not pay for the
  // longer barrier wait behind thread 0's walk
  constexpr int IT = 18;
  const int64_t tiles = (n + kSortThreads * IT - 1) / (kSortThreads * IT);
  launch_pdl(k_rle<IT>, (unsigned)tiles, kSortThreads, 0, s, kv, n, n_dev, sentinel, unique, seg, U_out, chunk_u0,
             chunk_log2, counter, status, epoch, epoch_off);
  return cudaGetLastError();
}

// The look-back epochs live in device memory and are advanced by a kernel in stream order
// (not baked into launch parameters), so a captured CUDA graph of a step can be replayed:
// every replay tags its status words with fresh epochs.
__global__ void k_epoch_advance(uint32_t* epoch, uint32_t n) {
  pdl_wait();
  *epoch += n;
}

cudaError_t launch_epoch_advance(uint32_t* epoch, uint32_t n, cudaStream_t s) {
  launch_pdl(k_epoch_advance, 1, 1, 0, s, epoch, n);
  return cudaGetLastError();
}

}  // namespace lirank
