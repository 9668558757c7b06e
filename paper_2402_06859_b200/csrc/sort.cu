// sort.cu -- a5 dedup: stable LSD radix sort of (row key, bag) pairs + run-length encode.
//
// The dedup gives, for every touched row, the CSR list of its occurrences in ascending
// occurrence order (the ordering is reading 16).  Keys are the
// stored-row index (< 2^31), invalid occurrences carry a sentinel key (= local rows) that
// sorts after every valid key and is cut off by the run-length encode.
//
// Design (B200): "onesweep" LSD radix sort -- one upfront histogram kernel for all digit
// passes, then ONE kernel per 8-bit digit pass that ranks a 4096-key tile in registers
// (warp match_any ranking, stable in index order), finds the tile's global digit offsets
// with a decoupled look-back over earlier tiles (64-bit epoch-tagged status words, so
// no per-step memset), and scatters.  Each pass moves 16 B per key (read key+value,
// write key+value).  Tiles are claimed in launch order through an atomic counter, so a
// look-back only ever waits on tiles that are already resident.
#include "common.cuh"
#include "kernels.h"

namespace lirank {

namespace {

constexpr unsigned long long kFlagAgg = 1ull << 30;
constexpr unsigned long long kFlagPrefix = 2ull << 30;
constexpr unsigned long long kCountMask = (1ull << 30) - 1;

__device__ __forceinline__ unsigned long long pack(uint32_t epoch, unsigned long long flag,
                                                   uint32_t count) {
  return ((unsigned long long)epoch << 32) | flag | (unsigned long long)count;
}

__device__ __forceinline__ void st_volatile(unsigned long long* p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// Exclusive prefix of everything before `tile` for the value published at
// status[tile * stride + slot]; publishes this tile's aggregate and then its inclusive
// prefix.  Called by one thread per slot.
__device__ __forceinline__ uint32_t lookback(unsigned long long* status, int64_t tile,
                                             int stride, int slot, uint32_t epoch,
                                             uint32_t aggregate) {
  unsigned long long* mine = status + tile * stride + slot;
  if (tile == 0) {
    st_volatile(mine, pack(epoch, kFlagPrefix, aggregate));
    return 0;
  }
  st_volatile(mine, pack(epoch, kFlagAgg, aggregate));
  uint32_t excl = 0;
  int64_t p = tile - 1;
  while (true) {
    const unsigned long long w = ld_volatile(status + p * stride + slot);
    if ((uint32_t)(w >> 32) != epoch || (w & (3ull << 30)) == 0) continue;  // not yet
    excl += (uint32_t)(w & kCountMask);
    if (w & kFlagPrefix) break;
    --p;
  }
  st_volatile(mine, pack(epoch, kFlagPrefix, excl + aggregate));
  return excl;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace

// Histogram of every digit pass in one read of the keys.
__global__ void __launch_bounds__(256)
k_radix_hist(const uint32_t* __restrict__ keys, int64_t n, int passes, uint32_t* hist) {
  __shared__ uint32_t sh[kMaxPasses * kRadixBins];
  for (int i = threadIdx.x; i < kMaxPasses * kRadixBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i - threadIdx.x < n;
       i += stride) {
    const bool in = i < n;
    const uint32_t k = in ? __ldg(keys + i) : 0u;
    const unsigned active = __ballot_sync(0xffffffffu, in);
    if (in) {
      for (int p = 0; p < passes; ++p) {
        const uint32_t d = (k >> (p * kRadixBits)) & (kRadixBins - 1);
        const unsigned peers = __match_any_sync(active, d);
        if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1))
          atomicAdd(&sh[p * kRadixBins + d], (uint32_t)__popc(peers));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadixBins; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, sh[i]);
}

// One digit pass.
__global__ void __launch_bounds__(kSortThreads)
k_onesweep(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
           uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n, int shift,
           const uint32_t* __restrict__ hist, uint32_t* tile_counter,
           unsigned long long* status, uint32_t epoch) {
  constexpr int NW = kSortThreads / 32;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t warp_hist[NW][kRadixBins];
  __shared__ uint32_t digit_base[kRadixBins];
  __shared__ uint32_t scan_tmp[kRadixBins];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < NW * kRadixBins; i += kSortThreads) (&warp_hist[0][0])[i] = 0;
  // exclusive scan of this pass's histogram (digit bases), Hillis-Steele in smem
  scan_tmp[tid] = hist[tid];
  __syncthreads();
  for (int off = 1; off < kRadixBins; off <<= 1) {
    const uint32_t v = tid >= off ? scan_tmp[tid - off] : 0u;
    __syncthreads();
    scan_tmp[tid] += v;
    __syncthreads();
  }
  const uint32_t hist_excl = scan_tmp[tid] - hist[tid];
  const int64_t tile = s_tile;
  const int64_t base = tile * kSortTile + (int64_t)warp * (kSortItems * 32);

  uint32_t k[kSortItems], v[kSortItems], r[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = base + i * 32 + lane;
    if (idx < n) {
      k[i] = __ldg(kin + idx);
      v[i] = __ldg(vin + idx);
    }
  }
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = base + i * 32 + lane;
    const uint32_t d = idx < n ? ((k[i] >> shift) & (kRadixBins - 1)) : (uint32_t)kRadixBins;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t cur = d < kRadixBins ? warp_hist[warp][d] : 0u;
    r[i] = cur + __popc(peers & lt);
    __syncwarp();
    if (d < kRadixBins && lane == __ffs(peers) - 1) warp_hist[warp][d] = cur + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit (thread tid = digit): exclusive prefix over warps, tile aggregate
  uint32_t total = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t c = warp_hist[w][tid];
    warp_hist[w][tid] = total;
    total += c;
  }
  const uint32_t excl = lookback(status, tile, kRadixBins, tid, epoch, total);
  digit_base[tid] = hist_excl + excl;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = base + i * 32 + lane;
    if (idx < n) {
      const uint32_t d = (k[i] >> shift) & (kRadixBins - 1);
      const uint32_t pos = digit_base[d] + warp_hist[warp][d] + r[i];
      kout[pos] = k[i];
      vout[pos] = v[i];
    }
  }
}

cudaError_t radix_sort_pairs(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, int64_t n,
                             int bits, const SortWs& ws, uint32_t epoch, int* passes_out,
                             bool* result_in_1, int64_t* launches, cudaStream_t s) {
  const int passes = (bits + kRadixBits - 1) / kRadixBits;
  *passes_out = passes;
  *result_in_1 = false;
  if (n == 0) return cudaSuccess;
  // hist and counters are adjacent (api.cu carve-up): one memset for both
  cudaError_t e = cudaMemsetAsync(ws.hist, 0, sizeof(uint32_t) * (kMaxPasses * kRadixBins + kMaxPasses + 2), s);
  if (e != cudaSuccess) return e;
  if (passes == 0) return cudaSuccess;
  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  if (tiles > ws.max_tiles) return cudaErrorInvalidValue;
  {
    int64_t want = (n + 255) / 256;
    const unsigned grid = (unsigned)(want < 148 * 8 ? want : 148 * 8);
    k_radix_hist<<<grid, 256, 0, s>>>(k0, n, passes, ws.hist);
    ++*launches;
  }
  uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
  for (int p = 0; p < passes; ++p) {
    k_onesweep<<<(unsigned)tiles, kSortThreads, 0, s>>>(ki, vi, ko, vo, n, p * kRadixBits,
                                                         ws.hist + p * kRadixBins,
                                                         ws.counters + p, ws.status, epoch + p);
    ++*launches;
    uint32_t* t;
    t = ki; ki = ko; ko = t;
    t = vi; vi = vo; vo = t;
  }
  *result_in_1 = (passes & 1) != 0;
  return cudaGetLastError();
}

// Run-length encode of the sorted keys (single pass, decoupled look-back over tiles).
// A "head" is the first occurrence of a key; the first sentinel (invalid) key is also a
// head, so its position is U and seg[U] = n_valid.  Without sentinels the tile holding
// item n-1 writes seg[U] = n.
__global__ void __launch_bounds__(kSortThreads)
k_rle(const uint32_t* __restrict__ keys, int64_t n, uint32_t sentinel, uint32_t* unique,
      uint32_t* seg, uint32_t* U_out, uint32_t* tile_counter, unsigned long long* status,
      uint32_t epoch) {
  constexpr int NW = kSortThreads / 32;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[NW];
  __shared__ uint32_t s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * kSortTile + (int64_t)warp * (kSortItems * 32);
  unsigned ball[kSortItems];
  uint32_t kk[kSortItems];
  uint32_t wcount = 0;
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = base + i * 32 + lane;
    bool head = false;
    uint32_t k = 0;
    if (idx < n) {
      k = __ldg(keys + idx);
      head = (idx == 0) || (__ldg(keys + idx - 1) != k);
    }
    kk[i] = k;
    ball[i] = __ballot_sync(0xffffffffu, head);
    wcount += __popc(ball[i]);
  }
  if (lane == 0) s_warp[warp] = wcount;
  __syncthreads();
  if (tid == 0) {
    uint32_t t = 0;
    for (int w = 0; w < NW; ++w) {
      const uint32_t c = s_warp[w];
      s_warp[w] = t;
      t += c;
    }
    s_excl = lookback(status, tile, kRadixBins, 0, epoch, t);
  }
  __syncthreads();
  uint32_t pos = s_excl + s_warp[warp];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = base + i * 32 + lane;
    if ((ball[i] >> lane) & 1u) {
      const uint32_t p = pos + __popc(ball[i] & lt);
      if (kk[i] != sentinel) unique[p] = kk[i];
      seg[p] = (uint32_t)idx;
    }
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

cudaError_t launch_rle(const uint32_t* keys, int64_t n, uint32_t sentinel, uint32_t* unique,
                       uint32_t* seg, uint32_t* U_out, uint32_t* counter,
                       unsigned long long* status, uint32_t epoch, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int64_t tiles = (n + kSortTile - 1) / kSortTile;
  k_rle<<<(unsigned)tiles, kSortThreads, 0, s>>>(keys, n, sentinel, unique, seg, U_out, counter,
                                                 status, epoch);
  return cudaGetLastError();
}

}  // namespace lirank
