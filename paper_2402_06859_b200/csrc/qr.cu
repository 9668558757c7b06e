// qr.cu -- NEXT-1: unlimited-dictionary ids.
//
// emb_hash_ids: MurmurHash3 x64-128 (seed 0) of id strings -> the int64 id (h1).  One
//   thread per string (ids are short: "member:1234"); each warp stages its 32 strings'
//   contiguous bytes in shared memory with 16-B loads, then every thread mixes its 16-byte
//   blocks as the algorithm defines, the 0..15-byte tail and fmix64.
// emb_qr_expand: the int64 is bitcast to two 32-bit numbers B (low) and C (high); each
//   indexes its own quotient/remainder table pair, and the rows are laid out in ONE
//   concatenated table [qB | rB | qC | rC] so the expanded bag goes through the ordinary
//   a2 / a5-a8 path (sum aggregation == SUM pooling over the expanded rows).  One thread
//   per id, vector stores of its 2 or 4 row ids; the quotient's "mod Q" is skipped when Q
//   covers every 32-bit n / R.
#include "handle.h"

namespace lirank {

namespace {

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

// 8 little-endian bytes at any byte address p of a shared-memory buffer: three aligned
// 32-bit loads and two funnel shifts (no byte loop).  Reads up to 11 bytes past p + 8.
__device__ __forceinline__ uint64_t le64_smem(const uint8_t* p) {
  const uintptr_t a = (uintptr_t)p;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
  const uint32_t sh = 8u * (uint32_t)(a & 3);
  const uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
  const uint32_t lo = __funnelshift_r(w0, w1, sh), hi = __funnelshift_r(w1, w2, sh);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t le64_global(const uint8_t* p) {
  uint64_t v = 0;
#pragma unroll
  for (int i = 7; i >= 0; --i) v = (v << 8) | (uint64_t)__ldg(p + i);
  return v;
}
// the low `nb` bytes (0..8) of x
__device__ __forceinline__ uint64_t low_bytes(uint64_t x, int nb) {
  return nb >= 8 ? x : (x & ((1ull << (8 * nb)) - 1ull));
}

// h1 of MurmurHash3 x64-128, seed 0, of key[0 .. len).  SMEM: key is in shared memory with
// at least 16 readable bytes past its end (the tail is read as two masked 8-byte words);
// otherwise key is global and the tail is assembled byte by byte.
template <bool SMEM>
__device__ __forceinline__ uint64_t murmur3_h1(const uint8_t* key, int64_t len) {
  constexpr uint64_t c1 = 0x87c37b91114253d5ULL, c2 = 0x4cf5ad432745937fULL;
  uint64_t h1 = 0, h2 = 0;
  const int64_t nblocks = len >> 4;
  for (int64_t b = 0; b < nblocks; ++b) {
    uint64_t k1 = SMEM ? le64_smem(key + 16 * b) : le64_global(key + 16 * b);
    uint64_t k2 = SMEM ? le64_smem(key + 16 * b + 8) : le64_global(key + 16 * b + 8);
    k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1;
    h1 = rotl64(h1, 27); h1 += h2; h1 = h1 * 5 + 0x52dce729;
    k2 *= c2; k2 = rotl64(k2, 33); k2 *= c1; h2 ^= k2;
    h2 = rotl64(h2, 31); h2 += h1; h2 = h2 * 5 + 0x38495ab5;
  }
  const uint8_t* tail = key + 16 * nblocks;
  const int rem = (int)(len & 15);
  uint64_t k1 = 0, k2 = 0;
  if (SMEM) {
    k1 = low_bytes(le64_smem(tail), min(rem, 8));
    k2 = low_bytes(le64_smem(tail + 8), max(rem - 8, 0));
  } else {
    for (int j = rem - 1; j >= 8; --j) k2 = (k2 << 8) | (uint64_t)__ldg(tail + j);
    for (int j = min(rem, 8) - 1; j >= 0; --j) k1 = (k1 << 8) | (uint64_t)__ldg(tail + j);
  }
  if (rem > 8) { k2 *= c2; k2 = rotl64(k2, 33); k2 *= c1; h2 ^= k2; }
  if (rem > 0) { k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1; }
  h1 ^= (uint64_t)len; h2 ^= (uint64_t)len;
  h1 += h2; h2 += h1;
  h1 = fmix64(h1); h2 = fmix64(h2);
  return h1 + h2;
}

// One thread per string.  A warp's 32 strings are one contiguous byte range; when it fits
// kWarpBytes it is staged in shared memory with 16-B loads (aligned down to 16 B, so the
// last load may touch up to 15 bytes past the range inside the same aligned 16-B block),
// and the threads hash from shared memory instead of issuing one byte load per byte.
constexpr int kHashWarps = 8;
constexpr int kWarpBytes = 2048;

__global__ void __launch_bounds__(32 * kHashWarps)
k_hash_ids(const uint8_t* __restrict__ bytes, const int64_t* __restrict__ str_off, int64_t n,
           uint64_t* __restrict__ out) {
  __shared__ __align__(16) uint8_t sbuf[kHashWarps][kWarpBytes + 32];  // + slack for tail reads
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * kHashWarps;
  for (int64_t base = ((int64_t)blockIdx.x * kHashWarps + w) * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    const int64_t last = min(base + 32, n);
    const int64_t s0 = __ldg(str_off + base), e0 = __ldg(str_off + last);
    const bool live = i < n;
    // dead lanes (past n) hash an empty string at the warp's first byte: every shared-memory
    // address below stays inside the staged range
    const int64_t si = live ? __ldg(str_off + i) : s0, len = live ? __ldg(str_off + i + 1) - si : 0;
    const uintptr_t a0 = (uintptr_t)(bytes + s0) & ~(uintptr_t)15;
    const int64_t span = (int64_t)((uintptr_t)(bytes + e0) - a0);
    uint64_t hv;
    if (span <= kWarpBytes) {  // warp-uniform
      for (int64_t k = lane; 16 * k < span; k += 32)
        reinterpret_cast<uint4*>(sbuf[w])[k] = __ldg(reinterpret_cast<const uint4*>(a0) + k);
      __syncwarp();
      hv = murmur3_h1<true>(sbuf[w] + ((uintptr_t)(bytes + si) - a0), len);
      __syncwarp();
    } else {
      hv = murmur3_h1<false>(bytes + si, len);
    }
    if (live) out[i] = hv;
  }
}

template <bool DUAL, bool WRAP>
__global__ void __launch_bounds__(256)
k_qr_expand(const uint64_t* __restrict__ h, const int32_t* __restrict__ offsets, int64_t nbags,
            int64_t nnz, uint32_t R, uint32_t Q, int32_t* __restrict__ ids_out,
            int32_t* __restrict__ offsets_out, bool vec) {
  constexpr int K = DUAL ? 4 : 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const uint64_t x = __ldg(h + i);
    const uint32_t nB = (uint32_t)x, nC = (uint32_t)(x >> 32);
    uint32_t qB = nB / R;
    const uint32_t rB = nB - qB * R;
    if (WRAP) qB %= Q;
    int32_t r[4];
    r[0] = (int32_t)qB;
    r[1] = (int32_t)(Q + rB);
    if (DUAL) {
      uint32_t qC = nC / R;
      const uint32_t rC = nC - qC * R;
      if (WRAP) qC %= Q;
      r[2] = (int32_t)(Q + R + qC);
      r[3] = (int32_t)(2 * Q + R + rC);
    }
    if (vec) {
      if (DUAL) reinterpret_cast<int4*>(ids_out)[i] = make_int4(r[0], r[1], r[2], r[3]);
      else reinterpret_cast<int2*>(ids_out)[i] = make_int2(r[0], r[1]);
    } else {
#pragma unroll
      for (int j = 0; j < K; ++j) ids_out[K * i + j] = r[j];
    }
  }
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nbags; b += stride)
    offsets_out[b] = K * __ldg(offsets + b);
}

unsigned grid_for(int64_t n) {
  const int64_t want = (n + 255) / 256;
  return (unsigned)(want < 1 ? 1 : (want < 148 * 8 ? want : 148 * 8));
}

}  // namespace

}  // namespace lirank

using namespace lirank;

extern "C" {

int64_t emb_qr_rows(int32_t R, int64_t Q, int32_t dual) {
  if (R < 1 || Q < 1) return -1;
  return (dual ? 2 : 1) * (Q + (int64_t)R);
}

emb_status emb_hash_ids(const uint8_t* bytes, const int64_t* str_offsets, int64_t n,
                        uint64_t* hashes, void* stream) {
  if (n < 0) return EMB_EINVAL;
  if (n == 0) return EMB_OK;
  if (!str_offsets || !hashes || !is_device_ptr(str_offsets) || !is_device_ptr(hashes))
    return EMB_EINVAL;
  if (bytes && !is_device_ptr(bytes)) return EMB_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  k_hash_ids<<<grid_for(n), 32 * kHashWarps, 0, s>>>(bytes, str_offsets, n, hashes);
  return cudaGetLastError() == cudaSuccess ? EMB_OK : EMB_ECUDA;
}

emb_status emb_qr_expand(const uint64_t* hashes, const int32_t* offsets, int64_t nbags,
                         int64_t nnz, int32_t R, int64_t Q, int32_t dual, int32_t* ids_out,
                         int32_t* offsets_out, void* stream) {
  const int64_t rows = emb_qr_rows(R, Q, dual);
  if (rows < 1 || rows >= ((int64_t)1 << 31) || nbags < 0 || nnz < 0) return EMB_EINVAL;
  if (!offsets || !offsets_out || !is_device_ptr(offsets) || !is_device_ptr(offsets_out))
    return EMB_EINVAL;
  if (nnz > 0 && (!hashes || !ids_out || !is_device_ptr(hashes) || !is_device_ptr(ids_out)))
    return EMB_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  // the quotient of a 32-bit n is at most (2^32 - 1) / R: no wrap needed when Q exceeds it
  const bool wrap = (uint64_t)Q <= (uint64_t)0xffffffffu / (uint32_t)R;
  const bool vec = aligned(ids_out, dual ? 16 : 8);
  const unsigned grid = grid_for(std::max<int64_t>(nnz, nbags + 1));
#define QRX(D, W) k_qr_expand<D, W><<<grid, 256, 0, s>>>(hashes, offsets, nbags, nnz, (uint32_t)R, \
                                                       (uint32_t)Q, ids_out, offsets_out, vec)
  if (dual) { if (wrap) QRX(true, true); else QRX(true, false); }
  else { if (wrap) QRX(false, true); else QRX(false, false); }
#undef QRX
  return cudaGetLastError() == cudaSuccess ? EMB_OK : EMB_ECUDA;
}

}  // extern "C"
