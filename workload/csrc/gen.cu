// gen.cu -- GPU copy of the seeded input generator of workload/gen.py (test/bench input
// plumbing, NOT part of the product library and holding none of the method's arithmetic).
// Bit-identical to the numpy implementation: SplitMix64 outputs addressed by counter,
// Irwin-Hall(4) sums of 22-bit uniforms scaled by 2^-shift (exact in fp32).
#include <cuda_runtime.h>
#include <stdint.h>

#define WL_API extern "C" __attribute__((visibility("default")))

static constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__host__ __device__ static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed + (stream + 1) * kGamma);
}

__device__ static inline float ih4(uint64_t key, uint64_t e, int shift) {
  const uint64_t h1 = mix64(key + (2 * e + 1) * kGamma);
  const uint64_t h2 = mix64(key + (2 * e + 2) * kGamma);
  const uint64_t m = (1ull << 22) - 1;
  const int64_t s = (int64_t)((h1 & m) + ((h1 >> 22) & m) + (h2 & m) + ((h2 >> 22) & m)) - (1ll << 23);
  return ldexpf((float)s, -shift);  // |s| <= 2^23: exact
}

// dst[r][d] (row pitch `pitch` floats) = value of (table, row0 + r, d), d < dim; pads = 0.
__global__ void k_fill_table(float* dst, int64_t nrows, int dim, int pitch, uint64_t key,
                             int64_t row0, int shift) {
  const int64_t total = nrows * pitch;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / pitch;
    const int d = (int)(i - r * pitch);
    dst[i] = d < dim ? ih4(key, (uint64_t)(row0 + r) * dim + d, shift) : 0.0f;
  }
}

// dst[b][f][d] = grad value of (sample0 + b, f, d).
__global__ void k_fill_grad(float* dst, int64_t batch, int F, int dim, uint64_t key,
                            int64_t sample0, int shift) {
  const int64_t total = batch * F * dim;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    dst[i] = ih4(key, (uint64_t)(sample0 * F * dim) + (uint64_t)i, shift);
  }
}

WL_API int wl_fill_table(float* dst, int64_t nrows, int dim, int pitch, uint64_t seed, int table,
                         int64_t row0, int shift, void* stream) {
  if (nrows <= 0) return 0;
  k_fill_table<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(dst, nrows, dim, pitch,
                                                           stream_key(seed, (uint64_t)table), row0, shift);
  return (int)cudaGetLastError();
}

WL_API int wl_fill_grad(float* dst, int64_t batch, int F, int dim, uint64_t seed, int64_t step,
                        int64_t sample0, int shift, void* stream) {
  if (batch <= 0) return 0;
  k_fill_grad<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(
      dst, batch, F, dim, stream_key(seed, (1ull << 32) + (uint64_t)step), sample0, shift);
  return (int)cudaGetLastError();
}

// Write a buffer larger than L2 (L2 flush between timed iterations).
__global__ void k_flush(uint4* p, int64_t n, uint32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(v, v, v, v);
}

WL_API int wl_flush(void* buf, int64_t bytes, uint32_t v, void* stream) {
  k_flush<<<148 * 8, 256, 0, (cudaStream_t)stream>>>((uint4*)buf, bytes / 16, v);
  return (int)cudaGetLastError();
}
