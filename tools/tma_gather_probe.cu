// tma_gather_probe.cu -- calibration only (not part of the product): random 96-B row gathers
// (the q8 row of a10) from a 12 GB table, register-staged LDG (4 lanes x 16 B + an 8-B meta
// load per row, UNR rows in flight per group: a10's scheme) vs cp.async.bulk into a
// per-group shared-memory ring of S slots (mbarrier complete_tx), to know whether TMA
// staging can raise a10's rows in flight.  Uniform ids (worst case for L2).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ids(uint32_t* ids, int64_t n, uint64_t rows, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (uint64_t)i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    ids[i] = (uint32_t)(z % rows);
  }
}

template <int UNR, int RB = 96>
__global__ void __launch_bounds__(256) k_ldg(const uint8_t* __restrict__ tab, const uint32_t* __restrict__ ids,
                                             int64_t n, float* out) {
  const int lane = threadIdx.x & 3;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 4;
  const int64_t G = (gridDim.x * (int64_t)blockDim.x) / 4;
  float acc = 0.f;
  for (int64_t i = g * UNR; i < n; i += G * UNR) {
    uint4 r[UNR];
    float2 m[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (i + u < n) {
        const uint8_t* row = tab + (size_t)__ldg(ids + i + u) * RB;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w) : "l"(row + 16 * lane));
        m[u] = *reinterpret_cast<const float2*>(row + 64);
      } else {
        r[u] = make_uint4(0, 0, 0, 0);
        m[u] = make_float2(0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += (float)(r[u].x ^ r[u].y ^ r[u].z ^ r[u].w) * m[u].x + m[u].y;
  }
  if (acc == 12345.f) out[0] = acc;
}

// 256-B rows (a2's fp32 D = 64 row): 8 lanes x 2 x 16 B, UNR rows in flight per group
template <int UNR>
__global__ void __launch_bounds__(256) k_ldg256(const uint8_t* __restrict__ tab, const uint32_t* __restrict__ ids,
                                                int64_t n, float* out) {
  const int lane = threadIdx.x & 7;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 8;
  const int64_t G = (gridDim.x * (int64_t)blockDim.x) / 8;
  float acc = 0.f;
  for (int64_t i = g * UNR; i < n; i += G * UNR) {
    float4 r[UNR][2];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const float4* row = reinterpret_cast<const float4*>(tab + (size_t)__ldg(ids + min(i + u, n - 1)) * 256);
#pragma unroll
      for (int v = 0; v < 2; ++v)
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r[u][v].x), "=f"(r[u][v].y), "=f"(r[u][v].z), "=f"(r[u][v].w) : "l"(row + lane + 8 * v));
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += r[u][0].x + r[u][1].y + r[u][0].z + r[u][1].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

// generic: a 4-lane group reads BYTES (<= 64, in 16-B lane pieces) of each random row at pitch RB
// -- the rows/s rate as a function of row size and pitch alignment
template <int UNR, int RB, int BYTES>
__global__ void __launch_bounds__(256) k_ldgn(const uint8_t* __restrict__ tab, const uint32_t* __restrict__ ids,
                                              int64_t n, float* out) {
  const int lane = threadIdx.x & 3;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 4;
  const int64_t G = (gridDim.x * (int64_t)blockDim.x) / 4;
  float acc = 0.f;
  for (int64_t i = g * UNR; i < n; i += G * UNR) {
    uint4 r[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      r[u] = make_uint4(0, 0, 0, 0);
      if (i + u < n && 16 * lane < BYTES) {
        const uint8_t* row = tab + (size_t)__ldg(ids + i + u) * RB;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w) : "l"(row + 16 * lane));
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += (float)(r[u].x ^ r[u].y ^ r[u].z ^ r[u].w);
  }
  if (acc == 12345.f) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S, int RB = 96>
__global__ void __launch_bounds__(256) k_tma(const uint8_t* __restrict__ tab, const uint32_t* __restrict__ ids,
                                             int64_t n, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int grp = threadIdx.x >> 2, lane = threadIdx.x & 3;  // 64 groups per CTA
  uint8_t* slots = sm + (size_t)grp * S * RB;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + 64 * S * RB) + grp * S;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 4;
  const int64_t G = (gridDim.x * (int64_t)blockDim.x) / 4;
  if (lane == 0)
    for (int q = 0; q < S; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[q])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int q, int64_t i) {
    const uint8_t* src = tab + (size_t)__ldg(ids + i) * RB;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[q])), "n"(RB) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(slots + q * RB)), "l"(src), "n"(RB), "r"(su32(&bars[q])) : "memory");
  };
  if (lane == 0)
    for (int q = 0; q < S; ++q)
      if (g + q * G < n) issue(q, g + q * G);
  float acc = 0.f;
  int it = 0;
  for (int64_t i = g; i < n; i += G, ++it) {
    const int q = it % S;
    const uint32_t par = (it / S) & 1;
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                     su32(&bars[q])), "r"(par) : "memory");
    const uint4 r = reinterpret_cast<const uint4*>(slots + q * RB)[lane];
    const float2 m = *reinterpret_cast<const float2*>(slots + q * RB + 64);
    __syncwarp(0xfu << (threadIdx.x & 28));
    if (lane == 0 && i + S * G < n) issue(q, i + S * G);
    acc += (float)(r.x ^ r.y ^ r.z ^ r.w) * m.x + m.y;
  }
  if (acc == 12345.f) out[0] = acc;
}

// per-lane LDGSTS (cp.async 16 B, L1 bypass) of each 96-B row into a per-group shared-memory ring
// of S slots, one commit group per row: rows in flight without registers
template <int S>
__global__ void __launch_bounds__(256) k_ldgsts(const uint8_t* __restrict__ tab, const uint32_t* __restrict__ ids,
                                                int64_t n, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int grp = threadIdx.x >> 2, lane = threadIdx.x & 3;
  uint8_t* slots = sm + (size_t)grp * S * 96;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 4;
  const int64_t G = (gridDim.x * (int64_t)blockDim.x) / 4;
  auto issue = [&](int q, int64_t i) {
    if (i < n) {
      const uint8_t* src = tab + (size_t)__ldg(ids + i) * 96;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(slots + q * 96 + 16 * lane)), "l"(src + 16 * lane)
                   : "memory");
      if (lane == 0)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(slots + q * 96 + 64)), "l"(src + 64)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int q = 0; q < S; ++q) issue(q, g + q * G);
  float acc = 0.f;
  int it = 0;
  for (int64_t i = g; i < n; i += G, ++it) {
    const int q = it % S;
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
    __syncwarp(0xfu << (threadIdx.x & 28));
    const uint4 r = reinterpret_cast<const uint4*>(slots + q * 96)[lane];
    const float2 m = *reinterpret_cast<const float2*>(slots + q * 96 + 64);
    __syncwarp(0xfu << (threadIdx.x & 28));
    issue(q, i + S * G);
    acc += (float)(r.x ^ r.y ^ r.z ^ r.w) * m.x + m.y;
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const int64_t n = 13238272;
  const uint64_t rows = 125000000;  // 12 GB of 96-B rows (Feed-1's q8 store)
  uint8_t* tab; cudaMalloc(&tab, rows * 96); cudaMemset(tab, 1, rows * 96);
  uint32_t* ids; cudaMalloc(&ids, n * 4);
  float* out; cudaMalloc(&out, 16);
  k_ids<<<1184, 256>>>(ids, n, rows, 7);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("%-28s %.3f ms  %.1f G rows/s\n", name, best, n / best / 1e6);
  };
  timeit("ldg UNR=4 (a10 scheme)", [&] { k_ldg<4><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  timeit("ldg UNR=8", [&] { k_ldg<8><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
#define T(S, CTAS)                                                                                   \
  {                                                                                                  \
    const int smem = 64 * S * 96 + 64 * S * 8;                                                       \
    cudaFuncSetAttribute(k_tma<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);               \
    int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tma<S>, 256, smem);           \
    char nm[64]; snprintf(nm, 64, "tma S=%d (%d CTA/SM)", S, per);                                   \
    timeit(nm, [&] { k_tma<S><<<148 * per * CTAS, 256, smem>>>(tab, ids, n, out); });                \
  }
  T(2, 1) T(4, 1) T(8, 1) T(4, 8) T(8, 8) T(16, 1)
#define L(S)                                                                                         \
  {                                                                                                  \
    const int smem = 64 * S * 96;                                                                    \
    cudaFuncSetAttribute(k_ldgsts<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);            \
    int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_ldgsts<S>, 256, smem);        \
    char nm[64]; snprintf(nm, 64, "ldgsts S=%d (%d CTA/SM)", S, per);                                \
    timeit(nm, [&] { k_ldgsts<S><<<148 * per, 256, smem>>>(tab, ids, n, out); });                    \
  }
  L(4) L(8) L(12) L(16)
  // rows/s by row size and pitch (the same 12 GB region, ids < rows): 16, 32, 64 B at pitch 96;
  // 64 B at pitch 64 (one atom, aligned) and 128 B rows at pitch 128 (1 line) from rows*96/128 rows
  timeit("16B of 96-B rows", [&] { k_ldgn<4, 96, 16><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  timeit("32B of 96-B rows", [&] { k_ldgn<4, 96, 32><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  timeit("64B of 96-B rows", [&] { k_ldgn<4, 96, 64><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  timeit("64B rows, pitch 64", [&] { k_ldgn<4, 64, 64><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  k_ids<<<1184, 256>>>(ids, n, rows * 96 / 128, 11);
  timeit("64B of 128-B rows", [&] { k_ldgn<4, 128, 64><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  timeit("64B of 128-B rows UNR8", [&] { k_ldgn<8, 128, 64><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  // the whole a10 row (64 codes + 8-B meta at +64) at a 128-B pitch: one 128-B line per row
  timeit("a10 row, pitch 128 UNR4", [&] { k_ldg<4, 128><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  timeit("a10 row, pitch 128 UNR8", [&] { k_ldg<8, 128><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  k_ids<<<1184, 256>>>(ids, n, rows, 7);
  timeit("a10 row, pitch 96 UNR4", [&] { k_ldg<4, 96><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  // even rows only at pitch 96 (rows that never straddle a 128-B line)
  k_ids<<<1184, 256>>>(ids, n, rows / 2, 7);
  timeit("a10 row, pitch 192 UNR4", [&] { k_ldg<4, 192><<<148 * 4 * 4, 256>>>(tab, ids, n, out); });
  // 256-B rows from a 32 GB table (a2's fp32 rows)
  uint8_t* tab2 = nullptr;
  const uint64_t rows2 = 125000000;
  cudaFree(tab);
  if (cudaMalloc(&tab2, rows2 * 256) == cudaSuccess) {
    cudaMemset(tab2, 1, rows2 * 256);
    k_ids<<<1184, 256>>>(ids, n, rows2, 9);
    timeit("256B ldg UNR=2 (a2 scheme)", [&] { k_ldg256<2><<<148 * 5 * 4, 256>>>(tab2, ids, n, out); });
    timeit("256B ldg UNR=4", [&] { k_ldg256<4><<<148 * 4 * 4, 256>>>(tab2, ids, n, out); });
#define T2(S)                                                                                        \
  {                                                                                                  \
    const int smem = 64 * S * 256 + 64 * S * 8;                                                      \
    cudaFuncSetAttribute(k_tma<S, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);          \
    int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tma<S, 256>, 256, smem);      \
    char nm[64]; snprintf(nm, 64, "256B tma S=%d (%d CTA/SM)", S, per);                              \
    timeit(nm, [&] { k_tma<S, 256><<<148 * per, 256, smem>>>(tab2, ids, n, out); });                 \
  }
    T2(2) T2(4) T2(6)
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
