// gather_probe.cu -- measures the random-row gather ceiling of this B200: n random rows of
// `row_bytes` gathered from a table of `table_gb` GB (uniform ids, max memory-level
// parallelism: ids precomputed, 8 independent 16-B loads in flight per thread, summed to
// defeat DCE).  Separates TLB/page-walk effects (table size) from pure DRAM/L2 effects.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_ids(uint32_t* ids, int64_t n, uint64_t rows, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (uint64_t)i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    ids[i] = (uint32_t)(z % rows);
  }
}

// LPR lanes per row, each lane one 16-B vector; UNR rows in flight per group.
template <int LPR, int UNR>
__global__ void __launch_bounds__(256) k_gather(const float4* __restrict__ tab, int vec_per_row,
                                                const uint32_t* __restrict__ ids, int64_t n, float* out) {
  const int lane = threadIdx.x % LPR;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR;
  const int64_t G = (gridDim.x * (int64_t)blockDim.x) / LPR;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t i = g * UNR; i < n; i += G * UNR) {
    float4 r[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (i + u < n) {
        const uint32_t id = __ldg(ids + i + u);
        const float4* p = tab + (size_t)id * vec_per_row + lane;
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r[u].x), "=f"(r[u].y), "=f"(r[u].z), "=f"(r[u].w) : "l"(p));
      } else r[u] = make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) { acc.x += r[u].x; acc.y += r[u].y; acc.z += r[u].z; acc.w += r[u].w; }
  }
  if (acc.x == 12345.f) out[0] = acc.y + acc.z + acc.w;
}

int main(int argc, char** argv) {
  const int64_t n = 13238272;
  float* out; cudaMalloc(&out, 16);
  uint32_t* ids; cudaMalloc(&ids, n * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double gbs[] = {0.5, 2, 8, 32, 64, 128};
  const int rbs[] = {256, 64};
  size_t maxb = (size_t)(128.0 * (1ull << 30));
  char* tab = nullptr;
  if (cudaMalloc(&tab, maxb) != cudaSuccess) { maxb = (size_t)64 << 30; cudaGetLastError(); cudaMalloc(&tab, maxb); }
  cudaMemset(tab, 0, maxb);
  for (int rb : rbs) for (double g : gbs) {
    size_t bytes = (size_t)(g * (1ull << 30));
    if (bytes > maxb) continue;
    uint64_t rows = bytes / rb;
    k_ids<<<1184, 256>>>(ids, n, rows, 12345);
    const int vpr = rb / 16;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      if (vpr == 16) k_gather<16, 8><<<148 * 8, 256>>>((const float4*)tab, vpr, ids, n, out);
      else k_gather<4, 8><<<148 * 8, 256>>>((const float4*)tab, vpr, ids, n, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    double alg = (double)n * (rb + 4);
    printf("row %3d B  table %6.1f GB  n %lld  %.3f ms  %.0f GB/s (alg)  %.2f Grows/s\n", rb, g, (long long)n, best, alg / best / 1e6, n / best / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
