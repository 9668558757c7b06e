// cub_sort_probe.cu -- calibration only (not part of the product): CUB DeviceRadixSort on
// n (key, value) pairs with `bits` key bits, Zipf-like keys, to know what a library onesweep
// achieves on this part for the dedup's sort.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>

__global__ void k_keys(uint32_t* k, uint32_t* v, int64_t n, uint32_t rows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
    uint32_t r = (uint32_t)(exp(log((double)rows) * u));  // log-uniform ~ Zipf(1)
    k[i] = (uint32_t)(((uint64_t)r * 2654435761ull) % rows);
    v[i] = (uint32_t)i;
  }
}

int main() {
  const int64_t n = 13238272;
  const uint32_t rows = 125000000;
  uint32_t *k0, *k1, *v0, *v1;
  cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
  k_keys<<<1184, 256>>>(k0, v0, n, rows);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, (int)n, 0, 27);
  void* t; cudaMalloc(&t, tmp);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bits : {27, 32}) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, v0, v1, (int)n, 0, bits);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("cub SortPairs n=%lld bits=%d: %.3f ms (%.1f G pairs/s)\n", (long long)n, bits, best, n / best / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
