// forward.cu -- a2 fp32 pooled lookup and a10 q8 pooled lookup (sm_100a).
//
// a2: out[b][f][:] = sum over j in bag(f,b), in bag order, of
// W[key_j][:]; MEAN divides by the bag length; empty bag -> 0; invalid ids skipped.
// a10: the same over the q8 store, each term fmaf(code, scale, middle).
//
// Design (B200): one group of LPB lanes per bag (D=64 -> half-warp), 128-bit row loads
// (ld.global.nc.L1::no_allocate: rows are streamed, L2 keeps Zipf-hot rows), ids of a
// bag loaded LPB at a time and broadcast by shuffle, row loads of UNR ids issued before
// the in-order adds.  Grid: one group per bag, 256-thread CTAs.  The fp32 kernel also
// emits the (row key, bag) pair of every occurrence for the backward's dedup, so the
// backward never re-reads ids/offsets (8 extra bytes written per id).
#include "common.cuh"
#include "kernels.h"

namespace lirank {

template <int LPB, int VPL, bool MEAN, bool EMIT>
__global__ void __launch_bounds__(256)
k_pool_fwd_f32(const float* __restrict__ W, int pitch, const int* __restrict__ ids,
               const int* __restrict__ offsets, int B, int F, int D,
               const FeatMeta* __restrict__ meta, float* __restrict__ out,
               uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
               uint32_t sentinel, uint32_t* status) {
  constexpr int UNR = (VPL == 1) ? 4 : (VPL == 2 ? 2 : 1);
  const int lane = threadIdx.x & (LPB - 1);
  const long long bag = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
  if (bag >= (long long)F * B) return;
  const unsigned gmask = group_mask<LPB>();
  const int f = (int)(bag / B);
  const int b = (int)(bag - (long long)f * B);
  const FeatMeta m = meta[f];
  const int lo = __ldg(offsets + bag);
  const int hi = __ldg(offsets + bag + 1);
  const int nvec = pitch >> 2;

  float4 acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);

  bool bad = false;
  for (int j0 = lo; j0 < hi; j0 += LPB) {
    const int j = j0 + lane;
    uint32_t key = sentinel;
    if (j < hi) {
      const int id = ld_nc_i32(ids + j);
      const bool valid = id >= 0 && id < m.rows;
      bad |= !valid;
      if (valid && id >= m.lo && id < m.hi) key = (uint32_t)(m.base + (id - m.lo));
      if (EMIT) {
        keys_out[j] = key;
        vals_out[j] = (uint32_t)bag;
      }
    }
    const int cnt = min(LPB, hi - j0);
    for (int jj = 0; jj < cnt; jj += UNR) {
      uint32_t k[UNR];
      float4 r[UNR][VPL];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        k[u] = __shfl_sync(gmask, key, (jj + u) & (LPB - 1), LPB);
        if (jj + u >= cnt) k[u] = sentinel;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (k[u] != sentinel) {
          const float* row = W + (size_t)k[u] * pitch;
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            const int vi = lane + v * LPB;
            r[u][v] = (VPL * LPB == 1 || vi < nvec) ? ld_nc_f4(row + 4 * vi)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (k[u] != sentinel) {
#pragma unroll
          for (int v = 0; v < VPL; ++v) acc[v] = f4_add_rn(acc[v], r[u][v]);
        }
    }
  }
  if (bad) set_status(status, kStIdRange);

  if (MEAN) {
    const int L = hi - lo;
    if (L > 0) {
      const float fl = (float)L;
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        acc[v] = make_float4(__fdiv_rn(acc[v].x, fl), __fdiv_rn(acc[v].y, fl),
                             __fdiv_rn(acc[v].z, fl), __fdiv_rn(acc[v].w, fl));
    }
  }
  float* o = out + ((size_t)b * F + f) * D;
  if ((D & 3) == 0) {
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int vi = lane + v * LPB;
      if (4 * vi < D) st_f4(o + 4 * vi, acc[v]);
    }
  } else {
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int d = 4 * (lane + v * LPB);
      if (d + 0 < D) o[d + 0] = acc[v].x;
      if (d + 1 < D) o[d + 1] = acc[v].y;
      if (d + 2 < D) o[d + 2] = acc[v].z;
      if (d + 3 < D) o[d + 3] = acc[v].w;
    }
  }
}

__device__ __forceinline__ float4 deq4(uint32_t w, float scale, float middle) {
  // X^dequant = X^middle + X^int * X^scale, one fmaf per element (reading 7)
  const float c0 = (float)(int)(int8_t)(w & 0xffu);
  const float c1 = (float)(int)(int8_t)((w >> 8) & 0xffu);
  const float c2 = (float)(int)(int8_t)((w >> 16) & 0xffu);
  const float c3 = (float)(int)(int8_t)(w >> 24);
  return make_float4(__fmaf_rn(c0, scale, middle), __fmaf_rn(c1, scale, middle),
                     __fmaf_rn(c2, scale, middle), __fmaf_rn(c3, scale, middle));
}

// a10.  Lane l of a group reads code words l, l+LPB, ... (4 codes each) of the row and the
// row's {middle, scale} (one broadcast 8-B load per group).
template <int LPB, int VPL, bool MEAN>
__global__ void __launch_bounds__(256)
k_pool_fwd_q8(const uint8_t* __restrict__ codes, int qpitch, const float2* __restrict__ qmeta,
              const int* __restrict__ ids, const int* __restrict__ offsets, int B, int F,
              int D, const FeatMeta* __restrict__ meta, float* __restrict__ out,
              uint32_t* status) {
  constexpr int UNR = (VPL == 1) ? 4 : (VPL == 2 ? 2 : 1);
  const int lane = threadIdx.x & (LPB - 1);
  const long long bag = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
  if (bag >= (long long)F * B) return;
  const unsigned gmask = group_mask<LPB>();
  const int f = (int)(bag / B);
  const int b = (int)(bag - (long long)f * B);
  const FeatMeta m = meta[f];
  const int lo = __ldg(offsets + bag);
  const int hi = __ldg(offsets + bag + 1);
  const int nw = (D + 3) >> 2;  // code words that carry dims < D
  constexpr uint32_t kNone = 0xffffffffu;

  float4 acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);

  bool bad = false;
  for (int j0 = lo; j0 < hi; j0 += LPB) {
    const int j = j0 + lane;
    uint32_t key = kNone;
    if (j < hi) {
      const int id = ld_nc_i32(ids + j);
      const bool valid = id >= 0 && id < m.rows;
      bad |= !valid;
      if (valid && id >= m.lo && id < m.hi) key = (uint32_t)(m.base + (id - m.lo));
    }
    const int cnt = min(LPB, hi - j0);
    for (int jj = 0; jj < cnt; jj += UNR) {
      uint32_t k[UNR];
      uint32_t w[UNR][VPL];
      float2 mt[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        k[u] = __shfl_sync(gmask, key, (jj + u) & (LPB - 1), LPB);
        if (jj + u >= cnt) k[u] = kNone;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (k[u] != kNone) {
          mt[u] = __ldg(qmeta + k[u]);
          const uint32_t* row = reinterpret_cast<const uint32_t*>(codes + (size_t)k[u] * qpitch);
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            const int wi = lane + v * LPB;
            w[u][v] = (wi < nw) ? (uint32_t)ld_nc_i32(reinterpret_cast<const int*>(row + wi)) : 0u;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (k[u] != kNone) {
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            acc[v] = f4_add_rn(acc[v], deq4(w[u][v], mt[u].y, mt[u].x));
        }
    }
  }
  if (bad) set_status(status, kStIdRange);

  if (MEAN) {
    const int L = hi - lo;
    if (L > 0) {
      const float fl = (float)L;
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        acc[v] = make_float4(__fdiv_rn(acc[v].x, fl), __fdiv_rn(acc[v].y, fl),
                             __fdiv_rn(acc[v].z, fl), __fdiv_rn(acc[v].w, fl));
    }
  }
  float* o = out + ((size_t)b * F + f) * D;
  if ((D & 3) == 0) {
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int vi = lane + v * LPB;
      if (4 * vi < D) st_f4(o + 4 * vi, acc[v]);
    }
  } else {
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int d = 4 * (lane + v * LPB);
      if (d + 0 < D) o[d + 0] = acc[v].x;
      if (d + 1 < D) o[d + 1] = acc[v].y;
      if (d + 2 < D) o[d + 2] = acc[v].z;
      if (d + 3 < D) o[d + 3] = acc[v].w;
    }
  }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------

#define LIRANK_GEOM_DISPATCH(G, KERNEL_LAUNCH)                              \
  do {                                                                      \
    if ((G).lpb == 1) { constexpr int L_ = 1, V_ = 1; KERNEL_LAUNCH; }      \
    else if ((G).lpb == 2) { constexpr int L_ = 2, V_ = 1; KERNEL_LAUNCH; } \
    else if ((G).lpb == 4) { constexpr int L_ = 4, V_ = 1; KERNEL_LAUNCH; } \
    else if ((G).lpb == 8) { constexpr int L_ = 8, V_ = 1; KERNEL_LAUNCH; } \
    else if ((G).lpb == 16) { constexpr int L_ = 16, V_ = 1; KERNEL_LAUNCH; } \
    else if ((G).vpl == 1) { constexpr int L_ = 32, V_ = 1; KERNEL_LAUNCH; } \
    else if ((G).vpl == 2) { constexpr int L_ = 32, V_ = 2; KERNEL_LAUNCH; } \
    else if ((G).vpl <= 4) { constexpr int L_ = 32, V_ = 4; KERNEL_LAUNCH; } \
    else { constexpr int L_ = 32, V_ = 8; KERNEL_LAUNCH; }                  \
  } while (0)

cudaError_t launch_pool_fwd_f32(const FwdArgs& a, cudaStream_t s) {
  const Geom g = geom_for(a.pitch);
  const long long bags = (long long)a.F * a.B;
  if (bags == 0) return cudaSuccess;
  const long long threads = bags * g.lpb;
  const unsigned grid = (unsigned)((threads + 255) / 256);
#define LAUNCH_F32(MEAN, EMIT)                                                             \
  LIRANK_GEOM_DISPATCH(g, (k_pool_fwd_f32<L_, V_, MEAN, EMIT><<<grid, 256, 0, s>>>(        \
                              a.W, a.pitch, a.ids, a.offsets, a.B, a.F, a.D, a.meta, a.out, \
                              a.keys_out, a.vals_out, a.sentinel, a.status)))
  if (a.mean) {
    if (a.keys_out) LAUNCH_F32(true, true); else LAUNCH_F32(true, false);
  } else {
    if (a.keys_out) LAUNCH_F32(false, true); else LAUNCH_F32(false, false);
  }
#undef LAUNCH_F32
  return cudaGetLastError();
}

cudaError_t launch_pool_fwd_q8(const FwdQ8Args& a, cudaStream_t s) {
  // geometry over 32-bit code words (4 dims each)
  const Geom g = geom_for(4 * ((a.D + 3) / 4));
  const long long bags = (long long)a.F * a.B;
  if (bags == 0) return cudaSuccess;
  const long long threads = bags * g.lpb;
  const unsigned grid = (unsigned)((threads + 255) / 256);
#define LAUNCH_Q8(MEAN)                                                                    \
  LIRANK_GEOM_DISPATCH(g, (k_pool_fwd_q8<L_, V_, MEAN><<<grid, 256, 0, s>>>(               \
                              a.codes, a.qpitch, a.qmeta, a.ids, a.offsets, a.B, a.F, a.D, \
                              a.meta, a.out, a.status)))
  if (a.mean) LAUNCH_Q8(true); else LAUNCH_Q8(false);
#undef LAUNCH_Q8
  return cudaGetLastError();
}

}  // namespace lirank
