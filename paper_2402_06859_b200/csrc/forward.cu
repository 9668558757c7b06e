// forward.cu -- a2 fp32 pooled lookup and a10 q8 pooled lookup (sm_100a).
//
// a2: out[b][f][:] = sum over j in bag(f,b), in bag order, of
// W[key_j][:]; MEAN divides by the bag length; empty bag -> 0; invalid ids skipped.
// a10: the same over the q8 store, each term fmaf(code, scale, middle).
//
// Design (B200).  One group of LPB lanes per bag (D=64 fp32: 8 lanes x two 128-bit loads
// = one 256-B row, 4 bags per warp).  The group loads LPB ids at once (one per lane) and broadcasts them by
// full-mask shuffles (the id loop runs to the longest bag of the warp, so every lane
// reaches every shuffle); it then issues the row loads of UNR ids back to back before
// adding them in bag order.  Row loads allocate in L1 and carry an L2 evict_last hint:
// Zipf-hot rows are re-read on every SM, and an SM-local L1 hit saves the L2 round trip and
// takes the hottest rows' traffic off their single L2 slice (measured against
// L1::no_allocate: Feed-1 a2 0.452 -> 0.389 ms, alpha 1.2 0.650 -> 0.331 ms, a10 0.307 ->
// 0.274 ms).  (Per-slot id loads by every lane made the id->row dependence
// chain 4x longer and were measurably slower.)  Measured
// (profiles/): a random 256-B row gather on this part is DRAM-activation bound at
// ~24 G rows/s (~6.3 TB/s) for uniform ids; this kernel runs the Feed-1 batch at that
// rate incl. its offsets/ids/outputs.  A CTA-staged variant (offsets + ids through shared
// memory, 4 bags per group) was slower (fewer independent groups in flight) and was
// dropped.  The fp32 kernel also emits, per occurrence, the packed {row key, grad row}
// pair the backward's dedup sorts (8 B per id), so the backward never re-reads ids or
// offsets.
#include "common.cuh"
#include "kernels.h"

namespace lirank {

namespace {

__device__ __forceinline__ uint32_t row_key(int id, const FeatMeta& m, uint32_t none, bool& bad) {
  const bool valid = id >= 0 && id < m.rows;
  bad |= !valid;
  return (valid && id >= m.lo && id < m.hi) ? (uint32_t)(m.base + (id - m.lo)) : none;
}

template <int N>
__device__ __forceinline__ void mean_div(float4 (&acc)[N], int L) {
  if (L <= 0) return;
  const float fl = (float)L;
#pragma unroll
  for (int v = 0; v < N; ++v)
    acc[v] = make_float4(__fdiv_rn(acc[v].x, fl), __fdiv_rn(acc[v].y, fl),
                         __fdiv_rn(acc[v].z, fl), __fdiv_rn(acc[v].w, fl));
}

__device__ __forceinline__ void store4(float* o, int d, int D, float4 a) {
  if ((D & 3) == 0) {
    if (d < D) st_f4(o + d, a);
  } else {
    if (d + 0 < D) o[d + 0] = a.x;
    if (d + 1 < D) o[d + 1] = a.y;
    if (d + 2 < D) o[d + 2] = a.z;
    if (d + 3 < D) o[d + 3] = a.w;
  }
}

// Output row of bag (f, b) where the F features form source blocks of Fb features each:
// out row = (blk * B + b) * Fb + (f % Fb).  Unsharded: Fb = F, row = b * F + f.
__device__ __forceinline__ size_t out_row(int f, int b, int B, int Fb) {
  const int blk = f / Fb;
  return ((size_t)blk * B + b) * Fb + (f - blk * Fb);
}

// Destination of the pooled row with block-order index grow (= out_row): `out` in block
// order, or (fused exchange) the source rank's buffer through its peer mapping.
template <bool PEER>
__device__ __forceinline__ float* dst_row(float* out, uint32_t grow, int B, int Fb, int D,
                                          const PeerOut& pm) {
  if (!PEER) return out + (size_t)grow * D;
  const uint32_t per = (uint32_t)B * (uint32_t)Fb;
  const uint32_t blk = grow / per, rem = grow - blk * per;
  const uint32_t b = rem / (uint32_t)Fb, j = rem - b * (uint32_t)Fb;
  return pm.base[blk] + ((size_t)((size_t)pm.slot * B + b) * pm.F_out + __ldg(pm.fcol + j)) * D;
}

}  // namespace

// FR (full rows: D == pitch == 4 * LPB * VPL, the D = 64 geometry): compile-time row size,
// no bounds logic on the row loads and stores (the bounds / address arithmetic was ~40% of
// the kernel's instructions on the ncu source page).
template <int LPB, int VPL, bool MEAN, bool EMIT, bool PEER, bool FR>
__global__ void __launch_bounds__(256)
k_pool_fwd_f32(const float* __restrict__ W, int pitch, const int* __restrict__ ids,
               const int* __restrict__ offsets, int B, int F, int Fb, int D,
               const FeatMeta* __restrict__ meta, float* __restrict__ out,
               uint2* __restrict__ kv_out, uint32_t sentinel, uint32_t* status,
              const uint32_t* __restrict__ order, bool skip_short, const PeerOut pm) {
  pdl_wait();
  // rows in flight per group (D = 64 full rows, measured: 2 -> 0.343 ms at 48 registers, 3 ->
  // 0.361 at 56, 4 -> 0.359 at 64; at alpha 0 all within 1%).  Occupancy (round 2): 6 CTAs/SM
  // at 40 registers spills, 0.351 ms; 7 at 32, 0.503 -- the default 5 at 48 stays.
  constexpr int UNR = (VPL == 1) ? 4 : (VPL == 2 ? 2 : 1);
  constexpr unsigned kFull = 0xffffffffu;
  if (FR) { D = 4 * LPB * VPL; pitch = D; }
  const int lane = threadIdx.x & (LPB - 1);
  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
  const bool in_range = gid < (long long)F * B;  // predicate, never return: shuffles below
  const long long bag = (order != nullptr && in_range) ? (long long)__ldg(order + gid) : gid;
  const int lo = in_range ? __ldg(offsets + bag) : 0;
  const int hi = in_range ? __ldg(offsets + bag + 1) : 0;
  // bags of <= 1 id are k_pool_short_f32's when skip_short (it batches LPB of them per group)
  const bool live = in_range && !(skip_short && hi - lo <= 1);
  const int len = live ? hi - lo : 0;
  const int f = live ? (int)(bag / B) : 0;
  const int b = live ? (int)(bag - (long long)f * B) : 0;
  const FeatMeta m = meta[f];
  const int nvec = pitch >> 2;
  const uint32_t grow = (uint32_t)out_row(f, b, B, Fb);
  const uint64_t pol_last = l2_policy_last();
  float4 acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  bool bad = false;
  // Warp-uniform trip count (the longest bag among the warp's groups): every lane reaches
  // every shuffle, so shuffles use the full mask; shorter bags are predicated.
  const int maxlen = __reduce_max_sync(kFull, len);
  // ids are loaded one batch ahead (one per lane, LPB per group), so the next batch's id
  // loads overlap this batch's row gathers instead of following them
  uint32_t key_next = sentinel;
  if (lane < len) {
    key_next = row_key(__ldg(ids + lo + lane), m, sentinel, bad);
    if (EMIT) kv_out[lo + lane] = make_uint2(key_next, grow);
  }
  for (int j0 = 0; j0 < maxlen; j0 += LPB) {
    const uint32_t key = key_next;
    const int jn = j0 + LPB + lane;
    key_next = sentinel;
    if (jn < len) {
      key_next = row_key(__ldg(ids + lo + jn), m, sentinel, bad);
      if (EMIT) kv_out[lo + jn] = make_uint2(key_next, grow);
    }
#pragma unroll
    for (int jj = 0; jj < LPB; jj += UNR) {
      uint32_t k[UNR];
      float4 r[UNR][VPL];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        k[u] = __shfl_sync(kFull, key, (jj + u) & (LPB - 1), LPB);
        if (jj + u >= LPB || j0 + jj + u >= len) k[u] = sentinel;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (k[u] != sentinel) {
          const float* row = W + (size_t)k[u] * pitch;
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            const int vi = lane + v * LPB;
            r[u][v] = (FR || vi < nvec) ? ld_l1_f4_hint(row + 4 * vi, pol_last) : make_float4(0.f, 0.f, 0.f, 0.f);
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
  if (!live) return;
  if (bad) set_status(status, kStIdRange);  // any lane: each lane validated its own ids
  if (PEER && pm.skip_empty && len == 0) return;
  if (MEAN) mean_div(acc, len);
  float* o = dst_row<PEER>(out, grow, B, Fb, D, pm);
  if ((D & 3) == 0) {
    const uint64_t pol_first = l2_policy_first();
#pragma unroll
    for (int v = 0; v < VPL; ++v)
      if (FR || 4 * (lane + v * LPB) < D) st_f4_hint(o + 4 * (lane + v * LPB), acc[v], pol_first);
  } else {
#pragma unroll
    for (int v = 0; v < VPL; ++v) store4(o, 4 * (lane + v * LPB), D, acc[v]);
  }
}

// Bags of at most one id (one-hot features, empty bags).  The main kernel gives each bag a
// lane group and keeps UNR of its ids' rows in flight; a one-id bag leaves one row in flight
// per group.  Here a group serves LPB consecutive (ordered) positions -- lane l resolves the
// bag at position LPB*g + l and loads its id -- and gathers their rows UNR at a time, so
// one-hot-heavy batches keep as many rows in flight as multi-hot ones.  Positions whose bag
// has more ids are left to the main kernel.  A one-id bag's pooled value is its row (SUM and
// MEAN alike); an empty bag's is 0.
template <int LPB, int VPL, bool EMIT, bool PEER, bool FR>
__global__ void __launch_bounds__(256)
k_pool_short_f32(const float* __restrict__ W, int pitch, const int* __restrict__ ids,
                 const int* __restrict__ offsets, int B, int F, int Fb, int D,
                 const FeatMeta* __restrict__ meta, float* __restrict__ out,
                 uint2* __restrict__ kv_out, uint32_t sentinel, uint32_t* status,
                 const uint32_t* __restrict__ order, const PeerOut pm) {
  pdl_wait();
  constexpr int UNR = VPL >= 4 ? 2 : 4;
  constexpr unsigned kFull = 0xffffffffu;
  if (FR) { D = 4 * LPB * VPL; pitch = D; }
  const int lane = threadIdx.x & (LPB - 1);
  const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
  const long long nb = (long long)F * B;
  const long long pos = g * LPB + lane;
  bool mine = pos < nb;
  const long long bag = mine ? (order != nullptr ? (long long)__ldg(order + pos) : pos) : 0;
  const int lo = mine ? __ldg(offsets + bag) : 0;
  const int len = mine ? __ldg(offsets + bag + 1) - lo : 2;
  mine = mine && len <= 1 && !(PEER && pm.skip_empty && len == 0);
  uint32_t key = sentinel, grow = 0;
  bool bad = false;
  if (mine) {
    const int f = (int)(bag / B), b = (int)(bag - (long long)f * B);
    grow = (uint32_t)out_row(f, b, B, Fb);
    if (len == 1) {
      key = row_key(__ldg(ids + lo), meta[f], sentinel, bad);
      if (EMIT) kv_out[lo] = make_uint2(key, grow);
    }
  }
  const int nvec = pitch >> 2;
  const uint64_t pol_last = l2_policy_last();
#pragma unroll
  for (int j = 0; j < LPB; j += UNR) {
    uint32_t k[UNR], gr[UNR];
    bool mm[UNR];
    float4 r[UNR][VPL];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int src = (j + u) & (LPB - 1);
      k[u] = __shfl_sync(kFull, key, src, LPB);
      gr[u] = __shfl_sync(kFull, grow, src, LPB);
      mm[u] = __shfl_sync(kFull, (int)mine, src, LPB) != 0 && j + u < LPB;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int vi = lane + v * LPB;
        r[u][v] = (mm[u] && k[u] != sentinel && (FR || vi < nvec)) ? ld_l1_f4_hint(W + (size_t)k[u] * pitch + 4 * vi, pol_last)
                                                          : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u)
      if (mm[u]) {
        float* o = dst_row<PEER>(out, gr[u], B, Fb, D, pm);
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);  // 0 + row, as the main kernel (-0 -> +0)
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          if (FR) st_f4(o + 4 * (lane + v * LPB), f4_add_rn(z, r[u][v]));
          else store4(o, 4 * (lane + v * LPB), D, f4_add_rn(z, r[u][v]));
        }
      }
  }
  if (bad) set_status(status, kStIdRange);
}

// X^dequant = X^middle + X^int * X^scale: one fmaf per element (reading 7).
// The int8 code becomes an exact float without a conversion instruction: with
// u = byte ^ 0x80 = code + 128, the float with bits 0x4B0000uu is 2^23 + u, so
// (2^23 + u) - (2^23 + 128) = code exactly.
// Min-max stores (NEXT-4) hold unsigned codes u directly: xmask = 0 and magic = 2^23.
// 4 codes (one 32-bit word) -> acc += base + code * scale, element by element (each element
// exactly fl(acc + fmaf(code, scale, base)); the magic subtraction, fma and add run paired,
// FADD2 / FFMA2, two elements per instruction).
__device__ __forceinline__ float code_bits(uint32_t x, uint32_t sel) {  // 2^23 + u
  return __int_as_float((int)__byte_perm(x, 0x4B000000u, sel));
}
__device__ __forceinline__ float4 deq4_add(float4 acc, uint32_t w, float scale, float middle,
                                           uint32_t xmask, float magic) {
  const uint32_t x = w ^ xmask;
  const float2 nm = make_float2(-magic, -magic), sc = make_float2(scale, scale),
               md = make_float2(middle, middle);
  const float2 c01 = f2_add_rn(make_float2(code_bits(x, 0x7540), code_bits(x, 0x7541)), nm);
  const float2 c23 = f2_add_rn(make_float2(code_bits(x, 0x7542), code_bits(x, 0x7543)), nm);
  const float2 a01 = f2_add_rn(make_float2(acc.x, acc.y), f2_fma_rn(c01, sc, md));
  const float2 a23 = f2_add_rn(make_float2(acc.z, acc.w), f2_fma_rn(c23, sc, md));
  return make_float4(a01.x, a01.y, a23.x, a23.y);
}
__device__ __forceinline__ uint4 ld_l1_u4_hint(const void* p, uint64_t pol) {  // L1-allocating
  uint4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint4 ld_nc_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// a10.  q8 row layout: [codes: D int8][pad to 8][middle f32][scale f32][pad to 32]
// (D=64: 96 B = 3 whole sectors).  Lane l of a group of LPB lanes reads 16-code vectors
// l, l+LPB, ... (one 16-B load each) and the row's {middle, scale} (8 B, same address for
// the group).  D=64: 4 lanes per bag, 8 bags per warp, 16 dims per lane.  As in the fp32
// kernel, ids are loaded LPB at a time and broadcast by full-mask shuffles over a
// warp-uniform trip count, so a lane spends its instructions on the dequant, not on
// per-slot key arithmetic.
template <int LPB, int VPL, bool MEAN, bool PEER>
__global__ void __launch_bounds__(256, 4)
k_pool_fwd_q8(const uint8_t* __restrict__ codes, int qpitch, int meta_off,
              const int* __restrict__ ids, const int* __restrict__ offsets, int B, int F, int Fb,
              int D, const FeatMeta* __restrict__ meta, float* __restrict__ out,
              uint32_t* status,
              const uint32_t* __restrict__ order, uint32_t xmask, float magic, bool skip_short,
              const PeerOut pm) {
  pdl_wait();
  constexpr int UNR = (VPL == 1) ? 4 : 2;
  constexpr uint32_t kNone = 0xffffffffu;
  constexpr unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & (LPB - 1);
  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
  const bool in_range = gid < (long long)F * B;  // predicate, never return: shuffles below
  const long long bag = (order != nullptr && in_range) ? (long long)__ldg(order + gid) : gid;
  const int lo = in_range ? __ldg(offsets + bag) : 0;
  const int hi = in_range ? __ldg(offsets + bag + 1) : 0;
  const bool live = in_range && !(skip_short && hi - lo <= 1);  // (skip_short: unused for a10)
  const int len = live ? hi - lo : 0;
  const int f = live ? (int)(bag / B) : 0;
  const int b = live ? (int)(bag - (long long)f * B) : 0;
  const FeatMeta m = meta[f];
  const int nv16 = (D + 15) >> 4;  // 16-code vectors carrying dims < D
  const uint64_t pol_last = l2_policy_last();  // q8 rows: Zipf-hot, keep in L2
  float4 acc[4 * VPL];
#pragma unroll
  for (int v = 0; v < 4 * VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  bool bad = false;
  const int maxlen = __reduce_max_sync(kFull, len);
  uint32_t key_next = lane < len ? row_key(__ldg(ids + lo + lane), m, kNone, bad) : kNone;
  for (int j0 = 0; j0 < maxlen; j0 += LPB) {  // ids one batch ahead, as in the fp32 kernel
    const uint32_t key = key_next;
    const int jn = j0 + LPB + lane;
    key_next = jn < len ? row_key(__ldg(ids + lo + jn), m, kNone, bad) : kNone;
#pragma unroll 1
    for (int jj = 0; jj < LPB; jj += UNR) {
      uint32_t k[UNR];
      uint4 w[UNR][VPL];
      float2 mt[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        k[u] = __shfl_sync(kFull, key, (jj + u) & (LPB - 1), LPB);
        if (jj + u >= LPB || j0 + jj + u >= len) k[u] = kNone;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (k[u] != kNone) {
          const uint8_t* row = codes + (size_t)k[u] * qpitch;
          mt[u] = *reinterpret_cast<const float2*>(row + meta_off);
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            const int vi = lane + v * LPB;
            w[u][v] = vi < nv16 ? ld_l1_u4_hint(row + 16 * vi, pol_last) : make_uint4(0u, 0u, 0u, 0u);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (k[u] != kNone) {
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            acc[4 * v + 0] = deq4_add(acc[4 * v + 0], w[u][v].x, mt[u].y, mt[u].x, xmask, magic);
            acc[4 * v + 1] = deq4_add(acc[4 * v + 1], w[u][v].y, mt[u].y, mt[u].x, xmask, magic);
            acc[4 * v + 2] = deq4_add(acc[4 * v + 2], w[u][v].z, mt[u].y, mt[u].x, xmask, magic);
            acc[4 * v + 3] = deq4_add(acc[4 * v + 3], w[u][v].w, mt[u].y, mt[u].x, xmask, magic);
          }
        }
    }
  }
  if (!live) return;
  if (bad) set_status(status, kStIdRange);  // any lane: each lane validated its own ids
  if (PEER && pm.skip_empty && len == 0) return;
  if (MEAN) mean_div(acc, len);
  // lane l holds dims 16*(l + v*LPB) .. +16
  float* o = PEER ? dst_row<true>(out, (uint32_t)out_row(f, b, B, Fb), B, Fb, D, pm)
                  : out + out_row(f, b, B, Fb) * D;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int d = 16 * (lane + v * LPB);
#pragma unroll
    if ((D & 3) == 0) {
      const uint64_t pol_first = l2_policy_first();  // outputs: written once
#pragma unroll
      for (int h = 0; h < 4; ++h)
        if (d + 4 * h < D) st_f4_hint(o + d + 4 * h, acc[4 * v + h], pol_first);
    } else {
#pragma unroll
      for (int h = 0; h < 4; ++h) store4(o, d + 4 * h, D, acc[4 * v + h]);
    }
  }
}

// ---------------------------------------------------------------------------
// Bag order, longest first (kernels.h kLenBins): bin = 255 - min(len, 255).  Group g of
// the pooling grid takes bag order[g], so the groups of a warp walk bags of about the same
// length and the longest bags start first.  Measured on Feed-1 (alpha 1.05): a2 0.549 ->
// 0.521 ms, a10 0.435 -> 0.388 ms (a per-CTA ordering of 64 consecutive bags gained ~2%).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int len_bin(const int* __restrict__ offsets, long long bag) {
  const int len = __ldg(offsets + bag + 1) - __ldg(offsets + bag);
  return kLenBins - 1 - min(max(len, 0), kLenBins - 1);
}

__global__ void __launch_bounds__(256)
k_len_hist(const int* __restrict__ offsets, long long nbags, uint32_t* __restrict__ hist) {
  pdl_wait();
  __shared__ uint32_t h[kLenBins];
  for (int i = threadIdx.x; i < kLenBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < nbags;
       g += (long long)gridDim.x * blockDim.x)
    atomicAdd(&h[len_bin(offsets, g)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < kLenBins; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, h[i]);
}

// Each CTA owns a contiguous range of bags: count per bin, reserve a range per bin with one
// global atomic, then place (order inside a bin is arbitrary; every bag's result is not).
__global__ void __launch_bounds__(256)
k_len_scatter(const int* __restrict__ offsets, long long nbags, const uint32_t* __restrict__ hist,
              uint32_t* __restrict__ cursor, uint32_t* __restrict__ order) {
  pdl_wait();
  __shared__ uint32_t h[kLenBins], base[kLenBins], start[kLenBins];
  const long long per = (nbags + gridDim.x - 1) / gridDim.x;
  const long long b0 = (long long)blockIdx.x * per;
  const long long b1 = min(nbags, b0 + per);
  for (int i = threadIdx.x; i < kLenBins; i += blockDim.x) { h[i] = 0; start[i] = hist[i]; }
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan of the 256 global bin counts
    uint32_t t = 0;
    for (int i = 0; i < kLenBins; ++i) { const uint32_t c = start[i]; start[i] = t; t += c; }
  }
  for (long long g = b0 + threadIdx.x; g < b1; g += blockDim.x) atomicAdd(&h[len_bin(offsets, g)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < kLenBins; i += blockDim.x) {
    base[i] = h[i] ? start[i] + atomicAdd(cursor + i, h[i]) : 0u;
    h[i] = 0;
  }
  __syncthreads();
  for (long long g = b0 + threadIdx.x; g < b1; g += blockDim.x) {
    const int bin = len_bin(offsets, g);
    order[base[bin] + atomicAdd(&h[bin], 1u)] = (uint32_t)g;
  }
}

// Returns the permutation (nullptr: identity) for `bags` bags of `offsets`.
static const uint32_t* bag_order(const int* offsets, long long bags, uint32_t* ws, cudaStream_t s) {
  if (ws == nullptr || bags < 2) return nullptr;
  uint32_t* hist = ws + bags;
  uint32_t* cursor = hist + kLenBins;
  if (cudaMemsetAsync(hist, 0, 2 * kLenBins * sizeof(uint32_t), s) != cudaSuccess) return nullptr;
  const long long want = (bags + 255) / 256;
  const unsigned grid = (unsigned)(want < 148 * 4 ? want : 148 * 4);
  launch_pdl(k_len_hist, grid, 256, 0, s, offsets, bags, hist);
  launch_pdl(k_len_scatter, grid, 256, 0, s, offsets, bags, (const uint32_t*)hist, cursor, ws);
  return ws;
}

const uint32_t* launch_bag_order(const int* offsets, long long bags, uint32_t* ws, cudaStream_t s) {
  return bag_order(offsets, bags, ws, s);
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

#define LIRANK_FWD_GEOM_DISPATCH(G, KERNEL_LAUNCH)                          \
  do {                                                                      \
    if ((G).lpb == 1) {                                                     \
      if ((G).vpl == 1) { constexpr int L_ = 1, V_ = 1; KERNEL_LAUNCH; }    \
      else { constexpr int L_ = 1, V_ = 2; KERNEL_LAUNCH; }                 \
    } else if ((G).lpb == 2) { constexpr int L_ = 2, V_ = 2; KERNEL_LAUNCH; } \
    else if ((G).lpb == 4) { constexpr int L_ = 4, V_ = 2; KERNEL_LAUNCH; } \
    else if ((G).lpb == 8) { constexpr int L_ = 8, V_ = 2; KERNEL_LAUNCH; } \
    else if ((G).lpb == 16) { constexpr int L_ = 16, V_ = 2; KERNEL_LAUNCH; } \
    else if ((G).vpl <= 2) { constexpr int L_ = 32, V_ = 2; KERNEL_LAUNCH; } \
    else if ((G).vpl <= 4) { constexpr int L_ = 32, V_ = 4; KERNEL_LAUNCH; } \
    else { constexpr int L_ = 32, V_ = 8; KERNEL_LAUNCH; }                  \
  } while (0)

// a2 geometry: about 2 float4 per lane (D=64: 8 lanes x 2 per row, 4 bags per warp).  Measured
// against 16 lanes x 1: Feed-1 a2 0.522 -> 0.491 ms, Ads (mostly one-hot bags) 4.17 -> 3.19 ms:
// more bags per warp keep more rows in flight when bags are short.
static Geom fwd_geom(int pitch) {
  const int nvec = pitch / 4;
  int lpb = 1;
  while (lpb * 2 < nvec && lpb < 32) lpb <<= 1;
  return Geom{lpb, (nvec + lpb - 1) / lpb};
}

cudaError_t launch_pool_fwd_f32(const FwdArgs& a, cudaStream_t s) {
  const Geom g = fwd_geom(a.pitch);
  const long long bags = (long long)a.F * a.B;
  if (bags == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((bags * g.lpb + 255) / 256);
  const int Fb = a.Fb > 0 ? a.Fb : a.F;
  const uint32_t* order = bag_order(a.offsets, bags, a.order_ws, s);
  const bool split = order != nullptr;  // short bags sit at the end of the ordered positions
  const bool peer = a.peer.base[0] != nullptr;  // fused exchange (sharded: SUM, recording)
  const bool fr = (a.D & 3) == 0 && a.pitch == a.D && a.D == 4 * g.lpb * g.vpl;
#define LAUNCH_F32(MEAN, EMIT, PEER)                                                       \
  LIRANK_FWD_GEOM_DISPATCH(g, (launch_pdl(fr ? k_pool_fwd_f32<L_, V_, MEAN, EMIT, PEER, true>          \
                                             : k_pool_fwd_f32<L_, V_, MEAN, EMIT, PEER, false>, grid, 256, 0, s, \
                              a.W, a.pitch, a.ids, a.offsets, a.B, a.F, Fb, a.D, a.meta,    \
                              a.out, a.kv_out, a.sentinel, a.status, order, split, a.peer)))
  if (peer) {
    if (a.mean || !a.kv_out) return cudaErrorInvalidValue;
    LAUNCH_F32(false, true, true);
  } else if (a.mean) {
    if (a.kv_out) LAUNCH_F32(true, true, false); else LAUNCH_F32(true, false, false);
  } else {
    if (a.kv_out) LAUNCH_F32(false, true, false); else LAUNCH_F32(false, false, false);
  }
#undef LAUNCH_F32
  if (split) {
    const unsigned sgrid = (unsigned)(((bags + g.lpb - 1) / g.lpb * g.lpb + 255) / 256);
#define LAUNCH_SHORT(EMIT, PEER)                                                             \
  LIRANK_FWD_GEOM_DISPATCH(g, (launch_pdl(fr ? k_pool_short_f32<L_, V_, EMIT, PEER, true>            \
                                             : k_pool_short_f32<L_, V_, EMIT, PEER, false>, sgrid, 256, 0, s, \
                              a.W, a.pitch, a.ids, a.offsets, a.B, a.F, Fb, a.D, a.meta,    \
                              a.out, a.kv_out, a.sentinel, a.status, order, a.peer)))
    if (peer) LAUNCH_SHORT(true, true);
    else if (a.kv_out) LAUNCH_SHORT(true, false);
    else LAUNCH_SHORT(false, false);
#undef LAUNCH_SHORT
  }
  return cudaGetLastError();
}

cudaError_t launch_pool_fwd_q8(const FwdQ8Args& a, cudaStream_t s) {
  // geometry over 16-code vectors (one 16-B load each)
  // (4 lanes x one 16-code vector for D = 64; 2 lanes x 2 vectors measured slower)
  const Geom g = geom_for(4 * ((a.D + 15) / 16));
  const long long bags = (long long)a.F * a.B;
  if (bags == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((bags * g.lpb + 255) / 256);
  const int Fb = a.Fb > 0 ? a.Fb : a.F;
  // any permutation of the bags is a correct order (the kernels read the current lengths);
  // reusing the last a2 forward's order on the same offsets only saves its two kernels
  const uint32_t* order = a.order_ready ? a.order_ws : bag_order(a.offsets, bags, a.order_ws, s);
  const uint32_t xmask = a.minmax ? 0u : 0x80808080u;
  const float magic = a.minmax ? 8388608.0f : 8388736.0f;
  // (no short-bag split here: a k_pool_short_f32-style q8 kernel measured slower -- Ads a10
  // 3.24 -> 3.79 ms -- the q8 groups already hold 8 bags per warp; nor a compile-time full-row
  // variant as a2 has: Feed-1 a10 0.274 -> 0.375 ms, serving 0.74 -> 0.92 ms; the meta pair
  // loaded with the rows' L2 evict_last hint too: unchanged, 0.2744 vs 0.2753 ms)
#define LAUNCH_Q8(MEAN, PEER)                                                              \
  LIRANK_GEOM_DISPATCH(g, (launch_pdl(k_pool_fwd_q8<L_, V_, MEAN, PEER>, grid, 256, 0, s,   \
                              a.codes, a.qpitch, a.meta_off, a.ids, a.offsets, a.B, a.F, Fb, \
                              a.D, a.meta, a.out, a.status, order, xmask, magic, false, a.peer)))
  if (a.peer.base[0] != nullptr) {
    if (a.mean) return cudaErrorInvalidValue;
    LAUNCH_Q8(false, true);
  } else if (a.mean) {
    LAUNCH_Q8(true, false);
  } else {
    LAUNCH_Q8(false, false);
  }
#undef LAUNCH_Q8
  return cudaGetLastError();
}

}  // namespace lirank
