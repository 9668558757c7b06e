// backward.cu -- a6 segment-reduce + norm partials, a7 global norm/clip, a8 clip+AdaGrad,
// a9 quantize (full table and fused re-quantize of updated rows).
//
// a6 ("the global gradient"):
//   G[u][d] = (float) sum_{occ in seg u, ascending} (double) grad[b][f][d] (x 1/L for MEAN)
// a7 ("clip the global gradient to have unit norm"; §8(c) step 5):
//   S = sum_u sum_d (double)G[u][d]^2 (+ extra, + other ranks); c = min(1, max_norm/sqrt S)
// a8 (north_star "row-wise AdaGrad"; §8(c) steps 6-7):
//   g = fl(G*c); row-wise: s = (float)(sum (double)g^2 / D), A' = A + s,
//   den = sqrtf(A') + eps, w' = w - (lr/den)*g ; element-wise: A' = A + g*g,
//   w' = w + (-lr*g)/(sqrtf(A') + eps)
// a9 (§8(c) step 8): middle-max 8-bit, half-away rounding, saturation.
//
// Design (B200):
// * segment-reduce is load-balanced by OCCURRENCES, not by segments: the sorted
//   occurrence list is cut into chunks of 2^chunk_log2 (32..128, chosen per call so a small
//   batch still spreads over every SM: chunk_log2_for), one lane group (LPB lanes, one
//   float4 of the 256-B grad row per lane at D=64) per chunk, fp64 accumulators in
//   registers, UNR grad-row gathers in flight.  Segments wholly inside a chunk are
//   finished in place; a segment cut by chunk boundaries leaves fp64 partials that a
//   fix-up pass sums in chunk order (long segments -- the Zipf head, ~10^5-10^6
//   occurrences -- by a whole CTA over contiguous chunk ranges combined in fixed order).
//   Every sum has a fixed order, so results are run-to-run deterministic with no float
//   atomics.
// * norm partials are one fp64 per chunk (+ one per fix-up), summed in index order.
// * the update is one persistent grid-stride kernel over the U unique rows (U is read
//   on the device, no host sync): read G, scale by c, read-modify-write w and A, and
//   optionally re-quantize the new row into the q8 store while it is in registers.
// * warp discipline: every shuffle uses the full mask with width LPB and is reached by
//   all 32 lanes (loops that contain shuffles have warp-uniform trip counts; inactive
//   groups are predicated, never returned), so no collective emulation code is emitted.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace lirank {

namespace {

constexpr int kFixLong = 8;           // spans of more chunks than this use a whole CTA
constexpr int kFixBig = 512;          // ... and of more than this, kLongPieces CTAs first
constexpr int kLongPieces = 8;
constexpr int kFixThreads = 1024;
constexpr unsigned kFull = 0xffffffffu;

template <int LPB>
__device__ __forceinline__ double group_sum(double x) {
#pragma unroll
  for (int o = LPB / 2; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o, LPB);
  return x;
}

// (the pooled-gradient rows are re-read once per id of their bag: kept in L2 with evict_last)
// FR (full rows: D == pitch == 4 * LPB * VPL): no bounds logic at all.
template <int VPL, bool FR>
__device__ __forceinline__ void load_grad_row(const float* __restrict__ grad, size_t row_off,
                                              int D, int lane, int LPB, float4 (&r)[VPL], uint64_t pol) {
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int d = 4 * (lane + v * LPB);
    if (FR) {
      r[v] = ld_nc_f4_hint(grad + row_off + d, pol);
    } else if ((D & 3) == 0) {
      r[v] = d < D ? ld_nc_f4_hint(grad + row_off + d, pol) : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      r[v].x = d + 0 < D ? __ldg(grad + row_off + d + 0) : 0.f;
      r[v].y = d + 1 < D ? __ldg(grad + row_off + d + 1) : 0.f;
      r[v].z = d + 2 < D ? __ldg(grad + row_off + d + 2) : 0.f;
      r[v].w = d + 3 < D ? __ldg(grad + row_off + d + 3) : 0.f;
    }
  }
}

template <int VPL>
__device__ __forceinline__ void zero(double (&acc)[VPL][4]) {
#pragma unroll
  for (int v = 0; v < VPL; ++v)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[v][e] = 0.0;
}

// 2^896: the fp32 bit pattern moved into an fp64 (widen_s) is the value x 2^-896
constexpr double kWidenScale = 0x1p896;

// chk += {x, y} * 0 on both halves (FFMA2): a NaN half marks an Inf / NaN element
__device__ __forceinline__ void chk2(unsigned long long& chk, float x, float y) {
  const unsigned long long v = (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(y) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(chk) : "l"(v), "l"(0ull));
}
__device__ __forceinline__ bool chk_bad(unsigned long long chk) {
  const float a = __uint_as_float((uint32_t)chk), b = __uint_as_float((uint32_t)(chk >> 32));
  return a != a || b != b;
}

// Scaled widening: the fp32 bits of x, sign kept at bit 63 and exponent | mantissa shifted
// into the fp64 exponent | mantissa fields, ARE the fp64 x * 2^-896 -- exactly, for every
// finite x: normals (biased exponent e -> e, i.e. 2^(e-127) -> 2^(e-1023)), zero and fp32
// subnormals (m * 2^-149 -> m * 2^-1045, an fp64 subnormal).  Two ALU instructions for the
// high word ((int)bits >> 3 keeps the sign in bits 31..28; & 0x8fffffff clears 30..28) and
// one for the low word.  Inf / NaN come out finite (exponent 255): callers detect them.
__device__ __forceinline__ double widen_s(float x) {
  const uint32_t b = __float_as_uint(x);
  const int hi = (int)((uint32_t)((int)b >> 3) & 0x8fffffffu);
  return __hiloint2double(hi, (int)(b << 29));
}

// acc += (double)r (x 1/L for MEAN).  HW: the F2F conversion (XU pipe: the pipe that bounds
// this kernel with it, ~70% busy on Feed-1).  !HW: SUM: fma(widen_s(r), 2^896, acc) -- the
// product is exactly (double)r, so the fused add rounds exactly as acc + (double)r does;
// MEAN: widen_s(r) * ((1/L) 2^896) is exactly (double)r * (1/L) rounded once, then the add --
// bit-identical sums either way (the build is -fmad=false: no other contraction), with the
// conversion on the ALU pipe.  chk: x * 0 + chk (FFMA2, two elements per instruction) turns
// NaN for an Inf / NaN element (the kernel then flags the batch for the exact re-run).
// (Round 2's first integer widening -- exponent re-biasing with a per-element zero /
// subnormal / non-finite test -- had five instructions plus the tests: 0.661 -> 0.942 ms.)
template <int VPL, bool MEAN, bool HW>
__device__ __forceinline__ void accumulate(double (&acc)[VPL][4], const float4 (&r)[VPL], double inv,
                                           unsigned long long& chk) {
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    if (!HW && !MEAN) {  // fma(x 2^-896, 2^896, acc): the exact x, one rounding of acc + x
      acc[v][0] = __fma_rn(widen_s(r[v].x), kWidenScale, acc[v][0]);
      acc[v][1] = __fma_rn(widen_s(r[v].y), kWidenScale, acc[v][1]);
      acc[v][2] = __fma_rn(widen_s(r[v].z), kWidenScale, acc[v][2]);
      acc[v][3] = __fma_rn(widen_s(r[v].w), kWidenScale, acc[v][3]);
      chk2(chk, r[v].x, r[v].y);
      chk2(chk, r[v].z, r[v].w);
    } else if (!HW) {  // MEAN: the exact product x * (1/L), rounded once, then the add
      acc[v][0] += widen_s(r[v].x) * inv;
      acc[v][1] += widen_s(r[v].y) * inv;
      acc[v][2] += widen_s(r[v].z) * inv;
      acc[v][3] += widen_s(r[v].w) * inv;
      chk2(chk, r[v].x, r[v].y);
      chk2(chk, r[v].z, r[v].w);
    } else if (MEAN) {
      acc[v][0] += (double)r[v].x * inv;
      acc[v][1] += (double)r[v].y * inv;
      acc[v][2] += (double)r[v].z * inv;
      acc[v][3] += (double)r[v].w * inv;
    } else {
      acc[v][0] += (double)r[v].x;
      acc[v][1] += (double)r[v].y;
      acc[v][2] += (double)r[v].z;
      acc[v][3] += (double)r[v].w;
    }
  }
}

// Finish a complete segment: G[u] = (float)acc, return this lane's sum of (double)G^2.  The
// norm's re-widening stays on F2F (once per unique row: the XU pipe has room now, the issue
// slots do not -- widen_s + the rescale there measured 0.567 -> 0.591 ms).
template <int VPL, bool FR>
__device__ __forceinline__ double write_G(float* G, int pitch, uint32_t u, int lane, int LPB,
                                          const double (&acc)[VPL][4]) {
  double nrm = 0.0;
  const int nvec = pitch >> 2;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int vi = lane + v * LPB;
    if (FR || vi < nvec) {
      float4 g = make_float4((float)acc[v][0], (float)acc[v][1], (float)acc[v][2],
                             (float)acc[v][3]);
      st_f4_hint(G + (size_t)u * pitch + 4 * vi, g, l2_policy_first());  // G: streamed to a8
      nrm += (double)g.x * (double)g.x;
      nrm += (double)g.y * (double)g.y;
      nrm += (double)g.z * (double)g.z;
      nrm += (double)g.w * (double)g.w;
    }
  }
  return nrm;
}

template <int VPL, bool FR>
__device__ __forceinline__ void write_partial(double* P, int pitch, int64_t c, int lane, int LPB,
                                              const double (&acc)[VPL][4]) {
  const int nvec = pitch >> 2;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int vi = lane + v * LPB;
    if (FR || vi < nvec) {
      double* p = P + (size_t)c * pitch + 4 * vi;
      reinterpret_cast<double2*>(p)[0] = make_double2(acc[v][0], acc[v][1]);
      reinterpret_cast<double2*>(p)[1] = make_double2(acc[v][2], acc[v][3]);
    }
  }
}

}  // namespace

// One lane group per chunk of 2^chunk_log2 sorted occurrences.  kv[k] = {row key, grad row}.
// MODE 1: ALU widening (widen_s); a lane that met an Inf / NaN input element sets *nf_flag
// (a G that overflows to Inf needs nothing: its norm term is the F2F one, Inf).  MODE 2: the re-run of such a batch with the F2F
// conversions (returns at once unless *nf_flag is set; the owner list is already complete).
// For finite batches MODE 1 alone gives the F2F results bit for bit; otherwise MODE 2 does.
template <int LPB, int VPL, bool MEAN, bool FR, int MODE>
__device__ __forceinline__ void segreduce_block(
    int64_t vb, const uint32_t* __restrict__ seg, const uint32_t* __restrict__ Up,
    const uint2* __restrict__ kv, const uint32_t* __restrict__ chunk_u0, const float* __restrict__ grad,
    const int* __restrict__ offsets, int B, int F, int D, int pitch, int64_t chunks, int chunk_log2,
    float* __restrict__ G, double* __restrict__ part_first, double* __restrict__ part_last,
    double* __restrict__ norm_main, double* __restrict__ norm_fix, uint32_t* __restrict__ owner_list,
    uint32_t* owner_count) {
  constexpr bool HW = MODE != 1;
  uint32_t* nf_flag = owner_count + 2;  // zeroed with the counts by launch_segreduce
  // rows in flight per group: D=64 (VPL 2) measured best at 2 with 4 CTAs/SM (64 registers:
  // 0.78 -> 0.72 ms on Feed-1; 1 -> 0.74, 4 -> 0.78 at 80 registers, 8 -> 1.5); key-derived
  // segment heads then took it to 0.69 ms)
  // (full-row kernel, round 2: 1 -> 0.643 ms, 2 -> 0.610, 4 -> 0.706 with spills)
  // (ALU widening, round 2: UNR 2 at 4 CTAs/SM 0.59 ms, 3 0.62, 4 at 3 CTAs/SM 0.62; groups of
  // 16 lanes x one float4 -- half the groups per warp, so less write-out divergence: UNR 4 or
  // 6 0.584 ms, 8 0.688 (spills) vs 8 x 2 0.565)
  constexpr int UNR = (VPL == 1) ? 8 : (VPL == 2 ? 2 : 2);
  if (FR) { D = 4 * LPB * VPL; pitch = D; }  // compile-time row geometry (the launcher checked)
  const uint64_t pol = l2_policy_last();
  const int lane = threadIdx.x & (LPB - 1);
  const int64_t c = (vb * blockDim.x + threadIdx.x) / LPB;
  const uint32_t U = *Up;
  const int64_t n_valid = seg[U];
  const int chunk = 1 << chunk_log2;
  const int64_t k0 = c << chunk_log2;
  const bool live = c < chunks && k0 < n_valid;
  const int64_t k1 = live ? min(k0 + (int64_t)chunk, n_valid) : k0;
  uint32_t u = live ? __ldg(chunk_u0 + c) : 0u;  // segment containing occurrence k0 (RLE)
  // the open segment started before this chunk (its sum is a part_first partial)
  bool first_open = live && (int64_t)__ldg(seg + u) < k0;
  const unsigned gshift = (threadIdx.x & 31) & ~(LPB - 1);  // this group's lanes in the warp

  double acc[VPL][4];
  zero(acc);
  double nrm = 0.0;
  unsigned long long chk = 0ull;  // two fp32 zeros
  // Warp-uniform loop (chunk/LPB batches for every group): each batch loads LPB {key,
  // grad row} pairs (one per lane) and broadcasts them with full-mask shuffles; slots
  // past k1 (last chunk, dead groups) are predicated.  Segment boundaries come from the
  // keys themselves (an occurrence whose key differs from its predecessor's starts a
  // segment), so no dependent load of the next boundary sits on the segment chain.
  uint32_t carry_key = 0;  // key of the occurrence before the batch (lane LPB-1's, last batch)
  // the {key, grad row} pairs are loaded one batch ahead of the gradient-row gathers
  uint2 kv_next = k0 + lane < k1 ? __ldg(kv + k0 + lane) : make_uint2(0u, 0u);
  for (int it = 0; it < chunk / LPB; ++it) {
    const int64_t kb = k0 + (int64_t)it * LPB;
    uint2 kvl = kv_next;
    kv_next = kb + LPB + lane < k1 ? __ldg(kv + kb + LPB + lane) : make_uint2(0u, 0u);
    double inv_l = 1.0;
    const bool in_l = kb + lane < k1;
    if (in_l) {
      if (MEAN) {
        const uint32_t bb = kvl.y / (uint32_t)F, ff = kvl.y - bb * (uint32_t)F;
        const uint32_t bag = ff * (uint32_t)B + bb;
        inv_l = 1.0 / (double)(__ldg(offsets + bag + 1) - __ldg(offsets + bag));
        if (!HW) inv_l *= kWidenScale;  // exact: a power of two
      }
    }
    uint32_t prev = __shfl_up_sync(kFull, kvl.x, 1, LPB);
    if (lane == 0) prev = carry_key;
    const bool head_l = in_l && kb + lane > k0 && kvl.x != prev;  // k0's segment is the open one
    const unsigned heads = (__ballot_sync(kFull, head_l) >> gshift) & ((LPB < 32) ? ((1u << LPB) - 1u) : kFull);
    carry_key = __shfl_sync(kFull, kvl.x, LPB - 1, LPB);
    const uint32_t grow_l = kvl.y;
#pragma unroll 1
    for (int jj = 0; jj < LPB; jj += UNR) {  // not unrolled: UNR rows in flight, not LPB
      float4 r[UNR][VPL];
      double iv[UNR];
      bool ok[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const uint32_t gq = __shfl_sync(kFull, grow_l, (jj + q) & (LPB - 1), LPB);
        iv[q] = MEAN ? __shfl_sync(kFull, inv_l, (jj + q) & (LPB - 1), LPB) : (HW ? 1.0 : kWidenScale);
        ok[q] = (jj + q < LPB) && (kb + jj + q < k1);
        if (ok[q]) load_grad_row<VPL, FR>(grad, (size_t)gq * D, D, lane, LPB, r[q], pol);
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        if (ok[q]) {
          if ((heads >> (jj + q)) & 1u) {  // segment u finished inside this chunk
            if (first_open) write_partial<VPL, FR>(part_first, pitch, c, lane, LPB, acc);
            else nrm += write_G<VPL, FR>(G, pitch, u, lane, LPB, acc);
            zero(acc);
            ++u;
            first_open = false;
          }
          accumulate<VPL, MEAN, HW>(acc, r[q], iv[q], chk);
        }
      }
    }
  }
  // the segment containing occurrence k1-1: it ends here iff k1 is the end of the valid
  // occurrences or starts another key
  bool owner = false;
  if (live) {
    if (first_open) {
      write_partial<VPL, FR>(part_first, pitch, c, lane, LPB, acc);  // continues or ends here
    } else if (k1 == n_valid || __ldg(&kv[k1].x) != __ldg(&kv[k1 - 1].x)) {
      nrm += write_G<VPL, FR>(G, pitch, u, lane, LPB, acc);
    } else {
      write_partial<VPL, FR>(part_last, pitch, c, lane, LPB, acc);  // starts here, spills over
      owner = true;
    }
  }
  nrm = group_sum<LPB>(nrm);  // all lanes converge here
  if (!HW && chk_bad(chk)) *nf_flag = 1u;  // an Inf / NaN in this lane's elements: re-run exactly
  if (lane == 0 && c < chunks) {
    norm_main[c] = nrm;
    norm_fix[c] = 0.0;
    if (owner && MODE != 2) {
      const uint32_t slot = atomicAdd(owner_count, 1u);
      owner_list[slot] = (uint32_t)c;
    }
  }
}

template <int LPB, int VPL, bool MEAN, bool FR, int MODE>
__global__ void __launch_bounds__(256, 4)
k_segreduce(const uint32_t* __restrict__ seg, const uint32_t* __restrict__ Up,
            const uint2* __restrict__ kv, const uint32_t* __restrict__ chunk_u0,
            const float* __restrict__ grad, const int* __restrict__ offsets, int B, int F, int D,
            int pitch, int64_t chunks, int chunk_log2, float* __restrict__ G, double* __restrict__ part_first,
            double* __restrict__ part_last, double* __restrict__ norm_main,
            double* __restrict__ norm_fix, uint32_t* __restrict__ owner_list,
            uint32_t* owner_count, int64_t nblocks) {
  pdl_wait();
  if (MODE != 2) {  // one block of chunks per CTA
    segreduce_block<LPB, VPL, MEAN, FR, MODE>(blockIdx.x, seg, Up, kv, chunk_u0, grad, offsets, B, F, D, pitch,
                                              chunks, chunk_log2, G, part_first, part_last, norm_main,
                                              norm_fix, owner_list, owner_count);
    return;
  }
  // the re-run: a small grid that returns at once unless the first pass flagged an Inf / NaN,
  // then strides over the same blocks (block-uniform loop: the shuffles stay full-warp)
  if (*(volatile uint32_t*)(owner_count + 2) == 0u) return;
  for (int64_t vb = blockIdx.x; vb < nblocks; vb += gridDim.x)
    segreduce_block<LPB, VPL, MEAN, FR, MODE>(vb, seg, Up, kv, chunk_u0, grad, offsets, B, F, D, pitch,
                                              chunks, chunk_log2, G, part_first, part_last, norm_main,
                                              norm_fix, owner_list, owner_count);
}

// Fix-up of segments spanning chunks.  Entry e = chunk c_s where segment u starts and
// spills over; its sum = part_last[c_s] + sum_{c = c_s+1 .. c_e} part_first[c].
// One lane group per entry for short spans; entries spanning > kFixLong chunks are left
// to k_fixup_long.  The entry loop is warp-uniform (see the file header).
template <int LPB, int VPL>
__global__ void __launch_bounds__(256)
k_fixup_short(const uint32_t* __restrict__ seg, const uint32_t* __restrict__ Up,
              const uint32_t* __restrict__ chunk_u0, int pitch, const double* __restrict__ part_first,
              const double* __restrict__ part_last, const uint32_t* __restrict__ owner_list,
              const uint32_t* __restrict__ owner_count, float* __restrict__ G,
              double* __restrict__ norm_fix, uint32_t* long_list, uint32_t* long_count, uint32_t* big_list,
              uint32_t* big_count, int chunk_log2) {
  pdl_wait();
  constexpr int GPW = 32 / LPB;  // groups per warp
  const int lane = threadIdx.x & (LPB - 1);
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;  // global warp
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) / 32;
  const int gin = (threadIdx.x & 31) / LPB;
  const uint32_t n_entries = *owner_count;
  const uint32_t U = *Up;
  const int nvec = pitch >> 2;
  for (int64_t eb = gw * GPW; eb < n_entries; eb += nwarps * GPW) {  // uniform per warp
    const int64_t e = eb + gin;
    bool live = e < n_entries;
    uint32_t cs = 0, u = 0;
    int64_t ce = 0;
    if (live) {
      cs = owner_list[e];
      // the segment spills into chunk cs+1, so it is the one containing that chunk's first
      // occurrence: chunk_u0[cs+1] (no binary search over seg[])
      u = __ldg(chunk_u0 + cs + 1);
      ce = ((int64_t)__ldg(seg + u + 1) - 1) >> chunk_log2;
      if (ce - cs > kFixLong) {
        if (lane == 0) {
          const uint32_t slot = atomicAdd(long_count, 1u);
          long_list[2 * slot] = cs;
          long_list[2 * slot + 1] = u;
          if (ce - cs > kFixBig) {  // the Zipf head: its partials are summed in pieces first
            const uint32_t b = atomicAdd(big_count, 1u);
            big_list[2 * b] = cs;
            big_list[2 * b + 1] = u;
          }
        }
        live = false;
      }
    }
    double nrm = 0.0;
    if (live) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int vi = lane + v * LPB;
        if (vi < nvec) {
          const double* p = part_last + (size_t)cs * pitch + 4 * vi;
          double a0 = p[0], a1 = p[1], a2 = p[2], a3 = p[3];
          for (int64_t cc = cs + 1; cc <= ce; cc += 4) {  // 4 partial rows in flight, added in order
            double2 x[4][2];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (cc + j <= ce) {
                const double2* q = reinterpret_cast<const double2*>(part_first + (size_t)(cc + j) * pitch + 4 * vi);
                x[j][0] = q[0];
                x[j][1] = q[1];
              }
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (cc + j <= ce) { a0 += x[j][0].x; a1 += x[j][0].y; a2 += x[j][1].x; a3 += x[j][1].y; }
          }
          const float4 g = make_float4((float)a0, (float)a1, (float)a2, (float)a3);
          st_f4(G + (size_t)u * pitch + 4 * vi, g);
          nrm += (double)g.x * g.x + (double)g.y * g.y + (double)g.z * g.z + (double)g.w * g.w;
        }
      }
    }
    nrm = group_sum<LPB>(nrm);
    if (lane == 0 && live) norm_fix[cs] = nrm;
  }
}

// First chunk of piece k of a span of nch chunks after chunk cs (k = kLongPieces: the end).
__device__ __forceinline__ int64_t piece_lo(int64_t cs, int64_t nch, int k) {
  return cs + 1 + (nch * k) / kLongPieces;
}

// The spans of more than kFixBig chunks (the hottest rows: up to ~10^4 chunks; one CTA alone
// walked the hottest one's partial rows in ~32 dependent rounds, 39 us of the step) are cut
// into kLongPieces contiguous pieces, one CTA each (a piece: its own sub-ranges combined in
// order, as below).  A piece's sum is stored over the partial of the piece's first chunk --
// read only by this piece, and already consumed -- so no other scratch; k_fixup_long then
// adds part_last + the pieces in piece order.  (Cutting EVERY long span into 8 pieces
// measured a6 0.549 -> 0.617 ms: a 1024-thread CTA and two barriers per piece of a few chunks.)
__global__ void __launch_bounds__(kFixThreads, 1)
k_fixup_long_pieces(const uint32_t* __restrict__ seg, int pitch, double* __restrict__ part_first,
                    const uint32_t* __restrict__ big_list, const uint32_t* __restrict__ big_count,
                    int chunk_log2) {
  pdl_wait();
  extern __shared__ double sm[];  // [nsplit * pitch]
  const uint32_t n_big = *big_count;
  const int nsplit = max(1, kFixThreads / pitch);
  for (int64_t w = blockIdx.x; w < (int64_t)n_big * kLongPieces; w += gridDim.x) {
    const int64_t e = w / kLongPieces;
    const int k = (int)(w % kLongPieces);
    const uint32_t cs = big_list[2 * e], u = big_list[2 * e + 1];
    const int64_t nch = (((int64_t)__ldg(seg + u + 1) - 1) >> chunk_log2) - cs;
    const int64_t lo = piece_lo(cs, nch, k), m = piece_lo(cs, nch, k + 1) - lo;  // m > 64
    for (int t = threadIdx.x; t < nsplit * pitch; t += blockDim.x) {
      const int el = t % pitch, sp = t / pitch;
      const int64_t a = lo + (m * sp) / nsplit, b = lo + (m * (sp + 1)) / nsplit;
      double acc = 0.0;
      int64_t cc = a;
      for (; cc + 16 <= b; cc += 16) {  // 16 loads in flight, adds in chunk order
        double x[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) x[q] = part_first[(size_t)(cc + q) * pitch + el];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc += x[q];
      }
      for (; cc < b; ++cc) acc += part_first[(size_t)cc * pitch + el];
      sm[sp * pitch + el] = acc;
    }
    __syncthreads();  // every read of the piece's partials is done
    for (int el = threadIdx.x; el < pitch; el += blockDim.x) {
      double acc = 0.0;
      for (int sp = 0; sp < nsplit; ++sp) acc += sm[sp * pitch + el];
      part_first[(size_t)lo * pitch + el] = acc;
    }
    __syncthreads();  // sm is reused by the next piece
  }
}

// Long spans: one CTA per entry.  Thread t owns element (t % pitch) of the row for chunk
// sub-range (t / pitch); sub-ranges are contiguous and combined in order.  A span of more
// than kFixBig chunks instead adds its kLongPieces piece sums (k_fixup_long_pieces) in order.
__global__ void __launch_bounds__(kFixThreads, 1)  // 1: 64 registers, all 16 loads in flight
k_fixup_long(const uint32_t* __restrict__ seg, int pitch, const double* __restrict__ part_first,
             const double* __restrict__ part_last, const uint32_t* __restrict__ long_list,
             const uint32_t* __restrict__ long_count, float* __restrict__ G,
             double* __restrict__ norm_fix, int chunk_log2) {
  pdl_wait();
  extern __shared__ double sm[];  // [max(nsplit * pitch, kFixThreads)]
  const uint32_t n_entries = *long_count;
  const int nsplit = max(1, kFixThreads / pitch);
  for (uint32_t e = blockIdx.x; e < n_entries; e += gridDim.x) {
    const uint32_t cs = long_list[2 * e], u = long_list[2 * e + 1];
    const int64_t s_end = __ldg(seg + u + 1);
    const int64_t ce = (s_end - 1) >> chunk_log2;
    const int64_t nch = ce - cs;  // chunks cs+1 .. ce
    const bool big = nch > kFixBig;  // (uniform over the CTA)
    for (int t = threadIdx.x; !big && t < nsplit * pitch; t += blockDim.x) {
      const int el = t % pitch, sp = t / pitch;
      const int64_t a = cs + 1 + (nch * sp) / nsplit;
      const int64_t b = cs + 1 + (nch * (sp + 1)) / nsplit;
      double s = 0.0;
      int64_t cc = a;
      for (; cc + 16 <= b; cc += 16) {  // 16 loads in flight, adds in chunk order
        double x[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) x[q] = __ldg(part_first + (size_t)(cc + q) * pitch + el);
#pragma unroll
        for (int q = 0; q < 16; ++q) s += x[q];
      }
      for (; cc < b; ++cc) s += part_first[(size_t)cc * pitch + el];
      sm[sp * pitch + el] = s;
    }
    __syncthreads();
    double nrm_part = 0.0;
    for (int el = threadIdx.x; el < pitch; el += blockDim.x) {
      double s = part_last[(size_t)cs * pitch + el];
      if (big) {
        for (int k = 0; k < kLongPieces; ++k) s += part_first[(size_t)piece_lo(cs, nch, k) * pitch + el];
      } else {
        for (int sp = 0; sp < nsplit; ++sp) s += sm[sp * pitch + el];
      }
      const float g = (float)s;
      G[(size_t)u * pitch + el] = g;
      nrm_part += (double)g * (double)g;
    }
    // deterministic block reduction of nrm_part (threads < pitch hold values): a fixed
    // shuffle tree per warp, then the warp partials in warp order (3 barriers, not 12)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm_part += __shfl_xor_sync(0xffffffffu, nrm_part, o);
    __syncthreads();  // this entry's reads of sm are done
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = nrm_part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sm[w];
      norm_fix[cs] = t;
    }
    __syncthreads();
  }
}

// S_local = sum over chunks of norm_main + norm_fix in a fixed order: each of up to
// kNormParts CTAs sums a contiguous range of chunks (fixed tree), the last CTA to finish
// adds the CTA partials in index order.  Deterministic for a given chunk count.
constexpr int kNormParts = 64;
__global__ void __launch_bounds__(256)
k_norm_partial(const double* __restrict__ norm_main, const double* __restrict__ norm_fix,
               int64_t chunks, double* __restrict__ parts, uint32_t* done, double* S_local) {
  pdl_wait();
  __shared__ double sm[256];
  __shared__ bool last;
  const int64_t per = (chunks + gridDim.x - 1) / gridDim.x;
  const int64_t a = (int64_t)blockIdx.x * per, b = min(chunks, a + per);
  double s = 0.0;
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
    s += norm_main[i];
    s += norm_fix[i];
  }
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = sm[0];
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double t = 0.0;
    for (unsigned p = 0; p < gridDim.x; ++p) t += ld_volatile_f64(parts + p);
    *S_local = t;
    *done = 0u;  // re-armed for the next launch
  }
}

// S = sum of rank partials in rank order + extra; c = (n > max_norm) ? max_norm/n : 1.
// Non-finite S: c = -1 (the update kernel then skips every row) + sticky status.
__global__ void k_norm_finalize(const double* parts, int nparts, double extra,
                                const double* extra_dev, float max_norm, double* S_global,
                                float* clip, float* clip_out, uint32_t* status) {
  pdl_wait();
  double S = 0.0;
  for (int r = 0; r < nparts; ++r) S += parts[r];
  S += extra;
  if (extra_dev) S += *extra_dev;
  *S_global = S;
  float c;
  if (!isfinite(S)) {
    c = -1.0f;
    atomicOr(status, kStNonFinite);
  } else {
    const double n = sqrt(S);
    c = (n > (double)max_norm) ? (float)((double)max_norm / n) : 1.0f;
  }
  *clip = c;
  if (clip_out) *clip_out = c;
}

// ---------------------------------------------------------------------------
// middle-max quantization of one row held by a lane group (used by a9 and REQUANT).
// Must be called by all 32 lanes of the warp; `live` predicates this group's stores.
// ---------------------------------------------------------------------------
// NaN-propagating min / max (PTX min.NaN / max.NaN, sm_80+): a NaN anywhere in the row
// reaches the row's extremes, so one isfinite() on them detects every non-finite element.
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// X^int of one element, exactly as the oracle: round-half-away((X - base) / X^scale),
// saturated to [lo, hi] (the IEEE quotient, used where the fast path cannot decide).
// Middle-max: base = X^middle, [-128, 127]; min-max (NEXT-4): base = X^min, [0, 255].
__device__ __forceinline__ uint32_t code_exact(float e, float base, float scale, float lo, float hi) {
  float r = roundf(__fdiv_rn(__fsub_rn(e, base), scale));
  r = fminf(fmaxf(r, lo), hi);
  return (uint32_t)((int)r) & 0xffu;
}

// rot (full rows only, D == 4 * LPB * VPL): this lane holds float4 (lane + v * LPB + rot) mod
// (LPB * VPL) of the row in x[v] (the TMA update's bank-conflict-free smem layout).
template <int LPB, int VPL>
__device__ __forceinline__ int rot_idx(int lane, int v, int rot) {
  return rot ? (lane + v * LPB + rot) % (LPB * VPL) : lane + v * LPB;
}
template <int LPB, int VPL>
__device__ __forceinline__ void quantize_group_row(const float4 (&x)[VPL], int D, int lane, bool live,
                                                   uint8_t* __restrict__ code_row,
                                                   int meta_off, int qpitch, bool minmax,
                                                   uint32_t* status, int rot = 0) {
  float mn = FLT_MAX, mx = -FLT_MAX;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int d = 4 * (rot_idx<LPB, VPL>(lane, v, rot));
    const float e[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
    if (d + 4 <= D) {
#pragma unroll
      for (int i = 0; i < 4; ++i) { mn = fmin_nan(mn, e[i]); mx = fmax_nan(mx, e[i]); }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (d + i < D) { mn = fmin_nan(mn, e[i]); mx = fmax_nan(mx, e[i]); }
    }
  }
#pragma unroll
  for (int o = LPB / 2; o > 0; o >>= 1) {
    mn = fmin_nan(mn, __shfl_xor_sync(kFull, mn, o, LPB));
    mx = fmax_nan(mx, __shfl_xor_sync(kFull, mx, o, LPB));
  }
  if (!live) return;
  float middle, scale;
  bool zero_codes;
  if (!isfinite(mn) || !isfinite(mx)) {
    middle = 0.f; scale = 0.f; zero_codes = true;
    if (lane == 0) atomicOr(status, kStNonFinite);
  } else if (mx == mn) {
    middle = mx; scale = 0.f; zero_codes = true;
  } else {
    // middle-max: X^middle = (X^max * 2^(b-1) + X^min * (2^(b-1) - 1)) / (2^b - 1), b = 8;
    // min-max (NEXT-4): the saved base is X^min itself ("middle" names the base below)
    middle = minmax ? mn
                    : __fdiv_rn(__fadd_rn(__fmul_rn(mx, 128.0f), __fmul_rn(mn, 127.0f)), 255.0f);
    // X^scale = (X^max - X^min) / (2^b - 1)
    scale = __fdiv_rn(__fsub_rn(mx, mn), 255.0f);
    zero_codes = scale == 0.0f;
  }
  const float qlo = minmax ? 0.0f : -128.0f, qhi = minmax ? 255.0f : 127.0f;
  // X^int = round((X - X^middle) / X^scale), half away from zero, saturated to [-128,127].
  // The IEEE quotient is only needed near a rounding boundary: q~ = (X - X^middle) *
  // RN(1/X^scale) is within 2^-23 relative (< 4e-5 absolute for |q| < 200) of the
  // correctly rounded quotient q, so when |q~ - rint(q~)| < 0.4999 both round to the same
  // integer (no tie is possible there, so half-even rint == half-away); and clamping q~ to
  // [-128, 127] before rounding equals rounding then saturating.  rint is the 1.5*2^23
  // trick, whose float bits hold the code in their low byte.  A lane with any element at
  // |q~ - rint(q~)| >= 0.4999 (about 2e-4 of elements) redoes its words exactly.
  const bool fast = scale >= 1.17549435e-38f && scale <= 4.2535296e37f;  // [2^-126, 2^125]
  const float rcp = fast ? __frcp_rn(scale) : 0.0f;
  uint32_t* words = reinterpret_cast<uint32_t*>(code_row);
  if (!zero_codes) {
    float err = fast ? 0.0f : 1.0f;
    uint32_t wv[VPL];
    // (paired FADD2 / FMUL2 arithmetic: each element exactly the scalar operation)
    const float2 nmid = make_float2(-middle, -middle), rc = make_float2(rcp, rcp);
    const float2 kbig = make_float2(12582912.0f, 12582912.0f), nkbig = make_float2(-12582912.0f, -12582912.0f);
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int d = 4 * (rot_idx<LPB, VPL>(lane, v, rot));
      float2 q[2] = {f2_mul_rn(f2_add_rn(make_float2(x[v].x, x[v].y), nmid), rc),
                     f2_mul_rn(f2_add_rn(make_float2(x[v].z, x[v].w), nmid), rc)};
      uint32_t bits[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        q[h] = make_float2(fminf(fmaxf(q[h].x, qlo), qhi), fminf(fmaxf(q[h].y, qlo), qhi));
        const float2 big = f2_add_rn(q[h], kbig);
        const float2 rq = f2_add_rn(big, nkbig);
        const float2 dq = f2_add_rn(q[h], make_float2(-rq.x, -rq.y));
        err = fmaxf(err, fmaxf(fabsf(dq.x), fabsf(dq.y)));
        bits[2 * h] = __float_as_uint(big.x);
        bits[2 * h + 1] = __float_as_uint(big.y);
      }
      uint32_t w = __byte_perm(__byte_perm(bits[0], bits[1], 0x0040),
                               __byte_perm(bits[2], bits[3], 0x0040), 0x5410);
      if (d + 4 > D) w &= D > d ? (1u << (8 * (D - d))) - 1u : 0u;  // codes past D are 0
      wv[v] = w;
    }
    if (err >= 0.4999f) {  // rare: exact quotient for this lane's elements
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int d = 4 * (rot_idx<LPB, VPL>(lane, v, rot));
        const float e[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
        uint32_t w = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (d + i < D) w |= code_exact(e[i], middle, scale, qlo, qhi) << (8 * i);
        wv[v] = w;
      }
    }
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int wi = rot_idx<LPB, VPL>(lane, v, rot);
      if (4 * wi < D) words[wi] = wv[v];
    }
  } else {
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int wi = rot_idx<LPB, VPL>(lane, v, rot);
      if (4 * wi < D) words[wi] = 0u;
    }
  }
  // The row tail [4*ceil(D/4), qpitch) -- pad, {middle, scale}, pad -- is written whole, so
  // every 32 B sector of the row is fully overwritten by this warp.
  for (int o = 4 * ((D + 3) / 4) + 4 * lane; o < qpitch; o += 4 * LPB)
    words[o >> 2] = o == meta_off ? __float_as_uint(middle)
                                  : (o == meta_off + 4 ? __float_as_uint(scale) : 0u);
}

// a9 over all rows.  Geometry: LPB lanes per row with VPL float4 each (D=64: 4 lanes x 4):
// few lanes per row keep the per-row reductions cheap; R rows per group per iteration.
template <int LPB, int VPL>
__global__ void __launch_bounds__(256, 4)
k_quantize(const float* __restrict__ W, int pitch, int64_t rows, int D,
           uint8_t* __restrict__ codes, int qpitch, int meta_off, bool minmax, uint32_t* status) {
  pdl_wait();
  // rows in flight per group; at 4 CTAs/SM (64 registers) one row per group streams best
  // (D=64: 7.99 ms for 125M rows vs 8.15 at 2 rows / 3 CTAs and 9.6 at 2 rows / 116 regs)
  constexpr int R = VPL >= 4 ? 1 : 2;
  const int lane = threadIdx.x & (LPB - 1);
  const int64_t gstride = ((int64_t)gridDim.x * blockDim.x) / LPB;
  const int64_t g0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
  const int64_t gbase = g0 - (threadIdx.x & 31) / LPB;  // first group of my warp
  const int nvec = pitch >> 2;
  for (int64_t rb = gbase; rb < rows; rb += R * gstride) {  // uniform per warp
    const int64_t r0 = g0 + (rb - gbase);
    float4 x[R][VPL];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int64_t r = r0 + q * gstride;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int vi = lane + v * LPB;
        x[q][v] = (r < rows && vi < nvec) ? ld_nc_f4(W + (size_t)r * pitch + 4 * vi)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int64_t r = r0 + q * gstride;
      const bool live = r < rows;
      uint8_t* row = codes + (size_t)(live ? r : 0) * qpitch;
      quantize_group_row<LPB, VPL>(x[q], D, lane, live, row, meta_off, qpitch, minmax, status);
    }
  }
}

// Fused clip + sparse AdaGrad on the U unique rows (+ optional re-quantize).  Each lane
// group handles R rows per iteration, all their loads issued before any update.
template <int LPB, int VPL, bool ROWWISE, bool REQUANT>
__global__ void __launch_bounds__(256, (REQUANT && !ROWWISE) ? 1 : 3)
k_adagrad(const uint32_t* __restrict__ unique, const uint32_t* __restrict__ Up,
          const float* __restrict__ G, const float* __restrict__ clip, float* __restrict__ Wt,
          float* __restrict__ A, int pitch, int D, float lr, float eps,
          uint8_t* __restrict__ codes, int qpitch, int meta_off, bool minmax, uint32_t* status) {
  pdl_wait();
  constexpr int R = VPL >= 4 ? 1 : 2;
  const float c = *clip;
  if (c < 0.0f) return;  // non-finite global norm: skip the step (uniform over the grid)
  const uint32_t U = *Up;
  const int lane = threadIdx.x & (LPB - 1);
  const int64_t gstride = ((int64_t)gridDim.x * blockDim.x) / LPB;
  const int64_t g0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
  const int64_t gbase = g0 - (threadIdx.x & 31) / LPB;
  const int nvec = pitch >> 2;
  const double dimD = (double)D;
  // the unique-row keys are loaded one iteration ahead: the key -> row-load dependence of
  // the next iteration overlaps this iteration's row loads and updates
  uint32_t key_next[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int64_t u = g0 + q * gstride;
    key_next[q] = u < U ? __ldg(unique + u) : 0u;
  }
  for (int64_t ub = gbase; ub < U; ub += R * gstride) {  // uniform per warp
    const int64_t u0 = g0 + (ub - gbase);
    uint32_t key[R];
    bool has[R];
    float4 g[R][VPL], w[R][VPL], av[ROWWISE ? 1 : R][VPL];
    float arow[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int64_t u = u0 + q * gstride;
      has[q] = u < U;
      key[q] = key_next[q];
      const int64_t un = u + R * gstride;
      key_next[q] = un < U ? __ldg(unique + un) : 0u;
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int64_t u = u0 + q * gstride;
      if (ROWWISE) arow[q] = has[q] ? __ldg(A + key[q]) : 0.f;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int vi = lane + v * LPB;
        if (has[q] && vi < nvec) {
          const float4 Gv = ld_nc_f4(G + (size_t)u * pitch + 4 * vi);
          g[q][v] = make_float4(__fmul_rn(Gv.x, c), __fmul_rn(Gv.y, c), __fmul_rn(Gv.z, c),
                                __fmul_rn(Gv.w, c));
          w[q][v] = ld_f4(Wt + (size_t)key[q] * pitch + 4 * vi);
          if (!ROWWISE) av[ROWWISE ? 0 : q][v] = ld_f4(A + (size_t)key[q] * pitch + 4 * vi);
        } else {
          g[q][v] = make_float4(0.f, 0.f, 0.f, 0.f);
          w[q][v] = g[q][v];
          if (!ROWWISE) av[ROWWISE ? 0 : q][v] = g[q][v];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if (ROWWISE) {
        double ss = 0.0;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          ss += (double)g[q][v].x * (double)g[q][v].x;
          ss += (double)g[q][v].y * (double)g[q][v].y;
          ss += (double)g[q][v].z * (double)g[q][v].z;
          ss += (double)g[q][v].w * (double)g[q][v].w;
        }
        ss = group_sum<LPB>(ss);  // all lanes (has[] only predicates)
        const float s = (float)(ss / dimD);
        const float a = __fadd_rn(arow[q], s);
        const float den = __fadd_rn(__fsqrt_rn(a), eps);
        const float mult = __fdiv_rn(lr, den);
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          w[q][v].x = __fsub_rn(w[q][v].x, __fmul_rn(mult, g[q][v].x));
          w[q][v].y = __fsub_rn(w[q][v].y, __fmul_rn(mult, g[q][v].y));
          w[q][v].z = __fsub_rn(w[q][v].z, __fmul_rn(mult, g[q][v].z));
          w[q][v].w = __fsub_rn(w[q][v].w, __fmul_rn(mult, g[q][v].w));
        }
        if (has[q] && lane == 0) A[key[q]] = a;
      } else if (has[q]) {
        const float nlr = -lr;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const int vi = lane + v * LPB;
          if (vi < nvec) {
            float4 a = av[ROWWISE ? 0 : q][v];
            const float4 gg = g[q][v];
            a.x = __fadd_rn(a.x, __fmul_rn(gg.x, gg.x));
            a.y = __fadd_rn(a.y, __fmul_rn(gg.y, gg.y));
            a.z = __fadd_rn(a.z, __fmul_rn(gg.z, gg.z));
            a.w = __fadd_rn(a.w, __fmul_rn(gg.w, gg.w));
            w[q][v].x = __fadd_rn(w[q][v].x, __fdiv_rn(__fmul_rn(nlr, gg.x), __fadd_rn(__fsqrt_rn(a.x), eps)));
            w[q][v].y = __fadd_rn(w[q][v].y, __fdiv_rn(__fmul_rn(nlr, gg.y), __fadd_rn(__fsqrt_rn(a.y), eps)));
            w[q][v].z = __fadd_rn(w[q][v].z, __fdiv_rn(__fmul_rn(nlr, gg.z), __fadd_rn(__fsqrt_rn(a.z), eps)));
            w[q][v].w = __fadd_rn(w[q][v].w, __fdiv_rn(__fmul_rn(nlr, gg.w), __fadd_rn(__fsqrt_rn(a.w), eps)));
            st_f4(A + (size_t)key[q] * pitch + 4 * vi, a);
          }
        }
      }
      if (has[q]) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const int vi = lane + v * LPB;
          if (vi < nvec) st_f4(Wt + (size_t)key[q] * pitch + 4 * vi, w[q][v]);
        }
      }
      if (REQUANT) {
        uint8_t* row = codes + (size_t)key[q] * qpitch;
        quantize_group_row<LPB, VPL>(w[q], D, lane, has[q], row, meta_off, qpitch, minmax, status);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// a8 (+ fused a9), row-wise AdaGrad at D = 64, with TMA bulk copies.  Each lane group of 4
// lanes owns a ring of kTmaStages shared-memory slots (its G row and W row, 256 B each) and
// one mbarrier per slot: lane 0 of the group issues the two cp.async.bulk copies of row i+S
// (global -> shared, completion counted in bytes on the slot's mbarrier) right after the
// group has read slot i, so S rows per group are in flight while the group updates and
// re-quantizes the current one -- without holding them in registers (the register-staged
// kernel above keeps one row per group in flight and only while it waits).  The unique-row
// keys and accumulators are loaded one stage ahead by lane 0.  Reading a slot: in one
// 128-bit shared load the 8 lanes of a quarter-warp are 2 groups; group g reads its row from
// float4 (lane + 4v + 4(g & 1)) mod 16, so the two groups hit disjoint banks.
// ---------------------------------------------------------------------------
constexpr int kTmaStages = 2;
// Grid: up to 48 resident waves of CTAs (sized from the occurrence count, U <= nnz), i.e.
// about two rows per group on Feed-1 -- both in flight at once -- with CTAs replacing each
// other as they finish.  Measured update time (Feed-1, alpha 1.05): 1 wave (persistent, ~16
// rows per group) 0.595 ms, 4 waves 0.564, 12 waves 0.532, 24 waves 0.522, 48 waves 0.517,
// 96 waves 0.572; the register-staged kernel 0.549.  alpha 0: 1.90 vs 2.04 ms; Ads 1.09 vs
// 1.17 ms; alpha 1.2 (U = 0.92M, one row per group) 0.206 vs 0.196 ms.  (Round 2: the top ncu
// stall, lane 0's accumulator address waiting on its key, moved by loading keys two rows
// ahead -- a8 unchanged, 0.4046 vs 0.4034 ms without requant: the rows' DRAM time dominates.)
constexpr int kTmaWaves = 48;
constexpr int kTmaRowBytes = 256;  // D = 64 fp32
constexpr size_t kTmaSmem = 8 /*warps*/ * kTmaStages * 8 /*groups*/ * 2 * kTmaRowBytes +
                            8 * kTmaStages * 8 * sizeof(unsigned long long);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <bool REQUANT>
__global__ void __launch_bounds__(256, 3)
k_adagrad_tma(const uint32_t* __restrict__ unique, const uint32_t* __restrict__ Up,
              const float* __restrict__ G, const float* __restrict__ clip, float* __restrict__ Wt,
              float* __restrict__ A, float lr, float eps, uint8_t* __restrict__ codes, int qpitch,
              int meta_off, bool minmax, uint32_t* status) {
  constexpr int LPB = 4, VPL = 4, S = kTmaStages, D = 64;
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_wait();
  const int warp = threadIdx.x >> 5, grp = (threadIdx.x & 31) >> 2, lane = threadIdx.x & 3;
  const float c = *clip;
  if (c < 0.0f) return;  // non-finite global norm: skip the step (uniform over the grid)
  const uint32_t U = *Up;
  // the grid is sized from the occurrence count (U is only known on the device): CTAs past
  // the unique rows leave before setting anything up
  if ((int64_t)blockIdx.x * (blockDim.x / 4) >= (int64_t)U) return;
  uint8_t* slots = smem + (size_t)(warp * S * 8) * 2 * kTmaRowBytes;  // [S][8 groups][G | W]
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(smem + (size_t)8 * S * 8 * 2 * kTmaRowBytes) + warp * S * 8;
  const int64_t gstride = ((int64_t)gridDim.x * blockDim.x) / LPB;
  const int64_t g0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
  const int64_t gbase = g0 - grp;  // first group of my warp
  if (lane == 0)
    for (int q = 0; q < S; ++q) mbar_init(&bars[q * 8 + grp], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int rot = (grp & 1) * 4;
  // lane 0's ring (S = 2, kept in named registers): key and accumulator of the row in each
  // slot; the key of the next row to issue
  static_assert(S == 2, "ring of two slots");
  uint32_t kr0 = 0, kr1 = 0, knext = 0;
  float ar0 = 0.f, ar1 = 0.f;
  auto issue = [&](int q, int64_t u, uint32_t key) {  // lane 0: row u into slot q
    uint8_t* sl = slots + (size_t)(q * 8 + grp) * 2 * kTmaRowBytes;
    // the group's generic-proxy reads of this slot (ordered before by __syncwarp) before the
    // async-proxy (TMA) writes that refill it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bars[q * 8 + grp], 2 * kTmaRowBytes);
    tma_load_1d(sl, G + (size_t)u * D, kTmaRowBytes, &bars[q * 8 + grp]);
    tma_load_1d(sl + kTmaRowBytes, Wt + (size_t)key * D, kTmaRowBytes, &bars[q * 8 + grp]);
  };
  if (lane == 0) {
    if (g0 < U) {
      kr0 = __ldg(unique + g0);
      ar0 = A[kr0];
      issue(0, g0, kr0);
    }
    if (g0 + gstride < U) {
      kr1 = __ldg(unique + g0 + gstride);
      ar1 = A[kr1];
      issue(1, g0 + gstride, kr1);
    }
    const int64_t un = g0 + S * gstride;
    knext = un < U ? __ldg(unique + un) : 0u;
  }
  const double dimD = (double)D;
  int it = 0;
  for (int64_t ub = gbase; ub < U; ub += gstride, ++it) {  // uniform per warp
    const int64_t u = g0 + (ub - gbase);
    const bool has = u < U;
    const int q = it & 1;
    const uint32_t par = (uint32_t)(it >> 1) & 1u;
    const uint32_t key = __shfl_sync(kFull, q ? kr1 : kr0, 0, LPB);
    const float arow = __shfl_sync(kFull, q ? ar1 : ar0, 0, LPB);
    float4 g[VPL], w[VPL];
    if (has) {
      mbar_wait(&bars[q * 8 + grp], par);
      const float4* sg = reinterpret_cast<const float4*>(slots + (size_t)(q * 8 + grp) * 2 * kTmaRowBytes);
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int fi = rot_idx<LPB, VPL>(lane, v, rot);
        const float4 Gv = sg[fi];
        g[v] = make_float4(__fmul_rn(Gv.x, c), __fmul_rn(Gv.y, c), __fmul_rn(Gv.z, c), __fmul_rn(Gv.w, c));
        w[v] = sg[16 + fi];
      }
    } else {
#pragma unroll
      for (int v = 0; v < VPL; ++v) g[v] = w[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();  // the group has read slot q: it may be refilled
    if (lane == 0) {
      const int64_t un = u + S * gstride;
      if (un < U) {
        const float an = A[knext];
        if (q) { kr1 = knext; ar1 = an; } else { kr0 = knext; ar0 = an; }
        issue(q, un, knext);
        const int64_t unn = un + gstride;
        knext = unn < U ? __ldg(unique + unn) : 0u;
      }
    }
    double ss = 0.0;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      ss += (double)g[v].x * (double)g[v].x;
      ss += (double)g[v].y * (double)g[v].y;
      ss += (double)g[v].z * (double)g[v].z;
      ss += (double)g[v].w * (double)g[v].w;
    }
    ss = group_sum<LPB>(ss);
    const float s2 = (float)(ss / dimD);
    const float a = __fadd_rn(arow, s2);
    const float den = __fadd_rn(__fsqrt_rn(a), eps);
    const float mult = __fdiv_rn(lr, den);
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      w[v].x = __fsub_rn(w[v].x, __fmul_rn(mult, g[v].x));
      w[v].y = __fsub_rn(w[v].y, __fmul_rn(mult, g[v].y));
      w[v].z = __fsub_rn(w[v].z, __fmul_rn(mult, g[v].z));
      w[v].w = __fsub_rn(w[v].w, __fmul_rn(mult, g[v].w));
    }
    if (has) {
      if (lane == 0) A[key] = a;
#pragma unroll
      for (int v = 0; v < VPL; ++v) st_f4(Wt + (size_t)key * D + 4 * rot_idx<LPB, VPL>(lane, v, rot), w[v]);
    }
    if (REQUANT)
      quantize_group_row<LPB, VPL>(w, D, lane, has, codes + (size_t)key * qpitch, meta_off, qpitch, minmax,
                                   status, rot);
  }
}

// ---------------------------------------------------------------------------
// launchers
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

static Geom geom_target(int pitch, int target);

#define LIRANK_GEOM4_DISPATCH(G, KERNEL_LAUNCH)                             \
  do {                                                                      \
    if ((G).lpb == 1) {                                                     \
      if ((G).vpl == 1) { constexpr int L_ = 1, V_ = 1; KERNEL_LAUNCH; }    \
      else if ((G).vpl == 2) { constexpr int L_ = 1, V_ = 2; KERNEL_LAUNCH; } \
      else { constexpr int L_ = 1, V_ = 4; KERNEL_LAUNCH; }                 \
    } else if ((G).lpb == 2) { constexpr int L_ = 2, V_ = 4; KERNEL_LAUNCH; } \
    else if ((G).lpb == 4) { constexpr int L_ = 4, V_ = 4; KERNEL_LAUNCH; } \
    else if ((G).lpb == 8) { constexpr int L_ = 8, V_ = 4; KERNEL_LAUNCH; } \
    else if ((G).lpb == 16) { constexpr int L_ = 16, V_ = 4; KERNEL_LAUNCH; } \
    else if ((G).vpl <= 4) { constexpr int L_ = 32, V_ = 4; KERNEL_LAUNCH; } \
    else { constexpr int L_ = 32, V_ = 8; KERNEL_LAUNCH; }                  \
  } while (0)

#define LIRANK_GEOM2_DISPATCH(G, KERNEL_LAUNCH)                             \
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

// Grid-stride kernels: by default one wave of exactly the CTAs that fit (148 SMs x the
// kernel's occupancy), so no partial last wave; fewer CTAs when there is less work.
// `waves` > 1 oversubscribes: for the random-access update, later CTAs fill SMs whose
// first CTAs finished early (measured 0.58 -> 0.55 ms at 8 CTAs/SM requested vs 3 resident).
static unsigned persistent_grid(const void* kernel, int64_t groups, int lpb, int waves = 1) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms < 1) sms = 148;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t want = (groups * lpb + 255) / 256;
  const int64_t cap = (int64_t)sms * (waves > 1 ? 8 : per_sm);
  return (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
}

cudaError_t launch_segreduce(const BwdArgs& a, int64_t* launches, cudaStream_t s) {
  if (a.nnz == 0) return cudaSuccess;
  const Geom g = geom_target(a.pitch, 2);  // D=64: 8 lanes x 2 float4 per occurrence
  cudaError_t e = cudaMemsetAsync(a.owner_count, 0, 4 * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)((a.chunks * g.lpb + 255) / 256);
  const bool full_row = (a.D & 3) == 0 && a.pitch == a.D && a.D == 4 * g.lpb * g.vpl;
  // the ALU-widening pass, then the exact re-run that returns at once unless a lane met an
  // Inf / NaN (Feed-1: 0.607 -> 0.567 ms; alpha = 0 0.840 -> 0.842; Ads 2.00 -> 1.967; the
  // re-run folded into the same kernel behind a warp vote measured 0.592 ms)
#define LAUNCH_SR(MEAN, MODE)                                                                     \
  LIRANK_GEOM2_DISPATCH(g, (launch_pdl(full_row ? k_segreduce<L_, V_, MEAN, true, MODE> : k_segreduce<L_, V_, MEAN, false, MODE>, \
                              MODE == 2 ? (grid < 148u ? grid : 148u) : grid, 256, 0, s, \
                              a.seg, a.U, a.kv, a.chunk_u0, a.grad, a.offsets, a.B, a.F, a.D, \
                              a.pitch, a.chunks, a.chunk_log2, a.G, a.part_first, a.part_last, \
                              a.norm_main, a.norm_fix, a.owner_list, a.owner_count, (int64_t)grid)))
  if (a.mean) { LAUNCH_SR(true, 1); LAUNCH_SR(true, 2); }
  else { LAUNCH_SR(false, 1); LAUNCH_SR(false, 2); }
  ++*launches;
#undef LAUNCH_SR
  ++*launches;
  uint32_t* long_count = a.owner_count + 1;
  uint32_t* long_list = a.owner_list + a.chunks;  // [2 * chunks] after the owner list
  uint32_t* big_count = a.owner_count + 3;
  uint32_t* big_list = a.owner_list + 3 * a.chunks;  // [2 * chunks / kFixBig] after the long list
  LIRANK_GEOM2_DISPATCH(g, (launch_pdl(k_fixup_short<L_, V_>, persistent_grid((const void*)k_fixup_short<L_, V_>, a.chunks, L_), 256, 0, s,
                              a.seg, a.U, a.chunk_u0, a.pitch, a.part_first, a.part_last,
                              a.owner_list, a.owner_count, a.G, a.norm_fix, long_list, long_count, big_list, big_count,
                              a.chunk_log2)));
  ++*launches;
  const int nsplit = a.pitch < kFixThreads ? kFixThreads / a.pitch : 1;
  const size_t smem = sizeof(double) * (size_t)(nsplit * a.pitch > kFixThreads ? nsplit * a.pitch : kFixThreads);
  launch_pdl(k_fixup_long_pieces, 148, kFixThreads, smem, s, a.seg, a.pitch, a.part_first, big_list, big_count,
             a.chunk_log2);
  launch_pdl(k_fixup_long, 148, kFixThreads, smem, s, a.seg, a.pitch, a.part_first, a.part_last,
             long_list, long_count, a.G, a.norm_fix, a.chunk_log2);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_norm_partial(const BwdArgs& a, cudaStream_t s) {
  const int64_t want = (a.chunks + 1023) / 1024;
  const unsigned grid = (unsigned)(want < 1 ? 1 : (want < kNormParts ? want : kNormParts));
  launch_pdl(k_norm_partial, grid, 256, 0, s, a.norm_main, a.norm_fix, a.chunks, a.norm_parts,
             a.norm_done, a.S_local);
  return cudaGetLastError();
}

cudaError_t launch_norm_finalize(const double* parts, int nparts, const BwdArgs& a,
                                 cudaStream_t s) {
  launch_pdl(k_norm_finalize, 1, 1, 0, s, parts, nparts, a.extra_sq_norm, a.extra_dev, a.max_norm,
             a.S_global, a.clip, a.clip_out, a.status);
  return cudaGetLastError();
}

cudaError_t launch_adagrad(const BwdArgs& a, cudaStream_t s) {
  if (a.nnz == 0) return cudaSuccess;
  // D=64: 16 lanes x 1 float4 per row without re-quantization; with it, 4 lanes x 4 float4
  // (the row's min/max and the per-row divides are then shared by 4 lanes, not 16) at 3
  // CTAs/SM (measured: 0.68 -> 0.55 ms on Feed-1).
  const bool rq = a.q8_codes != nullptr;
  if (a.rowwise && a.pitch == 64 && a.D == 64 && a.tma) {  // TMA-pipelined update (D = 64)
    // function attributes and occupancy are per device and per kernel variant: cached so
    // (per device, variant) they are set before any graph capture of a step
    static int per_sm_cache[kMaxDevices][2] = {};
    auto kern = rq ? (const void*)k_adagrad_tma<true> : (const void*)k_adagrad_tma<false>;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    const int dv = dev >= 0 && dev < kMaxDevices ? dev : 0;
    int& per_sm = per_sm_cache[dv][rq ? 1 : 0];
    if (per_sm == 0 || dev != dv) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
      int ps = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, 256, kTmaSmem) != cudaSuccess || ps < 1) ps = 1;
      per_sm = ps;
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (a.nnz * 4 + 255) / 256;
    const int64_t cap = (int64_t)sms * per_sm * kTmaWaves;
    const unsigned grid = (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
    if (rq)
      launch_pdl(k_adagrad_tma<true>, grid, 256, kTmaSmem, s, a.unique, a.U, a.G, a.clip, a.Wt, a.A, a.lr,
                 a.eps, a.q8_codes, a.qpitch, a.q8_meta_off, a.q8_minmax, a.status);
    else
      launch_pdl(k_adagrad_tma<false>, grid, 256, kTmaSmem, s, a.unique, a.U, a.G, a.clip, a.Wt, a.A, a.lr,
                 a.eps, a.q8_codes, a.qpitch, a.q8_meta_off, a.q8_minmax, a.status);
    return cudaGetLastError();
  }
  const Geom g = rq ? geom_target(a.pitch, 4) : geom_for(a.pitch);
#define LAUNCH_AG(DISPATCH, RW, RQ)                                                         \
  DISPATCH(g, (launch_pdl(k_adagrad<L_, V_, RW, RQ>, persistent_grid((const void*)k_adagrad<L_, V_, RW, RQ>, \
                                                            a.nnz, L_, 2), 256, 0, s,       \
                  a.unique, a.U, a.G, a.clip, a.Wt, a.A, a.pitch, a.D, a.lr, a.eps,         \
                  a.q8_codes, a.qpitch, a.q8_meta_off, a.q8_minmax, a.status)))
  if (a.rowwise) {
    if (rq) LAUNCH_AG(LIRANK_GEOM4_DISPATCH, true, true);
    else LAUNCH_AG(LIRANK_GEOM_DISPATCH, true, false);
  } else {
    if (rq) LAUNCH_AG(LIRANK_GEOM4_DISPATCH, false, true);
    else LAUNCH_AG(LIRANK_GEOM_DISPATCH, false, false);
  }
#undef LAUNCH_AG
  return cudaGetLastError();
}

// Geometry with about `target` float4 vectors per lane (fewer lanes per row: cheaper
// per-row reductions and more rows in flight per warp).
static Geom geom_target(int pitch, int target) {
  const int nvec = pitch / 4;
  int lpb = 1;
  while (lpb * target < nvec && lpb < 32) lpb <<= 1;
  return Geom{lpb, (nvec + lpb - 1) / lpb};
}
static Geom quant_geom(int pitch) { return geom_target(pitch, 4); }

cudaError_t launch_quantize(const float* W, int pitch, int64_t rows, int D, uint8_t* codes,
                            int qpitch, int meta_off, bool minmax, uint32_t* status, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  const Geom g = quant_geom(pitch);
#define LAUNCH_Q(L, V)                                                                 \
  launch_pdl(k_quantize<L, V>, persistent_grid((const void*)k_quantize<L, V>, rows, L), 256, 0, s, \
      W, pitch, rows, D, codes, qpitch, meta_off, minmax, status)
  if (g.lpb == 1) {
    if (g.vpl == 1) LAUNCH_Q(1, 1); else if (g.vpl == 2) LAUNCH_Q(1, 2); else if (g.vpl == 3) LAUNCH_Q(1, 3); else LAUNCH_Q(1, 4);
  } else if (g.lpb == 2) { if (g.vpl <= 3) LAUNCH_Q(2, 3); else LAUNCH_Q(2, 4); }
  else if (g.lpb == 4) { if (g.vpl <= 3) LAUNCH_Q(4, 3); else LAUNCH_Q(4, 4); }
  else if (g.lpb == 8) { if (g.vpl <= 3) LAUNCH_Q(8, 3); else LAUNCH_Q(8, 4); }
  else if (g.lpb == 16) { if (g.vpl <= 3) LAUNCH_Q(16, 3); else LAUNCH_Q(16, 4); }
  else { if (g.vpl <= 4) LAUNCH_Q(32, 4); else LAUNCH_Q(32, 8); }
#undef LAUNCH_Q
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// misc
// ---------------------------------------------------------------------------
__global__ void k_fill(float* p, int64_t n, float v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

cudaError_t launch_fill(float* p, int64_t n, float v, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_fill<<<148 * 8, 256, 0, s>>>(p, n, v);
  return cudaGetLastError();
}

}  // namespace lirank
