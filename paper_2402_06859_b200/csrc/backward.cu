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
//   occurrence list is cut into fixed chunks of kChunk, one lane group (LPB lanes, one
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
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace lirank {

namespace {

constexpr int kFixLong = 8;           // spans of more chunks than this use a whole CTA
constexpr int kFixThreads = 512;

template <int LPB>
__device__ __forceinline__ double group_sum(double x) {
  const unsigned m = group_mask<LPB>();
#pragma unroll
  for (int o = LPB / 2; o > 0; o >>= 1) x += __shfl_xor_sync(m, x, o, LPB);
  return x;
}

template <int VPL>
__device__ __forceinline__ void load_grad_row(const float* __restrict__ grad, size_t row_off,
                                              int D, int lane, int LPB, float4 (&r)[VPL]) {
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int d = 4 * (lane + v * LPB);
    if ((D & 3) == 0) {
      r[v] = d < D ? __ldg(reinterpret_cast<const float4*>(grad + row_off + d))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
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

// Finish a complete segment: G[u] = (float)acc, return this lane's sum of (double)G^2.
template <int VPL>
__device__ __forceinline__ double write_G(float* G, int pitch, uint32_t u, int lane, int LPB,
                                          const double (&acc)[VPL][4]) {
  double nrm = 0.0;
  const int nvec = pitch >> 2;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int vi = lane + v * LPB;
    if (vi < nvec) {
      float4 g = make_float4((float)acc[v][0], (float)acc[v][1], (float)acc[v][2],
                             (float)acc[v][3]);
      st_f4(G + (size_t)u * pitch + 4 * vi, g);
      nrm += (double)g.x * (double)g.x;
      nrm += (double)g.y * (double)g.y;
      nrm += (double)g.z * (double)g.z;
      nrm += (double)g.w * (double)g.w;
    }
  }
  return nrm;
}

template <int VPL>
__device__ __forceinline__ void write_partial(double* P, int pitch, int64_t c, int lane, int LPB,
                                              const double (&acc)[VPL][4]) {
  const int nvec = pitch >> 2;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int vi = lane + v * LPB;
    if (vi < nvec) {
      double* p = P + (size_t)c * pitch + 4 * vi;
      reinterpret_cast<double2*>(p)[0] = make_double2(acc[v][0], acc[v][1]);
      reinterpret_cast<double2*>(p)[1] = make_double2(acc[v][2], acc[v][3]);
    }
  }
}

}  // namespace

template <int LPB, int VPL, bool MEAN>
__global__ void __launch_bounds__(256)
k_segreduce(const uint32_t* __restrict__ seg, const uint32_t* __restrict__ Up,
            const uint32_t* __restrict__ vals, const float* __restrict__ grad,
            const int* __restrict__ offsets, int B, int F, int D, int pitch, int64_t chunks,
            float* __restrict__ G, double* __restrict__ part_first,
            double* __restrict__ part_last, double* __restrict__ norm_main,
            double* __restrict__ norm_fix, uint32_t* __restrict__ owner_list,
            uint32_t* owner_count) {
  constexpr int UNR = (VPL == 1) ? 4 : (VPL == 2 ? 2 : 1);
  const int lane = threadIdx.x & (LPB - 1);
  const unsigned gmask = group_mask<LPB>();
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
  if (c >= chunks) return;
  const uint32_t U = *Up;
  const int64_t n_valid = seg[U];
  const int64_t k0 = c * kChunk;
  if (k0 >= n_valid) {
    if (lane == 0) { norm_main[c] = 0.0; norm_fix[c] = 0.0; }
    return;
  }
  const int64_t k1 = min(k0 + (int64_t)kChunk, n_valid);
  // u0 = last segment with seg[u] <= k0
  uint32_t lo = 0, hi = U - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if ((int64_t)__ldg(seg + mid) <= k0) lo = mid; else hi = mid - 1;
  }
  uint32_t u = lo;
  int64_t s_start = __ldg(seg + u), s_end = __ldg(seg + u + 1);

  double acc[VPL][4];
  zero(acc);
  double nrm = 0.0;

  for (int64_t kb = k0; kb < k1; kb += LPB) {
    const int64_t kl = kb + lane;
    uint32_t bag = 0;
    double inv = 1.0;
    if (kl < k1) {
      bag = __ldg(vals + kl);
      if (MEAN) inv = 1.0 / (double)(__ldg(offsets + bag + 1) - __ldg(offsets + bag));
    }
    const int cnt = (int)min((int64_t)LPB, k1 - kb);
    for (int jj = 0; jj < cnt; jj += UNR) {
      float4 r[UNR][VPL];
      double iv[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const uint32_t bq = __shfl_sync(gmask, bag, (jj + q) & (LPB - 1), LPB);
        iv[q] = MEAN ? __shfl_sync(gmask, inv, (jj + q) & (LPB - 1), LPB) : 1.0;
        if (jj + q < cnt) {
          const uint32_t f = bq / (uint32_t)B, b = bq - f * (uint32_t)B;
          load_grad_row<VPL>(grad, ((size_t)b * F + f) * D, D, lane, LPB, r[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        if (jj + q < cnt) {
          const int64_t occ = kb + jj + q;
          if (occ == s_end) {  // segment u finished inside this chunk
            if (s_start < k0) write_partial<VPL>(part_first, pitch, c, lane, LPB, acc);
            else nrm += write_G<VPL>(G, pitch, u, lane, LPB, acc);
            zero(acc);
            ++u;
            s_start = s_end;
            s_end = __ldg(seg + u + 1);
          }
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            if (MEAN) {
              acc[v][0] += (double)r[q][v].x * iv[q];
              acc[v][1] += (double)r[q][v].y * iv[q];
              acc[v][2] += (double)r[q][v].z * iv[q];
              acc[v][3] += (double)r[q][v].w * iv[q];
            } else {
              acc[v][0] += (double)r[q][v].x;
              acc[v][1] += (double)r[q][v].y;
              acc[v][2] += (double)r[q][v].z;
              acc[v][3] += (double)r[q][v].w;
            }
          }
        }
      }
    }
  }
  // the segment containing occurrence k1-1
  bool owner = false;
  if (s_start < k0) {
    write_partial<VPL>(part_first, pitch, c, lane, LPB, acc);  // continues or ends here
  } else if (s_end <= k1) {
    nrm += write_G<VPL>(G, pitch, u, lane, LPB, acc);
  } else {
    write_partial<VPL>(part_last, pitch, c, lane, LPB, acc);  // starts here, spills over
    owner = true;
  }
  nrm = group_sum<LPB>(nrm);
  if (lane == 0) {
    norm_main[c] = nrm;
    norm_fix[c] = 0.0;
    if (owner) {
      const uint32_t slot = atomicAdd(owner_count, 1u);
      owner_list[slot] = (uint32_t)c;
    }
  }
}

// Fix-up of segments spanning chunks.  Entry e = chunk c_s where segment u starts and
// spills over; its sum = part_last[c_s] + sum_{c = c_s+1 .. c_e} part_first[c].
// One lane group per entry for short spans; entries spanning > kFixLong chunks are left
// to k_fixup_long.
template <int LPB, int VPL>
__global__ void __launch_bounds__(256)
k_fixup_short(const uint32_t* __restrict__ seg, const uint32_t* __restrict__ Up,
              int pitch, const double* __restrict__ part_first,
              const double* __restrict__ part_last, const uint32_t* __restrict__ owner_list,
              const uint32_t* __restrict__ owner_count, float* __restrict__ G,
              double* __restrict__ norm_fix, uint32_t* long_list, uint32_t* long_count) {
  const int lane = threadIdx.x & (LPB - 1);
  const int64_t gstride = ((int64_t)gridDim.x * blockDim.x) / LPB;
  const uint32_t n_entries = *owner_count;
  const uint32_t U = *Up;
  const int nvec = pitch >> 2;
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPB; e < n_entries;
       e += gstride) {
    const uint32_t cs = owner_list[e];
    const int64_t k0 = (int64_t)cs * kChunk;
    // segment that starts in chunk cs and spills over = the last segment with seg <= k0+kChunk-1
    uint32_t lo = 0, hi = U - 1;
    const int64_t kl = k0 + kChunk - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if ((int64_t)__ldg(seg + mid) <= kl) lo = mid; else hi = mid - 1;
    }
    const uint32_t u = lo;
    const int64_t s_end = __ldg(seg + u + 1);
    const int64_t ce = (s_end - 1) / kChunk;
    if (ce - cs > kFixLong) {
      if (lane == 0) {
        const uint32_t slot = atomicAdd(long_count, 1u);
        long_list[2 * slot] = cs;
        long_list[2 * slot + 1] = u;
      }
      continue;
    }
    double nrm = 0.0;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int vi = lane + v * LPB;
      if (vi < nvec) {
        const double* p = part_last + (size_t)cs * pitch + 4 * vi;
        double a0 = p[0], a1 = p[1], a2 = p[2], a3 = p[3];
        for (int64_t cc = cs + 1; cc <= ce; ++cc) {
          const double* q = part_first + (size_t)cc * pitch + 4 * vi;
          a0 += q[0]; a1 += q[1]; a2 += q[2]; a3 += q[3];
        }
        const float4 g = make_float4((float)a0, (float)a1, (float)a2, (float)a3);
        st_f4(G + (size_t)u * pitch + 4 * vi, g);
        nrm += (double)g.x * g.x + (double)g.y * g.y + (double)g.z * g.z + (double)g.w * g.w;
      }
    }
    nrm = group_sum<LPB>(nrm);
    if (lane == 0) norm_fix[cs] = nrm;
  }
}

// Long spans: one CTA per entry.  Thread t owns element (t % nelem) of the row for chunk
// sub-range (t / nelem); sub-ranges are contiguous and combined in order.
__global__ void __launch_bounds__(kFixThreads)
k_fixup_long(const uint32_t* __restrict__ seg, int pitch, const double* __restrict__ part_first,
             const double* __restrict__ part_last, const uint32_t* __restrict__ long_list,
             const uint32_t* __restrict__ long_count, float* __restrict__ G,
             double* __restrict__ norm_fix) {
  extern __shared__ double sm[];  // [nsplit][pitch]
  const uint32_t n_entries = *long_count;
  const int nsplit = max(1, kFixThreads / pitch);
  for (uint32_t e = blockIdx.x; e < n_entries; e += gridDim.x) {
    const uint32_t cs = long_list[2 * e], u = long_list[2 * e + 1];
    const int64_t s_end = __ldg(seg + u + 1);
    const int64_t ce = (s_end - 1) / kChunk;
    const int64_t nch = ce - cs;  // chunks cs+1 .. ce
    for (int t = threadIdx.x; t < nsplit * pitch; t += blockDim.x) {
      const int el = t % pitch, sp = t / pitch;
      const int64_t a = cs + 1 + (nch * sp) / nsplit;
      const int64_t b = cs + 1 + (nch * (sp + 1)) / nsplit;
      double s = 0.0;
      int64_t cc = a;
      for (; cc + 4 <= b; cc += 4) {
        const double x0 = part_first[(size_t)cc * pitch + el];
        const double x1 = part_first[(size_t)(cc + 1) * pitch + el];
        const double x2 = part_first[(size_t)(cc + 2) * pitch + el];
        const double x3 = part_first[(size_t)(cc + 3) * pitch + el];
        s += x0; s += x1; s += x2; s += x3;
      }
      for (; cc < b; ++cc) s += part_first[(size_t)cc * pitch + el];
      sm[sp * pitch + el] = s;
    }
    __syncthreads();
    double nrm_part = 0.0;
    for (int el = threadIdx.x; el < pitch; el += blockDim.x) {
      double s = part_last[(size_t)cs * pitch + el];
      for (int sp = 0; sp < nsplit; ++sp) s += sm[sp * pitch + el];
      const float g = (float)s;
      G[(size_t)u * pitch + el] = g;
      nrm_part += (double)g * (double)g;
    }
    // deterministic block reduction of nrm_part (threads < pitch hold values)
    __syncthreads();
    sm[threadIdx.x] = nrm_part;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) norm_fix[cs] = sm[0];
    __syncthreads();
  }
}

// S_local = sum over chunks (index order) of norm_main + norm_fix.  One CTA, fixed tree.
__global__ void __launch_bounds__(1024)
k_norm_partial(const double* __restrict__ norm_main, const double* __restrict__ norm_fix,
               int64_t chunks, double* S_local) {
  __shared__ double sm[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < chunks; i += blockDim.x) {
    s += norm_main[i];
    s += norm_fix[i];
  }
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *S_local = sm[0];
}

// S = sum of rank partials in rank order + extra; c = (n > max_norm) ? max_norm/n : 1.
// Non-finite S: c = -1 (the update kernel then skips every row) + sticky status.
__global__ void k_norm_finalize(const double* parts, int nparts, double extra, float max_norm,
                                double* S_global, float* clip, uint32_t* status) {
  double S = 0.0;
  for (int r = 0; r < nparts; ++r) S += parts[r];
  S += extra;
  *S_global = S;
  if (!isfinite(S)) {
    *clip = -1.0f;
    atomicOr(status, kStNonFinite);
    return;
  }
  const double n = sqrt(S);
  *clip = (n > (double)max_norm) ? (float)((double)max_norm / n) : 1.0f;
}

// ---------------------------------------------------------------------------
// middle-max quantization of one row held by a lane group (used by a9 and REQUANT)
// ---------------------------------------------------------------------------
template <int LPB, int VPL>
__device__ __forceinline__ void quantize_group_row(const float4 (&x)[VPL], int D, int lane,
                                                   uint8_t* __restrict__ code_row,
                                                   float2* __restrict__ meta_row,
                                                   uint32_t* status) {
  const unsigned gm = group_mask<LPB>();
  float mn = FLT_MAX, mx = -FLT_MAX;
  bool finite = true;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int d = 4 * (lane + v * LPB);
    const float e[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (d + i < D) {
        finite &= isfinite(e[i]);
        mn = fminf(mn, e[i]);
        mx = fmaxf(mx, e[i]);
      }
  }
#pragma unroll
  for (int o = LPB / 2; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(gm, mn, o, LPB));
    mx = fmaxf(mx, __shfl_xor_sync(gm, mx, o, LPB));
    finite = __shfl_xor_sync(gm, (int)finite, o, LPB) && finite;
  }
  float middle, scale;
  bool zero_codes;
  if (!finite) {
    middle = 0.f; scale = 0.f; zero_codes = true;
    if (lane == 0) atomicOr(status, kStNonFinite);
  } else if (mx == mn) {
    middle = mx; scale = 0.f; zero_codes = true;
  } else {
    // X^middle = (X^max * 2^(b-1) + X^min * (2^(b-1) - 1)) / (2^b - 1), b = 8
    middle = __fdiv_rn(__fadd_rn(__fmul_rn(mx, 128.0f), __fmul_rn(mn, 127.0f)), 255.0f);
    // X^scale = (X^max - X^min) / (2^b - 1)
    scale = __fdiv_rn(__fsub_rn(mx, mn), 255.0f);
    zero_codes = scale == 0.0f;
  }
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int wi = lane + v * LPB;
    const int d = 4 * wi;
    if (d < D) {
      const float e[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
      uint32_t word = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int code = 0;
        if (!zero_codes && d + i < D) {
          // X^int = round((X - X^middle) / X^scale): half away from zero, saturated
          float r = roundf(__fdiv_rn(__fsub_rn(e[i], middle), scale));
          r = fminf(fmaxf(r, -128.0f), 127.0f);
          code = (int)r;
        }
        word |= ((uint32_t)(code & 0xff)) << (8 * i);
      }
      reinterpret_cast<uint32_t*>(code_row)[wi] = word;
    }
  }
  if (lane == 0) *meta_row = make_float2(middle, scale);
}

template <int LPB, int VPL>
__global__ void __launch_bounds__(256)
k_quantize(const float* __restrict__ W, int pitch, int64_t rows, int D,
           uint8_t* __restrict__ codes, int qpitch, float2* __restrict__ qmeta,
           uint32_t* status) {
  const int lane = threadIdx.x & (LPB - 1);
  const int64_t gstride = ((int64_t)gridDim.x * blockDim.x) / LPB;
  const int nvec = pitch >> 2;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPB; r < rows;
       r += gstride) {
    float4 x[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int vi = lane + v * LPB;
      x[v] = vi < nvec ? ld_nc_f4(W + (size_t)r * pitch + 4 * vi) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    quantize_group_row<LPB, VPL>(x, D, lane, codes + (size_t)r * qpitch, qmeta + r, status);
  }
}

// Fused clip + sparse AdaGrad on the U unique rows (+ optional re-quantize).
template <int LPB, int VPL, bool ROWWISE, bool REQUANT>
__global__ void __launch_bounds__(256)
k_adagrad(const uint32_t* __restrict__ unique, const uint32_t* __restrict__ Up,
          const float* __restrict__ G, const float* __restrict__ clip, float* __restrict__ Wt,
          float* __restrict__ A, int pitch, int D, float lr, float eps,
          uint8_t* __restrict__ codes, int qpitch, float2* __restrict__ qmeta,
          uint32_t* status) {
  const float c = *clip;
  if (c < 0.0f) return;  // non-finite global norm: skip the step
  const uint32_t U = *Up;
  const int lane = threadIdx.x & (LPB - 1);
  const int64_t gstride = ((int64_t)gridDim.x * blockDim.x) / LPB;
  const int nvec = pitch >> 2;
  const double invD = (double)D;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPB; u < U; u += gstride) {
    const uint32_t key = __ldg(unique + u);
    float4 g[VPL], w[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int vi = lane + v * LPB;
      if (vi < nvec) {
        const float4 Gv = ld_nc_f4(G + (size_t)u * pitch + 4 * vi);
        g[v] = make_float4(__fmul_rn(Gv.x, c), __fmul_rn(Gv.y, c), __fmul_rn(Gv.z, c),
                           __fmul_rn(Gv.w, c));
        w[v] = ld_f4(Wt + (size_t)key * pitch + 4 * vi);
      } else {
        g[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        w[v] = g[v];
      }
    }
    if (ROWWISE) {
      double ss = 0.0;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        ss += (double)g[v].x * (double)g[v].x;
        ss += (double)g[v].y * (double)g[v].y;
        ss += (double)g[v].z * (double)g[v].z;
        ss += (double)g[v].w * (double)g[v].w;
      }
      ss = group_sum<LPB>(ss);
      const float s = (float)(ss / invD);
      const float a = __fadd_rn(__ldg(A + key), s);
      const float den = __fadd_rn(__fsqrt_rn(a), eps);
      const float mult = __fdiv_rn(lr, den);
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        w[v].x = __fsub_rn(w[v].x, __fmul_rn(mult, g[v].x));
        w[v].y = __fsub_rn(w[v].y, __fmul_rn(mult, g[v].y));
        w[v].z = __fsub_rn(w[v].z, __fmul_rn(mult, g[v].z));
        w[v].w = __fsub_rn(w[v].w, __fmul_rn(mult, g[v].w));
      }
      if (lane == 0) A[key] = a;
    } else {
      const float nlr = -lr;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int vi = lane + v * LPB;
        if (vi < nvec) {
          float* ap = A + (size_t)key * pitch + 4 * vi;
          float4 a = ld_f4(ap);
          a.x = __fadd_rn(a.x, __fmul_rn(g[v].x, g[v].x));
          a.y = __fadd_rn(a.y, __fmul_rn(g[v].y, g[v].y));
          a.z = __fadd_rn(a.z, __fmul_rn(g[v].z, g[v].z));
          a.w = __fadd_rn(a.w, __fmul_rn(g[v].w, g[v].w));
          w[v].x = __fadd_rn(w[v].x, __fdiv_rn(__fmul_rn(nlr, g[v].x), __fadd_rn(__fsqrt_rn(a.x), eps)));
          w[v].y = __fadd_rn(w[v].y, __fdiv_rn(__fmul_rn(nlr, g[v].y), __fadd_rn(__fsqrt_rn(a.y), eps)));
          w[v].z = __fadd_rn(w[v].z, __fdiv_rn(__fmul_rn(nlr, g[v].z), __fadd_rn(__fsqrt_rn(a.z), eps)));
          w[v].w = __fadd_rn(w[v].w, __fdiv_rn(__fmul_rn(nlr, g[v].w), __fadd_rn(__fsqrt_rn(a.w), eps)));
          st_f4(ap, a);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int vi = lane + v * LPB;
      if (vi < nvec) st_f4(Wt + (size_t)key * pitch + 4 * vi, w[v]);
    }
    if (REQUANT)
      quantize_group_row<LPB, VPL>(w, D, lane, codes + (size_t)key * qpitch, qmeta + key, status);
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

static unsigned persistent_grid(int64_t groups, int lpb) {
  // 148 SMs x 8 resident 256-thread CTAs
  const int64_t want = (groups * lpb + 255) / 256;
  const int64_t cap = 148 * 8;
  return (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
}

cudaError_t launch_segreduce(const BwdArgs& a, int64_t* launches, cudaStream_t s) {
  if (a.nnz == 0) return cudaSuccess;
  const Geom g = geom_for(a.pitch);
  cudaError_t e = cudaMemsetAsync(a.owner_count, 0, 2 * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)((a.chunks * g.lpb + 255) / 256);
#define LAUNCH_SR(MEAN)                                                                     \
  LIRANK_GEOM_DISPATCH(g, (k_segreduce<L_, V_, MEAN><<<grid, 256, 0, s>>>(                 \
                              a.seg, a.U, a.vals, a.grad, a.offsets, a.B, a.F, a.D, a.pitch, \
                              a.chunks, a.G, a.part_first, a.part_last, a.norm_main,        \
                              a.norm_fix, a.owner_list, a.owner_count)))
  if (a.mean) LAUNCH_SR(true); else LAUNCH_SR(false);
#undef LAUNCH_SR
  ++*launches;
  uint32_t* long_count = a.owner_count + 1;
  uint32_t* long_list = a.owner_list + a.chunks;  // [2 * chunks] after the owner list
  const unsigned fgrid = persistent_grid(a.chunks, g.lpb);
  LIRANK_GEOM_DISPATCH(g, (k_fixup_short<L_, V_><<<fgrid, 256, 0, s>>>(
                              a.seg, a.U, a.pitch, a.part_first, a.part_last, a.owner_list,
                              a.owner_count, a.G, a.norm_fix, long_list, long_count)));
  ++*launches;
  const int nsplit = a.pitch < kFixThreads ? kFixThreads / a.pitch : 1;
  const size_t smem = sizeof(double) * (size_t)(nsplit * a.pitch > kFixThreads ? nsplit * a.pitch : kFixThreads);
  k_fixup_long<<<148, kFixThreads, smem, s>>>(a.seg, a.pitch, a.part_first, a.part_last,
                                              long_list, long_count, a.G, a.norm_fix);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_norm_partial(const BwdArgs& a, cudaStream_t s) {
  k_norm_partial<<<1, 1024, 0, s>>>(a.norm_main, a.norm_fix, a.chunks, a.S_local);
  return cudaGetLastError();
}

cudaError_t launch_norm_finalize(const double* parts, int nparts, const BwdArgs& a,
                                 cudaStream_t s) {
  k_norm_finalize<<<1, 1, 0, s>>>(parts, nparts, a.extra_sq_norm, a.max_norm, a.S_global,
                                  a.clip, a.status);
  return cudaGetLastError();
}

cudaError_t launch_adagrad(const BwdArgs& a, cudaStream_t s) {
  if (a.nnz == 0) return cudaSuccess;
  const Geom g = geom_for(a.pitch);
  const unsigned grid = persistent_grid(a.nnz, g.lpb);
#define LAUNCH_AG(RW, RQ)                                                                   \
  LIRANK_GEOM_DISPATCH(g, (k_adagrad<L_, V_, RW, RQ><<<grid, 256, 0, s>>>(                 \
                              a.unique, a.U, a.G, a.clip, a.Wt, a.A, a.pitch, a.D, a.lr,    \
                              a.eps, a.q8_codes, a.qpitch, a.q8_meta, a.status)))
  const bool rq = a.q8_codes != nullptr;
  if (a.rowwise) {
    if (rq) LAUNCH_AG(true, true); else LAUNCH_AG(true, false);
  } else {
    if (rq) LAUNCH_AG(false, true); else LAUNCH_AG(false, false);
  }
#undef LAUNCH_AG
  return cudaGetLastError();
}

cudaError_t launch_quantize(const float* W, int pitch, int64_t rows, int D, uint8_t* codes,
                            int qpitch, float2* qmeta, uint32_t* status, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  const Geom g = geom_for(pitch);
  const unsigned grid = persistent_grid(rows, g.lpb);
  LIRANK_GEOM_DISPATCH(g, (k_quantize<L_, V_><<<grid, 256, 0, s>>>(W, pitch, rows, D, codes,
                                                                    qpitch, qmeta, status)));
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
