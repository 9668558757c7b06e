// incremental.cu -- NEXT-3: incremental training (Eq. 2-3).
//
// Total loss = loss_D(w) + lambda_f/2 [alpha (w-w0)^T H0 (w-w0) + (1-alpha)(w-w1)^T H1 (w-w1)]
// with diagonal H (empirical-FIM diagonal), w0 the cold-start model, w1 = w_{t-1}.
//
// k_cold_init: w = alpha w0 + (1-alpha) w1 over the whole local table, streamed
//   with 128-bit loads/stores (3 x 4 B per element: an HBM-bound pass).
// k_fim_penalty: after the segment-reduce, the penalty gradient
//   lambda [alpha H0 (w-w0) + (1-alpha) H1 (w-w1)] is added to G[u] of every TOUCHED row
//   (reading 30: lazy, only the rows a step updates) before the global norm, and the
//   row's squared norm is re-accumulated (the segment-reduce's partials are replaced):
//   one lane group per row, grid-stride with a fixed group count, one fp64 partial per
//   group in group order -> deterministic.
#include "common.cuh"
#include "kernels.h"

namespace lirank {

namespace {

__device__ __forceinline__ float pen1(float w, float a0, float h0, float a1, float h1, float alpha,
                                      float beta, float lambda, bool t0, bool t1) {
  const float p0 = t0 ? __fmul_rn(alpha, __fmul_rn(h0, __fsub_rn(w, a0))) : 0.0f;
  const float p1 = t1 ? __fmul_rn(beta, __fmul_rn(h1, __fsub_rn(w, a1))) : 0.0f;
  return __fmul_rn(lambda, __fadd_rn(p0, p1));
}

}  // namespace

__global__ void __launch_bounds__(256)
k_cold_init(const float4* __restrict__ w0, const float4* __restrict__ w1, int64_t n4, float alpha,
            float4* __restrict__ w) {
  const float beta = __fsub_rn(1.0f, alpha);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = ld_nc_f4(reinterpret_cast<const float*>(w0 + i));
    const float4 b = ld_nc_f4(reinterpret_cast<const float*>(w1 + i));
    float4 r;
    r.x = __fadd_rn(__fmul_rn(alpha, a.x), __fmul_rn(beta, b.x));
    r.y = __fadd_rn(__fmul_rn(alpha, a.y), __fmul_rn(beta, b.y));
    r.z = __fadd_rn(__fmul_rn(alpha, a.z), __fmul_rn(beta, b.z));
    r.w = __fadd_rn(__fmul_rn(alpha, a.w), __fmul_rn(beta, b.w));
    w[i] = r;
  }
}

template <int LPB, int VPL>
__global__ void __launch_bounds__(256)
k_fim_penalty(const uint32_t* __restrict__ unique, const uint32_t* __restrict__ Up,
              float* __restrict__ G, const float* __restrict__ W, const float* __restrict__ w0,
              const float* __restrict__ H0, const float* __restrict__ w1,
              const float* __restrict__ H1, int pitch, int D, float lambda, float alpha,
              int64_t ngroups, double* __restrict__ norm_part, double* __restrict__ norm_zero) {
  const uint32_t U = *Up;
  const int lane = threadIdx.x & (LPB - 1);
  const int64_t g0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPB;
  const int64_t gbase = g0 - (threadIdx.x & 31) / LPB;
  const int nvec = pitch >> 2;
  const bool t0 = w0 != nullptr && H0 != nullptr, t1 = w1 != nullptr && H1 != nullptr;
  const float beta = __fsub_rn(1.0f, alpha);
  double nrm = 0.0;
  for (int64_t ub = gbase; ub < U; ub += ngroups) {  // uniform per warp
    const int64_t u = g0 + (ub - gbase);
    if (u < U && g0 < ngroups) {
      const size_t row = (size_t)__ldg(unique + u) * pitch;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int vi = lane + v * LPB;
        if (vi < nvec) {
          const size_t o = row + 4 * vi;
          const float4 w = ld_f4(W + o);
          const float4 a0 = t0 ? ld_nc_f4(w0 + o) : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 h0 = t0 ? ld_nc_f4(H0 + o) : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 a1 = t1 ? ld_nc_f4(w1 + o) : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 h1 = t1 ? ld_nc_f4(H1 + o) : make_float4(0.f, 0.f, 0.f, 0.f);
          float* gp = G + (size_t)u * pitch + 4 * vi;
          float4 g = ld_f4(gp);
          g.x = __fadd_rn(g.x, pen1(w.x, a0.x, h0.x, a1.x, h1.x, alpha, beta, lambda, t0, t1));
          g.y = __fadd_rn(g.y, pen1(w.y, a0.y, h0.y, a1.y, h1.y, alpha, beta, lambda, t0, t1));
          g.z = __fadd_rn(g.z, pen1(w.z, a0.z, h0.z, a1.z, h1.z, alpha, beta, lambda, t0, t1));
          g.w = __fadd_rn(g.w, pen1(w.w, a0.w, h0.w, a1.w, h1.w, alpha, beta, lambda, t0, t1));
          const int d = 4 * vi;  // pads (d >= D) stay out of the norm
          if (d + 0 < D) nrm += (double)g.x * (double)g.x; else g.x = 0.f;
          if (d + 1 < D) nrm += (double)g.y * (double)g.y; else g.y = 0.f;
          if (d + 2 < D) nrm += (double)g.z * (double)g.z; else g.z = 0.f;
          if (d + 3 < D) nrm += (double)g.w * (double)g.w; else g.w = 0.f;
          st_f4(gp, g);
        }
      }
    }
  }
#pragma unroll
  for (int o = LPB / 2; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o, LPB);
  if (lane == 0 && g0 < ngroups) {
    norm_part[g0] = nrm;
    norm_zero[g0] = 0.0;
  }
}

cudaError_t launch_cold_init(const float* w0, const float* w1, int64_t n, float alpha, float* w,
                             cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t n4 = n / 4;  // n = rows * pitch, pitch % 4 == 0
  const int64_t want = (n4 + 255) / 256;
  const unsigned grid = (unsigned)(want < 148 * 8 ? (want < 1 ? 1 : want) : 148 * 8);
  k_cold_init<<<grid, 256, 0, s>>>(reinterpret_cast<const float4*>(w0),
                                   reinterpret_cast<const float4*>(w1), n4, alpha,
                                   reinterpret_cast<float4*>(w));
  return cudaGetLastError();
}

int64_t launch_fim_penalty(const BwdArgs& a, const FimArgs& f, cudaStream_t s) {
  if (a.nnz == 0) return 0;
  const Geom g = geom_for(a.pitch);
  // fixed number of lane groups (<= the chunk-partial capacity), independent of U
  const int64_t cap_groups = (int64_t)148 * 8 * 256 / g.lpb;
  const int64_t ngroups = a.chunks < cap_groups ? a.chunks : cap_groups;  // >= 1
  const unsigned grid = (unsigned)((ngroups * g.lpb + 255) / 256);  // groups past ngroups idle
#define FIMX(L, V)                                                                              \
  k_fim_penalty<L, V><<<grid, 256, 0, s>>>(a.unique, a.U, a.G, a.Wt, f.w0, f.H0, f.w1, f.H1,    \
                                           a.pitch, a.D, f.lambda, f.alpha, ngroups,            \
                                           a.norm_main, a.norm_fix)
  if (g.lpb == 1) FIMX(1, 1); else if (g.lpb == 2) FIMX(2, 1); else if (g.lpb == 4) FIMX(4, 1);
  else if (g.lpb == 8) FIMX(8, 1); else if (g.lpb == 16) FIMX(16, 1);
  else if (g.vpl == 1) FIMX(32, 1); else if (g.vpl == 2) FIMX(32, 2); else if (g.vpl <= 4) FIMX(32, 4);
  else FIMX(32, 8);
#undef FIMX
  return cudaGetLastError() == cudaSuccess ? ngroups : -1;
}

}  // namespace lirank
