// common.cuh -- shared device helpers for the LiRank embedding kernels (sm_100a).
//
// Numerics discipline (SURVEY.md §7 "bit-exactness discipline"): the library is built
// with -fmad=false and without fast-math, and every parity-critical float operation is
// written with an explicit round-to-nearest intrinsic (__fadd_rn, __fmul_rn, __fdiv_rn,
// __fsqrt_rn) so the operation order of SURVEY.md §8(c) is the one executed.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lirank {

constexpr int kWarp = 32;

// Sticky status bits (device word; emb_sync maps them to emb_status).
constexpr uint32_t kStIdRange = 1u;
constexpr uint32_t kStNonFinite = 2u;
constexpr uint32_t kStOverflow = 4u;
constexpr int kMaxDevices = 64;  // per-device caches of launch set-up (function attributes)  // sharded: received ids exceed a planned capacity

// ---------------------------------------------------------------------------
// Row-group geometry.  One "group" of LPB lanes (a power of two <= 32) owns one
// embedding row of nvec = pitch/4 float4 vectors; lane l holds vectors l, l+LPB, ...
// (VPL = ceil(nvec / LPB) per lane).  D=64: LPB=16, VPL=1 -> half-warp per row,
// one 128-bit load per lane, 256 B per row request.
// ---------------------------------------------------------------------------
struct Geom {
  int lpb;  // lanes per group
  int vpl;  // float4 vectors per lane
};

inline Geom geom_for(int pitch) {
  int nvec = pitch / 4;
  int lpb = 1;
  while (lpb < nvec && lpb < 32) lpb <<= 1;
  int vpl = (nvec + lpb - 1) / lpb;
  return Geom{lpb, vpl};
}

// Group-level shuffle helpers (width = LPB).
template <int LPB>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (LPB == 32) {
    return 0xffffffffu;
  } else {
    unsigned lane = threadIdx.x & 31;
    unsigned base = lane & ~(unsigned)(LPB - 1);
    return ((1u << LPB) - 1u) << base;
  }
}

// 128-bit streaming loads/stores.
__device__ __forceinline__ float4 ld_nc_f4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
// L2 eviction-priority hints (createpolicy + .L2::cache_hint): table rows that Zipf traffic
// re-reads are loaded evict_last, results written once are stored evict_first, so streaming
// outputs do not push the hot rows out of the 126 MB L2.
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_l1_f4_hint(const float* p, uint64_t pol) {  // L1-allocating
  float4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float4 ld_nc_f4_hint(const float* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_f4_hint(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ float4 ld_f4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ void st_f4(float* p, float4 v) {
  *reinterpret_cast<float4*>(p) = v;
}
__device__ __forceinline__ int ld_nc_i32(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ double ld_volatile_f64(const double* p) {
  return *reinterpret_cast<const volatile double*>(p);
}
// Paired fp32 arithmetic (sm_100a FADD2 / FFMA2 / FMUL2: two IEEE round-to-nearest fp32
// operations per instruction, each element exactly the scalar __fadd_rn / __fmaf_rn /
// __fmul_rn): half the issue slots of the scalar form on the same FP32 pipe.
__device__ __forceinline__ float2 f2_add_rn(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, r;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 r, a, b;\n\tmov.b64 {%0, %1}, r;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2_mul_rn(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, r;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mul.rn.f32x2 r, a, b;\n\tmov.b64 {%0, %1}, r;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2_fma_rn(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 a, b, c, r;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
      "fma.rn.f32x2 r, a, b, c;\n\tmov.b64 {%0, %1}, r;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
__device__ __forceinline__ float4 f4_add_rn(float4 a, float4 b) {
  const float2 lo = f2_add_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
  const float2 hi = f2_add_rn(make_float2(a.z, a.w), make_float2(b.z, b.w));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

// Programmatic dependent launch: a kernel launched with launch_pdl may be scheduled while its
// stream predecessor drains (its CTAs take SM slots as the predecessor's retire, instead of a
// full drain + launch gap); pdl_wait() -- its first statement -- blocks until the predecessor
// has completed and its memory is visible, so nothing before it may read predecessor output.
// In a kernel launched normally pdl_wait() returns at once.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                     cudaStream_t s, Args... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ void set_status(uint32_t* st, uint32_t bit) {
  // Rare path; one atomic per offending warp is plenty.
  atomicOr(st, bit);
}

// Per-feature metadata resolved on the host (row addressing).
// An id i of feature f is valid iff 0 <= i < rows; it is stored on this rank iff
// lo <= i < hi, at stored row base + (i - lo).
struct FeatMeta {
  int64_t base;  // stored row of global row `lo` of the feature's table (-1: not local)
  int32_t rows;  // global rows of the table
  int32_t lo;    // first global row stored here
  int32_t hi;    // one past the last global row stored here
  int32_t pad;
};

}  // namespace lirank
