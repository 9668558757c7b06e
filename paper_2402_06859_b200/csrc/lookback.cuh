// lookback.cuh -- decoupled look-back (single-pass prefix over tiles) and a device-wide
// exclusive scan built on it.  Status words are 64-bit {epoch:32 | flag:2 | count:30}:
// the epoch tag makes stale words from earlier launches invalid, so the status array is
// never cleared per step (it is zeroed once at emb_create).
#pragma once

#include <stdint.h>

namespace lirank {

constexpr unsigned long long kFlagAgg = 1ull << 30;
constexpr unsigned long long kFlagPrefix = 2ull << 30;
constexpr unsigned long long kCountMask = (1ull << 30) - 1;

__device__ __forceinline__ unsigned long long lb_pack(uint32_t epoch, unsigned long long flag,
                                                      uint32_t count) {
  return ((unsigned long long)epoch << 32) | flag | (unsigned long long)count;
}
__device__ __forceinline__ void st_volatile(unsigned long long* p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// Publish this tile's aggregate (tile 0 publishes its inclusive prefix directly).
__device__ __forceinline__ void lb_publish(unsigned long long* status, int64_t tile, int stride,
                                           int slot, uint32_t epoch, uint32_t aggregate) {
  st_volatile(status + tile * stride + slot,
              lb_pack(epoch, tile == 0 ? kFlagPrefix : kFlagAgg, aggregate));
}

// Exclusive prefix of everything before `tile`, then publish the inclusive prefix.  Looks
// back kLB predecessors per round (independent loads, one L2 round trip), walking from the
// nearest: adds aggregates until an inclusive prefix is found; a predecessor that has not
// published yet is re-polled from where the walk stopped.
template <int kLB = 8, int kSleepMax = 64>
__device__ __forceinline__ uint32_t lb_wait(unsigned long long* status, int64_t tile, int stride,
                                            int slot, uint32_t epoch, uint32_t aggregate) {
  if (tile == 0) return 0;
  uint32_t excl = 0;
  int64_t p = tile - 1;
  {  // fast path: the nearest predecessor has usually published its inclusive prefix already
    const unsigned long long w0 = ld_volatile(status + p * stride + slot);
    if ((uint32_t)(w0 >> 32) == epoch && (w0 & kFlagPrefix)) {
      excl = (uint32_t)(w0 & kCountMask);
      st_volatile(status + tile * stride + slot, lb_pack(epoch, kFlagPrefix, excl + aggregate));
      return excl;
    }
  }
  int sleep_ns = 64;
  while (true) {
    unsigned long long w[kLB];
#pragma unroll
    for (int i = 0; i < kLB; ++i)
      w[i] = p - i >= 0 ? ld_volatile(status + (p - i) * stride + slot) : 0ull;
    bool done = false;
    int i = 0;
    for (; i < kLB && p - i >= 0; ++i) {
      if ((uint32_t)(w[i] >> 32) != epoch || (w[i] & (3ull << 30)) == 0) break;  // not yet
      excl += (uint32_t)(w[i] & kCountMask);
      if (w[i] & kFlagPrefix) { done = true; break; }
    }
    if (done) break;
    if (i == 0) {  // nothing new: yield the issue slots to working warps (backing off)
      __nanosleep(sleep_ns);
      if (sleep_ns < kSleepMax) sleep_ns *= 2;
    }
    p -= i;
  }
  st_volatile(status + tile * stride + slot, lb_pack(epoch, kFlagPrefix, excl + aggregate));
  return excl;
}

// The same for one counter, walked by a whole warp (all 32 lanes call it): lane i reads the
// status of tile p - i, so one L2 round trip covers 32 predecessors.  The walk adds the
// aggregates up to the nearest inclusive prefix; if an unpublished tile comes first it adds
// the published ones before it and re-polls from there.  Lane 0 publishes the inclusive
// prefix; every lane returns the exclusive one.
template <int kSleepMax = 64>
__device__ __forceinline__ uint32_t lb_wait_warp(unsigned long long* status, int64_t tile, int stride,
                                                 int slot, uint32_t epoch, uint32_t aggregate, int lane) {
  if (tile == 0) return 0;
  uint32_t excl = 0;
  int64_t p = tile - 1;
  int sleep_ns = 32;
  while (true) {
    const unsigned long long w = p - lane >= 0 ? ld_volatile(status + (p - lane) * stride + slot) : 0ull;
    const bool valid = (uint32_t)(w >> 32) == epoch && (w & (3ull << 30)) != 0;
    const unsigned bad = __ballot_sync(0xffffffffu, !valid);
    const unsigned pref = __ballot_sync(0xffffffffu, valid && (w & kFlagPrefix));
    const int first_bad = bad ? __ffs(bad) - 1 : 32;
    const int first_pref = pref ? __ffs(pref) - 1 : 32;
    if (first_pref < first_bad) {  // lanes 0..first_pref: aggregates, then the prefix
      excl += __reduce_add_sync(0xffffffffu, lane <= first_pref ? (uint32_t)(w & kCountMask) : 0u);
      break;
    }
    excl += __reduce_add_sync(0xffffffffu, lane < first_bad ? (uint32_t)(w & kCountMask) : 0u);
    p -= first_bad;
    if (first_bad == 0) {
      __nanosleep(sleep_ns);
      if (sleep_ns < kSleepMax) sleep_ns *= 2;
    }
  }
  if (lane == 0) st_volatile(status + tile * stride + slot, lb_pack(epoch, kFlagPrefix, excl + aggregate));
  return excl;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace lirank
