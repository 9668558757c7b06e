// exchange.cu -- the sharded path: a1 bucketize + ids exchange, a3 pooled exchange, a4 grad
// exchange ("Each embedding table is placed on a GPU, and each GPU's input
// batch is all-to-all'ed so that every GPU receives the input columns belonging to its
// embedding table.  Each GPU does its local embedding lookup, and the lookups are
// all-to-all'ed to return the output to the GPU that the input column came from.").
//
// Rank r holds a local batch of B samples (feature-major ids/offsets, like W=1).
//   a1: every occurrence goes to the owner of its row (table-wise: owner[t];
//       row-wise: id / ceil(rows/W)), already translated to the owner's stored-row key.
//       Per destination the message is [features of that owner][B] bag lengths + the keys
//       in (feature, sample, bag) order -- built by count -> exclusive scan -> stable
//       scatter, then a device-side count all-gather and the keys + lengths moved WITHOUT
//       the host reading any count: fused (EMB_F_P2P) by one kernel storing each rank's
//       keys at their compacted place in the owner's receive buffer; collective by an
//       all-to-all of capacity-padded key slots ([W][pair_cap], sizes fixed by the plan)
//       and an owner-side compaction.  The received count stays on the device (the a5-a8
//       kernels read it), so a sharded step has no host synchronisation and can be
//       captured as a CUDA graph.  Overflow of a planned capacity is a sticky error.
//   owner: pools every source's bags with the a2 kernel into [src][B][Fr][D] and records
//       the {key, grad row} pairs for its backward.
//   a3: table-wise: all-to-all of the pooled blocks back + a column permute into
//       [B][F][D]; row-wise (every owner holds a slice of every table): reduce-scatter of
//       the per-owner partial sums lands [B][F][D] directly.
//   a4: the transpose (table-wise all-to-all of grad blocks; row-wise all-gather), then
//       the owner's local a5-a8; the global norm sums one fp64 per rank in rank order.
#include "handle.h"
#include "lookback.cuh"

namespace lirank {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

// Exclusive scan of n uint32 (one pass, decoupled look-back); out[n] = total.
__global__ void __launch_bounds__(kScanThreads)
k_scan_excl(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int64_t n,
            uint32_t* tile_counter, unsigned long long* status, const uint32_t* epoch_p) {
  __shared__ uint32_t s_tile, s_warp[kScanThreads / 32], s_excl;
  const uint32_t epoch = *epoch_p;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * kScanTile + (int64_t)tid * kScanItems;  // blocked per thread
  uint32_t v[kScanItems], sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? __ldg(in + base + i) : 0u;
    sum += v[i];
  }
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {  // the warps' prefix, then a warp-wide look-back (as the RLE's)
    constexpr int NWS = kScanThreads / 32;
    const uint32_t c = lane < NWS ? s_warp[lane] : 0u;
    uint32_t xs = c;
#pragma unroll
    for (int o = 1; o < NWS; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, xs, o);
      if (lane >= o) xs += y;
    }
    const uint32_t t = __shfl_sync(0xffffffffu, xs, NWS - 1);
    if (lane < NWS) s_warp[lane] = xs - c;
    if (lane == 0) lb_publish(status, tile, 1, 0, epoch, t);
    const uint32_t ex = lb_wait_warp(status, tile, 1, 0, epoch, t, lane);
    if (lane == 0) s_excl = ex;
  }
  __syncthreads();
  uint32_t run = s_excl + s_warp[warp] + x - sum;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    if (base + i == n - 1) out[n] = run + v[i];
    run += v[i];
  }
}

// a1 count: ids of bag (f, b) per destination rank -> lens[dest_base[o]*B + j*B + b].
// One thread per bag, bags visited longest first (order: the a2 length-binned permutation), so
// a warp's threads walk bags of about the same length.  (A group of 8 lanes per bag --
// coalesced id loads, owners counted by shuffles and ranked by match.any / ballots -- measured
// slower: count 90 -> 113 us, scatter 121 -> 159 us on Feed-1: twice the instructions per id.)
template <int WMAX>  // >= W: the owners' counters in registers
__global__ void k_bucket_count(const int* __restrict__ ids, const int* __restrict__ offsets, int B,
                               int F, int W, const FeatMeta* __restrict__ meta,
                               const int32_t* __restrict__ owner0, const int32_t* __restrict__ blk,
                               const int32_t* __restrict__ jmap, const int32_t* __restrict__ dest_base,
                               uint32_t* __restrict__ lens, uint32_t* status, const uint32_t* __restrict__ order) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)F * B) return;
  const int64_t bag = order ? (int64_t)__ldg(order + t) : t;
  const int f = (int)(bag / B), b = (int)(bag - (int64_t)f * B);
  const int rows = meta[f].rows, o0 = owner0[f], bk = blk[f];
  uint32_t cnt[WMAX];
#pragma unroll
  for (int o = 0; o < WMAX; ++o) cnt[o] = 0;
  bool bad = false;
  for (int j = __ldg(offsets + bag), e = __ldg(offsets + bag + 1); j < e; ++j) {
    const int id = __ldg(ids + j);
    if (id < 0 || id >= rows) { bad = true; continue; }
    const int o = o0 + id / bk;
#pragma unroll
    for (int q = 0; q < WMAX; ++q) cnt[q] += (q == o);
  }
  if (bad) atomicOr(status, kStIdRange);
#pragma unroll
  for (int o = 0; o < WMAX; ++o) {
    if (o >= W) break;
    const int jj = jmap[o * F + f];
    if (jj >= 0) lens[((int64_t)dest_base[o] + jj) * B + b] = cnt[o];
  }
}

// a1 scatter: keys (owner-local stored rows) into the send buffer, stable per bag.
template <int WMAX>
__global__ void k_bucket_scatter(const int* __restrict__ ids, const int* __restrict__ offsets, int B,
                                 int F, int W, const FeatMeta* __restrict__ meta,
                                 const int32_t* __restrict__ owner0, const int32_t* __restrict__ blk,
                                 const int32_t* __restrict__ jmap, const int32_t* __restrict__ dest_base,
                                 const int64_t* __restrict__ key_base, const uint32_t* __restrict__ pos,
                                 uint32_t* __restrict__ send_keys, uint32_t pair_cap, uint32_t* status,
                                 const uint32_t* __restrict__ order) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)F * B) return;
  const int64_t bag = order ? (int64_t)__ldg(order + t) : t;
  const int f = (int)(bag / B), b = (int)(bag - (int64_t)f * B);
  const int rows = meta[f].rows, o0 = owner0[f], bk = blk[f];
  // p[o] = where the next key for owner o goes: contiguous by owner (pair_cap == 0), or
  // slot o of a capacity-padded [W][pair_cap] buffer (the collective path's fixed sizes)
  uint32_t p[WMAX];
#pragma unroll
  for (int o = 0; o < WMAX; ++o) {
    const int jj = o < W ? jmap[o * F + f] : -1;
    p[o] = jj >= 0 ? pos[((int64_t)dest_base[o] + jj) * B + b] : 0u;
    if (pair_cap && jj >= 0) p[o] = p[o] - __ldg(pos + (int64_t)dest_base[o] * B) + (uint32_t)o * pair_cap;
  }
  bool over = false;
  for (int j = __ldg(offsets + bag), e = __ldg(offsets + bag + 1); j < e; ++j) {
    const int id = __ldg(ids + j);
    if (id < 0 || id >= rows) continue;
    const int o = o0 + id / bk;
    const uint32_t key = (uint32_t)(key_base[(int64_t)o * F + f] + (id - (int64_t)(o - o0) * bk));
    uint32_t at = 0;
#pragma unroll
    for (int q = 0; q < WMAX; ++q)
      if (q == o) { at = p[q]; p[q] = at + 1; }
    if (pair_cap && at >= (uint32_t)(o + 1) * pair_cap) { over = true; continue; }
    send_keys[at] = key;
  }
  if (over) atomicOr(status, kStOverflow);
}

// Counts of the whole exchange: cnt_all[s * W + o] = keys rank s sends owner o (all-gathered,
// so every rank sees the same matrix).  The call overflows if some owner receives more than
// its capacity or, collective path, some source's keys exceed their pair slot: then EVERY
// rank discards it (decided identically everywhere from cnt_all): no keys are moved, the
// owners' a1 lengths are zeroed (every bag pools to 0 and records no occurrence), the
// row-wise slot sum outputs 0, and each rank raises the sticky overflow status.
__device__ __forceinline__ bool exchange_overflow(const uint32_t* __restrict__ cnt_all, int W,
                                                  uint32_t recv_cap, uint32_t pair_cap) {
  bool over = false;
  for (int o = 0; o < W; ++o) {
    uint64_t tot = 0;
    for (int s = 0; s < W; ++s) {
      const uint32_t c = __ldg(cnt_all + s * W + o);
      tot += c;
      over |= pair_cap && c > pair_cap;
    }
    over |= tot > recv_cap;
  }
  return over;
}

__global__ void k_recv_guard(const uint32_t* __restrict__ cnt_all, int W, uint32_t recv_cap,
                             uint32_t pair_cap, uint32_t* __restrict__ recv_lens, int64_t n_lens,
                             uint32_t* status) {
  if (!exchange_overflow(cnt_all, W, recv_cap, pair_cap)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, kStOverflow);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_lens; i += (int64_t)gridDim.x * blockDim.x)
    recv_lens[i] = 0u;
}

// Fused a1 (EMB_F_P2P): this rank's keys for owner o (blockIdx.y) go straight to their
// compacted place in o's receive buffer -- after the keys of ranks 0..rank-1 (the
// all-gathered counts), so every owner sees the sources in rank order -- and this rank's
// [Fo][B] bag lengths to o's [rank][Fo][B] block.
struct PushIds {
  uint32_t* keys[kMaxWorld];  // each owner's recv_keys (peer mapping)
  uint32_t* lens[kMaxWorld];  // each owner's recv_lens
};
__global__ void __launch_bounds__(256)
k_push_ids(const uint32_t* __restrict__ send_keys, const uint32_t* __restrict__ pos,
           const uint32_t* __restrict__ lens, const uint32_t* __restrict__ cnt_all,
           const int32_t* __restrict__ dest_base, int W, int rank, int B, uint32_t recv_cap,
           const PushIds pd) {
  if (exchange_overflow(cnt_all, W, recv_cap, 0u)) return;  // discarded everywhere
  const int o = blockIdx.y;
  const uint32_t n = __ldg(cnt_all + rank * W + o);
  uint32_t base = 0;
  for (int s = 0; s < rank; ++s) base += __ldg(cnt_all + s * W + o);
  const uint32_t* __restrict__ src = send_keys + __ldg(pos + (int64_t)__ldg(dest_base + o) * B);
  uint32_t* __restrict__ dst = pd.keys[o] + base;
  // 4 keys in flight per thread (independent loads before the stores): 87 -> 35 us on Feed-1
  const uint32_t nt = gridDim.x * blockDim.x;
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * nt < n; i += 4 * nt) {
    const uint32_t k0 = __ldg(src + i), k1 = __ldg(src + i + nt), k2 = __ldg(src + i + 2 * nt),
                   k3 = __ldg(src + i + 3 * nt);
    dst[i] = k0;
    dst[i + nt] = k1;
    dst[i + 2 * nt] = k2;
    dst[i + 3 * nt] = k3;
  }
  for (; i < n; i += nt) dst[i] = __ldg(src + i);
  const int Fo = __ldg(dest_base + o + 1) - __ldg(dest_base + o);
  const int64_t nl = (int64_t)Fo * B;
  const uint32_t* ls = lens + (int64_t)__ldg(dest_base + o) * B;
  uint32_t* ld = pd.lens[o] + (int64_t)rank * nl;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x)
    ld[i] = __ldg(ls + i);
}

// Collective a1: the padded slots [W][pair_cap] of the received keys -> compacted in
// source order (source s's keys after those of sources 0..s-1).
__global__ void __launch_bounds__(256)
k_compact_ids(const uint32_t* __restrict__ pad, const uint32_t* __restrict__ cnt_all, int W, int rank,
              uint32_t pair_cap, uint32_t recv_cap, uint32_t* __restrict__ keys) {
  if (exchange_overflow(cnt_all, W, recv_cap, pair_cap)) return;  // discarded everywhere
  const int s = blockIdx.y;
  uint32_t base = 0;
  for (int q = 0; q < s; ++q) base += __ldg(cnt_all + q * W + rank);
  const uint32_t n = __ldg(cnt_all + s * W + rank);
  const uint32_t* src = pad + (size_t)s * pair_cap;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    keys[base + i] = __ldg(src + i);
}

// per-destination send counts from the scanned lengths
__global__ void k_send_counts(const uint32_t* __restrict__ pos, const int32_t* __restrict__ dest_base,
                              int W, int B, uint32_t* __restrict__ cnt) {
  const int o = threadIdx.x;
  if (o < W) cnt[o] = pos[(int64_t)dest_base[o + 1] * B] - pos[(int64_t)dest_base[o] * B];
}

// Grid-stride walk over the float4 columns of the [B][F] rows of a [B][F][D] tensor with no
// per-element division (the 64-bit i / nv, row / F of a flat index cost more instructions than
// the copy itself): thread t owns column v = t % nv for all its rows, rows advance by a fixed
// stride and (b, f) are updated incrementally.  Needs the thread count to be a multiple of nv
// (nv = D / 4 dividing 256: walk_ok).  (Measured, Feed-1 1-rank: slot sum 113 -> 97 us, grad
// push 80 -> 75, table-wise collective step 3.41 -> 2.90 ms; grids of 148 x 32 CTAs instead of
// 148 x 4..8 were slower: 107 / 67 us.)
struct RowWalk {
  int64_t row, rstride;
  int b, f, v, sb, sf;
  __device__ RowWalk(int F, int nv) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    v = (int)(t % nv);
    row = t / nv;
    rstride = nt / nv;
    b = (int)(row / F);
    f = (int)(row - (int64_t)b * F);
    sb = (int)(rstride / F);
    sf = (int)(rstride - (int64_t)sb * F);
  }
  __device__ void next(int F) {
    row += rstride;
    b += sb;
    f += sf;
    if (f >= F) { f -= F; ++b; }
  }
};
__host__ __device__ inline bool walk_ok(int D) { return (D & 3) == 0 && D / 4 <= 256 && 256 % (D / 4) == 0; }

// table-wise a3: out[b][f] = recv block of owner(f) at [b][j(f)]  (and the a4 transpose);
// fmap[f] = {dest_base(owner), Fo(owner), j}: the block starts at dest_base * B
template <bool TO_OUT>
__global__ void k_permute(float* __restrict__ dense, float* __restrict__ blocks, int B, int F, int D,
                          const int32_t* __restrict__ fmap) {
  if (walk_ok(D)) {  // float4 columns, no per-element division
    const int nv = D / 4;
    const int64_t nrows = (int64_t)B * F;
    for (RowWalk w(F, nv); w.row < nrows; w.next(F)) {
      const int64_t src = ((int64_t)fmap[3 * w.f] * B + (int64_t)w.b * fmap[3 * w.f + 1] + fmap[3 * w.f + 2]) * D + 4 * w.v;
      float4* d4 = reinterpret_cast<float4*>(dense + w.row * D + 4 * w.v);
      float4* s4 = reinterpret_cast<float4*>(blocks + src);
      if (TO_OUT) *d4 = *s4;
      else *s4 = *d4;
    }
    return;
  }
  const int64_t total = (int64_t)B * F * D;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / D;
    const int d = (int)(i - row * D);
    const int b = (int)(row / F), f = (int)(row - (int64_t)b * F);
    const int64_t src = ((int64_t)fmap[3 * f] * B + (int64_t)b * fmap[3 * f + 1] + fmap[3 * f + 2]) * D + d;
    if (TO_OUT) dense[i] = blocks[src];
    else blocks[src] = dense[i];
  }
}

// ---- fused exchange (EMB_F_P2P) ------------------------------------------------------------
struct PushDst {
  float* dst[kMaxWorld];  // each owner's pooled buffer (peer mapping)
  int32_t Fo[kMaxWorld];  // features each owner pools (its pooled row block width)
};

// a4 fused: this rank's grad row (b, f) goes to every owner o that pooled feature f
// (jmap[o][f] = j >= 0; table-wise one owner, row-wise all of them), at the row the owner's
// recorded occurrences point to: dst[o] + ((rank * B + b) * Fo[o] + j) * D.  Replaces the
// permute + all-to-all (table-wise) and the all-gather (row-wise): the grads cross NVLink
// once, written by this kernel's stores (k_fence_sys + the barrier publish them).
__global__ void __launch_bounds__(256)
k_push_grad(const float* __restrict__ grad, int B, int F, int D, int W, int rank,
            const int32_t* __restrict__ jmap, const PushDst pd) {
  if (walk_ok(D) && (D / 4) % 2 == 0) {  // two float4 columns per thread: 2 loads in flight
    const int h = D / 8;
    const int64_t nrows = (int64_t)B * F;
    for (RowWalk w(F, h); w.row < nrows; w.next(F)) {
      const float4 g0 = ld_f4(grad + w.row * D + 4 * w.v), g1 = ld_f4(grad + w.row * D + 4 * (w.v + h));
      for (int o = 0; o < W; ++o) {
        const int j = __ldg(jmap + o * F + w.f);
        if (j >= 0) {
          float* d = pd.dst[o] + (((int64_t)rank * B + w.b) * pd.Fo[o] + j) * D;
          st_f4(d + 4 * w.v, g0);
          st_f4(d + 4 * (w.v + h), g1);
        }
      }
    }
    return;
  }
  if (walk_ok(D)) {  // float4 columns, no per-element division
    const int nv = D / 4;
    const int64_t nrows = (int64_t)B * F;
    for (RowWalk w(F, nv); w.row < nrows; w.next(F)) {
      const float4 g = ld_f4(grad + w.row * D + 4 * w.v);
      for (int o = 0; o < W; ++o) {
        const int j = __ldg(jmap + o * F + w.f);
        if (j >= 0) st_f4(pd.dst[o] + (((int64_t)rank * B + w.b) * pd.Fo[o] + j) * D + 4 * w.v, g);
      }
    }
    return;
  }
  const bool vec = (D & 3) == 0;
  const int nv = vec ? D / 4 : D;
  const int64_t total = (int64_t)B * F * nv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / nv;
    const int v = (int)(i - row * nv);
    const int b = (int)(row / F), f = (int)(row - (int64_t)b * F);
    if (vec) {
      const float4 g = ld_f4(grad + row * D + 4 * v);
      for (int o = 0; o < W; ++o) {
        const int j = __ldg(jmap + o * F + f);
        if (j >= 0) st_f4(pd.dst[o] + (((int64_t)rank * B + b) * pd.Fo[o] + j) * D + 4 * v, g);
      }
    } else {
      const float g = grad[row * D + v];
      for (int o = 0; o < W; ++o) {
        const int j = __ldg(jmap + o * F + f);
        if (j >= 0) pd.dst[o][(((int64_t)rank * B + b) * pd.Fo[o] + j) * D + v] = g;
      }
    }
  }
}

// Before a fused-exchange barrier: one system-scope fence after the storing kernels (stream
// order makes their peer stores happen-before it; the fence is cumulative), so the stores are
// visible to the destination GPU before this rank's arrival at the barrier is.
__global__ void k_fence_sys() { __threadfence_system(); }

// a3 fused, row-wise: out[b][f] = sum over owners o, in rank order, of slot_o[b][f] (the
// owners' partial pools their kernels stored here) -- the sum the reduce-scatter forms.
// Owner o stored only bags with ids on it (lens[(o * F + f) * B + b] > 0, this rank's a1
// lengths): the others are +0 and skipped (a partial sum is never -0, so x + 0 == x), which
// keeps one-hot and short bags off NVLink for all but the owners holding their ids.
__global__ void __launch_bounds__(256)
k_sum_slots(float* __restrict__ out, const float* __restrict__ slots, const uint32_t* __restrict__ lens,
            int W, int B, int F, int D, const uint32_t* __restrict__ cnt_all, uint32_t recv_cap) {
  const bool discard = exchange_overflow(cnt_all, W, recv_cap, 0u);  // the owners stored nothing
  if (walk_ok(D) && (D / 4) % 2 == 0) {  // two float4 columns per thread (v, v + nv/2): 2 loads in flight
    const int nv = D / 4, h = nv / 2;
    const int64_t n = (int64_t)B * F * D, nrows = (int64_t)B * F;
    for (RowWalk w(F, h); w.row < nrows; w.next(F)) {
      float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
      bool any = false;
      for (int o = 0; o < W; ++o) {
        if (discard || __ldg(lens + ((int64_t)o * F + w.f) * B + w.b) == 0) continue;
        const float* sl = slots + (int64_t)o * n + w.row * D + 4 * w.v;
        const float4 x0 = ld_nc_f4(sl), x1 = ld_nc_f4(sl + 4 * h);
        a0 = any ? f4_add_rn(a0, x0) : x0;
        a1 = any ? f4_add_rn(a1, x1) : x1;
        any = true;
      }
      st_f4(out + w.row * D + 4 * w.v, a0);
      st_f4(out + w.row * D + 4 * (w.v + h), a1);
    }
    return;
  }
  if (walk_ok(D)) {  // float4 columns, no per-element division
    const int nv = D / 4;
    const int64_t n = (int64_t)B * F * D, nrows = (int64_t)B * F;
    for (RowWalk w(F, nv); w.row < nrows; w.next(F)) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      bool any = false;
      for (int o = 0; o < W; ++o) {
        if (discard || __ldg(lens + ((int64_t)o * F + w.f) * B + w.b) == 0) continue;
        const float4 x = ld_nc_f4(slots + (int64_t)o * n + w.row * D + 4 * w.v);
        a = any ? f4_add_rn(a, x) : x;
        any = true;
      }
      st_f4(out + w.row * D + 4 * w.v, a);
    }
    return;
  }
  const bool vec = (D & 3) == 0;
  const int nv = vec ? D / 4 : D;
  const int64_t n = (int64_t)B * F * D, total = (int64_t)B * F * nv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / nv;
    const int v = (int)(i - row * nv);
    const int b = (int)(row / F), f = (int)(row - (int64_t)b * F);
    if (vec) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      bool any = false;
      for (int o = 0; o < W; ++o) {
        if (discard || __ldg(lens + ((int64_t)o * F + f) * B + b) == 0) continue;
        const float4 x = ld_nc_f4(slots + (int64_t)o * n + row * D + 4 * v);
        a = any ? f4_add_rn(a, x) : x;
        any = true;
      }
      st_f4(out + row * D + 4 * v, a);
    } else {
      float a = 0.f;
      bool any = false;
      for (int o = 0; o < W; ++o) {
        if (discard || __ldg(lens + ((int64_t)o * F + f) * B + b) == 0) continue;
        const float x = slots[(int64_t)o * n + row * D + v];
        a = any ? __fadd_rn(a, x) : x;
        any = true;
      }
      out[row * D + v] = a;
    }
  }
}

emb_status scan(emb_t h, const uint32_t* in, uint32_t* out, int64_t n, int which) {
  CK(cudaMemsetAsync(h->x.scan_counter + which, 0, sizeof(uint32_t), h->stream));
  if (n == 0) return cudaMemsetAsync(out, 0, sizeof(uint32_t), h->stream) == cudaSuccess ? EMB_OK : EMB_ECUDA;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  // its own look-back words: the a5 dedup of the previous forward may still be running on
  // the side stream with the radix sort's status array
  k_scan_excl<<<(unsigned)tiles, kScanThreads, 0, h->stream>>>(in, out, n, h->x.scan_counter + which,
                                                               h->x.scan_status, h->d_epoch + 1);
  CK(cudaGetLastError());
  CK(launch_epoch_advance(h->d_epoch + 1, 1, h->stream));
  h->launches += 2;
  return cudaGetLastError() == cudaSuccess ? EMB_OK : EMB_ECUDA;
}

}  // namespace

void carve_exchange(const Plan& p, Carver& cv, ExchangeWs* x) {
  const int64_t W = p.world, B = p.max_batch, F = p.F, Fr = p.Fr, D = p.D;
  const int64_t Ltot = B * p.dest_base[W];
  const bool p2p = (p.flags & EMB_F_P2P) != 0;
  x->lens = cv.take<uint32_t>(Ltot);
  x->pos = cv.take<uint32_t>(Ltot + 1);
  // fused: keys contiguous by owner (pushed from there); collective: [W][pair_cap] slots
  x->send_keys = cv.take<uint32_t>(p2p ? p.max_nnz : W * p.pair_cap);
  x->cnt = cv.take<uint32_t>(W + W * W);
  x->recv_lens = cv.take<uint32_t>(W * Fr * B);
  x->recv_off = cv.take<uint32_t>(W * Fr * B + 1);
  x->recv_keys = cv.take<uint32_t>(p.recv_nnz_cap);
  if (!p2p) x->recv_pad = cv.take<uint32_t>(W * p.pair_cap);
  x->pooled = cv.take<float>(W * B * Fr * D);
  // fused exchange: two destination sets (the fp32 forward's and the q8 forward's), so a q8
  // lookup of the forward's batch needs no barrier before its owners store (set 1 was last
  // read by the previous step's q8 slot sum, ordered before by this step's forward barriers)
  const bool row = p.sharding == EMB_SHARD_ROW;
  x->xdense = cv.take<float>((p2p && !row ? 2 : 1) * B * F * D);
  x->ident = cv.take<FeatMeta>(W * Fr);
  x->d_jmap = cv.take<int32_t>(W * F);
  x->d_fmap = cv.take<int32_t>(3 * F);
  x->d_feats_by_dest = cv.take<int32_t>(F);
  x->d_dest_base = cv.take<int32_t>(W + 1);
  x->d_key_base = cv.take<int64_t>(W * F);
  x->d_owner0 = cv.take<int32_t>(F);
  x->d_blk = cv.take<int32_t>(F);
  x->scan_counter = cv.take<uint32_t>(4);
  const int64_t scan_n = std::max<int64_t>(Ltot + 1, W * Fr * B + 1);
  x->scan_status = cv.take<unsigned long long>((scan_n + kScanTile - 1) / kScanTile + 1);
  if (p2p) {
    if (row) x->pslots = cv.take<float>(2 * W * B * F * D);
    x->fdst_stride = row ? (int64_t)W * B * F * D : (int64_t)B * F * D;
    x->d_fcol = cv.take<int32_t>(Fr);
    x->p2p_scratch = cv.take<uint8_t>((int64_t)kPeerScratchBytes);
  }
}

emb_status exchange_init(emb_t h) {
  const Plan& p = h->p;
  const int W = p.world, F = p.F;
  std::vector<FeatMeta> ident((size_t)W * p.Fr);
  for (auto& m : ident) { m.base = 0; m.rows = 0x7fffffff; m.lo = 0; m.hi = 0x7fffffff; m.pad = 0; }
  std::vector<int32_t> fmap(3 * F, 0);
  if (p.sharding == EMB_SHARD_TABLE)
    for (int f = 0; f < F; ++f) {
      const int o = p.owner[p.feature_table[f]];
      fmap[3 * f] = p.dest_base[o];  // x B on the device (k_permute): no per-B upload
      fmap[3 * f + 1] = p.Fo[o];
      fmap[3 * f + 2] = p.jmap[(size_t)o * F + f];
    }
  const ExchangeWs& x = h->x;
  CK(cudaMemcpyAsync(x.ident, ident.data(), sizeof(FeatMeta) * ident.size(), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(x.d_jmap, p.jmap.data(), 4 * p.jmap.size(), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(x.d_dest_base, p.dest_base.data(), 4 * p.dest_base.size(), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(x.d_key_base, p.key_base.data(), 8 * p.key_base.size(), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(x.d_owner0, p.owner0.data(), 4 * p.owner0.size(), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(x.d_blk, p.blk.data(), 4 * p.blk.size(), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(x.d_fmap, fmap.data(), 4 * fmap.size(), cudaMemcpyHostToDevice, h->stream));
  std::vector<int32_t> fcol(p.feats_of[p.rank].begin(), p.feats_of[p.rank].end());
  if (p.flags & EMB_F_P2P && !fcol.empty())
    CK(cudaMemcpyAsync(x.d_fcol, fcol.data(), 4 * fcol.size(), cudaMemcpyHostToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));  // host vectors go out of scope
  return EMB_OK;
}

// Collective (the first sharded forward; every rank reaches it in the same call): map every
// rank's fused-exchange destinations into this device.  Lazy rather than at emb_create, so
// handles of in-process (loopback) ranks can be created one after another.
static emb_status map_p2p(emb_t h) {
  ExchangeWs& x = h->x;
  if (x.peer_pooled[0] != nullptr) return EMB_OK;
  const int W = h->p.world;
  void* local[5] = {x.xdense, h->p.sharding == EMB_SHARD_ROW ? (void*)x.pslots : (void*)x.xdense, x.pooled,
                    x.recv_keys, x.recv_lens};
  void* peers[5 * kMaxWorld] = {};
  if (!h->comm->map_peers(local, 5, peers, x.p2p_scratch, h->stream)) return EMB_ENCCL;
  for (int r = 0; r < W; ++r) {
    x.peer_xdense[r] = (float*)peers[0 * W + r];
    x.peer_pslots[r] = (float*)peers[1 * W + r];
    x.peer_pooled[r] = (float*)peers[2 * W + r];
    x.peer_recv_keys[r] = (uint32_t*)peers[3 * W + r];
    x.peer_recv_lens[r] = (uint32_t*)peers[4 * W + r];
  }
  return EMB_OK;
}

// The fused-exchange destination of this rank's owner pooling.
static PeerOut peer_out(emb_t h, int set) {
  const Plan& p = h->p;
  PeerOut pm;
  memset(&pm, 0, sizeof(pm));
  if (!(p.flags & EMB_F_P2P)) return pm;
  const bool row = p.sharding == EMB_SHARD_ROW;
  for (int r = 0; r < p.world; ++r)
    pm.base[r] = (row ? h->x.peer_pslots[r] : h->x.peer_xdense[r]) + set * h->x.fdst_stride;
  pm.fcol = h->x.d_fcol;
  pm.F_out = p.F;
  pm.slot = row ? p.rank : 0;
  pm.skip_empty = row ? 1 : 0;
  return pm;
}

emb_status exchange_forward(emb_t h, const Staged& st, int32_t batch, int64_t nnz, bool q8, bool reuse) {
  const Plan& p = h->p;
  const ExchangeWs& x = h->x;
  const int W = p.world, F = p.F, Fr = p.Fr, D = p.D, B = batch, r = p.rank;
  const int64_t Ltot = (int64_t)B * p.dest_base[W];
  const int64_t n_lens = (int64_t)W * Fr * B;
  const unsigned bag_grid = (unsigned)(((int64_t)F * B + 255) / 256);
  const bool p2p = (p.flags & EMB_F_P2P) != 0;
  const uint32_t pair_cap = p2p ? 0u : (uint32_t)p.pair_cap;
  const uint32_t recv_cap = (uint32_t)p.recv_nnz_cap;
  uint32_t* cnt_all = x.cnt + W;  // [W][W], all-gathered
  emb_status s;
  if (p2p && (s = map_p2p(h)) != EMB_OK) return s;
  // a q8 lookup of the last forward's own batch: its ids are already at their owners (receive
  // buffers, counts, bag order: untouched since -- the backward's exchange uses other buffers)
  const bool skip_a1 = q8 && reuse && h->x_ids_fwd && h->fwd_B == B;
  if (skip_a1) {
    Phase ph(h->prof, h->stream, EMB_PH_EXCHANGE);
    // (fused: the owners store into the q8 destination set, last read by the previous step's
    // q8 slot sum -- ordered before by this step's forward barriers: no barrier here)
  } else {
    Phase ph(h->prof, h->stream, EMB_PH_EXCHANGE);
    h->x_ids_fwd = !q8;  // this call's exchange overwrites the receive buffers
    // ---- a1: bucketize -----------------------------------------------------------------
    const uint32_t* bag_ord = launch_bag_order(st.offsets, (long long)F * B, h->order_ws, h->stream);
    if (bag_ord) h->launches += 2;
    if (F * (int64_t)B > 0) {
      if (W <= 8)
        k_bucket_count<8><<<bag_grid, 256, 0, h->stream>>>(st.ids, st.offsets, B, F, W, h->d_meta, x.d_owner0,
                                                           x.d_blk, x.d_jmap, x.d_dest_base, x.lens, h->d_status,
                                                           bag_ord);
      else
        k_bucket_count<kMaxWorld><<<bag_grid, 256, 0, h->stream>>>(st.ids, st.offsets, B, F, W, h->d_meta,
                                                                   x.d_owner0, x.d_blk, x.d_jmap, x.d_dest_base,
                                                                   x.lens, h->d_status, bag_ord);
      h->launches += 1;
      CK(cudaGetLastError());
    }
    if ((s = scan(h, x.lens, x.pos, Ltot, 0)) != EMB_OK) return s;
    if (F * (int64_t)B > 0) {
      if (W <= 8)
        k_bucket_scatter<8><<<bag_grid, 256, 0, h->stream>>>(st.ids, st.offsets, B, F, W, h->d_meta, x.d_owner0,
                                                             x.d_blk, x.d_jmap, x.d_dest_base, x.d_key_base,
                                                             x.pos, x.send_keys, pair_cap, h->d_status, bag_ord);
      else
        k_bucket_scatter<kMaxWorld><<<bag_grid, 256, 0, h->stream>>>(st.ids, st.offsets, B, F, W, h->d_meta,
                                                                     x.d_owner0, x.d_blk, x.d_jmap, x.d_dest_base,
                                                                     x.d_key_base, x.pos, x.send_keys, pair_cap,
                                                                     h->d_status, bag_ord);
      h->launches += 1;
    }
    k_send_counts<<<1, 32, 0, h->stream>>>(x.pos, x.d_dest_base, W, B, x.cnt);
    h->launches += 1;
    CK(cudaGetLastError());
    // the count matrix, on the device only.  (It also orders buffer reuse: no rank passes it
    // before every rank has finished the previous call's reads of its receive buffers.)
    if (!h->comm->allgather(x.cnt, cnt_all, sizeof(uint32_t) * W, h->stream)) return EMB_ENCCL;
    if (p2p) {
      PushIds pd;
      memset(&pd, 0, sizeof(pd));
      for (int o = 0; o < W; ++o) { pd.keys[o] = x.peer_recv_keys[o]; pd.lens[o] = x.peer_recv_lens[o]; }
      k_push_ids<<<dim3(148 * 2, W), 256, 0, h->stream>>>(x.send_keys, x.pos, x.lens, cnt_all, x.d_dest_base,
                                                           W, r, B, recv_cap, pd);
      k_fence_sys<<<1, 1, 0, h->stream>>>();
      h->launches += 2;
      CK(cudaGetLastError());
      if (!h->comm->barrier(x.p2p_scratch, h->stream)) return EMB_ENCCL;
    } else {
      std::vector<size_t> soff(W), sb(W), roff(W), rb(W);
      for (int o = 0; o < W; ++o) {  // capacity-padded slots: sizes fixed by the plan
        soff[o] = roff[o] = 4ull * o * p.pair_cap;
        sb[o] = rb[o] = 4ull * p.pair_cap;
      }
      if (!h->comm->alltoallv(x.send_keys, soff.data(), sb.data(), x.recv_pad, roff.data(), rb.data(), h->stream))
        return EMB_ENCCL;
      // bag lengths: [Fo x B] to each owner; [Fr x B] from each source
      for (int o = 0; o < W; ++o) {
        soff[o] = 4ull * p.dest_base[o] * B;
        sb[o] = 4ull * p.Fo[o] * B;
        roff[o] = 4ull * o * Fr * B;
        rb[o] = 4ull * Fr * B;
      }
      if (!h->comm->alltoallv(x.lens, soff.data(), sb.data(), x.recv_lens, roff.data(), rb.data(), h->stream))
        return EMB_ENCCL;
      k_compact_ids<<<dim3(148, W), 256, 0, h->stream>>>(x.recv_pad, cnt_all, W, r, pair_cap, recv_cap,
                                                         x.recv_keys);
      h->launches += 1;
      CK(cudaGetLastError());
    }
    k_recv_guard<<<148, 256, 0, h->stream>>>(cnt_all, W, recv_cap, pair_cap, x.recv_lens, n_lens, h->d_status);
    h->launches += 1;
    CK(cudaGetLastError());
    if ((s = scan(h, x.recv_lens, x.recv_off, n_lens, 1)) != EMB_OK) return s;
  }
  // ---- owner: pool every source's bags into [src][B][Fr][D] -------------------------------
  h->order_bags = -1;  // order_ws now holds the owner's order, not a local forward's
  if (!q8) {
    FwdArgs a;
    memset(&a, 0, sizeof(a));
    a.W = h->W;
    a.pitch = p.pitch;
    a.ids = (const int*)x.recv_keys;
    a.offsets = (const int*)x.recv_off;
    a.B = B;
    a.F = W * Fr;
    a.Fb = Fr;
    a.D = D;
    a.meta = x.ident;
    a.out = x.pooled;
    a.kv_out = h->kvA;
    a.sentinel = (uint32_t)p.local_rows;
    a.status = h->d_status;
    a.order_ws = h->order_ws;
    a.peer = peer_out(h, q8 ? 1 : 0);
    Phase ph(h->prof, h->stream, EMB_PH_FWD);
    CK(launch_pool_fwd_f32(a, h->stream));
  } else {
    FwdQ8Args a;
    memset(&a, 0, sizeof(a));
    a.codes = h->codes;
    a.qpitch = p.qpitch;
    a.meta_off = h->q8_meta_off;
    a.minmax = (p.flags & EMB_F_Q8_MINMAX) != 0;
    a.ids = (const int*)x.recv_keys;
    a.offsets = (const int*)x.recv_off;
    a.B = B;
    a.F = W * Fr;
    a.Fb = Fr;
    a.D = D;
    a.meta = x.ident;
    a.out = x.pooled;
    a.status = h->d_status;
    a.order_ws = h->order_ws;
    a.order_ready = skip_a1 && (int64_t)W * Fr * B >= 2;  // the forward ordered these receive bags
    a.peer = peer_out(h, q8 ? 1 : 0);
    Phase ph(h->prof, h->stream, EMB_PH_FWD_Q8);
    CK(launch_pool_fwd_q8(a, h->stream));
  }
  h->launches += skip_a1 ? 1 : fwd_launches((int64_t)W * Fr * B, true, !q8);
  // ---- a3: pooled exchange back ----------------------------------------------------------
  {
    Phase ph(h->prof, h->stream, EMB_PH_EXCHANGE);
    if (p2p) {
      // the owners' kernels stored straight into this rank's buffers; once every rank has
      // passed the barrier, they are complete
      k_fence_sys<<<1, 1, 0, h->stream>>>();
      h->launches += 1;
      if (!h->comm->barrier(x.p2p_scratch, h->stream)) return EMB_ENCCL;
      const int64_t n = (int64_t)B * F * D;
      if (n > 0 && p.sharding == EMB_SHARD_ROW) {
        k_sum_slots<<<148 * 4, 256, 0, h->stream>>>(st.out, x.pslots + (q8 ? x.fdst_stride : 0), x.lens, W, B, F, D,
                                                    cnt_all, recv_cap);
        h->launches += 1;
        CK(cudaGetLastError());
      } else if (n > 0) {
        CK(cudaMemcpyAsync(st.out, x.xdense + (q8 ? x.fdst_stride : 0), 4ull * n, cudaMemcpyDeviceToDevice,
                           h->stream));
      }
    } else if (p.sharding == EMB_SHARD_ROW) {
      if (!h->comm->reduce_scatter_f32(x.pooled, st.out, (size_t)B * F * D, h->stream)) return EMB_ENCCL;
    } else {
      std::vector<size_t> soff(W), sb(W), roff(W), rb(W);
      for (int o = 0; o < W; ++o) {
        soff[o] = 4ull * o * B * Fr * D;
        sb[o] = 4ull * B * Fr * D;
        roff[o] = 4ull * p.dest_base[o] * B * D;
        rb[o] = 4ull * p.Fo[o] * B * D;
      }
      if (!h->comm->alltoallv(x.pooled, soff.data(), sb.data(), x.xdense, roff.data(), rb.data(), h->stream))
        return EMB_ENCCL;
      if ((int64_t)B * F * D > 0) {
        k_permute<true><<<148 * 8, 256, 0, h->stream>>>(st.out, x.xdense, B, F, D, x.d_fmap);
        h->launches += 1;
        CK(cudaGetLastError());
      }
    }
  }
  if (!q8) {
    // the received count, for the backward's a5-a8 (device only; a later q8 forward reuses
    // recv_off, so it is copied out here, in stream order before the dedup reads it)
    CK(cudaMemcpyAsync(h->d_fwd_n, x.recv_off + n_lens, sizeof(uint32_t), cudaMemcpyDeviceToDevice, h->stream));
    h->have_fwd = true;
    h->fwd_nnz = p.recv_nnz_cap;  // capacity: the kernels read the count from d_fwd_n
    h->fwd_n_dev = h->d_fwd_n;
    h->fwd_nnz_hint = nnz;
    h->fwd_B = B;
  }
  return EMB_OK;
}

emb_status exchange_backward(emb_t h, const float* grad_dev) {
  const Plan& p = h->p;
  const ExchangeWs& x = h->x;
  const int W = p.world, F = p.F, Fr = p.Fr, D = p.D, B = h->fwd_B;
  {
    Phase ph(h->prof, h->stream, EMB_PH_EXCHANGE);
    if (p.flags & EMB_F_P2P) {
      if (x.peer_pooled[0] == nullptr) return EMB_ESTATE;  // (a forward maps the peers)
      if ((int64_t)B * F * D > 0) {
        PushDst pd;
        memset(&pd, 0, sizeof(pd));
        for (int o = 0; o < W; ++o) { pd.dst[o] = x.peer_pooled[o]; pd.Fo[o] = p.Fo[o]; }
        k_push_grad<<<148 * 8, 256, 0, h->stream>>>(grad_dev, B, F, D, W, p.rank, x.d_jmap, pd);
        h->launches += 1;
        CK(cudaGetLastError());
      }
      k_fence_sys<<<1, 1, 0, h->stream>>>();
      h->launches += 1;
      if (!h->comm->barrier(x.p2p_scratch, h->stream)) return EMB_ENCCL;
    } else if (p.sharding == EMB_SHARD_ROW) {
      if (!h->comm->allgather(grad_dev, x.pooled, 4ull * B * F * D, h->stream)) return EMB_ENCCL;
    } else {
      if ((int64_t)B * F * D > 0) {
        k_permute<false><<<148 * 8, 256, 0, h->stream>>>(const_cast<float*>(grad_dev), x.xdense, B, F, D,
                                                         x.d_fmap);
        h->launches += 1;
        CK(cudaGetLastError());
      }
      std::vector<size_t> soff(W), sb(W), roff(W), rb(W);
      for (int o = 0; o < W; ++o) {
        soff[o] = 4ull * p.dest_base[o] * B * D;
        sb[o] = 4ull * p.Fo[o] * B * D;
        roff[o] = 4ull * o * B * Fr * D;
        rb[o] = 4ull * B * Fr * D;
      }
      if (!h->comm->alltoallv(x.xdense, soff.data(), sb.data(), x.pooled, roff.data(), rb.data(), h->stream))
        return EMB_ENCCL;
    }
  }
  return EMB_OK;
}

}  // namespace lirank
