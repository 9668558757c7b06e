// api.cu -- C ABI (include/lirank_emb.h): planning, workspace carve-up, call sequencing.
//
// Host code only orchestrates: every step of the hot path runs in the kernels of
// forward.cu / sort.cu / backward.cu / exchange.cu.  No CPU fallback exists: without a
// CUDA device every compute call fails with EMB_ECUDA.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <vector>

#include "handle.h"

using namespace lirank;

namespace lirank {

namespace {

int bits_for(int64_t v) {  // smallest b with v < 2^b
  int b = 0;
  while (b < 63 && (int64_t(1) << b) <= v) ++b;
  return b;
}

// Rows of every table stored on rank r (table-wise: whole tables; row-wise: contiguous
// blocks of ceil(R/W) rows; unsharded: everything).
Layout layout_for(const Plan& p, int r) {
  Layout L;
  L.local_base.assign(p.T, -1);
  L.row_lo.assign(p.T, 0);
  L.row_hi.assign(p.T, 0);
  int64_t lr = 0;
  for (int t = 0; t < p.T; ++t) {
    const int64_t R = p.table_rows[t];
    int64_t lo = 0, hi = R;
    if (p.sharding == EMB_SHARD_TABLE) {
      if (p.owner[t] != r) continue;
    } else if (p.sharding == EMB_SHARD_ROW) {
      const int64_t blk = (R + p.world - 1) / p.world;
      lo = std::min<int64_t>(R, (int64_t)r * blk);
      hi = std::min<int64_t>(R, lo + blk);
    }
    L.local_base[t] = lr;
    L.row_lo[t] = lo;
    L.row_hi[t] = hi;
    lr += hi - lo;
  }
  L.local_rows = lr;
  return L;
}

}  // namespace

emb_status make_plan(const emb_config* c, Plan* p) {
  if (!c || !p) return EMB_EINVAL;
  if (c->abi_version != EMB_ABI_VERSION) return EMB_EINVAL;
  if (c->num_tables < 1 || !c->table_rows) return EMB_EINVAL;
  if (c->dim < 1 || c->dim > 1024) return EMB_EINVAL;
  if (c->num_features < 1 || !c->feature_table) return EMB_EINVAL;
  if (c->pooling != EMB_POOL_SUM && c->pooling != EMB_POOL_MEAN) return EMB_EINVAL;
  if (c->adagrad_mode != EMB_ADAGRAD_ROWWISE && c->adagrad_mode != EMB_ADAGRAD_ELEMENTWISE)
    return EMB_EINVAL;
  if (c->max_nnz < 0 || c->max_nnz >= (int64_t(1) << 30)) return EMB_EINVAL;
  if (c->max_batch < 0) return EMB_EINVAL;
  if ((int64_t)c->max_batch * c->num_features >= (int64_t(1) << 31) - 1) return EMB_EINVAL;
  if (!(c->eps >= 0.f) || !(c->max_norm > 0.f) || !(c->init_accumulator >= 0.f)) return EMB_EINVAL;
  if ((c->flags & EMB_F_REQUANT) && !(c->flags & EMB_F_Q8)) return EMB_EINVAL;
  if ((c->flags & EMB_F_Q8_MINMAX) && !(c->flags & EMB_F_Q8)) return EMB_EINVAL;
  if ((c->flags & EMB_F_Q8_ONLY) && (!(c->flags & EMB_F_Q8) || (c->flags & EMB_F_REQUANT)))
    return EMB_EINVAL;
  if (c->world_size < 1 || c->world_size > kMaxWorld || c->rank < 0 || c->rank >= c->world_size)
    return EMB_EINVAL;
  if (c->sharding != EMB_SHARD_NONE && c->sharding != EMB_SHARD_TABLE && c->sharding != EMB_SHARD_ROW)
    return EMB_EINVAL;
  if (c->world_size > 1 && c->sharding == EMB_SHARD_NONE) return EMB_EINVAL;
  if (c->world_size > 1 && c->pooling == EMB_POOL_MEAN) return EMB_EINVAL;  // DESIGN.md reading 24
  p->T = c->num_tables;
  p->D = c->dim;
  p->F = c->num_features;
  p->pitch = (int)round_up(c->dim, 4);
  // q8 row: [codes][pad to 8][middle, scale][pad to 32]: whole 32-B sectors, so the
  // fused re-quantize never partially writes a sector (no L2 fill reads)
  // q8 rows (reading 26): whole 64-B DRAM atoms when the store is rewritten every step (fused
  // requant: a partially written atom costs HBM a read-modify-write), whole 32-B sectors
  // otherwise (written once: 25% smaller; the 1B-row serving store measured slower at 128 B)
  p->qpitch = (int)round_up(round_up(c->dim, 8) + 8, (c->flags & EMB_F_REQUANT) ? 64 : 32);
  p->pooling = c->pooling;
  p->mode = c->adagrad_mode;
  p->exch = c->world_size > 1 || (c->flags & EMB_F_EXCHANGE);
  if (p->exch && c->sharding == EMB_SHARD_NONE) return EMB_EINVAL;
  if (p->exch && c->pooling == EMB_POOL_MEAN) return EMB_EINVAL;
  if ((c->flags & EMB_F_P2P) && !p->exch) return EMB_EINVAL;
  if ((c->flags & EMB_F_LOOPBACK) && (c->flags & EMB_F_HOSTCOMM)) return EMB_EINVAL;
  p->sharding = p->exch ? c->sharding : EMB_SHARD_NONE;
  p->rank = c->rank;
  p->world = c->world_size;
  p->flags = c->flags;
  p->A0 = c->init_accumulator;
  p->eps = c->eps;
  p->max_norm = c->max_norm;
  p->max_nnz = c->max_nnz;
  p->max_batch = c->max_batch;
  p->table_rows.assign(c->table_rows, c->table_rows + c->num_tables);
  p->feature_table.assign(c->feature_table, c->feature_table + c->num_features);
  for (int64_t r : p->table_rows)
    if (r < 0 || r >= (int64_t(1) << 31)) return EMB_EINVAL;
  for (int32_t t : p->feature_table)
    if (t < 0 || t >= p->T) return EMB_EINVAL;

  const int W = p->world, F = p->F;
  p->owner.assign(p->T, 0);
  if (p->sharding == EMB_SHARD_TABLE) {
    if (c->table_owner) {
      for (int t = 0; t < p->T; ++t) {
        if (c->table_owner[t] < 0 || c->table_owner[t] >= W) return EMB_EINVAL;
        p->owner[t] = c->table_owner[t];
      }
    } else {
      // greedy LPT by cost (cfg.table_cost, else rows; largest first, ties by table
      // index), each table to the least-loaded rank (ties to the lower rank)
      std::vector<double> cost(p->T);
      for (int t = 0; t < p->T; ++t) {
        cost[t] = c->table_cost ? c->table_cost[t] : (double)p->table_rows[t];
        if (!(cost[t] >= 0.0)) return EMB_EINVAL;
      }
      std::vector<int> order(p->T);
      for (int t = 0; t < p->T; ++t) order[t] = t;
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
      std::vector<double> load(W, 0.0);
      for (int t : order) {
        int best = 0;
        for (int r = 1; r < W; ++r)
          if (load[r] < load[best]) best = r;
        p->owner[t] = best;
        load[best] += cost[t];
      }
    }
  }
  p->layouts.clear();
  for (int r = 0; r < W; ++r) p->layouts.push_back(layout_for(*p, r));
  const Layout& me = p->layouts[p->rank];
  p->local_base = me.local_base;
  p->row_lo = me.row_lo;
  p->row_hi = me.row_hi;
  p->local_rows = me.local_rows;
  for (const Layout& L : p->layouts)
    if (L.local_rows >= (int64_t(1) << 31) - 1) return EMB_EINVAL;
  p->key_bits = bits_for(p->local_rows);  // keys in [0, local_rows], sentinel = local_rows

  // exchange maps (world > 1)
  p->feats_of.assign(W, {});
  p->Fo.assign(W, 0);
  p->dest_base.assign(W + 1, 0);
  p->jmap.assign((size_t)W * F, -1);
  p->key_base.assign((size_t)W * F, -1);
  p->owner0.assign(F, 0);
  p->blk.assign(F, 1);
  for (int o = 0; o < W; ++o) {
    for (int f = 0; f < F; ++f) {
      const int t = p->feature_table[f];
      const bool here = p->sharding == EMB_SHARD_TABLE ? p->owner[t] == o
                                                       : (W == 1 || p->layouts[o].local_base[t] >= 0);
      if (!here) continue;
      p->jmap[(size_t)o * F + f] = (int32_t)p->feats_of[o].size();
      p->feats_of[o].push_back(f);
      p->key_base[(size_t)o * F + f] = p->layouts[o].local_base[t];
    }
    p->Fo[o] = (int)p->feats_of[o].size();
    p->dest_base[o + 1] = p->dest_base[o] + p->Fo[o];
  }
  for (int f = 0; f < F; ++f) {
    const int t = p->feature_table[f];
    const int64_t R = p->table_rows[t];
    if (p->sharding == EMB_SHARD_TABLE) {
      p->owner0[f] = p->owner[t];
      p->blk[f] = (int32_t)std::max<int64_t>(R, 1);  // id / blk == 0 for every valid id
    } else {
      p->owner0[f] = 0;
      p->blk[f] = (int32_t)std::max<int64_t>((R + W - 1) / W, 1);
    }
  }
  p->Fr = p->Fo[p->rank];
  // Capacities: a rank can receive every id of every rank, and pools every bag of every rank
  // that reads its tables.  (Capacity, not expectation.)
  if (c->max_recv_nnz < 0 || c->max_recv_nnz >= (int64_t(1) << 30)) return EMB_EINVAL;
  p->recv_nnz_cap = !p->exch ? p->max_nnz
                  : c->max_recv_nnz > 0 ? c->max_recv_nnz
                                        : std::min<int64_t>(p->max_nnz * std::min(W, 2), (int64_t(1) << 30) - 1);
  p->owner_bags_cap = (int64_t)p->max_batch * (p->exch ? (int64_t)p->Fr * W : F);
  // collective a1: one key slot per (source, owner) pair, capacity-padded so the all-to-all
  // sizes are fixed by the plan (no host read of the counts); a source sends at most its
  // max_nnz ids, an owner receives at most recv_nnz_cap
  p->pair_cap = std::min<int64_t>(p->max_nnz, p->recv_nnz_cap);
  return EMB_OK;
}

namespace {

void carve(const Plan& p, Carver& cv, emb_handle* h) {
  const int64_t F = p.F, Bmax = p.max_batch, pitch = p.pitch;
  // a serving (q8-only) handle plans no training workspace (dedup, G, partials, staging)
  const bool train = !(p.flags & EMB_F_Q8_ONLY);
  const int64_t nnz_cap = train ? p.recv_nnz_cap : 1;  // occurrences pooled here per step
  const int64_t bags_cap = p.owner_bags_cap;
  const int64_t dense_cap = std::max<int64_t>(Bmax * F * p.D, 1);
  const int64_t tiles = (std::max<int64_t>(nnz_cap, bags_cap + Bmax * p.dest_base[p.world]) + kSortTileMin - 1) /
                            kSortTileMin + 1;
  const int64_t chunks = chunks_cap_for(nnz_cap);
  const int64_t max_unique = std::min<int64_t>(nnz_cap, p.local_rows) + 1;
  auto* meta = cv.take<FeatMeta>(F);
  int* stage_ids[2];
  int* stage_off[2];
  for (int k = 0; k < 2; ++k) {
    stage_ids[k] = cv.take<int>(p.max_nnz);
    stage_off[k] = cv.take<int>(F * Bmax + 1);
  }
  auto* stage_dense = cv.take<float>(dense_cap);  // also the device out of a host `out`
  auto* off_copy = cv.take<int>(F * Bmax + 1);
  auto* kvA = cv.take<uint2>(nnz_cap);
  auto* kvB = cv.take<uint2>(nnz_cap);
  auto* hist = cv.take<uint32_t>(kHistWords + kMaxPasses + 2);  // hist + counters
  auto* lb = cv.take<unsigned long long>(tiles * kRadixBinsMax);
  auto* cu0 = cv.take<uint32_t>(chunks);
  auto* unique = cv.take<uint32_t>(max_unique);
  auto* seg = cv.take<uint32_t>(max_unique + 1);
  auto* dU = cv.take<uint32_t>(4);
  auto* G = cv.take<float>(max_unique * pitch);
  auto* pf = cv.take<double>(chunks * pitch);
  auto* pl = cv.take<double>(chunks * pitch);
  auto* nm = cv.take<double>(chunks);
  auto* nf = cv.take<double>(chunks);
  auto* ol = cv.take<uint32_t>(3 * chunks + 2 * (chunks / 512 + 1));  // owners, long and big spans
  auto* oc = cv.take<uint32_t>(4);  // owner count, long count, a6 non-finite flag, pad
  auto* sp = cv.take<double>(std::max(p.world, 1));
  auto* sl = cv.take<double>(1);
  auto* nparts = cv.take<double>(64);     // k_norm_partial CTA partials (kNormParts)
  auto* ndone = cv.take<uint32_t>(1);     // its arrival counter (zeroed at create)
  auto* sg = cv.take<double>(1);
  auto* cl = cv.take<float>(1);
  auto* st = cv.take<uint32_t>(1);
  auto* ep = cv.take<uint32_t>(2);
  auto* fwdn = cv.take<uint32_t>(1);
  auto* order = cv.take<uint32_t>(kOrderWsWords(std::max<int64_t>(F * Bmax, bags_cap)));
  ExchangeWs x{};
  if (p.exch) carve_exchange(p, cv, &x);
  if (h) {
    h->order_ws = order;
    h->d_meta = meta;
    for (int k = 0; k < 2; ++k) {
      h->stage_ids[k] = stage_ids[k];
      h->stage_off[k] = stage_off[k];
    }
    h->stage_dense = stage_dense;
    h->off_copy = off_copy;
    h->kvA = kvA; h->kvB = kvB; h->chunk_u0 = cu0;
    h->sort.hist = hist;
    h->sort.counters = hist + kHistWords;
    h->sort.status = lb;
    h->sort.max_tiles = tiles;
    h->unique = unique;
    h->seg = seg;
    h->d_U = dU;
    h->G = G;
    h->part_first = pf; h->part_last = pl; h->norm_main = nm; h->norm_fix = nf;
    h->owner_list = ol; h->owner_count = oc;
    h->chunks_cap = chunks;
    h->S_parts = sp; h->S_local = sl; h->S_global = sg; h->d_clip = cl; h->d_status = st;
    h->d_epoch = ep;
    h->d_fwd_n = fwdn;
    h->norm_parts = nparts; h->norm_done = ndone;
    h->x = x;
  }
}

std::vector<FeatMeta> feat_meta(const Plan& p) {
  std::vector<FeatMeta> m(p.F);
  for (int f = 0; f < p.F; ++f) {
    const int t = p.feature_table[f];
    m[f].base = p.local_base[t];
    m[f].rows = (int32_t)p.table_rows[t];
    m[f].lo = (int32_t)p.row_lo[t];
    m[f].hi = (int32_t)p.row_hi[t];
    m[f].pad = 0;
  }
  return m;
}

}  // namespace

bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

emb_status stage_inputs(emb_t h, const int32_t* ids, const int32_t* offsets, int32_t batch,
                        int64_t nnz, float* out, Staged* s) {
  const int64_t nbags = (int64_t)h->p.F * batch;
  s->ids = ids;
  s->offsets = offsets;
  s->out = out;
  s->host_out = false;
  s->slot = -1;
  // argument errors first: nothing is enqueued for a call that fails
  const bool dev_out = is_device_ptr(out);
  if (dev_out && (h->p.D & 3) == 0 && !aligned(out, 16)) return EMB_EINVAL;
  const bool host_ids = nnz > 0 && !is_device_ptr(ids), host_off = !is_device_ptr(offsets);
  if (host_ids || host_off) {
    // copy stream, double-buffered slot: waits only for the slot's previous readers
    const int k = h->stage_next;
    h->stage_next ^= 1;
    if (k == h->last_slot) {  // the last forward's staged batch is overwritten
      h->last_ids = nullptr;
      h->last_off = nullptr;
      h->last_slot = -1;
    }
    CK(cudaStreamWaitEvent(h->copy, h->ev_free[k], 0));
    if (host_ids) {
      CK(cudaMemcpyAsync(h->stage_ids[k], ids, sizeof(int) * nnz, cudaMemcpyHostToDevice, h->copy));
      s->ids = h->stage_ids[k];
    }
    if (host_off) {
      CK(cudaMemcpyAsync(h->stage_off[k], offsets, sizeof(int) * (nbags + 1), cudaMemcpyHostToDevice, h->copy));
      s->offsets = h->stage_off[k];
    }
    CK(cudaEventRecord(h->ev_ready[k], h->copy));
    CK(cudaStreamWaitEvent(h->stream, h->ev_ready[k], 0));
    s->slot = k;
  }
  if (!dev_out) {
    s->out = h->stage_dense;
    s->host_out = true;
  }
  return EMB_OK;
}

emb_status release_stage(emb_t h, const Staged& s) {
  if (s.slot >= 0) CK(cudaEventRecord(h->ev_free[s.slot], h->stream));
  return EMB_OK;
}

// a5-a8 on this rank's recorded occurrences; grad is the pooled-gradient input in the
// layout of the recorded bags (unsharded: [B][F][D]; owner: [src][B][Fr][D]).  With W > 1
// the rank partials of the global squared norm are all-gathered and summed in rank order.
emb_status launch_dedup(emb_t h) {
  const Plan& p = h->p;
  const int64_t n = h->fwd_nnz;  // exact (unsharded) or the capacity (sharded: count on device)
  const uint2* kres = h->kvA;
  // segment-reduce chunk: sized for the call's ids (small batches still fill every SM), and
  // large enough that a capacity's worth of chunks fits the planned partials
  int cl = chunk_log2_for(h->fwd_nnz_hint);
  while (cl < kChunkLog2Max && ((n + (int64_t(1) << cl) - 1) >> cl) + 1 > h->chunks_cap) ++cl;
  h->chunk_log2 = cl;
  CK(cudaEventRecord(h->ev_kv, h->stream));
  CK(cudaStreamWaitEvent(h->side, h->ev_kv, 0));
  if (n > 0) {
    int passes = 0;
    bool in1 = false;
    {
      Phase ph(h->prof, h->side, EMB_PH_SORT);
      CK(radix_sort_pairs(h->kvA, h->kvB, n, h->fwd_n_dev, p.key_bits, h->sort, h->d_epoch, &passes, &in1,
                          &h->launches, h->side));
    }
    if (in1) kres = h->kvB;
    Phase ph(h->prof, h->side, EMB_PH_RLE);
    CK(launch_rle(kres, n, h->fwd_n_dev, (uint32_t)p.local_rows, h->unique, h->seg, h->d_U, h->chunk_u0, cl,
                  h->sort.counters + kMaxPasses, h->sort.status, h->d_epoch, (uint32_t)passes, h->side));
    CK(launch_epoch_advance(h->d_epoch, (uint32_t)passes + 1, h->side));
    h->launches += 2;
  } else {
    CK(cudaMemsetAsync(h->d_U, 0, sizeof(uint32_t), h->side));
    CK(cudaMemsetAsync(h->seg, 0, sizeof(uint32_t), h->side));
  }
  CK(cudaEventRecord(h->ev_dedup, h->side));
  h->dedup_pending = true;
  h->sorted_kv = kres;
  return EMB_OK;
}

emb_status join_dedup(emb_t h) {
  if (!h->dedup_pending) return EMB_OK;
  CK(cudaStreamWaitEvent(h->stream, h->ev_dedup, 0));
  h->dedup_pending = false;
  return EMB_OK;
}

emb_status backward_local(emb_t h, const float* grad_dev, float lr, double extra,
                          const double* extra_dev, float* clip_out) {
  const Plan& p = h->p;
  const int64_t n = h->fwd_nnz;
  emb_status js = join_dedup(h);  // a5 ran on the side stream since the forward
  if (js != EMB_OK) return js;
  const uint2* kres = h->sorted_kv;

  BwdArgs a;
  memset(&a, 0, sizeof(a));
  a.unique = h->unique;
  a.seg = h->seg;
  a.U = h->d_U;
  a.kv = kres;
  a.chunk_u0 = h->chunk_u0;
  a.nnz = n;
  a.grad = grad_dev;
  a.offsets = h->off_copy;
  a.B = h->fwd_B;
  a.F = p.F;
  a.D = p.D;
  a.pitch = p.pitch;
  a.mean = p.pooling == EMB_POOL_MEAN;
  a.G = h->G;
  a.part_first = h->part_first;
  a.part_last = h->part_last;
  a.norm_main = h->norm_main;
  a.norm_fix = h->norm_fix;
  a.owner_list = h->owner_list;
  a.owner_count = h->owner_count;
  a.chunk_log2 = h->chunk_log2;
  a.chunks = (n + (int64_t(1) << a.chunk_log2) - 1) >> a.chunk_log2;
  a.S_local = h->S_local;
  a.norm_parts = h->norm_parts;
  a.norm_done = h->norm_done;
  a.S_global = h->S_global;
  a.clip = h->d_clip;
  a.status = h->d_status;
  a.extra_sq_norm = extra;
  a.extra_dev = extra_dev;
  a.clip_out = clip_out;
  a.max_norm = p.max_norm;
  a.Wt = h->W;
  a.A = h->A;
  a.rowwise = p.mode == EMB_ADAGRAD_ROWWISE;
  a.lr = lr;
  a.eps = p.eps;
  a.q8_codes = (p.flags & EMB_F_REQUANT) ? h->codes : nullptr;
  a.q8_meta_off = h->q8_meta_off;
  a.q8_minmax = (p.flags & EMB_F_Q8_MINMAX) != 0;
  a.tma = LIRANK_TMA_UPDATE;
  a.qpitch = p.qpitch;

  {
    Phase ph(h->prof, h->stream, EMB_PH_SEGREDUCE);
    CK(launch_segreduce(a, &h->launches, h->stream));
  }
  {
    Phase ph(h->prof, h->stream, EMB_PH_NORM);
    if (h->fim_on && n > 0) {  // NEXT-3: penalty gradient of the touched rows, norm re-formed
      const int64_t ng = launch_fim_penalty(a, h->fim, h->stream);
      if (ng < 0) return EMB_ECUDA;
      a.chunks = ng;
      h->launches += 1;
    }
    CK(launch_norm_partial(a, h->stream));
    h->launches += 1;
    const double* parts = h->S_local;
    int np = 1;
    if (p.exch) {
      if (!h->comm->allgather(h->S_local, h->S_parts, sizeof(double), h->stream)) return EMB_ENCCL;
      parts = h->S_parts;
      np = p.world;
    }
    CK(launch_norm_finalize(parts, np, a, h->stream));
    h->launches += 1;
  }
  {
    Phase ph(h->prof, h->stream, EMB_PH_UPDATE);
    CK(launch_adagrad(a, h->stream));
    h->launches += n > 0;
  }
  if ((p.flags & EMB_F_REQUANT) && n > 0) h->have_q8 = true;
  return EMB_OK;
}

}  // namespace lirank

namespace api_detail {

emb_status check_batch_args(emb_t h, const int32_t* ids, const int32_t* offsets, int32_t batch,
                            int64_t nnz, const float* out) {
  if (!h || !offsets || !out) return EMB_EINVAL;
  if (batch < 0 || batch > h->p.max_batch) return EMB_EINVAL;
  if (nnz < 0 || nnz > h->p.max_nnz) return EMB_EINVAL;
  if (nnz > 0 && !ids) return EMB_EINVAL;
  return EMB_OK;
}

__global__ void k_gather_rows_b(const uint8_t* src, int64_t pitch_bytes, const int64_t* rows,
                                int64_t n, int64_t row_bytes, uint8_t* dst) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x)
    for (int64_t b = threadIdx.x; b < row_bytes; b += blockDim.x)
      dst[i * row_bytes + b] = src[rows[i] * pitch_bytes + b];
}
__global__ void k_scatter_rows_b(uint8_t* dst, int64_t pitch_bytes, const int64_t* rows,
                                 int64_t n, int64_t row_bytes, const uint8_t* src) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x)
    for (int64_t b = threadIdx.x; b < row_bytes; b += blockDim.x)
      dst[rows[i] * pitch_bytes + b] = src[i * row_bytes + b];
}

emb_status stored_rows(emb_t h, int32_t table, const int64_t* rows, int64_t n, std::vector<int64_t>* out) {
  const Plan& p = h->p;
  if (table < 0 || table >= p.T || n < 0 || (n > 0 && !rows)) return EMB_EINVAL;
  if (p.local_base[table] < 0 && n > 0) return EMB_EINVAL;
  out->resize(n);
  for (int64_t i = 0; i < n; ++i) {
    if (rows[i] < p.row_lo[table] || rows[i] >= p.row_hi[table]) return EMB_EINVAL;
    (*out)[i] = p.local_base[table] + rows[i] - p.row_lo[table];
  }
  return EMB_OK;
}

// Generic gather (dir=0) / scatter (dir=1) of n rows of `row_bytes` out of a device array
// with pitch `pitch_bytes`, through a temporary device buffer (not a hot path).
emb_status move_rows(emb_t h, void* dev, int64_t pitch_bytes, const std::vector<int64_t>& r,
                     int64_t row_bytes, void* host, int dir) {
  const int64_t n = (int64_t)r.size();
  if (n == 0) return EMB_OK;
  int64_t* d_rows = nullptr;
  uint8_t* d_buf = nullptr;
  CK(cudaMalloc(&d_rows, sizeof(int64_t) * n));
  if (cudaMalloc(&d_buf, row_bytes * n) != cudaSuccess) { cudaFree(d_rows); return EMB_ECUDA; }
  emb_status s = EMB_OK;
  do {
    if (cudaMemcpyAsync(d_rows, r.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, h->stream) != cudaSuccess) { s = EMB_ECUDA; break; }
    const unsigned grid = (unsigned)std::min<int64_t>(n, 65535);
    if (dir == 0) {
      k_gather_rows_b<<<grid, 128, 0, h->stream>>>((const uint8_t*)dev, pitch_bytes, d_rows, n, row_bytes, d_buf);
      if (cudaMemcpyAsync(host, d_buf, row_bytes * n, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess) { s = EMB_ECUDA; break; }
    } else {
      if (cudaMemcpyAsync(d_buf, host, row_bytes * n, cudaMemcpyHostToDevice, h->stream) != cudaSuccess) { s = EMB_ECUDA; break; }
      k_scatter_rows_b<<<grid, 128, 0, h->stream>>>((uint8_t*)dev, pitch_bytes, d_rows, n, row_bytes, d_buf);
    }
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(h->stream) != cudaSuccess) s = EMB_ECUDA;
  } while (0);
  cudaFree(d_rows);
  cudaFree(d_buf);
  return s;
}

}  // namespace api_detail

using namespace api_detail;

extern "C" {

int32_t emb_abi_version(void) { return EMB_ABI_VERSION; }

const char* emb_status_string(emb_status s) {
  switch (s) {
    case EMB_OK: return "ok";
    case EMB_EINVAL: return "invalid argument";
    case EMB_ENOMEM: return "buffer too small";
    case EMB_ECUDA: return "CUDA error";
    case EMB_ENCCL: return "NCCL / transport error";
    case EMB_EIDRANGE: return "id out of range (skipped)";
    case EMB_ENONFINITE: return "non-finite value (update skipped / row zeroed)";
    case EMB_ESTATE: return "call out of order";
  }
  return "unknown status";
}

emb_status emb_plan(const emb_config* cfg, emb_sizes* out) {
  if (!out) return EMB_EINVAL;
  Plan p;
  emb_status s = make_plan(cfg, &p);
  if (s != EMB_OK) return s;
  Carver cv(nullptr);
  carve(p, cv, nullptr);
  const bool serving = (p.flags & EMB_F_Q8_ONLY) != 0;
  out->weights_bytes = serving ? 0 : std::max<int64_t>(p.local_rows * p.pitch * 4, 4);
  out->accum_bytes = serving ? 0 : std::max<int64_t>(
      p.mode == EMB_ADAGRAD_ROWWISE ? p.local_rows * 4 : p.local_rows * p.pitch * 4, 4);
  out->q8_codes_bytes = (p.flags & EMB_F_Q8) ? std::max<int64_t>(p.local_rows * p.qpitch, 16) : 0;
  out->q8_meta_bytes = 0;  // {middle, scale} live inside the q8 rows
  out->workspace_bytes = round_up(cv.off, kAlign);
  out->local_rows = p.local_rows;
  out->row_pitch = p.pitch;
  out->q8_pitch = p.qpitch;
  return EMB_OK;
}

emb_status emb_local_layout(const emb_config* cfg, int64_t* local_base, int64_t* row_lo,
                            int64_t* row_hi) {
  Plan p;
  emb_status s = make_plan(cfg, &p);
  if (s != EMB_OK) return s;
  for (int t = 0; t < p.T; ++t) {
    if (local_base) local_base[t] = p.local_base[t];
    if (row_lo) row_lo[t] = p.row_lo[t];
    if (row_hi) row_hi[t] = p.row_hi[t];
  }
  return EMB_OK;
}

emb_status emb_nccl_unique_id(void* out128) {
  if (!out128) return EMB_EINVAL;
  return nccl_get_unique_id(out128) ? EMB_OK : EMB_ENCCL;
}

emb_status emb_loopback_hub_create(int32_t world, void** hub) {
  if (!hub || world < 1 || world > kMaxWorld) return EMB_EINVAL;
  *hub = loopback_hub_create(world);
  return *hub ? EMB_OK : EMB_ENOMEM;
}

emb_status emb_loopback_hub_destroy(void* hub) {
  if (!hub) return EMB_EINVAL;
  loopback_hub_destroy(hub);
  return EMB_OK;
}

emb_status emb_create(const emb_config* cfg, const emb_buffers* buf, emb_t* out) {
  if (!cfg || !buf || !out) return EMB_EINVAL;
  *out = nullptr;
  emb_handle* h = new (std::nothrow) emb_handle();
  if (!h) return EMB_ENOMEM;
  emb_status s = make_plan(cfg, &h->p);
  if (s != EMB_OK) { delete h; return s; }
  const Plan& p = h->p;
  const bool serving = (p.flags & EMB_F_Q8_ONLY) != 0;
  if ((!serving && (!buf->weights || !buf->accum)) || !buf->workspace) { delete h; return EMB_EINVAL; }
  if ((p.flags & EMB_F_Q8) && !buf->q8_codes) { delete h; return EMB_EINVAL; }
  const void* ptrs[5] = {buf->weights, buf->accum, buf->workspace, buf->q8_codes, buf->q8_meta};
  for (const void* q : ptrs)
    if (q && !aligned(q, kAlign)) { delete h; return EMB_EINVAL; }
  if (p.exch && !cfg->nccl_unique_id) { delete h; return EMB_EINVAL; }
  h->stream = (cudaStream_t)cfg->stream;
  h->W = serving ? nullptr : (float*)buf->weights;
  h->A = serving ? nullptr : (float*)buf->accum;
  h->codes = (uint8_t*)buf->q8_codes;
  h->q8_meta_off = (int)round_up(p.D, 8);
  Carver cv(buf->workspace);
  carve(p, cv, h);
  // device init: feature metadata, accumulators = A0, status = 0, look-back words = 0
  std::vector<FeatMeta> m = feat_meta(p);
  cudaError_t e = cudaMemcpyAsync(h->d_meta, m.data(), sizeof(FeatMeta) * m.size(),
                                  cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) {
    const int64_t na = serving ? 0 : (p.mode == EMB_ADAGRAD_ROWWISE ? p.local_rows : p.local_rows * p.pitch);
    if (na > 0) e = launch_fill(h->A, na, p.A0, h->stream);
    h->launches += na > 0;
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(h->d_status, 0, sizeof(uint32_t), h->stream);
  const uint32_t epoch0[2] = {1u, 1u};  // status words are zeroed: epoch 0 is never current
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h->d_epoch, epoch0, sizeof(epoch0), cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->norm_done, 0, sizeof(uint32_t), h->stream);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(h->sort.status, 0, sizeof(unsigned long long) * h->sort.max_tiles * kRadixBinsMax, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // `m` goes out of scope
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_kv, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_dedup, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->copy, cudaStreamNonBlocking);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&h->ev_ready[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_free[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_free[k], h->stream);  // slots start free
  }
  if (e != cudaSuccess) { delete h; return EMB_ECUDA; }
  if (p.exch) {
    h->comm = (p.flags & EMB_F_LOOPBACK)   ? make_loopback_transport((void*)cfg->nccl_unique_id, p.rank)
              : (p.flags & EMB_F_HOSTCOMM) ? make_host_transport(cfg->nccl_unique_id, p.rank, p.world)
                                           : make_nccl_transport(cfg->nccl_unique_id, p.rank, p.world);
    if (!h->comm) { delete h; return EMB_ENCCL; }
    if ((s = exchange_init(h)) != EMB_OK) { delete h->comm; delete h; return s; }
  }
  *out = h;
  return EMB_OK;
}

emb_status emb_destroy(emb_t h) {
  if (!h) return EMB_EINVAL;
  if (h->side) {
    cudaStreamSynchronize(h->side);
    cudaStreamDestroy(h->side);
  }
  if (h->ev_kv) cudaEventDestroy(h->ev_kv);
  if (h->ev_dedup) cudaEventDestroy(h->ev_dedup);
  if (h->copy) {
    cudaStreamSynchronize(h->copy);
    cudaStreamDestroy(h->copy);
  }
  for (int k = 0; k < 2; ++k) {
    if (h->ev_ready[k]) cudaEventDestroy(h->ev_ready[k]);
    if (h->ev_free[k]) cudaEventDestroy(h->ev_free[k]);
  }
  delete h->comm;
  delete h;
  return EMB_OK;
}

int64_t emb_kernel_launches(emb_t h) { return h ? h->launches : -1; }

emb_status emb_profile(emb_t h, int32_t enable) {
  if (!h) return EMB_EINVAL;
  h->prof.on = enable != 0;
  return EMB_OK;
}

emb_status emb_profile_read(emb_t h, double* ms, int64_t* count, int32_t reset) {
  if (!h) return EMB_EINVAL;
  Prof& pr = h->prof;
  if (reset) {
    for (int i = 0; i < EMB_PH_COUNT; ++i) { pr.ms[i] = 0; pr.n[i] = 0; }
  }
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaStreamSynchronize(h->side));
  for (auto& r : pr.pending) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) {
      pr.ms[r.ph] += t;
      pr.n[r.ph] += 1;
    }
    pr.pool.push_back(r.a);
    pr.pool.push_back(r.b);
  }
  pr.pending.clear();
  for (int i = 0; i < EMB_PH_COUNT; ++i) {
    if (ms) ms[i] = pr.ms[i];
    if (count) count[i] = pr.n[i];
  }
  return EMB_OK;
}

emb_status emb_sync(emb_t h) {
  if (!h) return EMB_EINVAL;
  CK(cudaStreamSynchronize(h->side));
  CK(cudaStreamSynchronize(h->stream));
  uint32_t st = 0;
  CK(cudaMemcpy(&st, h->d_status, sizeof(st), cudaMemcpyDeviceToHost));
  CK(cudaMemsetAsync(h->d_status, 0, sizeof(uint32_t), h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (st & kStOverflow) return EMB_ENOMEM;
  if (st & kStNonFinite) return EMB_ENONFINITE;
  if (st & kStIdRange) return EMB_EIDRANGE;
  return EMB_OK;
}

// --------------------------------------------------------------------------------------
// forward
// --------------------------------------------------------------------------------------

emb_status emb_forward(emb_t h, const int32_t* ids, const int32_t* offsets, int32_t batch,
                       int64_t nnz, float* out) {
  emb_status s = check_batch_args(h, ids, offsets, batch, nnz, out);
  if (s != EMB_OK) return s;
  const Plan& p = h->p;
  if (!h->W) return EMB_ESTATE;  // serving (q8-only) handle
  if ((s = join_dedup(h)) != EMB_OK) return s;  // the previous dedup may still read kvA/kvB
  Staged st;
  {
    Phase ph(h->prof, h->stream, EMB_PH_COPY);
    s = stage_inputs(h, ids, offsets, batch, nnz, out, &st);
  }
  if (s != EMB_OK) return s;
  h->last_ids = st.ids;  // (device) inputs of this forward, for emb_forward_q8(NULL, NULL)
  h->last_off = st.offsets;
  h->last_B = batch;
  h->last_nnz = nnz;
  h->last_slot = st.slot;
  if (p.exch) {
    s = exchange_forward(h, st, batch, nnz, /*q8=*/false);
    if (s != EMB_OK) return s;
    if ((s = launch_dedup(h)) != EMB_OK) return s;
  } else {
    FwdArgs a;
    memset(&a, 0, sizeof(a));
    a.W = h->W;
    a.pitch = p.pitch;
    a.ids = st.ids;
    a.offsets = st.offsets;
    a.B = batch;
    a.F = p.F;
    a.D = p.D;
    a.meta = h->d_meta;
    a.out = st.out;
    a.kv_out = h->kvA;
    a.sentinel = (uint32_t)p.local_rows;
    a.status = h->d_status;
    a.mean = p.pooling == EMB_POOL_MEAN;
    a.order_ws = h->order_ws;
    h->order_offsets = st.offsets;
    h->order_bags = (int64_t)p.F * batch;
    {
      Phase ph(h->prof, h->stream, EMB_PH_FWD);
      CK(launch_pool_fwd_f32(a, h->stream));
    }
    h->launches += fwd_launches((int64_t)p.F * batch, true, true);
    if (a.mean) {
      Phase ph(h->prof, h->stream, EMB_PH_COPY);
      CK(cudaMemcpyAsync(h->off_copy, st.offsets, sizeof(int) * ((int64_t)p.F * batch + 1),
                         cudaMemcpyDeviceToDevice, h->stream));
    }
    h->have_fwd = true;
    h->fwd_nnz = nnz;
    h->fwd_n_dev = nullptr;
    h->fwd_nnz_hint = nnz;
    h->fwd_B = batch;
    if ((s = launch_dedup(h)) != EMB_OK) return s;  // a5 starts now, on the side stream
  }
  if ((s = release_stage(h, st)) != EMB_OK) return s;
  if (st.host_out) {
    Phase ph(h->prof, h->stream, EMB_PH_COPY);
    CK(cudaMemcpyAsync(out, st.out, sizeof(float) * (int64_t)batch * p.F * p.D,
                       cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));  // a host `out` is complete when the call returns
  }
  return EMB_OK;
}

emb_status emb_forward_q8(emb_t h, const int32_t* ids, const int32_t* offsets, int32_t batch,
                          int64_t nnz, float* out) {
  // ids == offsets == NULL: the batch of the most recent emb_forward (its staged copy when
  // it came from host memory), e.g. serving the q8 store on the batch just trained on
  const bool reuse = h && !ids && !offsets;
  if (reuse) {
    if (!h->last_off) return EMB_ESTATE;
    if (batch != h->last_B || nnz != h->last_nnz) return EMB_EINVAL;
    ids = h->last_ids;
    offsets = h->last_off;
  }
  emb_status s = check_batch_args(h, ids, offsets, batch, nnz, out);
  if (s != EMB_OK) return s;
  const Plan& p = h->p;
  if (!(p.flags & EMB_F_Q8) || !h->have_q8) return EMB_ESTATE;
  Staged st;
  {
    Phase ph(h->prof, h->stream, EMB_PH_COPY);
    s = stage_inputs(h, ids, offsets, batch, nnz, out, &st);
  }
  if (s != EMB_OK) return s;
  if (reuse) st.slot = h->last_slot;  // the forward's staged batch: its slot is read again
  if (p.exch) {
    s = exchange_forward(h, st, batch, nnz, /*q8=*/true, reuse);
    if (s != EMB_OK) return s;
  } else {
    FwdQ8Args a;
    memset(&a, 0, sizeof(a));
    a.codes = h->codes;
    a.qpitch = p.qpitch;
    a.meta_off = h->q8_meta_off;
    a.minmax = (p.flags & EMB_F_Q8_MINMAX) != 0;
    a.ids = st.ids;
    a.offsets = st.offsets;
    a.B = batch;
    a.F = p.F;
    a.D = p.D;
    a.meta = h->d_meta;
    a.out = st.out;
    a.status = h->d_status;
    a.mean = p.pooling == EMB_POOL_MEAN;
    a.order_ws = h->order_ws;
    a.order_ready = h->order_offsets == st.offsets && h->order_bags == (int64_t)p.F * batch &&
                    h->order_bags >= 2;
    {
      Phase ph(h->prof, h->stream, EMB_PH_FWD_Q8);
      CK(launch_pool_fwd_q8(a, h->stream));
    }
    h->launches += a.order_ready ? 1 : fwd_launches((int64_t)p.F * batch, true, false);
  }
  if ((s = release_stage(h, st)) != EMB_OK) return s;
  if (st.host_out) {
    Phase ph(h->prof, h->stream, EMB_PH_COPY);
    CK(cudaMemcpyAsync(out, st.out, sizeof(float) * (int64_t)batch * p.F * p.D,
                       cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));  // a host `out` is complete when the call returns
  }
  return EMB_OK;
}

// --------------------------------------------------------------------------------------
// backward
// --------------------------------------------------------------------------------------

static emb_status backward_common(emb_t h, const float* grad_out, float lr, double extra_sq_norm,
                                  const double* extra_dev, float* clip_out) {
  if (!h || !grad_out) return EMB_EINVAL;
  if (!h->have_fwd) return EMB_ESTATE;
  if (!(lr >= 0.f) || !(extra_sq_norm >= 0.0)) return EMB_EINVAL;
  if ((extra_dev && !is_device_ptr(extra_dev)) || (clip_out && !is_device_ptr(clip_out)))
    return EMB_EINVAL;
  const Plan& p = h->p;
  const float* g = grad_out;
  if (!is_device_ptr(grad_out)) {
    Phase ph(h->prof, h->stream, EMB_PH_COPY);
    CK(cudaMemcpyAsync(h->stage_dense, grad_out, sizeof(float) * (int64_t)h->fwd_B * p.F * p.D,
                       cudaMemcpyHostToDevice, h->stream));
    g = h->stage_dense;
  } else if ((p.D & 3) == 0 && !aligned(grad_out, 16)) {
    return EMB_EINVAL;
  }
  if (p.exch) {
    emb_status s = exchange_backward(h, g);
    if (s != EMB_OK) return s;
    return backward_local(h, h->x.pooled, lr, extra_sq_norm, extra_dev, clip_out);
  }
  return backward_local(h, g, lr, extra_sq_norm, extra_dev, clip_out);
}

emb_status emb_backward_adagrad(emb_t h, const float* grad_out, float lr, double extra_sq_norm,
                                double* sq_norm_out) {
  emb_status s = backward_common(h, grad_out, lr, extra_sq_norm, nullptr, nullptr);
  if (s != EMB_OK) return s;
  if (sq_norm_out) {
    CK(cudaMemcpyAsync(sq_norm_out, h->S_global, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  return EMB_OK;
}

emb_status emb_allreduce_f32(emb_t h, float* data, int64_t count) {
  if (!h || count < 0 || (count > 0 && !data)) return EMB_EINVAL;
  const Plan& p = h->p;
  if (count == 0 || !p.exch) return EMB_OK;
  if (!is_device_ptr(data)) return EMB_EINVAL;
  Phase ph(h->prof, h->stream, EMB_PH_EXCHANGE);
  return h->comm->allreduce_sum_f32(data, (size_t)count, h->stream) ? EMB_OK : EMB_ENCCL;
}

emb_status emb_backward_adagrad_dev(emb_t h, const float* grad_out, float lr,
                                    const double* extra_sq_norm_dev, float* clip_out_dev,
                                    double* sq_norm_out_dev) {
  emb_status s = backward_common(h, grad_out, lr, 0.0, extra_sq_norm_dev, clip_out_dev);
  if (s != EMB_OK) return s;
  if (sq_norm_out_dev) {
    if (!is_device_ptr(sq_norm_out_dev)) return EMB_EINVAL;
    CK(cudaMemcpyAsync(sq_norm_out_dev, h->S_global, sizeof(double), cudaMemcpyDeviceToDevice,
                       h->stream));
  }
  return EMB_OK;
}

// --------------------------------------------------------------------------------------
// quantize
// --------------------------------------------------------------------------------------

emb_status emb_quantize_mm8(emb_t h) {
  if (!h) return EMB_EINVAL;
  const Plan& p = h->p;
  if (!(p.flags & EMB_F_Q8) || !h->W) return EMB_ESTATE;
  {
    Phase ph(h->prof, h->stream, EMB_PH_QUANTIZE);
    CK(launch_quantize(h->W, p.pitch, p.local_rows, p.D, h->codes, p.qpitch, h->q8_meta_off,
                       (p.flags & EMB_F_Q8_MINMAX) != 0,
                       h->d_status, h->stream));
  }
  h->launches += p.local_rows > 0;
  h->have_q8 = true;
  return EMB_OK;
}

emb_status emb_quantize_block(emb_t h, int32_t table, int64_t row0, int64_t n, const float* rows,
                              int64_t ld) {
  if (!h) return EMB_EINVAL;
  const Plan& p = h->p;
  if (!(p.flags & EMB_F_Q8)) return EMB_ESTATE;
  if (table < 0 || table >= p.T || n < 0 || row0 < 0 || ld < p.D || (ld & 3)) return EMB_EINVAL;
  if (n == 0) return EMB_OK;
  if (!rows || !is_device_ptr(rows) || !aligned(rows, 16)) return EMB_EINVAL;
  if (p.local_base[table] < 0 || row0 < p.row_lo[table] || row0 + n > p.row_hi[table])
    return EMB_EINVAL;  // not stored (entirely) on this rank
  const int64_t local = p.local_base[table] + (row0 - p.row_lo[table]);
  {
    Phase ph(h->prof, h->stream, EMB_PH_QUANTIZE);
    CK(launch_quantize(rows, (int)ld, n, p.D, h->codes + local * p.qpitch, p.qpitch, h->q8_meta_off,
                       (p.flags & EMB_F_Q8_MINMAX) != 0, h->d_status, h->stream));
  }
  h->launches += 1;
  h->have_q8 = true;
  return EMB_OK;
}

// --------------------------------------------------------------------------------------
// introspection
// --------------------------------------------------------------------------------------

// Rows of D floats <-> stored rows of `pitch` floats (pads stay as they are on write).
emb_status emb_read_rows(emb_t h, int32_t table, const int64_t* rows, int64_t n, float* w,
                         float* acc) {
  if (!h || (n > 0 && !w)) return EMB_EINVAL;
  if (!h->W) return EMB_ESTATE;
  std::vector<int64_t> r;
  emb_status s = stored_rows(h, table, rows, n, &r);
  if (s != EMB_OK) return s;
  const Plan& p = h->p;
  CK(cudaStreamSynchronize(h->stream));
  s = move_rows(h, h->W, (int64_t)p.pitch * 4, r, (int64_t)p.D * 4, w, 0);
  if (s != EMB_OK || !acc) return s;
  if (p.mode == EMB_ADAGRAD_ROWWISE) return move_rows(h, h->A, 4, r, 4, acc, 0);
  return move_rows(h, h->A, (int64_t)p.pitch * 4, r, (int64_t)p.D * 4, acc, 0);
}

emb_status emb_write_rows(emb_t h, int32_t table, const int64_t* rows, int64_t n, const float* w,
                          const float* acc) {
  if (!h) return EMB_EINVAL;
  if (!h->W) return EMB_ESTATE;
  std::vector<int64_t> r;
  emb_status s = stored_rows(h, table, rows, n, &r);
  if (s != EMB_OK) return s;
  const Plan& p = h->p;
  if (w) {
    s = move_rows(h, h->W, (int64_t)p.pitch * 4, r, (int64_t)p.D * 4, (void*)w, 1);
    if (s != EMB_OK) return s;
  }
  if (acc) {
    if (p.mode == EMB_ADAGRAD_ROWWISE) return move_rows(h, h->A, 4, r, 4, (void*)acc, 1);
    return move_rows(h, h->A, (int64_t)p.pitch * 4, r, (int64_t)p.D * 4, (void*)acc, 1);
  }
  return EMB_OK;
}

emb_status emb_read_q8(emb_t h, int32_t table, const int64_t* rows, int64_t n, int8_t* codes,
                       float* middle, float* scale) {
  if (!h) return EMB_EINVAL;
  const Plan& p = h->p;
  if (!(p.flags & EMB_F_Q8)) return EMB_ESTATE;
  std::vector<int64_t> r;
  emb_status s = stored_rows(h, table, rows, n, &r);
  if (s != EMB_OK) return s;
  CK(cudaStreamSynchronize(h->stream));
  if (codes) {
    s = move_rows(h, h->codes, p.qpitch, r, p.D, codes, 0);
    if (s != EMB_OK) return s;
  }
  if (middle || scale) {
    std::vector<float> mt(2 * n);
    s = move_rows(h, h->codes + h->q8_meta_off, p.qpitch, r, 8, mt.data(), 0);
    if (s != EMB_OK) return s;
    for (int64_t i = 0; i < n; ++i) {
      if (middle) middle[i] = mt[2 * i];
      if (scale) scale[i] = mt[2 * i + 1];
    }
  }
  return EMB_OK;
}

emb_status emb_last_dedup(emb_t h, int32_t* unique, int32_t* seg_offsets, int64_t cap,
                          int32_t* sorted_bags, int64_t cap_occ, int64_t* n_unique,
                          int64_t* n_valid) {
  if (!h) return EMB_EINVAL;
  if (!h->sorted_kv) return EMB_ESTATE;
  CK(cudaStreamSynchronize(h->side));
  CK(cudaStreamSynchronize(h->stream));
  uint32_t U = 0, nv = 0;
  CK(cudaMemcpy(&U, h->d_U, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&nv, h->seg + U, 4, cudaMemcpyDeviceToHost));
  if (n_unique) *n_unique = U;
  if (n_valid) *n_valid = nv;
  if ((unique || seg_offsets) && cap < (int64_t)U) return EMB_ENOMEM;
  if (sorted_bags && cap_occ < (int64_t)nv) return EMB_ENOMEM;
  if (unique && U) CK(cudaMemcpy(unique, h->unique, 4ull * U, cudaMemcpyDeviceToHost));
  if (seg_offsets) CK(cudaMemcpy(seg_offsets, h->seg, 4ull * (U + 1), cudaMemcpyDeviceToHost));
  if (sorted_bags && nv) {
    std::vector<uint2> tmp(nv);
    CK(cudaMemcpy(tmp.data(), h->sorted_kv, 8ull * nv, cudaMemcpyDeviceToHost));
    // the pairs carry the grad row (b*F + f); report the bag index f*B + b
    const uint32_t F = (uint32_t)h->p.F, B = (uint32_t)h->fwd_B;
    for (uint32_t i = 0; i < nv; ++i) {
      const uint32_t r = tmp[i].y;
      sorted_bags[i] = (int32_t)(h->p.exch ? r : (r % F) * B + r / F);
    }
  }
  return EMB_OK;
}

emb_status emb_set_incremental(emb_t h, const float* w0, const float* H0, const float* w1,
                               const float* H1, float lambda_f, float alpha) {
  if (!h) return EMB_EINVAL;
  if (!h->W) return EMB_ESTATE;
  if (!(lambda_f >= 0.f) || !(alpha >= 0.f && alpha <= 1.f)) return EMB_EINVAL;
  if ((w0 == nullptr) != (H0 == nullptr) || (w1 == nullptr) != (H1 == nullptr)) return EMB_EINVAL;
  for (const float* p : {w0, H0, w1, H1})
    if (p && (!is_device_ptr(p) || !aligned(p, 16))) return EMB_EINVAL;
  h->fim = FimArgs{w0, H0, w1, H1, lambda_f, alpha};
  h->fim_on = lambda_f > 0.f && (w0 != nullptr || w1 != nullptr);
  return EMB_OK;
}

emb_status emb_cold_weight_init(emb_t h, const float* w0, const float* w1, float alpha) {
  if (!h || !w0 || !w1) return EMB_EINVAL;
  if (!h->W) return EMB_ESTATE;
  if (!(alpha >= 0.f && alpha <= 1.f)) return EMB_EINVAL;
  if (!is_device_ptr(w0) || !is_device_ptr(w1) || !aligned(w0, 16) || !aligned(w1, 16))
    return EMB_EINVAL;
  const Plan& p = h->p;
  CK(launch_cold_init(w0, w1, p.local_rows * p.pitch, alpha, h->W, h->stream));
  h->launches += p.local_rows > 0;
  return EMB_OK;
}

emb_status emb_last_stats(emb_t h, double* sq_norm, float* clip, int64_t* n_unique) {
  if (!h) return EMB_EINVAL;
  CK(cudaStreamSynchronize(h->side));
  CK(cudaStreamSynchronize(h->stream));
  if (sq_norm) CK(cudaMemcpy(sq_norm, h->S_global, 8, cudaMemcpyDeviceToHost));
  if (clip) CK(cudaMemcpy(clip, h->d_clip, 4, cudaMemcpyDeviceToHost));
  if (n_unique) {
    uint32_t U = 0;
    CK(cudaMemcpy(&U, h->d_U, 4, cudaMemcpyDeviceToHost));
    *n_unique = U;
  }
  return EMB_OK;
}

}  // extern "C"
