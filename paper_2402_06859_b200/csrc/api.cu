// api.cu -- C ABI (include/lirank_emb.h): planning, workspace carve-up, call sequencing.
//
// Host code only orchestrates: every step of the hot path runs in the kernels of
// forward.cu / sort.cu / backward.cu.  No CPU fallback exists: without a CUDA device
// every compute call fails with EMB_ECUDA.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <vector>

#include "../../include/lirank_emb.h"
#include "comm.h"
#include "common.cuh"
#include "kernels.h"

using namespace lirank;

namespace {

constexpr int64_t kAlign = 256;

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Bump allocator over the caller's workspace; with base == nullptr it only sizes.
struct Carver {
  uint8_t* base;
  int64_t off = 0;
  explicit Carver(void* b) : base((uint8_t*)b) {}
  template <class T>
  T* take(int64_t count) {
    off = round_up(off, kAlign);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += (int64_t)sizeof(T) * std::max<int64_t>(count, 1);
    return p;
  }
};

struct Plan {
  int T = 0, D = 0, F = 0, pitch = 0, qpitch = 0;
  int pooling = 0, mode = 0, sharding = 0, rank = 0, world = 1;
  uint32_t flags = 0;
  float A0 = 0.f, eps = 0.f, max_norm = 0.f;
  int64_t max_nnz = 0;
  int max_batch = 0;
  std::vector<int64_t> table_rows, local_base, row_lo, row_hi;
  std::vector<int32_t> feature_table, owner;
  int64_t local_rows = 0;
  int key_bits = 0;
  // exchange capacities (world > 1)
  int64_t recv_nnz_cap = 0;   // ids this rank may receive per step
  int64_t owner_bags_cap = 0; // bags this rank may pool per step (sum over sources)
};

int bits_for(int64_t v) {  // smallest b with v < 2^b
  int b = 0;
  while (b < 63 && (int64_t(1) << b) <= v) ++b;
  return b;
}

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
  if (c->world_size < 1 || c->rank < 0 || c->rank >= c->world_size) return EMB_EINVAL;
  if (c->world_size == 1 && c->sharding != EMB_SHARD_NONE && c->sharding != EMB_SHARD_TABLE &&
      c->sharding != EMB_SHARD_ROW)
    return EMB_EINVAL;
  if (c->world_size > 1 && c->sharding != EMB_SHARD_TABLE && c->sharding != EMB_SHARD_ROW)
    return EMB_EINVAL;
  p->T = c->num_tables;
  p->D = c->dim;
  p->F = c->num_features;
  p->pitch = (int)round_up(c->dim, 4);
  // q8 row: [codes][pad to 8][middle, scale][pad to 32]: whole 32-B sectors, so the
  // fused re-quantize never partially writes a sector (no L2 fill reads)
  p->qpitch = (int)round_up(round_up(c->dim, 8) + 8, 32);
  p->pooling = c->pooling;
  p->mode = c->adagrad_mode;
  p->sharding = c->world_size > 1 ? c->sharding : EMB_SHARD_NONE;
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

  const int W = p->world;
  p->owner.assign(p->T, 0);
  p->local_base.assign(p->T, -1);
  p->row_lo.assign(p->T, 0);
  p->row_hi.assign(p->T, 0);
  if (p->sharding == EMB_SHARD_TABLE) {
    if (c->table_owner) {
      for (int t = 0; t < p->T; ++t) {
        if (c->table_owner[t] < 0 || c->table_owner[t] >= W) return EMB_EINVAL;
        p->owner[t] = c->table_owner[t];
      }
    } else {
      // greedy LPT by rows (largest first, ties by table index), to the least-loaded rank
      std::vector<int> order(p->T);
      for (int t = 0; t < p->T; ++t) order[t] = t;
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return p->table_rows[a] > p->table_rows[b];
      });
      std::vector<int64_t> load(W, 0);
      for (int t : order) {
        int best = 0;
        for (int r = 1; r < W; ++r)
          if (load[r] < load[best]) best = r;
        p->owner[t] = best;
        load[best] += p->table_rows[t];
      }
    }
  }
  int64_t lr = 0;
  for (int t = 0; t < p->T; ++t) {
    const int64_t R = p->table_rows[t];
    int64_t lo = 0, hi = R;
    bool mine = true;
    if (p->sharding == EMB_SHARD_TABLE) {
      mine = p->owner[t] == p->rank;
    } else if (p->sharding == EMB_SHARD_ROW) {
      const int64_t blk = (R + W - 1) / W;
      lo = std::min<int64_t>(R, (int64_t)p->rank * blk);
      hi = std::min<int64_t>(R, lo + blk);
    }
    if (!mine) {
      p->local_base[t] = -1;
      p->row_lo[t] = 0;
      p->row_hi[t] = 0;
      continue;
    }
    p->local_base[t] = lr;
    p->row_lo[t] = lo;
    p->row_hi[t] = hi;
    lr += hi - lo;
  }
  if (lr >= (int64_t(1) << 31) - 1) return EMB_EINVAL;
  p->local_rows = lr;
  p->key_bits = bits_for(lr);  // keys in [0, lr], sentinel = lr
  // Exchange capacities: a rank can receive at most every id of every rank, and pools at
  // most every bag of every rank.  (Capacity, not expectation.)
  p->recv_nnz_cap = W > 1 ? p->max_nnz * W : p->max_nnz;
  p->owner_bags_cap = (int64_t)p->max_batch * p->F * W;
  if (p->recv_nnz_cap >= (int64_t(1) << 30)) p->recv_nnz_cap = (int64_t(1) << 30) - 1;
  return EMB_OK;
}

}  // namespace

// CUDA-event phase profiler (emb_profile / emb_profile_read).
struct Prof {
  bool on = false;
  struct Rec { int ph; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  double ms[EMB_PH_COUNT] = {};
  int64_t n[EMB_PH_COUNT] = {};
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  ~Prof() {
    for (auto& r : pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// RAII phase marker: records a start event now and an end event at scope exit.
struct Phase {
  Prof* pr;
  cudaStream_t s;
  int ph;
  cudaEvent_t a = nullptr;
  Phase(Prof& p, cudaStream_t st, int phase) : pr(p.on ? &p : nullptr), s(st), ph(phase) {
    if (pr) { a = pr->get(); cudaEventRecord(a, s); }
  }
  ~Phase() {
    if (pr) {
      cudaEvent_t b = pr->get();
      cudaEventRecord(b, s);
      pr->pending.push_back({ph, a, b});
    }
  }
};

struct emb_handle {
  Plan p;
  Prof prof;
  cudaStream_t stream = nullptr;
  float* W = nullptr;
  float* A = nullptr;
  uint8_t* codes = nullptr;
  int q8_meta_off = 0;  // byte offset of {middle, scale} inside a q8 row
  // workspace
  FeatMeta* d_meta = nullptr;
  int* stage_ids = nullptr;
  int* stage_off = nullptr;
  float* stage_dense = nullptr;
  int* off_copy = nullptr;
  uint2 *kvA = nullptr, *kvB = nullptr;  // {row key, bag} per occurrence (sort ping-pong)
  uint32_t* chunk_u0 = nullptr;
  SortWs sort{};
  uint32_t* unique = nullptr;
  uint32_t* seg = nullptr;
  uint32_t* d_U = nullptr;
  float* G = nullptr;
  double *part_first = nullptr, *part_last = nullptr, *norm_main = nullptr, *norm_fix = nullptr;
  uint32_t* owner_list = nullptr;
  uint32_t* owner_count = nullptr;
  int64_t chunks_cap = 0;
  double* S_parts = nullptr;  // [world]
  double* S_local = nullptr;
  double* S_global = nullptr;
  float* d_clip = nullptr;
  uint32_t* d_status = nullptr;
  // exchange buffers (world > 1)
  ExchangeWs xws{};
  Comm* comm = nullptr;
  // state
  bool have_fwd = false;
  bool have_q8 = false;
  int64_t fwd_nnz = 0;       // occurrences recorded (local pooling input) by the last forward
  int fwd_B = 0;             // pooling batch of the last forward (B_global for table-wise)
  int fwd_B_local = 0;
  const uint2* sorted_kv = nullptr;
  uint32_t epoch = 1;
  int64_t launches = 0;
};

namespace {

void carve(const Plan& p, Carver& cv, emb_handle* h) {
  const int64_t F = p.F, Bmax = p.max_batch, pitch = p.pitch;
  const int64_t nnz_cap = p.recv_nnz_cap;            // occurrences pooled here per step
  const int64_t bags_cap = p.world > 1 ? p.owner_bags_cap : F * Bmax;
  const int64_t dense_cap = std::max<int64_t>(Bmax * F * p.D, 1);
  const int64_t tiles = (nnz_cap + kSortTile - 1) / kSortTile + 1;
  const int64_t chunks = (nnz_cap + kChunk - 1) / kChunk + 1;
  const int64_t max_unique = std::min<int64_t>(nnz_cap, p.local_rows) + 1;
  auto* meta = cv.take<FeatMeta>(F);
  auto* stage_ids = cv.take<int>(p.max_nnz);
  auto* stage_off = cv.take<int>(F * Bmax + 1);
  auto* stage_dense = cv.take<float>(dense_cap);
  auto* off_copy = cv.take<int>(bags_cap + 1);
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
  auto* ol = cv.take<uint32_t>(3 * chunks);
  auto* oc = cv.take<uint32_t>(2);
  auto* sp = cv.take<double>(std::max(p.world, 1));
  auto* sl = cv.take<double>(1);
  auto* sg = cv.take<double>(1);
  auto* cl = cv.take<float>(1);
  auto* st = cv.take<uint32_t>(1);
  ExchangeWs x{};
  if (p.world > 1) carve_exchange(p.world, p.F, p.max_batch, p.max_nnz, nnz_cap, bags_cap, p.D, cv.base, &cv.off, &x);
  if (h) {
    h->d_meta = meta;
    h->stage_ids = stage_ids;
    h->stage_off = stage_off;
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
    h->xws = x;
  }
}

bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

bool aligned(const void* ptr, uintptr_t a) { return ((uintptr_t)ptr % a) == 0; }

#define CK(x)                                  \
  do {                                         \
    cudaError_t e_ = (x);                      \
    if (e_ != cudaSuccess) return EMB_ECUDA;   \
  } while (0)

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

extern "C" {

int32_t emb_abi_version(void) { return EMB_ABI_VERSION; }

const char* emb_status_string(emb_status s) {
  switch (s) {
    case EMB_OK: return "ok";
    case EMB_EINVAL: return "invalid argument";
    case EMB_ENOMEM: return "buffer too small";
    case EMB_ECUDA: return "CUDA error";
    case EMB_ENCCL: return "NCCL error";
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
  out->weights_bytes = std::max<int64_t>(p.local_rows * p.pitch * 4, 4);
  out->accum_bytes = std::max<int64_t>(
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

emb_status emb_create(const emb_config* cfg, const emb_buffers* buf, emb_t* out) {
  if (!cfg || !buf || !out) return EMB_EINVAL;
  *out = nullptr;
  emb_handle* h = new (std::nothrow) emb_handle();
  if (!h) return EMB_ENOMEM;
  emb_status s = make_plan(cfg, &h->p);
  if (s != EMB_OK) { delete h; return s; }
  const Plan& p = h->p;
  if (!buf->weights || !buf->accum || !buf->workspace) { delete h; return EMB_EINVAL; }
  if ((p.flags & EMB_F_Q8) && !buf->q8_codes) { delete h; return EMB_EINVAL; }
  const void* ptrs[5] = {buf->weights, buf->accum, buf->workspace, buf->q8_codes, buf->q8_meta};
  for (const void* q : ptrs)
    if (q && !aligned(q, kAlign)) { delete h; return EMB_EINVAL; }
  h->stream = (cudaStream_t)cfg->stream;
  h->W = (float*)buf->weights;
  h->A = (float*)buf->accum;
  h->codes = (uint8_t*)buf->q8_codes;
  h->q8_meta_off = (int)round_up(p.D, 8);
  Carver cv(buf->workspace);
  carve(p, cv, h);
  // device init: feature metadata, accumulators = A0, status = 0, look-back words = 0
  std::vector<FeatMeta> m = feat_meta(p);
  cudaError_t e = cudaMemcpyAsync(h->d_meta, m.data(), sizeof(FeatMeta) * m.size(),
                                  cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) {
    const int64_t na = p.mode == EMB_ADAGRAD_ROWWISE ? p.local_rows : p.local_rows * p.pitch;
    e = launch_fill(h->A, na, p.A0, h->stream);
    h->launches += na > 0;
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(h->d_status, 0, sizeof(uint32_t), h->stream);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(h->sort.status, 0, sizeof(unsigned long long) * h->sort.max_tiles * kRadixBinsMax, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // `m` goes out of scope
  if (e != cudaSuccess) { delete h; return EMB_ECUDA; }
  if (p.world > 1) {
    if (!cfg->nccl_unique_id) { delete h; return EMB_EINVAL; }
    h->comm = comm_create(cfg->nccl_unique_id, p.rank, p.world);
    if (!h->comm) { delete h; return EMB_ENCCL; }
  }
  *out = h;
  return EMB_OK;
}

emb_status emb_destroy(emb_t h) {
  if (!h) return EMB_EINVAL;
  if (h->comm) comm_destroy(h->comm);
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
  CK(cudaStreamSynchronize(h->stream));
  uint32_t st = 0;
  CK(cudaMemcpy(&st, h->d_status, sizeof(st), cudaMemcpyDeviceToHost));
  CK(cudaMemsetAsync(h->d_status, 0, sizeof(uint32_t), h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (st & kStNonFinite) return EMB_ENONFINITE;
  if (st & kStIdRange) return EMB_EIDRANGE;
  return EMB_OK;
}

// --------------------------------------------------------------------------------------
// forward
// --------------------------------------------------------------------------------------

static emb_status check_batch_args(emb_t h, const int32_t* ids, const int32_t* offsets,
                                   int32_t batch, int64_t nnz, const float* out) {
  if (!h || !offsets || !out) return EMB_EINVAL;
  if (batch < 0 || batch > h->p.max_batch) return EMB_EINVAL;
  if (nnz < 0 || nnz > h->p.max_nnz) return EMB_EINVAL;
  if (nnz > 0 && !ids) return EMB_EINVAL;
  return EMB_OK;
}

struct Staged {
  const int* ids;
  const int* offsets;
  float* out;
  bool host_out;
};

static emb_status stage_inputs(emb_t h, const int32_t* ids, const int32_t* offsets,
                               int32_t batch, int64_t nnz, float* out, Staged* s) {
  const int64_t nbags = (int64_t)h->p.F * batch;
  s->ids = ids;
  s->offsets = offsets;
  s->out = out;
  s->host_out = false;
  if (nnz > 0 && !is_device_ptr(ids)) {
    CK(cudaMemcpyAsync(h->stage_ids, ids, sizeof(int) * nnz, cudaMemcpyHostToDevice, h->stream));
    s->ids = h->stage_ids;
  }
  if (!is_device_ptr(offsets)) {
    CK(cudaMemcpyAsync(h->stage_off, offsets, sizeof(int) * (nbags + 1), cudaMemcpyHostToDevice,
                       h->stream));
    s->offsets = h->stage_off;
  }
  if (!is_device_ptr(out)) {
    s->out = h->stage_dense;
    s->host_out = true;
  } else if ((h->p.D & 3) == 0 && !aligned(out, 16)) {
    return EMB_EINVAL;
  }
  return EMB_OK;
}

emb_status emb_forward(emb_t h, const int32_t* ids, const int32_t* offsets, int32_t batch,
                       int64_t nnz, float* out) {
  emb_status s = check_batch_args(h, ids, offsets, batch, nnz, out);
  if (s != EMB_OK) return s;
  const Plan& p = h->p;
  if (p.world > 1) return exchange_forward(h, ids, offsets, batch, nnz, out, /*q8=*/false);
  Staged st;
  {
    Phase ph(h->prof, h->stream, EMB_PH_COPY);
    s = stage_inputs(h, ids, offsets, batch, nnz, out, &st);
  }
  if (s != EMB_OK) return s;
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
  {
    Phase ph(h->prof, h->stream, EMB_PH_FWD);
    CK(launch_pool_fwd_f32(a, h->stream));
  }
  h->launches += (int64_t)p.F * batch > 0;
  if (a.mean || st.host_out) {
    Phase ph(h->prof, h->stream, EMB_PH_COPY);
    if (a.mean)
      CK(cudaMemcpyAsync(h->off_copy, st.offsets, sizeof(int) * ((int64_t)p.F * batch + 1),
                         cudaMemcpyDeviceToDevice, h->stream));
    if (st.host_out)
      CK(cudaMemcpyAsync(out, st.out, sizeof(float) * (int64_t)batch * p.F * p.D,
                         cudaMemcpyDeviceToHost, h->stream));
  }
  h->have_fwd = true;
  h->fwd_nnz = nnz;
  h->fwd_B = batch;
  h->fwd_B_local = batch;
  return EMB_OK;
}

emb_status emb_forward_q8(emb_t h, const int32_t* ids, const int32_t* offsets, int32_t batch,
                          int64_t nnz, float* out) {
  emb_status s = check_batch_args(h, ids, offsets, batch, nnz, out);
  if (s != EMB_OK) return s;
  const Plan& p = h->p;
  if (!(p.flags & EMB_F_Q8) || !h->have_q8) return EMB_ESTATE;
  if (p.world > 1) return exchange_forward(h, ids, offsets, batch, nnz, out, /*q8=*/true);
  Staged st;
  {
    Phase ph(h->prof, h->stream, EMB_PH_COPY);
    s = stage_inputs(h, ids, offsets, batch, nnz, out, &st);
  }
  if (s != EMB_OK) return s;
  FwdQ8Args a;
  memset(&a, 0, sizeof(a));
  a.codes = h->codes;
  a.qpitch = p.qpitch;
  a.meta_off = h->q8_meta_off;
  a.ids = st.ids;
  a.offsets = st.offsets;
  a.B = batch;
  a.F = p.F;
  a.D = p.D;
  a.meta = h->d_meta;
  a.out = st.out;
  a.status = h->d_status;
  a.mean = p.pooling == EMB_POOL_MEAN;
  {
    Phase ph(h->prof, h->stream, EMB_PH_FWD_Q8);
    CK(launch_pool_fwd_q8(a, h->stream));
  }
  h->launches += (int64_t)p.F * batch > 0;
  if (st.host_out) {
    Phase ph(h->prof, h->stream, EMB_PH_COPY);
    CK(cudaMemcpyAsync(out, st.out, sizeof(float) * (int64_t)batch * p.F * p.D,
                       cudaMemcpyDeviceToHost, h->stream));
  }
  return EMB_OK;
}

// --------------------------------------------------------------------------------------
// backward
// --------------------------------------------------------------------------------------

// a5-a8 on this rank's recorded occurrences; grad is the pooled-gradient input in the
// layout of the recorded bags ([B][F][D] with B = fwd_B).  Used by the W=1 path and,
// after the gradient exchange, by the sharded path.
emb_status backward_local(emb_t h, const float* grad_dev, float lr, double extra,
                          const double* S_parts_dev, int nparts, bool do_allgather) {
  const Plan& p = h->p;
  const int64_t n = h->fwd_nnz;
  const uint2* kres = h->kvA;
  if (n > 0) {
    int passes = 0;
    bool in1 = false;
    {
      Phase ph(h->prof, h->stream, EMB_PH_SORT);
      CK(radix_sort_pairs(h->kvA, h->kvB, n, p.key_bits, h->sort, h->epoch, &passes,
                          &in1, &h->launches, h->stream));
    }
    h->epoch += (uint32_t)passes;
    if (in1) kres = h->kvB;
    Phase ph(h->prof, h->stream, EMB_PH_RLE);
    CK(launch_rle(kres, n, (uint32_t)p.local_rows, h->unique, h->seg, h->d_U, h->chunk_u0,
                  h->sort.counters + kMaxPasses, h->sort.status, h->epoch, h->stream));
    h->epoch += 1;
    h->launches += 1;
  } else {
    CK(cudaMemsetAsync(h->d_U, 0, sizeof(uint32_t), h->stream));
    CK(cudaMemsetAsync(h->seg, 0, sizeof(uint32_t), h->stream));
  }
  h->sorted_kv = kres;

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
  a.chunks = (n + kChunk - 1) / kChunk;
  a.S_local = h->S_local;
  a.S_global = h->S_global;
  a.clip = h->d_clip;
  a.status = h->d_status;
  a.extra_sq_norm = extra;
  a.max_norm = p.max_norm;
  a.Wt = h->W;
  a.A = h->A;
  a.rowwise = p.mode == EMB_ADAGRAD_ROWWISE;
  a.lr = lr;
  a.eps = p.eps;
  a.q8_codes = (p.flags & EMB_F_REQUANT) ? h->codes : nullptr;
  a.q8_meta_off = h->q8_meta_off;
  a.qpitch = p.qpitch;

  {
    Phase ph(h->prof, h->stream, EMB_PH_SEGREDUCE);
    CK(launch_segreduce(a, &h->launches, h->stream));
  }
  Phase ph_norm(h->prof, h->stream, EMB_PH_NORM);
  CK(launch_norm_partial(a, h->stream));
  h->launches += 1;
  const double* parts = h->S_local;
  int np = 1;
  if (do_allgather) {
    if (!comm_allgather_f64(h->comm, h->S_local, h->S_parts, h->stream)) return EMB_ENCCL;
    parts = h->S_parts;
    np = p.world;
  } else if (S_parts_dev) {
    parts = S_parts_dev;
    np = nparts;
  }
  CK(launch_norm_finalize(parts, np, a, h->stream));
  h->launches += 1;
  ph_norm.~Phase();
  new (&ph_norm) Phase(h->prof, h->stream, EMB_PH_UPDATE);
  CK(launch_adagrad(a, h->stream));
  h->launches += n > 0;
  if ((p.flags & EMB_F_REQUANT) && n > 0) h->have_q8 = true;
  return EMB_OK;
}

emb_status emb_backward_adagrad(emb_t h, const float* grad_out, float lr, double extra_sq_norm,
                                double* sq_norm_out) {
  if (!h || !grad_out) return EMB_EINVAL;
  if (!h->have_fwd) return EMB_ESTATE;
  if (!(lr >= 0.f) || !(extra_sq_norm >= 0.0)) return EMB_EINVAL;
  const Plan& p = h->p;
  emb_status s;
  if (p.world > 1) {
    s = exchange_backward(h, grad_out, lr, extra_sq_norm);
  } else {
    const float* g = grad_out;
    if (!is_device_ptr(grad_out)) {
      Phase ph(h->prof, h->stream, EMB_PH_COPY);
      CK(cudaMemcpyAsync(h->stage_dense, grad_out, sizeof(float) * (int64_t)h->fwd_B * p.F * p.D,
                         cudaMemcpyHostToDevice, h->stream));
      g = h->stage_dense;
    } else if ((p.D & 3) == 0 && !aligned(grad_out, 16)) {
      return EMB_EINVAL;
    }
    s = backward_local(h, g, lr, extra_sq_norm, nullptr, 0, false);
  }
  if (s != EMB_OK) return s;
  if (sq_norm_out) {
    CK(cudaMemcpyAsync(sq_norm_out, h->S_global, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  return EMB_OK;
}

// --------------------------------------------------------------------------------------
// quantize
// --------------------------------------------------------------------------------------

emb_status emb_quantize_mm8(emb_t h) {
  if (!h) return EMB_EINVAL;
  const Plan& p = h->p;
  if (!(p.flags & EMB_F_Q8)) return EMB_ESTATE;
  {
    Phase ph(h->prof, h->stream, EMB_PH_QUANTIZE);
    CK(launch_quantize(h->W, p.pitch, p.local_rows, p.D, h->codes, p.qpitch, h->q8_meta_off, h->d_status,
                       h->stream));
  }
  h->launches += p.local_rows > 0;
  h->have_q8 = true;
  return EMB_OK;
}

// --------------------------------------------------------------------------------------
// introspection
// --------------------------------------------------------------------------------------

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

static emb_status stored_rows(emb_t h, int32_t table, const int64_t* rows, int64_t n,
                              std::vector<int64_t>* out) {
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
static emb_status move_rows(emb_t h, void* dev, int64_t pitch_bytes, const std::vector<int64_t>& r,
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

// Rows of D floats <-> stored rows of `pitch` floats (pads stay as they are on write).
emb_status emb_read_rows(emb_t h, int32_t table, const int64_t* rows, int64_t n, float* w,
                         float* acc) {
  if (!h || (n > 0 && !w)) return EMB_EINVAL;
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
      sorted_bags[i] = (int32_t)(h->p.world > 1 ? r : (r % F) * B + r / F);
    }
  }
  return EMB_OK;
}

emb_status emb_last_stats(emb_t h, double* sq_norm, float* clip, int64_t* n_unique) {
  if (!h) return EMB_EINVAL;
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
