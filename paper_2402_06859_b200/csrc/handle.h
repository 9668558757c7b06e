// handle.h -- internal: the plan, the handle, and helpers shared by api.cu and exchange.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "../../include/lirank_emb.h"
#include "comm.h"
#include "common.cuh"
#include "kernels.h"

namespace lirank {

constexpr int64_t kAlign = 256;
constexpr int kMaxWorld = 16;

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

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

// Where the rows of every table live on one rank.
struct Layout {
  std::vector<int64_t> local_base, row_lo, row_hi;  // per table (-1 base: not stored here)
  int64_t local_rows = 0;
};

struct Plan {
  int T = 0, D = 0, F = 0, pitch = 0, qpitch = 0;
  int pooling = 0, mode = 0, sharding = 0, rank = 0, world = 1;
  uint32_t flags = 0;
  float A0 = 0.f, eps = 0.f, max_norm = 0.f;
  int64_t max_nnz = 0;
  int max_batch = 0;
  std::vector<int64_t> table_rows, local_base, row_lo, row_hi;  // this rank's layout
  std::vector<int32_t> feature_table, owner;                    // owner: table-wise plan
  int64_t local_rows = 0;
  int key_bits = 0;
  // ---- sharded exchange (world > 1), identical on every rank --------------------------
  std::vector<Layout> layouts;              // [world]
  std::vector<std::vector<int>> feats_of;   // [world]: features whose table has rows there
  std::vector<int> Fo;                      // [world] = feats_of[o].size()
  std::vector<int> dest_base;               // [world+1]: prefix of Fo (units of B bags)
  std::vector<int32_t> jmap;                // [world][F]: index of f in feats_of[o] or -1
  std::vector<int64_t> key_base;            // [world][F]: local base of t(f) on o or -1
  std::vector<int32_t> owner0, blk;         // [F]: owner(id) = owner0 + id / blk
  int Fr = 0;                               // = Fo[rank]
  bool exch = false;                        // run the exchange path (world > 1, or forced)
  int64_t recv_nnz_cap = 0;                 // occurrences this rank may pool per step
  int64_t pair_cap = 0;                     // collective a1: key slot per (source, owner)
  int64_t owner_bags_cap = 0;               // bags this rank may pool per step
};

emb_status make_plan(const emb_config* c, Plan* p);

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

// Device buffers of the sharded exchange (carved from the workspace when world > 1).
struct ExchangeWs {
  uint32_t* lens = nullptr;       // [sum_o Fo * B] ids per (dest, feature, sample)
  uint32_t* pos = nullptr;        // [.. + 1] exclusive scan of lens = send positions
  uint32_t* send_keys = nullptr;  // [max_nnz] owner-local row keys, grouped by dest
  uint32_t* cnt = nullptr;        // [world] send counts, then [world][world] all counts
  uint32_t* recv_lens = nullptr;  // [world * Fr * B]
  uint32_t* recv_off = nullptr;   // [world * Fr * B + 1]
  uint32_t* recv_keys = nullptr;  // [recv_nnz_cap] received keys, compacted in source order
  uint32_t* recv_pad = nullptr;   // collective: [world][pair_cap] received key slots
  float* pooled = nullptr;        // [world][B][Fr][D]: owner partials / owner grads
  float* xdense = nullptr;        // [B][F][D]: table-wise return / grad send blocks
  FeatMeta* ident = nullptr;      // [world * Fr] identity metas for the owner's pooling
  int32_t* d_jmap = nullptr;      // [world][F]
  int32_t* d_fmap = nullptr;      // [F][3]: {dest_base(owner), Fo(owner), j} (table-wise)
  int32_t* d_feats_by_dest = nullptr;  // [F]: feats_of concatenated by dest (table-wise)
  int32_t* d_dest_base = nullptr;      // [world+1]
  int64_t* d_key_base = nullptr;       // [world][F]
  int32_t* d_owner0 = nullptr;         // [F]
  int32_t* d_blk = nullptr;            // [F]
  uint32_t* scan_counter = nullptr;    // [4] tile counters of the exchange scans
  unsigned long long* scan_status = nullptr;  // look-back words of the exchange scans
  // fused exchange (EMB_F_P2P)
  float* pslots = nullptr;        // row-wise: [2][world][B][F][D] owner partials, summed in rank order
  int64_t fdst_stride = 0;        // fused: floats between the two destination sets (fp32 / q8 forward)
  int32_t* d_fcol = nullptr;      // [Fr]: global feature of owner-local feature j
  uint8_t* p2p_scratch = nullptr; // [kPeerScratchBytes] transport scratch (barrier, mapping)
  float* peer_xdense[kMaxWorld] = {};  // table-wise: each rank's xdense (fwd destination)
  float* peer_pslots[kMaxWorld] = {};  // row-wise: each rank's pslots (fwd destination)
  float* peer_pooled[kMaxWorld] = {};  // each rank's pooled (bwd grad destination)
  uint32_t* peer_recv_keys[kMaxWorld] = {};  // each rank's recv_keys (a1 key destination)
  uint32_t* peer_recv_lens[kMaxWorld] = {};  // each rank's recv_lens
};

}  // namespace lirank

struct emb_handle {
  lirank::Plan p;
  lirank::Prof prof;
  cudaStream_t stream = nullptr;
  // a5 dedup runs on a side stream as soon as the forward has recorded the occurrences,
  // overlapping whatever the caller does before emb_backward_adagrad (the dense tower).
  cudaStream_t side = nullptr;
  cudaEvent_t ev_kv = nullptr;     // forward wrote kvA (main stream)
  cudaEvent_t ev_dedup = nullptr;  // dedup finished (side stream)
  bool dedup_pending = false;      // dedup of the last forward was launched on `side`
  float* W = nullptr;
  float* A = nullptr;
  uint8_t* codes = nullptr;
  int q8_meta_off = 0;  // byte offset of {middle, scale} inside a q8 row
  // workspace
  uint32_t* order_ws = nullptr;  // bag order of the pooling kernels (kOrderWsWords)
  const int* order_offsets = nullptr;  // offsets (device) + bag count the order was built for by
  int64_t order_bags = -1;             // the last unsharded a2 forward (a10 reuses it)
  lirank::FeatMeta* d_meta = nullptr;
  // host inputs are staged into one of two slots on the copy stream (double-buffered: the
  // next call's host-to-device copy overlaps this call's kernels on the main stream)
  int* stage_ids[2] = {nullptr, nullptr};
  int* stage_off[2] = {nullptr, nullptr};
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr};  // slot filled (copy stream)
  cudaEvent_t ev_free[2] = {nullptr, nullptr};   // slot's last reader done (main stream)
  int stage_next = 0;                            // slot the next host input goes to
  int last_slot = -1;                            // slot holding the last forward's inputs
  float* stage_dense = nullptr;
  int* off_copy = nullptr;
  uint2 *kvA = nullptr, *kvB = nullptr;  // {row key, grad row} per occurrence (sort ping-pong)
  uint32_t* chunk_u0 = nullptr;
  lirank::SortWs sort{};
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
  double* norm_parts = nullptr;
  uint32_t* norm_done = nullptr;
  double* S_global = nullptr;
  float* d_clip = nullptr;
  uint32_t* d_status = nullptr;
  // sharded exchange
  lirank::ExchangeWs x{};
  lirank::Transport* comm = nullptr;
  uint32_t* d_fwd_n = nullptr;  // sharded: occurrences the last fp32 forward pooled here
  // NEXT-3 incremental-training penalty (emb_set_incremental)
  lirank::FimArgs fim{};
  bool fim_on = false;
  // inputs of the last emb_forward (device: the caller's or the staged copy)
  const int* last_ids = nullptr;
  const int* last_off = nullptr;
  int last_B = -1;
  int64_t last_nnz = -1;
  // state
  bool have_fwd = false;
  bool have_q8 = false;
  int64_t fwd_nnz = 0;  // occurrences recorded (pooled on this rank) by the last forward;
                        // sharded: the capacity, the count itself is on the device:
  const uint32_t* fwd_n_dev = nullptr;  // (sharded) device count, read by the a5-a6 kernels
  int64_t fwd_nnz_hint = 0;  // the ids of the forward call (picks the segment-reduce chunk)
  int chunk_log2 = lirank::kChunkLog2Max;  // segment-reduce chunk of the last dedup
  int fwd_B = 0;        // local batch of the last forward
  bool x_ids_fwd = false;  // the receive buffers hold the last (fp32) forward's exchanged ids
  const uint2* sorted_kv = nullptr;
  // look-back epochs in device memory: [0] the dedup (side stream), [1] the exchange scans
  // (main stream); read by the kernels, advanced by k_epoch_advance (graph-replayable)
  uint32_t* d_epoch = nullptr;
  int64_t launches = 0;
};

namespace lirank {

bool is_device_ptr(const void* ptr);
inline bool aligned(const void* ptr, uintptr_t a) { return ((uintptr_t)ptr % a) == 0; }

#define CK(x)                                  \
  do {                                         \
    cudaError_t e_ = (x);                      \
    if (e_ != cudaSuccess) return EMB_ECUDA;   \
  } while (0)

struct Staged {
  const int* ids;
  const int* offsets;
  float* out;
  bool host_out;
  int slot;  // staging slot the inputs were copied to (-1: device inputs, nothing staged)
};
// after the kernels of a call that read staged inputs: the slot may be refilled
emb_status release_stage(emb_t h, const Staged& s);
emb_status stage_inputs(emb_t h, const int32_t* ids, const int32_t* offsets, int32_t batch,
                        int64_t nnz, float* out, Staged* s);

// a5-a8 on this rank's recorded occurrences (see api.cu).
emb_status backward_local(emb_t h, const float* grad_dev, float lr, double extra,
                          const double* extra_dev, float* clip_out);
// a5 (sort + run-length encode) of the recorded occurrences on the side stream.
emb_status launch_dedup(emb_t h);
// make the main stream wait for a pending dedup (before reusing kvA or reading its output)
emb_status join_dedup(emb_t h);

// sharded forward / backward (exchange.cu)
// reuse: a q8 forward of the last forward's batch (emb_forward_q8(NULL, NULL)): the ids
// exchange of that forward is still in the receive buffers, so a1 is skipped
emb_status exchange_forward(emb_t h, const Staged& st, int32_t batch, int64_t nnz, bool q8, bool reuse = false);
emb_status exchange_backward(emb_t h, const float* grad_dev);
void carve_exchange(const Plan& p, Carver& cv, ExchangeWs* x);
emb_status exchange_init(emb_t h);  // upload the exchange maps (emb_create)

}  // namespace lirank
