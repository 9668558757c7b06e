// comm.cu -- NCCL and loopback transports for the sharded exchange (see comm.h).
#include "comm.h"

#include "../../include/lirank_emb.h"

#include <dlfcn.h>
#include <string.h>

#include <condition_variable>
#include <mutex>
#include <vector>

namespace lirank {

// ---------------------------------------------------------------------------
// NCCL (dlopen'ed: the library has no link-time NCCL dependency; inside a PyTorch process
// this binds to the already-loaded torch NCCL, 2.28.x).  Types/values of nccl.h (2.x ABI).
// ---------------------------------------------------------------------------
namespace nccl {
typedef struct { char internal[128]; } UniqueId;
typedef void* Comm;
typedef int Result;                  // ncclSuccess = 0
enum { kUint8 = 1, kFloat32 = 7 };   // ncclUint8, ncclFloat32
enum { kSum = 0 };                   // ncclSum
struct Api {
  Result (*GetUniqueId)(UniqueId*) = nullptr;
  Result (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  Result (*CommDestroy)(Comm) = nullptr;
  Result (*GroupStart)() = nullptr;
  Result (*GroupEnd)() = nullptr;
  Result (*Send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  Result (*Recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  Result (*AllGather)(const void*, void*, size_t, int, Comm, cudaStream_t) = nullptr;
  Result (*ReduceScatter)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  Result (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  bool ok = false;
};
static Api& api() {
  static Api a = [] {
    Api x;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return x;
    x.GetUniqueId = (Result(*)(UniqueId*))dlsym(lib, "ncclGetUniqueId");
    x.CommInitRank = (Result(*)(Comm*, int, UniqueId, int))dlsym(lib, "ncclCommInitRank");
    x.CommDestroy = (Result(*)(Comm))dlsym(lib, "ncclCommDestroy");
    x.GroupStart = (Result(*)())dlsym(lib, "ncclGroupStart");
    x.GroupEnd = (Result(*)())dlsym(lib, "ncclGroupEnd");
    x.Send = (Result(*)(const void*, size_t, int, int, Comm, cudaStream_t))dlsym(lib, "ncclSend");
    x.Recv = (Result(*)(void*, size_t, int, int, Comm, cudaStream_t))dlsym(lib, "ncclRecv");
    x.AllGather = (Result(*)(const void*, void*, size_t, int, Comm, cudaStream_t))dlsym(lib, "ncclAllGather");
    x.ReduceScatter =
        (Result(*)(const void*, void*, size_t, int, int, Comm, cudaStream_t))dlsym(lib, "ncclReduceScatter");
    x.AllReduce =
        (Result(*)(const void*, void*, size_t, int, int, Comm, cudaStream_t))dlsym(lib, "ncclAllReduce");
    x.ok = x.GetUniqueId && x.CommInitRank && x.CommDestroy && x.GroupStart && x.GroupEnd &&
           x.Send && x.Recv && x.AllGather && x.ReduceScatter && x.AllReduce;
    return x;
  }();
  return a;
}
}  // namespace nccl

// cuMemGetAddressRange (driver API, dlopen'ed): the base of the allocation a pointer lies
// in -- CUDA IPC handles name whole allocations (torch sub-allocates its segments).
static bool alloc_base(const void* p, void** base) {
  typedef int (*Fn)(unsigned long long*, size_t*, unsigned long long);
  static Fn fn = [] {
    void* lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    return lib ? (Fn)dlsym(lib, "cuMemGetAddressRange_v2") : (Fn) nullptr;
  }();
  unsigned long long b = 0;
  size_t sz = 0;
  if (!fn || fn(&b, &sz, (unsigned long long)(uintptr_t)p) != 0) return false;
  *base = (void*)(uintptr_t)b;
  return true;
}

struct NcclTransport : Transport {
  nccl::Comm comm = nullptr;
  int world = 1, rank = 0;
  std::vector<void*> opened;  // IPC mappings of peer allocations (closed at destroy)
  ~NcclTransport() override {
    for (void* q : opened) cudaIpcCloseMemHandle(q);
    if (comm) nccl::api().CommDestroy(comm);
  }
  bool barrier(void* scratch, cudaStream_t s) override {
    // an all-gather of one word completes on a rank only after every rank has enqueued it,
    // i.e. after every rank's stream finished the work before it (the exchange enqueues a
    // system-scope fence after its peer-storing kernels)
    uint8_t* q = (uint8_t*)scratch;
    return nccl::api().AllGather(q, q + 256, 4, nccl::kUint8, comm, s) == 0;
  }
  // all ranks agree on `ok` (logical AND over ranks)
  bool agree(bool ok, void* scratch, cudaStream_t s) {
    uint8_t* q = (uint8_t*)scratch;
    int32_t mine = ok ? 1 : 0;
    std::vector<int32_t> all(world, 0);
    if (cudaMemcpyAsync(q, &mine, 4, cudaMemcpyHostToDevice, s) != cudaSuccess) return false;
    if (nccl::api().AllGather(q, q + 256, 4, nccl::kUint8, comm, s) != 0) return false;
    if (cudaMemcpyAsync(all.data(), q + 256, 4ull * world, cudaMemcpyDeviceToHost, s) != cudaSuccess) return false;
    if (cudaStreamSynchronize(s) != cudaSuccess) return false;
    for (int32_t v : all) ok &= v == 1;
    return ok;
  }
  bool map_peers(void* const* local, int n, void** peers, void* scratch, cudaStream_t s) override {
    struct Rec { cudaIpcMemHandle_t h; int64_t off; int32_t ok, pad; };
    const size_t per = sizeof(Rec) * (size_t)n, rbase = 1024;
    if (rbase + per * world > kPeerScratchBytes) return false;  // same on every rank
    std::vector<Rec> mine(n), all((size_t)n * world);
    for (int i = 0; i < n; ++i) {
      memset(&mine[i], 0, sizeof(Rec));
      void* base = nullptr;
      mine[i].ok = alloc_base(local[i], &base) && cudaIpcGetMemHandle(&mine[i].h, base) == cudaSuccess;
      mine[i].off = (int64_t)((uint8_t*)local[i] - (uint8_t*)base);
    }
    uint8_t* q = (uint8_t*)scratch;
    bool ok = cudaMemcpyAsync(q, mine.data(), per, cudaMemcpyHostToDevice, s) == cudaSuccess &&
              nccl::api().AllGather(q, q + rbase, per, nccl::kUint8, comm, s) == 0 &&
              cudaMemcpyAsync(all.data(), q + rbase, per * world, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
              cudaStreamSynchronize(s) == cudaSuccess;
    for (size_t k = 0; ok && k < all.size(); ++k) ok &= all[k].ok == 1;
    std::vector<std::pair<cudaIpcMemHandle_t, void*>> cache;  // one mapping per peer allocation
    std::vector<void*> mapped;
    for (int r = 0; ok && r < world; ++r)
      for (int i = 0; ok && i < n; ++i) {
        if (r == rank) { peers[(size_t)i * world + r] = local[i]; continue; }
        const Rec& x = all[(size_t)r * n + i];
        void* b = nullptr;
        for (auto& c : cache)
          if (memcmp(&c.first, &x.h, sizeof(x.h)) == 0) b = c.second;
        if (!b) {
          ok = cudaIpcOpenMemHandle(&b, x.h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
          if (!ok) break;
          cache.push_back({x.h, b});
          mapped.push_back(b);
        }
        peers[(size_t)i * world + r] = (uint8_t*)b + x.off;
      }
    ok = agree(ok, scratch, s);
    if (!ok) {
      for (void* b : mapped) cudaIpcCloseMemHandle(b);
      cudaGetLastError();
      return false;
    }
    opened.insert(opened.end(), mapped.begin(), mapped.end());
    return true;
  }
  bool allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    return nccl::api().AllGather(send, recv, bytes, nccl::kUint8, comm, s) == 0;
  }
  bool reduce_scatter_f32(const float* send, float* recv, size_t count, cudaStream_t s) override {
    return nccl::api().ReduceScatter(send, recv, count, nccl::kFloat32, nccl::kSum, comm, s) == 0;
  }
  bool allreduce_sum_f32(float* data, size_t count, cudaStream_t s) override {
    return nccl::api().AllReduce(data, data, count, nccl::kFloat32, nccl::kSum, comm, s) == 0;
  }
  bool alltoallv(const void* send, const size_t* soff, const size_t* sbytes, void* recv,
                 const size_t* roff, const size_t* rbytes, cudaStream_t s) override {
    auto& a = nccl::api();
    if (a.GroupStart() != 0) return false;
    bool ok = true;
    for (int r = 0; r < world; ++r) {
      if (sbytes[r]) ok &= a.Send((const uint8_t*)send + soff[r], sbytes[r], nccl::kUint8, r, comm, s) == 0;
      if (rbytes[r]) ok &= a.Recv((uint8_t*)recv + roff[r], rbytes[r], nccl::kUint8, r, comm, s) == 0;
    }
    ok &= a.GroupEnd() == 0;
    return ok;
  }
};

bool nccl_get_unique_id(void* out128) {
  auto& a = nccl::api();
  if (!a.ok) return false;
  nccl::UniqueId id;
  if (a.GetUniqueId(&id) != 0) return false;
  memcpy(out128, &id, sizeof(id));
  return true;
}

Transport* make_nccl_transport(const void* unique_id, int rank, int world) {
  auto& a = nccl::api();
  if (!a.ok || !unique_id) return nullptr;
  nccl::UniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  auto* t = new NcclTransport();
  t->world = world;
  t->rank = rank;
  if (a.CommInitRank(&t->comm, world, id, rank) != 0) {
    t->comm = nullptr;
    delete t;
    return nullptr;
  }
  return t;
}

// ---------------------------------------------------------------------------
// Loopback: W ranks = W threads of one process on one device.
// ---------------------------------------------------------------------------
namespace {

struct Slot {
  const void* send = nullptr;
  const size_t* soff = nullptr;
  const size_t* sbytes = nullptr;
  void* const* ptrs = nullptr;  // map_peers
  cudaEvent_t ready = nullptr;
  cudaEvent_t done = nullptr;
};

struct Hub {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<Slot> slots;
  explicit Hub(int w) : world(w), slots(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const int64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

__global__ void k_add_f32(float* __restrict__ dst, const float* __restrict__ src, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __fadd_rn(dst[i], src[i]);
}

struct LoopbackTransport : Transport {
  Hub* hub;
  int rank;
  cudaEvent_t ready = nullptr, done = nullptr;
  LoopbackTransport(Hub* h, int r) : hub(h), rank(r) {
    cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
  }
  ~LoopbackTransport() override {
    cudaEventDestroy(ready);
    cudaEventDestroy(done);
    if (scratch) cudaFree(scratch);
  }
  // phase 1: publish + barrier; caller issues its reads; phase 2: done + barriers.
  void publish(const void* send, const size_t* soff, const size_t* sbytes, cudaStream_t s) {
    Slot& me = hub->slots[rank];
    me.send = send;
    me.soff = soff;
    me.sbytes = sbytes;
    cudaEventRecord(ready, s);
    me.ready = ready;
    me.done = done;
    hub->barrier();
  }
  void finish(cudaStream_t s) {
    cudaEventRecord(done, s);
    hub->barrier();
    for (int r = 0; r < hub->world; ++r)
      if (r != rank) cudaStreamWaitEvent(s, hub->slots[r].done, 0);
    hub->barrier();
  }
  bool allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    publish(send, nullptr, nullptr, s);
    bool ok = true;
    for (int r = 0; r < hub->world; ++r) {
      ok &= cudaStreamWaitEvent(s, hub->slots[r].ready, 0) == cudaSuccess;
      ok &= cudaMemcpyAsync((uint8_t*)recv + r * bytes, hub->slots[r].send, bytes,
                            cudaMemcpyDeviceToDevice, s) == cudaSuccess;
    }
    finish(s);
    return ok;
  }
  bool reduce_scatter_f32(const float* send, float* recv, size_t count, cudaStream_t s) override {
    publish(send, nullptr, nullptr, s);
    bool ok = true;
    for (int r = 0; r < hub->world; ++r) {  // rank order: deterministic sum
      ok &= cudaStreamWaitEvent(s, hub->slots[r].ready, 0) == cudaSuccess;
      const float* src = (const float*)hub->slots[r].send + (size_t)rank * count;
      if (r == 0) {
        ok &= cudaMemcpyAsync(recv, src, count * sizeof(float), cudaMemcpyDeviceToDevice, s) == cudaSuccess;
      } else if (count) {
        k_add_f32<<<148 * 4, 256, 0, s>>>(recv, src, count);
        ok &= cudaGetLastError() == cudaSuccess;
      }
    }
    finish(s);
    return ok;
  }
  float* scratch = nullptr;  // allreduce staging (grown on demand: a test transport)
  size_t scratch_floats = 0;
  bool allreduce_sum_f32(float* data, size_t count, cudaStream_t s) override {
    if (count > scratch_floats) {
      if (cudaStreamSynchronize(s) != cudaSuccess) return false;
      if (scratch) cudaFree(scratch);
      scratch = nullptr;
      scratch_floats = 0;
      if (cudaMalloc(&scratch, count * sizeof(float)) != cudaSuccess) return false;
      scratch_floats = count;
    }
    publish(data, nullptr, nullptr, s);
    bool ok = true;
    for (int r = 0; r < hub->world; ++r) {  // rank order: every rank forms the same sum
      ok &= cudaStreamWaitEvent(s, hub->slots[r].ready, 0) == cudaSuccess;
      const float* src = (const float*)hub->slots[r].send;
      if (r == 0) {
        ok &= cudaMemcpyAsync(scratch, src, count * sizeof(float), cudaMemcpyDeviceToDevice, s) == cudaSuccess;
      } else if (count) {
        k_add_f32<<<148 * 4, 256, 0, s>>>(scratch, src, count);
        ok &= cudaGetLastError() == cudaSuccess;
      }
    }
    finish(s);  // every rank has read every `data` before any overwrites its own
    ok &= cudaMemcpyAsync(data, scratch, count * sizeof(float), cudaMemcpyDeviceToDevice, s) == cudaSuccess;
    return ok;
  }
  bool alltoallv(const void* send, const size_t* soff, const size_t* sbytes, void* recv,
                 const size_t* roff, const size_t* rbytes, cudaStream_t s) override {
    publish(send, soff, sbytes, s);
    bool ok = true;
    for (int r = 0; r < hub->world; ++r) {
      const Slot& src = hub->slots[r];
      const size_t n = src.sbytes[rank];
      ok &= n == rbytes[r];
      ok &= cudaStreamWaitEvent(s, src.ready, 0) == cudaSuccess;
      if (n)
        ok &= cudaMemcpyAsync((uint8_t*)recv + roff[r], (const uint8_t*)src.send + src.soff[rank], n,
                              cudaMemcpyDeviceToDevice, s) == cudaSuccess;
    }
    finish(s);
    return ok;
  }
  bool map_peers(void* const* local, int n, void** peers, void*, cudaStream_t) override {
    hub->slots[rank].ptrs = local;
    hub->barrier();
    for (int r = 0; r < hub->world; ++r)
      for (int i = 0; i < n; ++i) peers[(size_t)i * hub->world + r] = hub->slots[r].ptrs[i];
    hub->barrier();  // the slots' pointer arrays may go out of scope after this
    return true;
  }
  bool barrier(void*, cudaStream_t s) override {
    publish(nullptr, nullptr, nullptr, s);
    finish(s);
    return true;
  }
};

}  // namespace

void* loopback_hub_create(int world) { return world >= 1 ? new Hub(world) : nullptr; }
void loopback_hub_destroy(void* hub) { delete (Hub*)hub; }
Transport* make_loopback_transport(void* hub, int rank) {
  if (!hub) return nullptr;
  return new LoopbackTransport((Hub*)hub, rank);
}

// ---------------------------------------------------------------------------
// Host transport: one rank per process (any device, e.g. several processes sharing one
// GPU in a test); the bytes of every collective go device -> host -> caller's host
// all-gather -> host -> device, after the stream has drained.  Synchronous by design (a
// test transport: the point is to run the sharded protocol, the CUDA IPC peer mappings and
// the fused-exchange fences across real process boundaries without any kernel waiting on
// another rank's kernel -- which two processes time-sliced on one GPU cannot guarantee).
// ---------------------------------------------------------------------------
namespace {

struct HostTransport : Transport {
  // every copy is enqueued on the caller's stream and waited for: a plain cudaMemcpy runs on
  // the legacy stream (which non-blocking streams do not order against) and, host to device
  // from pageable memory, may return before its DMA has landed
  static bool copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind k, cudaStream_t s) {
    return !bytes || (cudaMemcpyAsync(dst, src, bytes, k, s) == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess);
  }
  emb_host_comm hc;
  int world = 1, rank = 0;
  std::vector<void*> opened;
  float* tmp = nullptr;  // device staging for the reductions ([world][count] floats)
  size_t tmp_floats = 0;
  ~HostTransport() override {
    for (void* q : opened) cudaIpcCloseMemHandle(q);
    if (tmp) cudaFree(tmp);
  }
  bool gather(const void* mine, void* all, size_t bytes) {
    return hc.allgather(hc.ctx, mine, all, (int64_t)bytes) == 0;
  }
  bool dev_tmp(size_t floats) {
    if (floats <= tmp_floats) return true;
    if (tmp) cudaFree(tmp);
    tmp = nullptr;
    tmp_floats = 0;
    if (cudaMalloc(&tmp, floats * sizeof(float)) != cudaSuccess) return false;
    tmp_floats = floats;
    return true;
  }
  bool allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    std::vector<uint8_t> h(bytes), all(bytes * world);
    if (cudaStreamSynchronize(s) != cudaSuccess) return false;
    if (!copy(h.data(), send, bytes, cudaMemcpyDeviceToHost, s)) return false;
    if (!gather(h.data(), all.data(), bytes)) return false;
    return !bytes || cudaMemcpyAsync(recv, all.data(), bytes * world, cudaMemcpyHostToDevice, s) == cudaSuccess &&
                         cudaStreamSynchronize(s) == cudaSuccess;
  }
  // reduce W device vectors (host-gathered, [world][count] in tmp) in rank order into dst
  bool sum_ranks(float* dst, size_t count, cudaStream_t s) {
    if (cudaMemcpyAsync(dst, tmp, count * sizeof(float), cudaMemcpyDeviceToDevice, s) != cudaSuccess) return false;
    for (int r = 1; r < world && count; ++r) {
      k_add_f32<<<148 * 4, 256, 0, s>>>(dst, tmp + (size_t)r * count, count);
      if (cudaGetLastError() != cudaSuccess) return false;
    }
    return cudaStreamSynchronize(s) == cudaSuccess;
  }
  bool reduce_scatter_f32(const float* send, float* recv, size_t count, cudaStream_t s) override {
    const size_t n = count * world;
    std::vector<float> h(n), all(n * world), mine(n);
    if (cudaStreamSynchronize(s) != cudaSuccess) return false;
    if (!copy(h.data(), send, n * 4, cudaMemcpyDeviceToHost, s)) return false;
    if (!gather(h.data(), all.data(), n * 4)) return false;
    for (int r = 0; r < world; ++r)  // rank r's slice for this rank
      memcpy(mine.data() + (size_t)r * count, all.data() + (size_t)r * n + (size_t)rank * count, count * 4);
    if (!dev_tmp(n)) return false;
    if (!copy(tmp, mine.data(), n * 4, cudaMemcpyHostToDevice, s)) return false;
    return sum_ranks(recv, count, s);
  }
  bool allreduce_sum_f32(float* data, size_t count, cudaStream_t s) override {
    std::vector<float> h(count), all(count * world);
    if (cudaStreamSynchronize(s) != cudaSuccess) return false;
    if (!copy(h.data(), data, count * 4, cudaMemcpyDeviceToHost, s)) return false;
    if (!gather(h.data(), all.data(), count * 4)) return false;
    if (!dev_tmp(count * world)) return false;
    if (!copy(tmp, all.data(), count * world * 4, cudaMemcpyHostToDevice, s)) return false;
    return sum_ranks(data, count, s);
  }
  bool alltoallv(const void* send, const size_t* soff, const size_t* sbytes, void* recv,
                 const size_t* roff, const size_t* rbytes, cudaStream_t s) override {
    // every rank publishes [world sizes][its payloads for ranks 0..W-1], padded to the
    // largest rank's size (one all-gather of the sizes first)
    if (cudaStreamSynchronize(s) != cudaSuccess) return false;
    int64_t tot = 0;
    for (int r = 0; r < world; ++r) tot += (int64_t)sbytes[r];
    std::vector<int64_t> tots(world);
    if (!gather(&tot, tots.data(), sizeof(int64_t))) return false;
    int64_t mx = 0;
    for (int64_t t : tots) mx = t > mx ? t : mx;
    const size_t hdr = sizeof(int64_t) * world, per = hdr + (size_t)mx;
    std::vector<uint8_t> mine(per, 0), all(per * world);
    int64_t at = 0;
    for (int r = 0; r < world; ++r) {
      const int64_t b = (int64_t)sbytes[r];
      memcpy(mine.data() + sizeof(int64_t) * r, &b, sizeof(b));
      if (!copy(mine.data() + hdr + at, (const uint8_t*)send + soff[r], b, cudaMemcpyDeviceToHost, s)) return false;
      at += b;
    }
    if (!gather(mine.data(), all.data(), per)) return false;
    for (int src = 0; src < world; ++src) {
      const uint8_t* blk = all.data() + per * src;
      int64_t off = 0, b = 0;
      for (int r = 0; r <= rank; ++r) {
        memcpy(&b, blk + sizeof(int64_t) * r, sizeof(b));
        if (r < rank) off += b;
      }
      if ((size_t)b != rbytes[src]) return false;
      if ((size_t)b && !copy((uint8_t*)recv + roff[src], blk + hdr + off, b, cudaMemcpyHostToDevice, s)) return false;
    }
    return true;
  }
  bool barrier(void*, cudaStream_t s) override {
    if (cudaStreamSynchronize(s) != cudaSuccess) return false;
    uint8_t one = 1;
    std::vector<uint8_t> all(world);
    return gather(&one, all.data(), 1);
  }
  bool map_peers(void* const* local, int n, void** peers, void*, cudaStream_t s) override {
    struct Rec { cudaIpcMemHandle_t h; int64_t off; int32_t ok, pad; };
    if (cudaStreamSynchronize(s) != cudaSuccess) return false;
    std::vector<Rec> mine(n), all((size_t)n * world);
    for (int i = 0; i < n; ++i) {
      memset(&mine[i], 0, sizeof(Rec));
      void* base = nullptr;
      mine[i].ok = alloc_base(local[i], &base) && cudaIpcGetMemHandle(&mine[i].h, base) == cudaSuccess;
      mine[i].off = (int64_t)((uint8_t*)local[i] - (uint8_t*)base);
    }
    bool ok = gather(mine.data(), all.data(), sizeof(Rec) * n);
    for (size_t k = 0; ok && k < all.size(); ++k) ok &= all[k].ok == 1;
    std::vector<std::pair<cudaIpcMemHandle_t, void*>> cache;
    std::vector<void*> mapped;
    for (int r = 0; ok && r < world; ++r)
      for (int i = 0; ok && i < n; ++i) {
        if (r == rank) { peers[(size_t)i * world + r] = local[i]; continue; }
        const Rec& x = all[(size_t)r * n + i];
        void* b = nullptr;
        for (auto& c : cache)
          if (memcmp(&c.first, &x.h, sizeof(x.h)) == 0) b = c.second;
        if (!b) {
          ok = cudaIpcOpenMemHandle(&b, x.h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
          if (!ok) break;
          cache.push_back({x.h, b});
          mapped.push_back(b);
        }
        peers[(size_t)i * world + r] = (uint8_t*)b + x.off;
      }
    int32_t me = ok ? 1 : 0;  // agree on the verdict
    std::vector<int32_t> v(world, 0);
    if (!gather(&me, v.data(), sizeof(me))) ok = false;
    for (int32_t q : v) ok &= q == 1;
    if (!ok) {
      for (void* b : mapped) cudaIpcCloseMemHandle(b);
      cudaGetLastError();
      return false;
    }
    opened.insert(opened.end(), mapped.begin(), mapped.end());
    return true;
  }
};

}  // namespace

Transport* make_host_transport(const void* host_comm, int rank, int world) {
  if (!host_comm) return nullptr;
  const emb_host_comm* hc = (const emb_host_comm*)host_comm;
  if (!hc->allgather) return nullptr;
  auto* t = new HostTransport();
  t->hc = *hc;
  t->rank = rank;
  t->world = world;
  return t;
}

}  // namespace lirank
