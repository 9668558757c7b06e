// comm.h -- transports of the sharded exchange (a1/a3/a4 and the norm exchange).
//
// Three implementations behind one interface:
// * NcclTransport: NCCL (torch's libnccl.so.2, dlopen'ed) over NVLink/NVSwitch, one rank
//   per GPU, communicator created from a 128-B ncclUniqueId the caller distributes.
// * LoopbackTransport: W ranks as W host threads of ONE process (test transport): every
//   collective is a host rendezvous plus cudaMemcpyAsync between the ranks' buffers,
//   ordered with CUDA events (no kernel ever waits on another rank's kernel).
// * HostTransport: one rank per PROCESS, any devices (test transport for several processes
//   on one GPU): every collective waits for the stream, moves the bytes through host memory
//   with a caller-supplied host all-gather (e.g. torch.distributed over gloo), and copies
//   them back; peer memory is mapped with CUDA IPC.  Kernels never wait on another rank.
// All calls enqueue on the caller's stream and are collective (same order on all ranks).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace lirank {

struct Transport {
  virtual ~Transport() {}
  // recv[r * bytes .. (r+1) * bytes) = send of rank r.
  virtual bool allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  // recv[0..count) = sum over ranks r of send_r[rank * count ..], fp32.
  virtual bool reduce_scatter_f32(const float* send, float* recv, size_t count, cudaStream_t s) = 0;
  // to every rank r: sbytes[r] bytes from send + soff[r]; from every rank r: rbytes[r]
  // bytes into recv + roff[r] (sizes must match pairwise; host arrays of length world).
  virtual bool alltoallv(const void* send, const size_t* soff, const size_t* sbytes, void* recv,
                         const size_t* roff, const size_t* rbytes, cudaStream_t s) = 0;
  // data[0..count) = sum over ranks of data_r (fp32; every rank gets the same values).
  virtual bool allreduce_sum_f32(float* data, size_t count, cudaStream_t s) = 0;
  // ---- fused exchange (EMB_F_P2P): peer memory ------------------------------------------
  // Collective, host-blocking.  Every rank passes n pointers into its own device buffers;
  // on success peers[i * world + r] is rank r's i-th pointer, addressable by this device's
  // kernels (own rank: the local pointer; NCCL: CUDA IPC mappings over NVLink; loopback:
  // the other handle's buffer on the same device).  Every rank returns the same verdict.
  // `scratch` is a device buffer of >= kPeerScratchBytes the transport may use meanwhile.
  virtual bool map_peers(void* const* local, int n, void** peers, void* scratch, cudaStream_t s) = 0;
  // Collective, stream-ordered: work enqueued on s after the barrier starts only once every
  // rank's stream has reached it, i.e. after every rank's earlier kernels (and their peer
  // stores) have completed.  `scratch`: device, >= kPeerScratchBytes.
  virtual bool barrier(void* scratch, cudaStream_t s) = 0;
};

constexpr size_t kPeerScratchBytes = 16384;

// NCCL: returns nullptr (and a reason) if libnccl.so.2 cannot be loaded or init fails.
Transport* make_nccl_transport(const void* unique_id, int rank, int world);
bool nccl_get_unique_id(void* out128);

// Loopback hub shared by the W in-process ranks.
void* loopback_hub_create(int world);
void loopback_hub_destroy(void* hub);
Transport* make_loopback_transport(void* hub, int rank);

// Host transport over a caller-supplied host all-gather (emb_host_comm in the header).
Transport* make_host_transport(const void* host_comm, int rank, int world);

}  // namespace lirank
