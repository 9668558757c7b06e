// comm.h -- multi-GPU exchange (a1/a3/a4) for world_size > 1.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lirank_emb.h"

namespace lirank {

struct Comm;

// Device buffers of the sharded exchange, carved from the workspace.
struct ExchangeWs {
  int64_t bytes = 0;
};

Comm* comm_create(const void* nccl_unique_id, int rank, int world);
void comm_destroy(Comm* c);
// dst[r] = src of rank r (one double per rank), enqueued on s.
bool comm_allgather_f64(Comm* c, const double* src, double* dst, cudaStream_t s);

void carve_exchange(int world, int F, int max_batch, int64_t max_nnz, int64_t nnz_cap,
                    int64_t bags_cap, int D, uint8_t* base, int64_t* off, ExchangeWs* x);

}  // namespace lirank

emb_status exchange_forward(emb_t h, const int32_t* ids, const int32_t* offsets, int32_t batch,
                            int64_t nnz, float* out, bool q8);
emb_status exchange_backward(emb_t h, const float* grad_out, float lr, double extra_sq_norm);
