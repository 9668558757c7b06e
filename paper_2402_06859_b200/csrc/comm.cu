// comm.cu -- multi-GPU exchange.  Round-1 state: the sharded path is not built yet;
// world_size > 1 handles are refused at emb_create (EMB_ENCCL) and the exchange entry
// points return EMB_EINVAL.
#include "comm.h"

namespace lirank {

struct Comm {
  int rank = 0, world = 1;
};

Comm* comm_create(const void*, int, int) { return nullptr; }
void comm_destroy(Comm* c) { delete c; }
bool comm_allgather_f64(Comm*, const double*, double*, cudaStream_t) { return false; }
void carve_exchange(int, int, int, int64_t, int64_t, int64_t, int, uint8_t*, int64_t*,
                    ExchangeWs* x) {
  x->bytes = 0;
}

}  // namespace lirank

emb_status exchange_forward(emb_t, const int32_t*, const int32_t*, int32_t, int64_t, float*,
                            bool) {
  return EMB_EINVAL;
}
emb_status exchange_backward(emb_t, const float*, float, double) { return EMB_EINVAL; }
