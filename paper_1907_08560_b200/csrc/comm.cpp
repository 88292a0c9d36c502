#include "internal.h"
namespace ghsvd {
ghsvd_status comm_init(Ctx* ctx) {
  ctx->err = "multi-GPU: not implemented yet";
  return GHSVD_E_NCCL;
}
void comm_destroy(Ctx*) {}
ghsvd_status comm_exchange(Ctx* ctx, int, int, int, const int*, const int*) {
  ctx->err = "multi-GPU: not implemented yet";
  return GHSVD_E_NCCL;
}
ghsvd_status comm_allreduce_counters(Ctx* ctx, DevCounters*) {
  ctx->err = "multi-GPU: not implemented yet";
  return GHSVD_E_NCCL;
}
}  // namespace ghsvd
