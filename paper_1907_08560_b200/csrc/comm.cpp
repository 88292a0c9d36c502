#include "internal.h"
namespace ghsvd {
ghsvd_status comm_init(Ctx* ctx) {
  ctx->err = "multi-GPU: not implemented yet";
  return GHSVD_E_NCCL;
}
void comm_destroy(Ctx*) {}
}  // namespace ghsvd
