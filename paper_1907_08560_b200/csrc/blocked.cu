#include "internal.h"
namespace ghsvd {
size_t blk_scratch_bytes(const ghsvd_options*, int64_t, int64_t) { return 0; }
ghsvd_status blk_sweep(Ctx* ctx, ghsvd_stats*) {
  ctx->err = "blocked: not implemented yet";
  return GHSVD_E_STATE;
}
}  // namespace ghsvd
