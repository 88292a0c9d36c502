#include "internal.h"
namespace ghsvd {
size_t phase2_scratch_bytes(int64_t m, int64_t n) { return (size_t)m * 16 + 4096; }
ghsvd_status phase2_reduce(Ctx* ctx) {
  ctx->err = "reduce: not implemented yet";
  return GHSVD_E_STATE;
}
}  // namespace ghsvd
