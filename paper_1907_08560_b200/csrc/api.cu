// api.cu -- the C ABI of include/ghsvd.h: workspace layout, state machine,
// argument checking, host<->device staging and the sweep driver (a5).
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <new>
#include <string>

#include "internal.h"

using namespace ghsvd;

struct ghsvd_ctx_s {
  Ctx c;
};

#define CTX_CUDA(call)                                                            \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);              \
      return GHSVD_E_CUDA;                                                        \
    }                                                                             \
  } while (0)

#define TRY(x)                     \
  do {                             \
    ghsvd_status s_ = (x);         \
    if (s_ != GHSVD_OK) return s_; \
  } while (0)

static const size_t ALIGN = 256;
static size_t al(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

namespace ghsvd {
// defined in comm.cpp
ghsvd_status comm_init(Ctx* ctx);
void comm_destroy(Ctx* ctx);
}  // namespace ghsvd

static Layout make_layout(const ghsvd_options* o, int64_t m, int64_t n, int64_t nl) {
  Layout L;
  const int64_t ldm = round_up(m + 1, 16), ncol = n + 1, ldn = round_up(n + 1, 16);
  const size_t fg = al((size_t)ldm * ncol * 16);
  const size_t z = al((size_t)ldn * ncol * 16);
  const bool blocked = o->variant == GHSVD_BLOCKED_BO || o->variant == GHSVD_BLOCKED_FB;
  size_t off = 0;
  L.off_F = off; off += fg;
  L.off_G = off; off += fg;
  L.off_Z = off; off += z;
  L.off_Z2 = off; off += z;
  if (o->want_x) {
    L.off_W = off; off += z;
    L.off_X = off; off += z;
  } else {
    L.off_W = L.off_X = (size_t)-1;
  }
  // no shadow copies of F, G: the blocked updates are in place
  L.off_F2 = L.off_G2 = (size_t)-1;
  size_t scr = phase2_scratch_bytes(m, n);
  if (nl > 0) scr = std::max(scr, phase1_scratch_bytes(m, n, nl));
  if (blocked) scr = std::max(scr, blk_scratch_bytes(o, m, n));
  L.scr_bytes = al(scr);
  L.off_scr = off; off += L.scr_bytes;
  L.off_misc = off;
  off += al(sizeof(DevCounters)) + al((size_t)ldm) + al((size_t)ldm * 4) + al((size_t)ncol * 8) +
         3 * al((size_t)ncol * 8) + al(64);
  L.total = off;
  return L;
}

extern "C" {

const char* ghsvd_version(void) { return "ghsvd-b200 0.1 (sm_100a)"; }

void ghsvd_default_options(ghsvd_options* o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->device = 0;
  o->stream = nullptr;
  o->world_size = 1;
  o->rank = 0;
  o->nccl_id = nullptr;
  o->variant = GHSVD_POINTWISE;
  o->ordering = GHSVD_ORDER_ROUND_ROBIN;
  o->nblocks = 0;
  o->max_sweeps = 30;
  o->criterion = GHSVD_CRIT_RELATIVE;
  o->eps = 0.0;
  o->cluster = 0;
  o->threads = 0;
  o->use_graph = 1;
  o->kernel = 0;
  o->detail_timing = 0;
  o->want_x = 0;
  o->exchange_overlap = 0;
  // experiment knobs of the tools: seeded from the environment HERE only (the library
  // reads nothing else from the environment)
  auto env = [](const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
  };
  o->schedule = (env("GHSVD_SERIAL", 0) ? GHSVD_SCHED_SERIAL : 0) | (env("GHSVD_PRIO", 1) ? 0 : GHSVD_SCHED_NO_PRIO) |
                (env("GHSVD_SPLIT_BND", 0) ? GHSVD_SCHED_SPLIT_BND : 0) |
                (env("GHSVD_GRAM3M", 1) ? 0 : GHSVD_SCHED_GRAM4M) | (env("GHSVD_UPD4M", 0) ? GHSVD_SCHED_UPD4M : 0) |
                (env("GHSVD_PIVOT_CL", 0) ? GHSVD_SCHED_PIVOT_CL : 0) |
                (env("GHSVD_SPLIT_FACTOR", 0) ? GHSVD_SCHED_SPLIT_FACTOR : 0);
  o->groups = env("GHSVD_GROUPS", 0);
  o->gram_splits = env("GHSVD_NSPLIT", 0);
  const char* tp = getenv("GHSVD_TRACE");
  o->trace_path = tp && *tp ? tp : nullptr;
}

static bool opts_ok(const ghsvd_options* o) {
  if (!o) return false;
  if (o->world_size < 1 || o->rank < 0 || o->rank >= o->world_size) return false;
  if (o->variant < 0 || o->variant > 2) return false;
  if (o->ordering < GHSVD_ORDER_ROUND_ROBIN || o->ordering > GHSVD_ORDER_HIER) return false;
  if (o->ordering != GHSVD_ORDER_ROUND_ROBIN && o->variant == GHSVD_POINTWISE) return false;
  if (o->super_blocks < 0 || (o->super_blocks & 1)) return false;
  if (o->max_sweeps < 1 || o->max_sweeps > 64) return false;
  if (o->criterion != 0 && o->criterion != 1) return false;
  if (o->nblocks < 0 || (o->nblocks & 1)) return false;
  if (o->world_size > 1 && o->nccl_id == nullptr) return false;
  if (o->world_size > 1 && o->variant == GHSVD_POINTWISE) return false;
  if (o->exchange_overlap < 0 || o->exchange_overlap > 1 || o->schedule < 0 || o->schedule > 127 || o->groups < 0 ||
      o->gram_splits < 0)
    return false;
  return true;
}

size_t ghsvd_workspace_bytes(const ghsvd_options* opts, int64_t m, int64_t n, int64_t nl) {
  if (!opts_ok(opts) || m < 1 || n < 1 || m < n || nl < 0) return 0;
  return make_layout(opts, m, n, nl).total;
}

ghsvd_status ghsvd_create(const ghsvd_options* opts, int64_t m, int64_t n, int64_t nl, void* workspace,
                          size_t bytes, ghsvd_ctx* out) {
  if (!out) return GHSVD_E_INVALID_ARG;
  *out = nullptr;
  if (!opts_ok(opts) || m < 1 || n < 1 || m < n || nl < 0 || !workspace) return GHSVD_E_INVALID_ARG;
  Layout L = make_layout(opts, m, n, nl);
  if (bytes < L.total) return GHSVD_E_WORKSPACE;
  ghsvd_ctx h = new (std::nothrow) ghsvd_ctx_s();
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  ctx->o = *opts;
  if (ctx->o.eps <= 0) ctx->o.eps = 0x1p-53;
  ctx->trace_path = opts->trace_path ? opts->trace_path : "";
  ctx->o.trace_path = ctx->trace_path.empty() ? nullptr : ctx->trace_path.c_str();
  ctx->stream = (cudaStream_t)opts->stream;
  ctx->ws = (char*)workspace;
  ctx->ws_bytes = bytes;
  ctx->L = L;
  ctx->m_cap = m;
  ctx->n_cap = n;
  ctx->nl_cap = nl;
  ctx->ldm = round_up(m + 1, 16);
  ctx->ldn = round_up(n + 1, 16);
  ctx->state = 0;
  ctx->F = (double2*)(ctx->ws + L.off_F);
  ctx->G = (double2*)(ctx->ws + L.off_G);
  ctx->Z = (double2*)(ctx->ws + L.off_Z);
  ctx->Z2 = (double2*)(ctx->ws + L.off_Z2);
  ctx->F2 = L.off_F2 == (size_t)-1 ? nullptr : (double2*)(ctx->ws + L.off_F2);
  ctx->G2 = L.off_G2 == (size_t)-1 ? nullptr : (double2*)(ctx->ws + L.off_G2);
  ctx->W = L.off_W == (size_t)-1 ? nullptr : (double2*)(ctx->ws + L.off_W);
  ctx->Xo = L.off_X == (size_t)-1 ? nullptr : (double2*)(ctx->ws + L.off_X);
  ctx->scr = ctx->ws + L.off_scr;
  char* p = ctx->ws + L.off_misc;
  ctx->cnt = (DevCounters*)p; p += al(sizeof(DevCounters));
  ctx->J = (int8_t*)p; p += al((size_t)ctx->ldm);
  ctx->rowdest = (int*)p; p += al((size_t)ctx->ldm * 4);
  ctx->p2 = (int64_t*)p; p += al((size_t)(n + 1) * 8);
  ctx->lam = (double*)p; p += al((size_t)(n + 1) * 8);
  ctx->sf = (double*)p; p += al((size_t)(n + 1) * 8);
  ctx->sg = (double*)p; p += al((size_t)(n + 1) * 8);
  ctx->graph = nullptr;
  ctx->comm = nullptr;
  cudaError_t e = cudaSetDevice(opts->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev2);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev3);
  if (e != cudaSuccess) {
    delete h;
    return GHSVD_E_CUDA;
  }
  // a communicator is built whenever an id is given (also for world_size == 1, which
  // runs the NCCL code path with a single rank)
  if (opts->world_size > 1 || (opts->nccl_id && opts->variant != GHSVD_POINTWISE)) {
    ghsvd_status s = comm_init(ctx);
    if (s != GHSVD_OK) {
      delete h;
      return s;
    }
  }
  *out = h;
  return GHSVD_OK;
}

const char* ghsvd_last_error(ghsvd_ctx h) { return h ? h->c.err.c_str() : "null context"; }

void ghsvd_destroy(ghsvd_ctx h) {
  if (!h) return;
  Ctx* ctx = &h->c;
  cudaSetDevice(ctx->o.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
  if (ctx->aux_stream2) cudaStreamDestroy(ctx->aux_stream2);
  for (cudaStream_t g : ctx->grp_streams) cudaStreamDestroy(g);
  for (cudaStream_t h : ctx->hi_stream)
    if (h) cudaStreamDestroy(h);
  for (cudaStream_t h : ctx->mid_stream)
    if (h) cudaStreamDestroy(h);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->ev2) cudaEventDestroy(ctx->ev2);
  if (ctx->ev3) cudaEventDestroy(ctx->ev3);
  comm_destroy(ctx);
  phase2_release(ctx);
  delete h;
}

// Zero F, G (all columns incl. the border column) before a new problem.
static ghsvd_status clear_factors(Ctx* ctx) {
  const size_t fg = (size_t)ctx->ldm * (ctx->n_cap + 1) * 16;
  CTX_CUDA(cudaMemsetAsync(ctx->F, 0, fg, ctx->stream));
  CTX_CUDA(cudaMemsetAsync(ctx->G, 0, fg, ctx->stream));
  return GHSVD_OK;
}

static void reset_problem(Ctx* ctx) {
  ctx->state = 0;
  ctx->bordered = false;
  ctx->z_init = false;
  ctx->have_p2 = false;
}

ghsvd_status ghsvd_set_factors(ghsvd_ctx h, int64_t m, int64_t n, const void* F, int64_t ldf, const int8_t* J,
                               const void* G, int64_t ldg) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  reset_problem(ctx);
  if (!F || !G || !J || m < 1 || n < 1 || m < n || ldf < m || ldg < m || m > ctx->m_cap || n > ctx->n_cap) {
    ctx->err = "set_factors: bad arguments (need m >= n >= 1, ld >= m, within the context's capacity)";
    return GHSVD_E_INVALID_ARG;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(clear_factors(ctx));
  // J -> device scratch, stable sort destinations (+ first)
  int8_t* Jin = (int8_t*)ctx->scr;
  int64_t* npos_dev = (int64_t*)(ctx->scr + al((size_t)m));
  CTX_CUDA(cudaMemcpyAsync(Jin, J, (size_t)m, cudaMemcpyDefault, ctx->stream));
  TRY(launch_sort_dest(ctx, Jin, m, false, ctx->rowdest, ctx->J, npos_dev));
  long long npos = 0;
  CTX_CUDA(cudaMemcpyAsync(&npos, npos_dev, 8, cudaMemcpyDeviceToHost, ctx->stream));
  // F -> G buffer (unsorted), then scatter rows into F; then G -> G buffer.
  CTX_CUDA(cudaMemcpy2DAsync(ctx->G, (size_t)ctx->ldm * 16, F, (size_t)ldf * 16, (size_t)m * 16, (size_t)n,
                             cudaMemcpyDefault, ctx->stream));
  TRY(launch_row_scatter(ctx, ctx->G, ctx->ldm, ctx->F, ctx->ldm, ctx->rowdest, m, n));
  CTX_CUDA(cudaMemcpy2DAsync(ctx->G, (size_t)ctx->ldm * 16, G, (size_t)ldg * 16, (size_t)m * 16, (size_t)n,
                             cudaMemcpyDefault, ctx->stream));
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  if (npos < 0) {
    ctx->err = "set_factors: J entries must be +1 or -1";
    return GHSVD_E_INVALID_ARG;
  }
  ctx->m = ctx->m_user = m;
  ctx->n = ctx->n_user = n;
  ctx->npos = npos;
  ctx->state = 1;
  return GHSVD_OK;
}

ghsvd_status ghsvd_factor(ghsvd_ctx h, int64_t NA, int64_t NL, int64_t NG, const void* A, const void* B,
                          const double* U, const void* TAA, const void* TAB, const void* TBB) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  reset_problem(ctx);
  const int64_t m = 2 * NA * NL;
  if (!A || !B || !U || !TAA || !TAB || !TBB || NA < 1 || NL < 1 || NG < 1 || m < NG || m > ctx->m_cap ||
      NG > ctx->n_cap || NL > ctx->nl_cap) {
    ctx->err = "factor: bad arguments (need 2*NA*NL >= NG, within capacity, NL <= nl of ghsvd_create)";
    return GHSVD_E_INVALID_ARG;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(clear_factors(ctx));
  TRY(phase1_factor(ctx, NA, NL, NG, A, B, U, TAA, TAB, TBB));
  ctx->m = ctx->m_user = m;
  ctx->n = ctx->n_user = NG;
  ctx->state = 1;
  return GHSVD_OK;
}

int64_t ghsvd_reduce_fallback_col(ghsvd_ctx h) { return h ? h->c.p2_fallback_col : -1; }

ghsvd_status ghsvd_reduce(ghsvd_ctx h, int flags) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  if (ctx->state != 1 || ctx->have_p2) {
    ctx->err = "reduce: must follow factor/set_factors (once) and precede sweep";
    return GHSVD_E_STATE;
  }
  if ((flags & ~(GHSVD_REDUCE_COLPIV | GHSVD_REDUCE_UNBLOCKED | GHSVD_REDUCE_BLOCKED | GHSVD_REDUCE_COLSEARCH |
                 GHSVD_REDUCE_OWN_QR)) ||
      ((flags & GHSVD_REDUCE_UNBLOCKED) && (flags & GHSVD_REDUCE_BLOCKED))) {
    ctx->err = "reduce: unknown flags";
    return GHSVD_E_INVALID_ARG;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  // a get_factors before reduce may have bordered the factors and set Z' = I: reduce works
  // on the unbordered m_user x n_user factors, zeroes both buffers, and bordering / Z' are
  // redone by the next prepare()
  ctx->m = ctx->m_user;
  ctx->n = ctx->n_user;
  ctx->p2_fallback_col = -2;   // no planned JQR (yet)
  ctx->p2_fallback_qr = -1;
  TRY(phase2_reduce(ctx, flags));
  ctx->have_p2 = true;
  ctx->bordered = false;
  ctx->z_init = false;
  return GHSVD_OK;
}

// Bordering (Sec 6.3.2, reading C-10) and Z' = I before the first sweep.
static ghsvd_status prepare(Ctx* ctx) {
  if (ctx->z_init) return GHSVD_OK;
  if (!ctx->have_p2) {
    // identity P2 so extract can treat both cases alike
  }
  if (ctx->n_user & 1) {
    const int64_t m = ctx->m_user, n = ctx->n_user;
    // zero row m (all n+1 columns) and column n, then F[m,n] = G[m,n] = 1, J[m] = -1
    // (the border row goes last so the +/- sorted form is kept; its sign does not
    // interact with any other column, C-10).
    CTX_CUDA(cudaMemset2DAsync(ctx->F + m, (size_t)ctx->ldm * 16, 0, 16, (size_t)(n + 1), ctx->stream));
    CTX_CUDA(cudaMemset2DAsync(ctx->G + m, (size_t)ctx->ldm * 16, 0, 16, (size_t)(n + 1), ctx->stream));
    CTX_CUDA(cudaMemsetAsync(ctx->F + n * ctx->ldm, 0, (size_t)ctx->ldm * 16, ctx->stream));
    CTX_CUDA(cudaMemsetAsync(ctx->G + n * ctx->ldm, 0, (size_t)ctx->ldm * 16, ctx->stream));
    static const double2 one = {1.0, 0.0};
    static const int8_t minus1 = -1;
    CTX_CUDA(cudaMemcpyAsync(ctx->F + n * ctx->ldm + m, &one, 16, cudaMemcpyHostToDevice, ctx->stream));
    CTX_CUDA(cudaMemcpyAsync(ctx->G + n * ctx->ldm + m, &one, 16, cudaMemcpyHostToDevice, ctx->stream));
    CTX_CUDA(cudaMemcpyAsync(ctx->J + m, &minus1, 1, cudaMemcpyHostToDevice, ctx->stream));
    ctx->m = m + 1;
    ctx->n = n + 1;
    ctx->bordered = true;
  } else {
    ctx->m = ctx->m_user;
    ctx->n = ctx->n_user;
  }
  TRY(launch_set_identity(ctx, ctx->Z, ctx->ldn, ctx->n));
  if (ctx->W) TRY(launch_set_identity(ctx, ctx->W, ctx->ldn, ctx->n));
  TRY(pw_configure(ctx));
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->z_init = true;
  return GHSVD_OK;
}

ghsvd_status ghsvd_get_factors(ghsvd_ctx h, int64_t* m, int64_t* n, void* F, int64_t ldf, int8_t* J, void* G,
                               int64_t ldg, int64_t* p2) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  // a size-only query (all buffers NULL) is also allowed after a sweep
  const bool size_only = !F && !J && !G && !p2;
  if (ctx->state != 1 && !(size_only && ctx->state == 2)) {
    ctx->err = "get_factors: must follow factor/set_factors/reduce and precede sweep";
    return GHSVD_E_STATE;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(prepare(ctx));
  if (m) *m = ctx->m;
  if (n) *n = ctx->n;
  if ((F && ldf < ctx->m) || (G && ldg < ctx->m)) {
    ctx->err = "get_factors: ld too small";
    return GHSVD_E_INVALID_ARG;
  }
  if (F)
    CTX_CUDA(cudaMemcpy2DAsync(F, (size_t)ldf * 16, ctx->F, (size_t)ctx->ldm * 16, (size_t)ctx->m * 16,
                               (size_t)ctx->n, cudaMemcpyDefault, ctx->stream));
  if (G)
    CTX_CUDA(cudaMemcpy2DAsync(G, (size_t)ldg * 16, ctx->G, (size_t)ctx->ldm * 16, (size_t)ctx->m * 16,
                               (size_t)ctx->n, cudaMemcpyDefault, ctx->stream));
  if (J) CTX_CUDA(cudaMemcpyAsync(J, ctx->J, (size_t)ctx->m, cudaMemcpyDefault, ctx->stream));
  if (p2) {
    if (ctx->have_p2) {
      CTX_CUDA(cudaMemcpyAsync(p2, ctx->p2, (size_t)ctx->n_user * 8, cudaMemcpyDefault, ctx->stream));
    } else {
      CTX_CUDA(cudaStreamSynchronize(ctx->stream));
      int64_t* tmp = new int64_t[ctx->n_user];
      for (int64_t i = 0; i < ctx->n_user; i++) tmp[i] = i;
      cudaError_t e = cudaMemcpy(p2, tmp, (size_t)ctx->n_user * 8, cudaMemcpyDefault);
      delete[] tmp;
      CTX_CUDA(e);
    }
  }
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  return GHSVD_OK;
}

static ghsvd_status map_err(Ctx* ctx, int e) {
  switch (e) {
    case -6: ctx->err = "S numerically indefinite (s_pp <= 0 or |s_pq| >= 1 after prescaling)"; return GHSVD_E_INDEFINITE_S;
    case -7: ctx->err = "rank-deficient block pivot"; return GHSVD_E_RANK_DEFICIENT;
    case -8: ctx->err = "non-finite value in a Gram or transformation"; return GHSVD_E_NONFINITE;
    default: ctx->err = "device error " + std::to_string(e); return GHSVD_E_CUDA;
  }
}

ghsvd_status ghsvd_run_steps(ghsvd_ctx h, int64_t s0, int64_t ns, uint64_t* all, uint64_t* big) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  if (ctx->state < 1) {
    ctx->err = "run_steps: no factors";
    return GHSVD_E_STATE;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(prepare(ctx));
  const bool blocked = ctx->o.variant != GHSVD_POINTWISE;
  if (!blocked && (s0 < 0 || ns < 0 || s0 + ns > ctx->n - 1)) {
    ctx->err = "run_steps: step range outside [0, n-2]";
    return GHSVD_E_INVALID_ARG;
  }
  CTX_CUDA(cudaMemsetAsync(ctx->cnt, 0, sizeof(DevCounters), ctx->stream));
  if (blocked) {
    TRY(blk_run_steps(ctx, s0, ns));  // block steps of the Level-2 round-robin
  } else {
    TRY(pw_run_steps(ctx, s0, ns));
  }
  DevCounters c;
  CTX_CUDA(cudaMemcpyAsync(&c, ctx->cnt, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  if (all) *all = c.all;
  if (big) *big = c.big;
  if (c.err) return map_err(ctx, c.err);
  ctx->state = 2;
  return GHSVD_OK;
}

ghsvd_status ghsvd_sweep(ghsvd_ctx h, ghsvd_stats* out) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  if (ctx->state != 1 && ctx->state != 2) {
    ctx->err = "sweep: must follow factor/set_factors/reduce (or a previous sweep, to resume)";
    return GHSVD_E_STATE;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(prepare(ctx));
  ghsvd_stats st;
  memset(&st, 0, sizeof(st));
  if (ctx->o.variant != GHSVD_POINTWISE) {
    TRY(blk_sweep(ctx, &st));
  } else {
    const uint64_t pairs = (uint64_t)ctx->n * (ctx->n - 1) / 2;
    const uint64_t bT = 128ull * ctx->m + 64ull * ctx->n, bS = 64ull * ctx->m;
    CTX_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    for (int sw = 0; sw < ctx->o.max_sweeps; sw++) {
      CTX_CUDA(cudaMemsetAsync(ctx->cnt, 0, sizeof(DevCounters), ctx->stream));
      CTX_CUDA(cudaEventRecord(ctx->ev2, ctx->stream));
      TRY(pw_sweep_launch(ctx));
      CTX_CUDA(cudaEventRecord(ctx->ev3, ctx->stream));
      DevCounters c;
      CTX_CUDA(cudaMemcpyAsync(&c, ctx->cnt, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
      CTX_CUDA(cudaStreamSynchronize(ctx->stream));
      if (c.err) return map_err(ctx, c.err);
      float kms = 0;
      CTX_CUDA(cudaEventElapsedTime(&kms, ctx->ev2, ctx->ev3));
      st.kernel_seconds += kms * 1e-3;
      st.launches += (uint64_t)(ctx->n - 1);
      st.alg_bytes += c.all * bT + (pairs - c.all) * bS;
      if (sw < 64) {
        st.all_per_sweep[sw] = c.all;
        st.big_per_sweep[sw] = c.big;
      }
      st.sweeps = sw + 1;
      st.pairs_visited += pairs;
      st.transforms_all += c.all;
      st.transforms_big += c.big;
      double off;
      memcpy(&off, &c.off_bits, 8);
      st.max_offdiag_last = off;
      if (c.big == 0) {
        st.converged = 1;
        break;
      }
    }
    CTX_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    CTX_CUDA(cudaEventSynchronize(ctx->ev1));
    float ms = 0;
    CTX_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    st.seconds = ms * 1e-3;
  }
  ctx->state = 2;
  if (out) *out = st;
  return st.converged ? GHSVD_OK : GHSVD_NOT_CONVERGED;
}

ghsvd_status ghsvd_extract(ghsvd_ctx h, double* lambda, double* sigma_f, double* sigma_g, void* Z, int64_t ldz,
                           int64_t* col_ids) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  if (ctx->state < 1) {
    ctx->err = "extract: no factors";
    return GHSVD_E_STATE;
  }
  if (Z && ldz < ctx->n_user) {
    ctx->err = "extract: ldz < n";
    return GHSVD_E_INVALID_ARG;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(prepare(ctx));
  TRY(launch_extract(ctx));
  if (ctx->comm && ctx->state == 2 && !ctx->blk_start.empty())
    TRY(comm_finalize_outputs(ctx, (int)ctx->blk_start.size(), ctx->blk_start.data(), ctx->blk_width.data(),
                              ctx->lam, ctx->sf, ctx->sg, ctx->Z2, ctx->ldn, ctx->o.want_x ? ctx->Xo : nullptr));
  const int64_t n = ctx->n_user;
  if (lambda) CTX_CUDA(cudaMemcpyAsync(lambda, ctx->lam, (size_t)n * 8, cudaMemcpyDefault, ctx->stream));
  if (sigma_f) CTX_CUDA(cudaMemcpyAsync(sigma_f, ctx->sf, (size_t)n * 8, cudaMemcpyDefault, ctx->stream));
  if (sigma_g) CTX_CUDA(cudaMemcpyAsync(sigma_g, ctx->sg, (size_t)n * 8, cudaMemcpyDefault, ctx->stream));
  if (Z)
    CTX_CUDA(cudaMemcpy2DAsync(Z, (size_t)ldz * 16, ctx->Z2, (size_t)ctx->ldn * 16, (size_t)n * 16, (size_t)n,
                               cudaMemcpyDefault, ctx->stream));
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  if (col_ids) {
    for (int64_t i = 0; i < n; i++) col_ids[i] = i;
  }
  return GHSVD_OK;
}

ghsvd_status ghsvd_extract_local(ghsvd_ctx h, double* lambda, double* sigma_f, double* sigma_g, void* Z,
                                 int64_t ldz, int64_t* col_ids, int64_t* ncols) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  if (ctx->state < 1) {
    ctx->err = "extract_local: no factors";
    return GHSVD_E_STATE;
  }
  if ((Z && (ldz < ctx->n_user || !col_ids)) || !ncols) {
    ctx->err = "extract_local: ldz < n, or Z without col_ids, or ncols NULL";
    return GHSVD_E_INVALID_ARG;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(prepare(ctx));
  TRY(launch_extract(ctx));
  const bool dist = ctx->comm && ctx->state == 2 && !ctx->blk_start.empty();
  if (dist)   // lambda, Sigma_F, Sigma_G combined over ranks; Z not
    TRY(comm_finalize_outputs(ctx, (int)ctx->blk_start.size(), ctx->blk_start.data(), ctx->blk_width.data(),
                              ctx->lam, ctx->sf, ctx->sg, nullptr, ctx->ldn, nullptr));
  const int64_t n = ctx->n_user;
  // the columns of this rank, in block order (one rank: all columns)
  std::vector<int64_t> cols;
  if (dist) {
    std::vector<int> blocks;
    comm_owned_blocks(ctx, (int)ctx->blk_start.size(), blocks);
    for (int b : blocks)
      for (int c = 0; c < ctx->blk_width[b]; c++)
        if (ctx->blk_start[b] + c < n) cols.push_back(ctx->blk_start[b] + c);
  } else {
    for (int64_t i = 0; i < n; i++) cols.push_back(i);
  }
  if (lambda) CTX_CUDA(cudaMemcpyAsync(lambda, ctx->lam, (size_t)n * 8, cudaMemcpyDefault, ctx->stream));
  if (sigma_f) CTX_CUDA(cudaMemcpyAsync(sigma_f, ctx->sf, (size_t)n * 8, cudaMemcpyDefault, ctx->stream));
  if (sigma_g) CTX_CUDA(cudaMemcpyAsync(sigma_g, ctx->sg, (size_t)n * 8, cudaMemcpyDefault, ctx->stream));
  if (Z) {
    // block columns are contiguous runs of columns: one 2D copy per run
    size_t j = 0;
    while (j < cols.size()) {
      size_t e = j + 1;
      while (e < cols.size() && cols[e] == cols[e - 1] + 1) e++;
      CTX_CUDA(cudaMemcpy2DAsync((double2*)Z + j * (size_t)ldz, (size_t)ldz * 16, ctx->Z2 + cols[j] * ctx->ldn,
                                 (size_t)ctx->ldn * 16, (size_t)n * 16, e - j, cudaMemcpyDefault, ctx->stream));
      j = e;
    }
  }
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  if (col_ids)
    for (size_t j = 0; j < cols.size(); j++) col_ids[j] = cols[j];
  *ncols = (int64_t)cols.size();
  return GHSVD_OK;
}

ghsvd_status ghsvd_extract_x(ghsvd_ctx h, void* X, int64_t ldx) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  if (!ctx->o.want_x || !ctx->W || ctx->state != 2) {
    ctx->err = "extract_x: needs opts.want_x and a completed sweep";
    return GHSVD_E_STATE;
  }
  if (!X || ldx < ctx->n_user) {
    ctx->err = "extract_x: bad X / ldx";
    return GHSVD_E_INVALID_ARG;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(launch_extract(ctx));
  if (ctx->comm && !ctx->blk_start.empty())
    TRY(comm_finalize_outputs(ctx, (int)ctx->blk_start.size(), ctx->blk_start.data(), ctx->blk_width.data(),
                              ctx->lam, ctx->sf, ctx->sg, ctx->Z2, ctx->ldn, ctx->Xo));
  const int64_t n = ctx->n_user;
  CTX_CUDA(cudaMemcpy2DAsync(X, (size_t)ldx * 16, ctx->Xo, (size_t)ctx->ldn * 16, (size_t)n * 16, (size_t)n,
                             cudaMemcpyDefault, ctx->stream));
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  return GHSVD_OK;
}

ghsvd_status ghsvd_get_transformed(ghsvd_ctx h, void* F, int64_t ldf, void* G, int64_t ldg, void* Zp,
                                   int64_t ldz) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  if (ctx->state < 1) return GHSVD_E_STATE;
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(prepare(ctx));
  if (F)
    CTX_CUDA(cudaMemcpy2DAsync(F, (size_t)ldf * 16, ctx->F, (size_t)ctx->ldm * 16, (size_t)ctx->m * 16,
                               (size_t)ctx->n, cudaMemcpyDefault, ctx->stream));
  if (G)
    CTX_CUDA(cudaMemcpy2DAsync(G, (size_t)ldg * 16, ctx->G, (size_t)ctx->ldm * 16, (size_t)ctx->m * 16,
                               (size_t)ctx->n, cudaMemcpyDefault, ctx->stream));
  if (Zp)
    CTX_CUDA(cudaMemcpy2DAsync(Zp, (size_t)ldz * 16, ctx->Z, (size_t)ctx->ldn * 16, (size_t)ctx->n * 16,
                               (size_t)ctx->n, cudaMemcpyDefault, ctx->stream));
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  return GHSVD_OK;
}

ghsvd_status ghsvd_get_state(ghsvd_ctx h, void* F, int64_t ldf, void* G, int64_t ldg, void* Zp, int64_t ldz,
                             void* W, int64_t ldw) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  if (ctx->state < 1) {
    ctx->err = "get_state: no factors";
    return GHSVD_E_STATE;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(prepare(ctx));   // bordered sizes m, n
  if ((F && ldf < ctx->m) || (G && ldg < ctx->m) || (Zp && ldz < ctx->n) || (W && (ldw < ctx->n || !ctx->W))) {
    ctx->err = "get_state: bad leading dimension, or W without want_x";
    return GHSVD_E_INVALID_ARG;
  }
  const size_t m = (size_t)ctx->m, n = (size_t)ctx->n;
  if (F)
    CTX_CUDA(cudaMemcpy2DAsync(F, (size_t)ldf * 16, ctx->F, (size_t)ctx->ldm * 16, m * 16, n, cudaMemcpyDefault,
                               ctx->stream));
  if (G)
    CTX_CUDA(cudaMemcpy2DAsync(G, (size_t)ldg * 16, ctx->G, (size_t)ctx->ldm * 16, m * 16, n, cudaMemcpyDefault,
                               ctx->stream));
  if (Zp)
    CTX_CUDA(cudaMemcpy2DAsync(Zp, (size_t)ldz * 16, ctx->Z, (size_t)ctx->ldn * 16, n * 16, n, cudaMemcpyDefault,
                               ctx->stream));
  if (W)
    CTX_CUDA(cudaMemcpy2DAsync(W, (size_t)ldw * 16, ctx->W, (size_t)ctx->ldn * 16, n * 16, n, cudaMemcpyDefault,
                               ctx->stream));
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  return GHSVD_OK;
}

ghsvd_status ghsvd_set_state(ghsvd_ctx h, const void* F, int64_t ldf, const void* G, int64_t ldg, const void* Zp,
                             int64_t ldz, const void* W, int64_t ldw) {
  if (!h) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  if (ctx->state < 1) {
    ctx->err = "set_state: set up the same problem first (factor / set_factors / reduce)";
    return GHSVD_E_STATE;
  }
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(prepare(ctx));   // bordering and J of the problem, as when the state was saved
  if (!F || !G || !Zp || ldf < ctx->m || ldg < ctx->m || ldz < ctx->n || (!W) != (!ctx->W) ||
      (W && ldw < ctx->n)) {
    ctx->err = "set_state: F, G, Z' required (W iff want_x); bad leading dimension";
    return GHSVD_E_INVALID_ARG;
  }
  const size_t m = (size_t)ctx->m, n = (size_t)ctx->n;
  CTX_CUDA(cudaMemcpy2DAsync(ctx->F, (size_t)ctx->ldm * 16, F, (size_t)ldf * 16, m * 16, n, cudaMemcpyDefault,
                             ctx->stream));
  CTX_CUDA(cudaMemcpy2DAsync(ctx->G, (size_t)ctx->ldm * 16, G, (size_t)ldg * 16, m * 16, n, cudaMemcpyDefault,
                             ctx->stream));
  CTX_CUDA(cudaMemcpy2DAsync(ctx->Z, (size_t)ctx->ldn * 16, Zp, (size_t)ldz * 16, n * 16, n, cudaMemcpyDefault,
                             ctx->stream));
  if (W)
    CTX_CUDA(cudaMemcpy2DAsync(ctx->W, (size_t)ctx->ldn * 16, W, (size_t)ldw * 16, n * 16, n, cudaMemcpyDefault,
                               ctx->stream));
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->state = 2;   // a sweep resumes from the loaded state
  return GHSVD_OK;
}

ghsvd_status ghsvd_hz2x2_batch(ghsvd_ctx h, int64_t count, const double* in, double tol, int criterion,
                               double* out, int* kind) {
  if (!h || !in || !out || !kind || count < 0) return GHSVD_E_INVALID_ARG;
  Ctx* ctx = &h->c;
  CTX_CUDA(cudaSetDevice(ctx->o.device));
  TRY(launch_hz2x2_batch(ctx, count, in, tol, criterion, out, kind));
  CTX_CUDA(cudaStreamSynchronize(ctx->stream));
  return GHSVD_OK;
}

}  // extern "C"
