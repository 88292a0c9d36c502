// comm.cpp -- multi-GPU layer of the blocked variant.
//
// P ranks (one per GPU) run the Level-2 round-robin over nblk = 2 P K block
// columns; rank r owns slots [r K, (r+1) K) of every block step (a slot holds one
// block pair).  Every rank keeps full-size F, G, Z buffers, but only the block
// columns it currently owns are up to date.  After block step s the block columns
// whose owner changes for step s' are moved with grouped ncclSend / ncclRecv
// (the paper's physical block-column exchange, over
// NVLink/NVSwitch), and once per sweep the counters are combined with
// ncclAllReduce so every rank takes the same stop decision.
// NCCL is loaded with dlopen("libnccl.so.2") (torch's copy when torch is loaded),
// so the library itself has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <chrono>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"
#include "ordering.h"

namespace ghsvd {

// ------------------------------------------------------------------ schedule
// owner[b] = rank owning block b in step s of the block ordering (ordering.h)
static void owners(int ord, int nsup, int nblk, int world, long long s, std::vector<int>& own) {
  own.assign(nblk, -1);
  const int K = nblk / 2 / world;
  for (int k = 0; k < nblk / 2; k++) {
    long long p, q;
    blk_order_pair(ord, nblk, nsup, s, k, &p, &q);
    own[p] = own[q] = k / K;
  }
}

static bool plan_args_ok(int ord, int nblk, int nsup, int world) {
  return world >= 1 && blk_order_check(ord, nblk, nsup) == 0 && (nblk / 2) % world == 0;
}

static int exchange_plan(int ord, int nblk, int nsup, int world, int rank, long long s, long long s_next,
                         int64_t* send_blk, int64_t* send_peer, int64_t* nsend, int64_t* recv_blk,
                         int64_t* recv_peer, int64_t* nrecv) {
  if (!plan_args_ok(ord, nblk, nsup, world) || rank < 0 || rank >= world) return -1;
  const long long nst = blk_order_steps(ord, nblk, nsup);
  if (s < 0 || s >= nst || s_next < 0 || s_next >= nst) return -1;
  std::vector<int> o1, o2;
  owners(ord, nsup, nblk, world, s, o1);
  owners(ord, nsup, nblk, world, s_next, o2);
  int64_t ns = 0, nr = 0;
  for (int b = 0; b < nblk; b++) {
    if (o1[b] == rank && o2[b] != rank) {
      send_blk[ns] = b;
      send_peer[ns] = o2[b];
      ns++;
    }
    if (o2[b] == rank && o1[b] != rank) {
      recv_blk[nr] = b;
      recv_peer[nr] = o1[b];
      nr++;
    }
  }
  *nsend = ns;
  *nrecv = nr;
  return 0;
}

// true if some block column changes rank between steps s and s_next (the same on every rank)
bool comm_step_moves(const Ctx* ctx, int nblk, long long s, long long s_next) {
  const int world = ctx->o.world_size;
  if (world <= 1) return false;
  std::vector<int> o1, o2;
  owners(ctx->o.ordering, ctx->blk_nsup, nblk, world, s, o1);
  owners(ctx->o.ordering, ctx->blk_nsup, nblk, world, s_next, o2);
  return o1 != o2;
}

}  // namespace ghsvd

extern "C" {

// Rank owning block column b in block step s (nblk even, world | nblk/2).  -1 on bad args.
int ghsvd_block_owner(int nblk, int world, int s, int b) {
  return ghsvd_block_owner_ord(GHSVD_ORDER_ROUND_ROBIN, nblk, 0, world, s, b);
}

// Exchange plan of `rank` between block steps s and s_next: blocks it sends
// (send_blk[i] to send_peer[i]) and receives (recv_blk[i] from recv_peer[i]),
// in increasing block order.  Arrays must hold nblk entries.  Returns 0 / -1.
int ghsvd_exchange_plan(int nblk, int world, int rank, int s, int s_next, int64_t* send_blk, int64_t* send_peer,
                        int64_t* nsend, int64_t* recv_blk, int64_t* recv_peer, int64_t* nrecv) {
  return ghsvd::exchange_plan(GHSVD_ORDER_ROUND_ROBIN, nblk, 0, world, rank, s, s_next, send_blk, send_peer, nsend,
                              recv_blk, recv_peer, nrecv);
}

int64_t ghsvd_order_steps(int ordering, int nblk, int nsup) {
  if (ghsvd::blk_order_check(ordering, nblk, nsup)) return -1;
  return ghsvd::blk_order_steps(ordering, nblk, nsup);
}

int ghsvd_order_pair(int ordering, int nblk, int nsup, int64_t s, int64_t k, int64_t* p, int64_t* q) {
  if (ghsvd::blk_order_check(ordering, nblk, nsup) || s < 0 || s >= ghsvd::blk_order_steps(ordering, nblk, nsup) ||
      k < 0 || k >= nblk / 2 || !p || !q)
    return -1;
  long long a, b;
  ghsvd::blk_order_pair(ordering, nblk, nsup, s, k, &a, &b);
  *p = a;
  *q = b;
  return 0;
}

int ghsvd_block_owner_ord(int ordering, int nblk, int nsup, int world, int64_t s, int b) {
  if (!ghsvd::plan_args_ok(ordering, nblk, nsup, world) || s < 0 ||
      s >= ghsvd::blk_order_steps(ordering, nblk, nsup) || b < 0 || b >= nblk)
    return -1;
  std::vector<int> own;
  ghsvd::owners(ordering, nsup, nblk, world, s, own);
  return own[b];
}

int ghsvd_exchange_plan_ord(int ordering, int nblk, int nsup, int world, int rank, int64_t s, int64_t s_next,
                            int64_t* send_blk, int64_t* send_peer, int64_t* nsend, int64_t* recv_blk,
                            int64_t* recv_peer, int64_t* nrecv) {
  return ghsvd::exchange_plan(ordering, nblk, nsup, world, rank, s, s_next, send_blk, send_peer, nsend, recv_blk,
                              recv_peer, nrecv);
}

}  // extern "C"

namespace ghsvd {

// ------------------------------------------------------------------ NCCL (dlopen)
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static Nccl* load_nccl() {
  static Nccl n;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (n.h) break;
  }
  if (!n.h) return nullptr;
  n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.h, "ncclGetUniqueId");
  n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.h, "ncclCommInitRank");
  n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
  n.CommSplit = (decltype(n.CommSplit))dlsym(n.h, "ncclCommSplit");
  n.Send = (decltype(n.Send))dlsym(n.h, "ncclSend");
  n.Recv = (decltype(n.Recv))dlsym(n.h, "ncclRecv");
  n.GroupStart = (decltype(n.GroupStart))dlsym(n.h, "ncclGroupStart");
  n.GroupEnd = (decltype(n.GroupEnd))dlsym(n.h, "ncclGroupEnd");
  n.AllReduce = (decltype(n.AllReduce))dlsym(n.h, "ncclAllReduce");
  n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.h, "ncclGetErrorString");
  if (!n.GetUniqueId || !n.CommInitRank || !n.CommSplit || !n.Send || !n.Recv || !n.GroupStart || !n.GroupEnd || !n.AllReduce) {
    dlclose(n.h);
    n.h = nullptr;
    return nullptr;
  }
  return &n;
}

// loaded once (thread-safe static initialisation: loopback ranks call in from several threads)
static Nccl* nccl() {
  static Nccl* const n = load_nccl();
  return n;
}

#define NCCL_CALL(x)                                                                            \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess) {                                                                    \
      ctx->err = std::string(#x) + ": " + (N->GetErrorString ? N->GetErrorString(r_) : "error"); \
      return GHSVD_E_NCCL;                                                                      \
    }                                                                                           \
  } while (0)

// ------------------------------------------------------------------ loopback transport
// Test transport (include/ghsvd.h, "loopback id"): the world_size ranks are contexts of
// ONE process on one device, each driven by its own host thread.  The exchange and the
// reductions are the NCCL calls' effect written as device copies between the contexts'
// workspaces, ordered by CUDA events and a host barrier; no kernel ever waits on another
// rank's kernel, so the ranks' streams may share a GPU.  Everything above the transport
// (ownership, halves schedule, events, stop decision) is the multi-GPU code path itself.
struct LoopGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;
  std::vector<Ctx*> ctx;
  std::vector<cudaEvent_t> ev_done, ev_copy;
  std::vector<DevCounters> cnt;
  // host barrier over the group's ranks; false on timeout (a rank failed) -- the group
  // is then broken and every later barrier fails at once
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      gen++;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(600), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct CommHandle {
  int kind;                           // 1 NCCL, 2 loopback
  ncclComm_t nccl;                    // F, G exchange, counters, outputs (context stream)
  ncclComm_t nccl_zw;                 // Z', W exchange (aux stream; split of nccl)
  std::shared_ptr<LoopGroup> loop;
};

static const char kLoopTag[16] = {'G', 'H', 'S', 'V', 'D', '-', 'L', 'O', 'O', 'P', 'B', 'A', 'C', 'K', 0, 0};
static std::mutex g_loop_mu;
static std::map<std::string, std::weak_ptr<LoopGroup>> g_loop_groups;

static CommHandle* handle(Ctx* ctx) { return (CommHandle*)ctx->comm; }

static ghsvd_status loop_init(Ctx* ctx, const char* id) {
  const std::string key(id + 16, 112);
  std::shared_ptr<LoopGroup> g;
  {
    std::lock_guard<std::mutex> lk(g_loop_mu);
    auto it = g_loop_groups.find(key);
    if (it != g_loop_groups.end()) g = it->second.lock();
    if (!g || g->broken) {
      g = std::make_shared<LoopGroup>();
      g->world = ctx->o.world_size;
      g->ctx.assign(g->world, nullptr);
      g->ev_done.assign(g->world, nullptr);
      g->ev_copy.assign(g->world, nullptr);
      g->cnt.assign(g->world, DevCounters{});
      g_loop_groups[key] = g;
    }
  }
  {
    std::lock_guard<std::mutex> lk(g->mu);
    const int r = ctx->o.rank;
    if (g->world != ctx->o.world_size || g->ctx[r]) {
      ctx->err = "loopback: world_size mismatch or rank joined twice";
      return GHSVD_E_INVALID_ARG;
    }
    g->ctx[r] = ctx;
    GH_CUDA(cudaEventCreateWithFlags(&g->ev_done[r], cudaEventDisableTiming));
    GH_CUDA(cudaEventCreateWithFlags(&g->ev_copy[r], cudaEventDisableTiming));
  }
  CommHandle* c = new CommHandle{2, nullptr, nullptr, g};
  ctx->comm = c;
  return GHSVD_OK;
}

ghsvd_status comm_init(Ctx* ctx) {
  if (ctx->o.nccl_id && memcmp(ctx->o.nccl_id, kLoopTag, 16) == 0) return loop_init(ctx, (const char*)ctx->o.nccl_id);
  Nccl* N = nccl();
  if (!N) {
    ctx->err = "multi-GPU: libnccl.so.2 could not be loaded";
    return GHSVD_E_NCCL;
  }
  ncclUniqueId id;
  memcpy(&id, ctx->o.nccl_id, sizeof(id));
  ncclComm_t c, cz;
  NCCL_CALL(N->CommInitRank(&c, ctx->o.world_size, id, ctx->o.rank));
  cz = nullptr;
  if (ctx->o.exchange_overlap) {
    // opt-in second communicator for the Z', W block columns: their exchange runs on
    // another stream, concurrently with the F, G traffic and the next step's kernels
    ncclResult_t r = N->CommSplit(c, 0, ctx->o.rank, &cz, nullptr);
    if (r != ncclSuccess) {
      N->CommDestroy(c);
      ctx->err = std::string("ncclCommSplit: ") + (N->GetErrorString ? N->GetErrorString(r) : "error");
      return GHSVD_E_NCCL;
    }
  }
  ctx->comm = new CommHandle{1, c, cz, nullptr};
  return GHSVD_OK;
}

void comm_destroy(Ctx* ctx) {
  CommHandle* c = handle(ctx);
  if (!c) return;
  if (c->kind == 1) {
    Nccl* N = nccl();
    if (N && N->CommDestroy) {
      if (c->nccl_zw) N->CommDestroy(c->nccl_zw);
      N->CommDestroy(c->nccl);
    }
  } else if (c->loop) {
    LoopGroup* g = c->loop.get();
    std::lock_guard<std::mutex> lk(g->mu);
    const int r = ctx->o.rank;
    if (g->ev_done[r]) cudaEventDestroy(g->ev_done[r]);
    if (g->ev_copy[r]) cudaEventDestroy(g->ev_copy[r]);
    g->ev_done[r] = g->ev_copy[r] = nullptr;
    g->ctx[r] = nullptr;
  }
  delete c;
  ctx->comm = nullptr;
}

static ghsvd_status loop_broken(Ctx* ctx) {
  ctx->err = "loopback: another rank did not reach the barrier (failed or timed out)";
  return GHSVD_E_NCCL;
}

// The NCCL exchange's effect: every rank pulls the block columns it receives from the
// sending rank's buffers once that rank's step is complete (ev_done), and no rank writes
// its buffers again before every pull of this exchange is done (ev_copy of all ranks).
static ghsvd_status loop_exchange(Ctx* ctx, const int64_t* rb, const int64_t* rp, int64_t nr, const int* bstart,
                                  const int* bwidth, int part, cudaStream_t st) {
  LoopGroup* g = handle(ctx)->loop.get();
  const int r = ctx->o.rank;
  GH_CUDA(cudaEventRecord(g->ev_done[r], st));
  if (!g->barrier()) return loop_broken(ctx);
  for (int64_t i = 0; i < nr; i++) {
    const Ctx* pc = g->ctx[rp[i]];
    if (!pc || pc->ldm != ctx->ldm || pc->ldn != ctx->ldn || pc->m != ctx->m || pc->n != ctx->n) {
      ctx->err = "loopback: ranks hold different problem shapes";
      return GHSVD_E_INVALID_ARG;
    }
    GH_CUDA(cudaStreamWaitEvent(st, g->ev_done[rp[i]], 0));
    const size_t b = (size_t)rb[i], c0 = (size_t)bstart[b], w = (size_t)bwidth[b];
    const cudaMemcpyKind k = cudaMemcpyDeviceToDevice;
    if (part & XCH_FG) {
      GH_CUDA(cudaMemcpyAsync(ctx->F + c0 * ctx->ldm, pc->F + c0 * pc->ldm, w * ctx->ldm * 16, k, st));
      GH_CUDA(cudaMemcpyAsync(ctx->G + c0 * ctx->ldm, pc->G + c0 * pc->ldm, w * ctx->ldm * 16, k, st));
    }
    if (part & XCH_ZW) {
      GH_CUDA(cudaMemcpyAsync(ctx->Z + c0 * ctx->ldn, pc->Z + c0 * pc->ldn, w * ctx->ldn * 16, k, st));
      if (ctx->o.want_x && ctx->W && pc->W)
        GH_CUDA(cudaMemcpyAsync(ctx->W + c0 * ctx->ldn, pc->W + c0 * pc->ldn, w * ctx->ldn * 16, k, st));
    }
  }
  GH_CUDA(cudaEventRecord(g->ev_copy[r], st));
  if (!g->barrier()) return loop_broken(ctx);
  for (int p = 0; p < g->world; p++)
    if (p != r) GH_CUDA(cudaStreamWaitEvent(st, g->ev_copy[p], 0));
  return GHSVD_OK;
}

// Move the block columns whose owner changes between block steps s_now and s_next, on
// stream st: part XCH_FG = F and G (m rows), XCH_ZW = Z' and W (n rows).  A block column
// is contiguous in each buffer.  Every rank issues the parts in the same order.
ghsvd_status comm_exchange(Ctx* ctx, int nblk, int s_now, int s_next, const int* bstart, const int* bwidth, int part,
                           cudaStream_t st) {
  Nccl* N = nccl();
  if (!ctx->comm || (!N && handle(ctx)->kind == 1)) {
    ctx->err = "multi-GPU: no communicator";
    return GHSVD_E_NCCL;
  }
  // nothing moves on any rank (e.g. inside an outer step of a Level-3 ordering)
  if (!comm_step_moves(ctx, nblk, s_now, s_next)) return GHSVD_OK;
  std::vector<int64_t> sb(nblk), sp(nblk), rb(nblk), rp(nblk);
  int64_t ns = 0, nr = 0;
  if (exchange_plan(ctx->o.ordering, nblk, ctx->blk_nsup, ctx->o.world_size, ctx->o.rank, s_now, s_next, sb.data(),
                    sp.data(), &ns, rb.data(), rp.data(), &nr)) {
    ctx->err = "multi-GPU: bad exchange plan arguments";
    return GHSVD_E_INVALID_ARG;
  }
  if (handle(ctx)->kind == 2) return loop_exchange(ctx, rb.data(), rp.data(), nr, bstart, bwidth, part, st);
  if (ns == 0 && nr == 0) return GHSVD_OK;
  ncclComm_t comm = (part == XCH_ZW && handle(ctx)->nccl_zw) ? handle(ctx)->nccl_zw : handle(ctx)->nccl;
  NCCL_CALL(N->GroupStart());
  auto xfer = [&](int64_t b, int peer, bool send) -> ncclResult_t {
    const size_t w = (size_t)bwidth[b], c0 = (size_t)bstart[b];
    double2* bufs[4] = {part & XCH_FG ? ctx->F + c0 * ctx->ldm : nullptr,
                        part & XCH_FG ? ctx->G + c0 * ctx->ldm : nullptr,
                        part & XCH_ZW ? ctx->Z + c0 * ctx->ldn : nullptr,
                        (part & XCH_ZW) && ctx->o.want_x && ctx->W ? ctx->W + c0 * ctx->ldn : nullptr};
    const size_t cnt[4] = {w * ctx->ldm * 2, w * ctx->ldm * 2, w * ctx->ldn * 2, w * ctx->ldn * 2};  // doubles
    for (int t = 0; t < 4; t++) {
      if (!bufs[t]) continue;
      ncclResult_t r = send ? N->Send(bufs[t], cnt[t], ncclFloat64, peer, comm, st)
                            : N->Recv(bufs[t], cnt[t], ncclFloat64, peer, comm, st);
      if (r != ncclSuccess) return r;
    }
    return ncclSuccess;
  };
  for (int64_t i = 0; i < ns; i++) NCCL_CALL(xfer(sb[i], (int)sp[i], true));
  for (int64_t i = 0; i < nr; i++) NCCL_CALL(xfer(rb[i], (int)rp[i], false));
  NCCL_CALL(N->GroupEnd());
  return GHSVD_OK;
}

// Sum all/big, max off, min err over ranks (one small allreduce group per sweep).
ghsvd_status comm_allreduce_counters(Ctx* ctx, DevCounters* c) {
  Nccl* N = nccl();
  if (!ctx->comm || (!N && handle(ctx)->kind == 1)) {
    ctx->err = "multi-GPU: no communicator";
    return GHSVD_E_NCCL;
  }
  if (handle(ctx)->kind == 2) {
    // *c holds this rank's counters (read back by the caller); combine in rank order
    LoopGroup* g = handle(ctx)->loop.get();
    g->cnt[ctx->o.rank] = *c;
    if (!g->barrier()) return loop_broken(ctx);
    DevCounters t{};
    for (int p = 0; p < g->world; p++) {
      const DevCounters& q = g->cnt[p];
      t.all += q.all;
      t.big += q.big;
      t.off_bits = q.off_bits > t.off_bits ? q.off_bits : t.off_bits;
      t.err = q.err < t.err ? q.err : t.err;
    }
    if (!g->barrier()) return loop_broken(ctx);
    *c = t;
    return GHSVD_OK;
  }
  ncclComm_t comm = handle(ctx)->nccl;
  cudaStream_t st = ctx->stream;
  DevCounters* d = ctx->cnt;  // device copy (already holds this rank's values)
  NCCL_CALL(N->GroupStart());
  NCCL_CALL(N->AllReduce(&d->all, &d->all, 2, ncclUint64, ncclSum, comm, st));
  NCCL_CALL(N->AllReduce(&d->off_bits, &d->off_bits, 1, ncclUint64, ncclMax, comm, st));
  NCCL_CALL(N->AllReduce(&d->err, &d->err, 1, ncclInt32, ncclMin, comm, st));
  NCCL_CALL(N->GroupEnd());
  GH_CUDA(cudaMemcpyAsync(c, d, sizeof(DevCounters), cudaMemcpyDeviceToHost, st));
  GH_CUDA(cudaStreamSynchronize(st));
  return GHSVD_OK;
}

// Block columns this rank owns after a completed sweep (ownership of block step 0, which
// the final exchange of every sweep restores).
void comm_owned_blocks(const Ctx* ctx, int nblk, std::vector<int>& blocks) {
  std::vector<int> own;
  owners(ctx->o.ordering, ctx->blk_nsup, nblk, ctx->o.world_size, 0, own);
  blocks.clear();
  for (int b = 0; b < nblk; b++)
    if (own[b] == ctx->o.rank) blocks.push_back(b);
}

// Complete the extracted outputs on every rank (Zout may be NULL: Z stays distributed): zero the columns this rank does
// not own after the final exchange (ownership of block step 0), then sum.
ghsvd_status comm_finalize_outputs(Ctx* ctx, int nblk, const int* bstart, const int* bwidth, double* lam, double* sf,
                                   double* sg, double2* Zout, int64_t ldz, double2* Xout) {
  Nccl* N = nccl();
  if (!ctx->comm || (!N && handle(ctx)->kind == 1)) {
    ctx->err = "multi-GPU: no communicator";
    return GHSVD_E_NCCL;
  }
  std::vector<int> own;
  owners(ctx->o.ordering, ctx->blk_nsup, nblk, ctx->o.world_size, 0, own);
  cudaStream_t st = ctx->stream;
  if (handle(ctx)->kind == 2) {
    // the sum of the disjointly owned outputs, as a gather from each column's owner
    // (the outputs are the owners' context buffers: lam, sf, sg, Z2, Xo)
    LoopGroup* g = handle(ctx)->loop.get();
    const int r = ctx->o.rank;
    GH_CUDA(cudaEventRecord(g->ev_done[r], st));
    if (!g->barrier()) return loop_broken(ctx);
    for (int b = 0; b < nblk; b++) {
      const int p = own[b];
      if (p == r) continue;
      const Ctx* pc = g->ctx[p];
      GH_CUDA(cudaStreamWaitEvent(st, g->ev_done[p], 0));
      const size_t c0 = (size_t)bstart[b], w = (size_t)bwidth[b];
      GH_CUDA(cudaMemcpyAsync(lam + c0, pc->lam + c0, w * 8, cudaMemcpyDeviceToDevice, st));
      GH_CUDA(cudaMemcpyAsync(sf + c0, pc->sf + c0, w * 8, cudaMemcpyDeviceToDevice, st));
      GH_CUDA(cudaMemcpyAsync(sg + c0, pc->sg + c0, w * 8, cudaMemcpyDeviceToDevice, st));
      if (Zout)
        GH_CUDA(cudaMemcpyAsync(Zout + c0 * ldz, pc->Z2 + c0 * ldz, w * ldz * 16, cudaMemcpyDeviceToDevice, st));
      if (Xout && pc->Xo)
        GH_CUDA(cudaMemcpy2DAsync(Xout + c0, (size_t)ldz * 16, pc->Xo + c0, (size_t)ldz * 16, w * 16,
                                  (size_t)ctx->n, cudaMemcpyDeviceToDevice, st));
    }
    GH_CUDA(cudaEventRecord(g->ev_copy[r], st));
    if (!g->barrier()) return loop_broken(ctx);
    for (int p = 0; p < g->world; p++)
      if (p != r) GH_CUDA(cudaStreamWaitEvent(st, g->ev_copy[p], 0));
    return GHSVD_OK;
  }
  for (int b = 0; b < nblk; b++) {
    if (own[b] == ctx->o.rank) continue;
    const size_t c0 = (size_t)bstart[b], w = (size_t)bwidth[b];
    GH_CUDA(cudaMemsetAsync(lam + c0, 0, w * 8, st));
    GH_CUDA(cudaMemsetAsync(sf + c0, 0, w * 8, st));
    GH_CUDA(cudaMemsetAsync(sg + c0, 0, w * 8, st));
    if (Zout) GH_CUDA(cudaMemsetAsync(Zout + c0 * ldz, 0, w * ldz * 16, st));
    if (Xout)  // rows c0 .. c0+w-1 of X belong to this block column of W^T
      GH_CUDA(cudaMemset2DAsync(Xout + c0, (size_t)ldz * 16, 0, w * 16, (size_t)ctx->n, st));
  }
  ncclComm_t comm = handle(ctx)->nccl;
  const size_t n = (size_t)ctx->n;
  NCCL_CALL(N->GroupStart());
  NCCL_CALL(N->AllReduce(lam, lam, n, ncclFloat64, ncclSum, comm, st));
  NCCL_CALL(N->AllReduce(sf, sf, n, ncclFloat64, ncclSum, comm, st));
  NCCL_CALL(N->AllReduce(sg, sg, n, ncclFloat64, ncclSum, comm, st));
  if (Zout) NCCL_CALL(N->AllReduce(Zout, Zout, n * ldz * 2, ncclFloat64, ncclSum, comm, st));
  if (Xout) NCCL_CALL(N->AllReduce(Xout, Xout, n * ldz * 2, ncclFloat64, ncclSum, comm, st));
  NCCL_CALL(N->GroupEnd());
  return GHSVD_OK;
}

}  // namespace ghsvd

extern "C" {

// Fill 128 bytes with a fresh ncclUniqueId (rank 0 calls this and broadcasts it).
// Returns 0, or -4 if NCCL cannot be loaded.
int ghsvd_nccl_unique_id(void* out128) {
  ghsvd::Nccl* N = ghsvd::nccl();
  if (!N || !out128) return -4;
  ncclUniqueId id;
  if (N->GetUniqueId(&id) != ncclSuccess) return -4;
  memcpy(out128, &id, sizeof(id));
  return 0;
}

}  // extern "C"
