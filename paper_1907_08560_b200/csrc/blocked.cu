// blocked.cu -- Level-2 blocked HZ (BO / FB variants), Sec 6.4
// (lines 1815-2040); SURVEY 8(a) row a6, and the slot bookkeeping of a7.
//
// Partition (Sec 6.4.1): nblk (even) block columns of widths w or w-1,
// non-increasing.  Outer ordering: round-robin over block columns (reading
// C-11).  Per block step s, for every block pair (bp, bq) owned by this rank:
//   k_blk_gram   H_blk = F_pair^* J F_pair, S_blk = G_pair^* G_pair (k x k,
//                k = w_p + w_q <= 64), lower-triangle 8x8 tiles on the FP64
//                tensor cores (mma.sync m8n8k4 f64 = DMMA, 3M complex product),
//                J folded into the A operand, split over row chunks; the last
//                CTA of a (pair, H|S) sums the partials in fixed order and
//                factorizes: HEBPJ(H_blk) -> F^, J^ (Sec 4.2-4.3) or pivoted
//                Cholesky(S_blk) -> G^;
//   k_blk_pivot  one CTA: F^, G^ in shared memory, border to even order, inner
//                Level-1 one-sided HZ sweep(s) (BO: 1 sweep; FB: until no
//                transformation, <= 30) accumulating Z_blk (Sec 6.4.2); counters;
//   k_blk_update F_pair <- F_pair Z_blk, G_pair <- G_pair Z_blk, Z_pair <-
//                Z_pair Z_blk in place, row tiles on DMMA (Sec 6.4.3, the
//                paper's three ZGEMMs; no shadow copy is needed on one GPU
//                because every CTA reads its row tile before writing it).
// blk_sweep schedules a step as two halves of the pairs on prioritized streams
// (DESIGN.md 6); multi-GPU (comm.cpp) exchanges block columns between the steps.
// Kernels: blk_gram.cuh (Grams + factorizations), blk_pivot.cuh (inner sweep),
// blk_update.cuh (updates), blk_common.cuh (shared helpers); this file: host side.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <string>
#include <vector>

#include "internal.h"
#include "ordering.h"
// the kernels (one translation unit: these files are included only here)
#include "blk_common.cuh"
#include "blk_gram.cuh"
#include "blk_pivot.cuh"
#include "blk_update.cuh"

namespace ghsvd {

namespace {

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

int resolve_nsup(const ghsvd_options* o, int64_t nb_rr);

// the round-robin partition: width w <= 32 -> block pivots of order <= 64
int64_t auto_nblk_rr(int64_t n, const ghsvd_options* o) {
  if (o->nblocks > 0) return o->nblocks;
  int64_t nb = (n + 31) / 32;
  nb += nb & 1;
  const int64_t P = std::max(1, o->world_size);
  return std::max<int64_t>(2, round_up(nb, 2 * P));
}

// tuning knobs (experiments only; defaults are the measured best)
int auto_nblk(int64_t n, const ghsvd_options* o) {
  if (o->nblocks > 0) return o->nblocks;
  int64_t nb = auto_nblk_rr(n, o);
  const int64_t P = std::max(1, o->world_size);
  // Level-3 orderings: whole super blocks (HIER: an even number of block columns in each)
  const int64_t ns = resolve_nsup(o, nb);
  if (ns != nb) {   // (ns == nb: one block column per super block, nothing to round)
    if (o->ordering == GHSVD_ORDER_LEVEL3) nb = round_up(nb, std::lcm<int64_t>(2 * P, std::max<int64_t>(2, ns)));
    if (o->ordering == GHSVD_ORDER_HIER) nb = round_up(nb, std::lcm<int64_t>(2 * P, 2 * std::max<int64_t>(2, ns)));
  }
  if (o->ordering != GHSVD_ORDER_ROUND_ROBIN && nb > n) nb = n - (n & 1);
  return (int)std::max<int64_t>(2, nb);
}


struct BlkPlan {
  int nblk, K, slot0, nsplit;
  long long split_rows;
  int nsup;   // super blocks of a LEVEL3 / HIER ordering (0 for the round-robin)
  int nst;    // block steps per sweep
};

// super blocks of the LEVEL3 / HIER orderings: the option, else one super pair per rank; on
// one GPU 4, or (small problems, < 32 block columns in the round-robin partition) one super
// block per block column, which IS the round-robin (rounding the partition up to whole even
// super blocks would only shrink the blocks)
int resolve_nsup(const ghsvd_options* o, int64_t nb_rr) {
  if (o->ordering == GHSVD_ORDER_ROUND_ROBIN) return 0;
  if (o->super_blocks > 0) return o->super_blocks;
  if (o->world_size > 1) return 2 * o->world_size;
  return nb_rr >= 32 ? 4 : (int)nb_rr;
}

BlkPlan make_plan(const Ctx* ctx) {
  BlkPlan p;
  p.nblk = auto_nblk(ctx->n, &ctx->o);
  const int P = std::max(1, ctx->o.world_size);
  p.K = p.nblk / 2 / P;
  p.slot0 = ctx->o.rank * p.K;
  p.nsup = resolve_nsup(&ctx->o, auto_nblk_rr(ctx->n, &ctx->o));
  p.nst = blk_order_check(ctx->o.ordering, p.nblk, p.nsup) ? -1 : (int)blk_order_steps(ctx->o.ordering, p.nblk, p.nsup);
  // Row split of the Gram launches, chosen against wave quantization: a launch covers
  // M = 2 * (pairs per launch) matrices x nsplit CTAs with R CTAs resident at once;
  // cost ~ waves x (32-row stages per CTA + fill/partial overhead).  Deterministic for a
  // given (m, K, device) since the sum of the split partials has a fixed order.
  int dev = 0, sms = 148, per_sm = 2;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // M from the GLOBAL pair count, so the split (and the partial-sum order) is the same
  // for every world size: a P-GPU run stays bitwise equal to the 1-GPU run
  const long long Kg = p.nblk / 2;
  const long long M = 2LL * (Kg >= 2 ? Kg / 2 : Kg);
  const long long R = (long long)sms * per_sm;
  long long best = -1;
  double best_cost = 0.0;
  for (int ns = 1; ns <= MAX_SPLIT; ns++) {
    const long long rows = round_up((ctx->m + ns - 1) / ns, RTG);
    const int nseff = (int)((ctx->m + rows - 1) / rows);
    if (nseff != ns) continue;
    const double waves = (double)((M * ns + R - 1) / R);
    const double cost = waves * (double)(rows / RTG + 3);
    if (best < 0 || cost < best_cost - 1e-9) {
      best = ns;
      best_cost = cost;
    }
  }
  p.nsplit = (int)std::max<long long>(1, best);
  if (ctx->o.gram_splits > 0) p.nsplit = std::min(MAX_SPLIT, ctx->o.gram_splits);
  const long long rows_per = (ctx->m + p.nsplit - 1) / p.nsplit;
  p.split_rows = round_up(std::max<long long>(rows_per, 1), RTG);
  p.nsplit = (int)((ctx->m + p.split_rows - 1) / p.split_rows);
  return p;
}

}  // namespace

// scratch carved by blk_setup for K block pairs per rank out of nblk block columns
static size_t blk_scratch_for(int64_t K, int64_t nb, bool want_x) {
  return al256((size_t)K * 2 * MAX_SPLIT * KM * KM * 16) + al256((size_t)2 * K * KM * KM * 16) +
         al256((size_t)2 * K * 4) + 2 * al256((size_t)(nb + 2) * 4) + 2 * al256((size_t)K * KM * KM * 16) +
         al256((size_t)K * KM) + al256((size_t)2 * K * 4) + (want_x ? al256((size_t)2 * K * KM * KM * 16) : 0) +
         al256((size_t)(2 * nb + 2) * TRACE_SLOTS * 16) + al256((size_t)2 * K * 4) + al256((size_t)(2 * nb + 2) * 8) +
         al256((size_t)(2 * nb + 2) * (nb / 2) * 16) + 4096;
}

// workspace bound at ghsvd_create for factors of up to n columns: the sweep may see
// n + 1 columns (odd n is bordered, Sec 6.3.2); a single rank holds all nblk/2 pairs
size_t blk_scratch_bytes(const ghsvd_options* o, int64_t m, int64_t n) {
  (void)m;
  const int64_t nb = auto_nblk(n + 1, o);
  return blk_scratch_for(nb / 2, nb, o->want_x != 0);
}

// in comm.cpp

struct BlkSetup {
  BlkPlan pl;
  BlkArgs a;
  std::vector<int> bs_h, bw_h;
  size_t smem_g, smem_p, smem_u, smem_f;
  bool fused;   // block-pivot factorization fused into the Gram's last CTAs (default; not GHSVD_SCHED_SPLIT_FACTOR)
  int tF, tZ, sms;
  bool upd4m, gram3m, pivot_cl;
  size_t smem_pc;
  unsigned long long* trace_buf;
};

static ghsvd_status blk_setup(Ctx* ctx, BlkSetup& S) {
  BlkPlan& pl = S.pl;
  BlkArgs& a = S.a;
  pl = make_plan(ctx);
  if (pl.nblk % 2 || pl.nblk < 2 || pl.nblk > ctx->n || pl.K < 1 ||
      pl.nblk % (2 * std::max(1, ctx->o.world_size))) {
    ctx->err = "blocked: nblocks must be even, <= n and a multiple of 2*world_size";
    return GHSVD_E_INVALID_ARG;
  }
  if (pl.nst < 1) {
    ctx->err = "blocked: invalid block ordering (super_blocks must be even and divide nblocks; HIER needs an even "
               "number of block columns per super block, or 1)";
    return GHSVD_E_INVALID_ARG;
  }
  const int64_t w = (ctx->n + pl.nblk - 1) / pl.nblk;
  if (2 * w > KM) {
    ctx->err = "blocked: block width " + std::to_string(w) + " > 32 (increase nblocks)";
    return GHSVD_E_INVALID_ARG;
  }
  if (blk_scratch_for(pl.K, pl.nblk, ctx->o.want_x != 0) > ctx->L.scr_bytes) {
    ctx->err = "blocked: workspace scratch too small (create the context with a blocked variant)";
    return GHSVD_E_WORKSPACE;
  }
  cudaStream_t str = ctx->stream;
  char* p = ctx->scr;
  a.gpart = (double2*)p; p += al256((size_t)pl.K * 2 * MAX_SPLIT * KM * KM * 16);
  a.zblk = (double2*)p; p += al256((size_t)2 * pl.K * KM * KM * 16);   // double-buffered by step parity
  a.applied = (int*)p; p += al256((size_t)2 * pl.K * 4);
  int* bstart = (int*)p; p += al256((size_t)(pl.nblk + 2) * 4);
  int* bwidth = (int*)p; p += al256((size_t)(pl.nblk + 2) * 4);
  a.fhat = (double2*)p; p += al256((size_t)pl.K * KM * KM * 16);
  a.ghat = (double2*)p; p += al256((size_t)pl.K * KM * KM * 16);
  a.jhat = (signed char*)p; p += al256((size_t)pl.K * KM);
  a.fact_ok = (int*)p; p += al256((size_t)2 * pl.K * 4);
  a.gcnt = (int*)p; p += al256((size_t)2 * pl.K * 4);
  a.W = ctx->o.want_x ? ctx->W : nullptr;
  if (a.W) {
    a.zinvT = (double2*)p; p += al256((size_t)2 * pl.K * KM * KM * 16);   // double-buffered like zblk
  } else {
    a.zinvT = nullptr;
  }
  // step-indexed arrays: a sweep has at most 2 nblk block steps (LEVEL3: (2Q-1)(2B-1) < 4QB)
  S.trace_buf = (unsigned long long*)p; p += al256((size_t)(2 * pl.nblk + 2) * TRACE_SLOTS * 16);
  a.upd_k2 = (unsigned long long*)p; p += al256((size_t)(2 * pl.nblk + 2) * 8);
  int4* ptab = (int4*)p; p += al256((size_t)(2 * pl.nblk + 2) * (pl.nblk / 2) * 16);
  a.trace = nullptr;
  a.trace_id = 0;
  k_blk_partition<<<1, 32, 0, str>>>(bstart, bwidth, pl.nblk, ctx->n);
  GH_CUDA(cudaMemsetAsync(a.gcnt, 0, (size_t)2 * pl.K * 4, str));
  GH_CUDA(cudaMemsetAsync(a.upd_k2, 0, (size_t)(2 * pl.nblk + 2) * 8, str));
  GH_CUDA(cudaGetLastError());
  S.bs_h.assign(pl.nblk, 0);
  S.bw_h.assign(pl.nblk, 0);
  GH_CUDA(cudaMemcpyAsync(S.bs_h.data(), bstart, pl.nblk * 4, cudaMemcpyDeviceToHost, str));
  GH_CUDA(cudaMemcpyAsync(S.bw_h.data(), bwidth, pl.nblk * 4, cudaMemcpyDeviceToHost, str));
  GH_CUDA(cudaStreamSynchronize(str));
  ctx->blk_start = S.bs_h;
  ctx->blk_width = S.bw_h;
  {
    // pair table of the whole block sweep: the kernels read their block pair from it
    std::vector<int4> t((size_t)pl.nst * (pl.nblk / 2));
    for (int s = 0; s < pl.nst; s++)
      for (int k = 0; k < pl.nblk / 2; k++) {
        long long bp, bq;
        blk_order_pair(ctx->o.ordering, pl.nblk, pl.nsup, s, k, &bp, &bq);
        t[(size_t)s * (pl.nblk / 2) + k] = make_int4(S.bs_h[bp], S.bw_h[bp], S.bs_h[bq], S.bw_h[bq]);
      }
    GH_CUDA(cudaMemcpyAsync(ptab, t.data(), t.size() * sizeof(int4), cudaMemcpyHostToDevice, str));
    GH_CUDA(cudaStreamSynchronize(str));
  }
  a.ptab = ptab;
  a.F = ctx->F;
  a.G = ctx->G;
  a.Z = ctx->Z;
  a.ldm = ctx->ldm;
  a.ldn = ctx->ldn;
  a.m = ctx->m;
  a.n = ctx->n;
  a.npos = ctx->npos;
  a.nblk = pl.nblk;
  a.ord = ctx->o.ordering;
  a.nsup = pl.nsup;
  ctx->blk_nsup = pl.nsup;
  a.slot0 = pl.slot0;
  a.npairs = pl.K;
  a.bstart = bstart;
  a.bwidth = bwidth;
  a.nsplit = pl.nsplit;
  a.split_rows = pl.split_rows;
  a.cnt = ctx->cnt;
  a.eps = ctx->o.eps;
  a.literal = ctx->o.criterion == GHSVD_CRIT_LITERAL;
  a.inner_sweeps = ctx->o.variant == GHSVD_BLOCKED_FB ? 30 : 1;
  a.pair0 = 0;
  S.fused = (ctx->o.schedule & GHSVD_SCHED_SPLIT_FACTOR) == 0;
  S.smem_g = (size_t)GSTAGES * KM * (S.fused ? GS_FUSED : GS) * 16;
  S.smem_f = BLK_FACTOR_SMEM;
  S.smem_p = (size_t)3 * KM * KM * 16;
  S.smem_u = (size_t)(KM * US + KM * ZS) * 16;
  GH_CUDA(cudaFuncSetAttribute(k_blk_gram<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_g));
  GH_CUDA(cudaFuncSetAttribute(k_blk_gram<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_g));
  GH_CUDA(cudaFuncSetAttribute(k_blk_gram<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_g));
  GH_CUDA(cudaFuncSetAttribute(k_blk_gram<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_g));
  GH_CUDA(cudaFuncSetAttribute(k_blk_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_f));
  S.gram3m = (ctx->o.schedule & GHSVD_SCHED_GRAM4M) == 0;
  S.pivot_cl = (ctx->o.schedule & GHSVD_SCHED_PIVOT_CL) != 0;
  S.smem_pc = (size_t)3 * KM * RB * 16;
  GH_CUDA(cudaFuncSetAttribute(k_blk_zinv, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * KM * KM * 16));
  GH_CUDA(cudaFuncSetAttribute(k_blk_pivot_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_pc));
  GH_CUDA(cudaFuncSetAttribute(k_blk_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_p));
  GH_CUDA(cudaFuncSetAttribute(k_blk_update<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_u));
  GH_CUDA(cudaFuncSetAttribute(k_blk_update<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_u));
  S.upd4m = (ctx->o.schedule & GHSVD_SCHED_UPD4M) != 0;
  S.tF = (int)((ctx->m + RT - 1) / RT);
  S.tZ = (int)((ctx->n + RT - 1) / RT);
  {
    int dev = 0;
    S.sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&S.sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return GHSVD_OK;
}

// Block-pivot launch over pairs [a.pair0, a.pair0 + np): the two-CTA cluster kernel (then,
// for want_x, the Gauss-Jordan inverse of each Z_blk), or the one-CTA kernel.
static void launch_pivot(const BlkSetup& S, const BlkArgs& a, int np, cudaStream_t st) {
  if (S.pivot_cl) {
    k_blk_pivot_cl<<<2 * np, NT_PC, S.smem_pc, st>>>(a);
    if (a.zinvT) k_blk_zinv<<<np, NT_P, (size_t)2 * KM * KM * 16, st>>>(a);
  } else {
    k_blk_pivot<<<np, NT_P, S.smem_p, st>>>(a);
  }
}

// Gram launch over pairs [a.pair0, a.pair0 + np): grid (row split, H|S, pair).
static void launch_gram(const BlkSetup& S, const BlkArgs& a, int np, cudaStream_t st) {
  const dim3 g(S.pl.nsplit, 2, np);
  if (S.fused) {
    if (S.gram3m)
      k_blk_gram<true, true><<<g, NT_G, S.smem_g, st>>>(a);
    else
      k_blk_gram<false, true><<<g, NT_G, S.smem_g, st>>>(a);
  } else {
    if (S.gram3m)
      k_blk_gram<true, false><<<g, NT_G, S.smem_g, st>>>(a);
    else
      k_blk_gram<false, false><<<g, NT_G, S.smem_g, st>>>(a);
  }
}

// Block-pivot factorization launch over pairs [a.pair0, a.pair0 + np): grid (H|S, pair)
// (nothing to launch when the Gram kernel factors in its last CTAs).
static void launch_factor(const BlkSetup& S, const BlkArgs& a, int np, cudaStream_t st) {
  if (!S.fused) k_blk_factor<<<dim3(2, np), NT_F, S.smem_f, st>>>(a);
}

// Update launch: pairs [pair0, pair0 + np), row tiles [tbeg, tend) (see k_blk_update).
static void launch_update(const BlkSetup& S, BlkArgs a, int pair0, int np, int tbeg, int tend, int wmode,
                          cudaStream_t st) {
  a.pair0 = pair0;
  if (np <= 0 || tend <= tbeg) return;
  if (S.upd4m)
    k_blk_update<true><<<dim3(np, tend - tbeg), NT_U, S.smem_u, st>>>(a, S.tF, tbeg, wmode);
  else
    k_blk_update<false><<<dim3(np, tend - tbeg), NT_U, S.smem_u, st>>>(a, S.tF, tbeg, wmode);
}

// Diagnostic: block steps [s0, s0+ns) of the first block sweep, one stream, no overlap.
ghsvd_status blk_run_steps(Ctx* ctx, int64_t s0, int64_t ns) {
  BlkSetup S;
  ghsvd_status e = blk_setup(ctx, S);
  if (e) return e;
  if (s0 < 0 || ns < 0 || s0 + ns > S.pl.nst) {
    ctx->err = "run_steps: block step range outside the block sweep";
    return GHSVD_E_INVALID_ARG;
  }
  if (ctx->o.world_size > 1) {
    ctx->err = "run_steps: single-rank diagnostic";
    return GHSVD_E_INVALID_ARG;
  }
  cudaStream_t str = ctx->stream;
  BlkArgs a = S.a;
  for (int64_t s = s0; s < s0 + ns; s++) {
    a.s = (int)s;
    launch_gram(S, a, S.pl.K, str);
    launch_factor(S, a, S.pl.K, str);
    launch_pivot(S, a, S.pl.K, str);
    launch_update(S, a, 0, S.pl.K, 0, 2 * S.tF + S.tZ, 0, str);
    if (a.W) launch_update(S, a, 0, S.pl.K, 0, S.tZ, 1, str);
    GH_CUDA(cudaGetLastError());
  }
  return GHSVD_OK;
}

// One-GPU block sweep, pipelined over pair groups (Sec 6.4 run on one device).
//
// Round-robin dependency structure (reading C-11 applied to block columns): the block
// columns of slot k at step s+1 are those of slots k-1 and k+1 at step s (slot 0 also
// keeps the fixed column n-1, slot K-1 the column it shares with itself).  So the
// slots are cut into G contiguous groups, each group's chain
//     Gram -> factor -> pivot -> update (F, G and Z' rows)
// runs on its own stream, and group g at step s waits only for the updates of groups
// g-1, g, g+1 at step s-1.  While one group is in its latency-bound factor / inner
// sweep phase the other groups' Gram and update kernels keep the tensor pipes busy,
// and step s+1 of the first groups starts while the last groups finish step s.  The
// per-pair work and its arithmetic are exactly those of the step-synchronous
// schedule, so the results are bitwise identical to it.
static ghsvd_status blk_sweep_groups(Ctx* ctx, ghsvd_stats* st, BlkSetup& S, int G) {
  BlkPlan& pl = S.pl;
  BlkArgs a = S.a;

  const int tF = S.tF, tZ = S.tZ;
  cudaStream_t str = ctx->stream;
  const uint64_t pairs = (uint64_t)ctx->n * (ctx->n - 1) / 2;
  const int nst = pl.nst;
  while ((int)ctx->grp_streams.size() < G) {
    cudaStream_t t;
    GH_CUDA(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
    ctx->grp_streams.push_back(t);
  }
  std::vector<int> g0(G + 1);
  for (int g = 0; g <= G; g++) g0[g] = (int)((long long)g * pl.K / G);
  std::vector<cudaEvent_t> ev_upd(2 * G), tev;
  for (auto& e : ev_upd) GH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // detail timing: per (step, group) events around Gram, factor + pivot, update on the
  // group's stream (kernels of other groups run concurrently inside these intervals)
  const bool timing = ctx->o.detail_timing != 0;
  if (timing) {
    tev.resize((size_t)nst * G * 4);
    for (auto& e : tev) GH_CUDA(cudaEventCreate(&e));
  }
  auto destroy_events = [&]() {
    for (auto e : ev_upd) cudaEventDestroy(e);
    for (auto e : tev) cudaEventDestroy(e);
  };
  double fl_gram_sweep = 0.0;
  for (int s = 0; s < nst; s++)
    for (int kk = pl.slot0; kk < pl.slot0 + pl.K; kk++) {
      long long bp, bq;
      blk_order_pair(a.ord, pl.nblk, pl.nsup, s, kk, &bp, &bq);
      const double kq = S.bw_h[bp] + S.bw_h[bq];
      fl_gram_sweep += 8.0 * kq * (kq + 1) * ctx->m;
    }
  std::vector<unsigned long long> k2(nst);
  GH_CUDA(cudaEventRecord(ctx->ev0, str));
  for (int sw = 0; sw < ctx->o.max_sweeps; sw++) {
    GH_CUDA(cudaMemsetAsync(ctx->cnt, 0, sizeof(DevCounters), str));
    GH_CUDA(cudaMemsetAsync(a.upd_k2, 0, (size_t)nst * 8, str));
    GH_CUDA(cudaEventRecord(ctx->ev2, str));
    for (int g = 0; g < G; g++) GH_CUDA(cudaStreamWaitEvent(ctx->grp_streams[g], ctx->ev2, 0));
    for (int s = 0; s < nst; s++) {
      const int b = s & 1;
      a.s = s;
      for (int g = 0; g < G; g++) {
        cudaStream_t sh = ctx->grp_streams[g];
        const int np = g0[g + 1] - g0[g];
        if (np <= 0) continue;
        if (s > 0) {
          if (g > 0) GH_CUDA(cudaStreamWaitEvent(sh, ev_upd[2 * (g - 1) + (b ^ 1)], 0));
          if (g + 1 < G) GH_CUDA(cudaStreamWaitEvent(sh, ev_upd[2 * (g + 1) + (b ^ 1)], 0));
        }
        a.pair0 = g0[g];
        cudaEvent_t* te = timing ? &tev[((size_t)s * G + g) * 4] : nullptr;
        if (te) GH_CUDA(cudaEventRecord(te[0], sh));
        launch_gram(S, a, np, sh);
        if (te) GH_CUDA(cudaEventRecord(te[1], sh));
        launch_factor(S, a, np, sh);
        launch_pivot(S, a, np, sh);
        if (te) GH_CUDA(cudaEventRecord(te[2], sh));
        launch_update(S, a, g0[g], np, 0, 2 * tF + tZ, 0, sh);
        if (a.W) launch_update(S, a, g0[g], np, 0, tZ, 1, sh);
        if (te) GH_CUDA(cudaEventRecord(te[3], sh));
        GH_CUDA(cudaEventRecord(ev_upd[2 * g + b], sh));
      }
      GH_CUDA(cudaGetLastError());
    }
    for (int g = 0; g < G; g++)
      if (g0[g + 1] > g0[g]) GH_CUDA(cudaStreamWaitEvent(str, ev_upd[2 * g + ((nst - 1) & 1)], 0));
    GH_CUDA(cudaEventRecord(ctx->ev3, str));
    DevCounters c;
    GH_CUDA(cudaMemcpyAsync(&c, ctx->cnt, sizeof(c), cudaMemcpyDeviceToHost, str));
    GH_CUDA(cudaMemcpyAsync(k2.data(), a.upd_k2, (size_t)nst * 8, cudaMemcpyDeviceToHost, str));
    GH_CUDA(cudaStreamSynchronize(str));
    if (c.err) {
      destroy_events();
      ctx->err = c.err == -7 ? "blocked: rank-deficient block pivot (HEBPJ)"
                 : c.err == -6 ? "blocked: indefinite / singular S block pivot"
                               : "blocked: non-finite value in a block pivot";
      return c.err == -7 ? GHSVD_E_RANK_DEFICIENT : c.err == -6 ? GHSVD_E_INDEFINITE_S : GHSVD_E_NONFINITE;
    }
    float kms = 0;
    GH_CUDA(cudaEventElapsedTime(&kms, ctx->ev2, ctx->ev3));
    st->kernel_seconds += kms * 1e-3;
    st->launches += (uint64_t)((a.W ? 4 : 3) + (S.fused ? 0 : 1)) * G * nst;
    st->flops_gram += fl_gram_sweep;
    double fl_upd_sweep = 0.0;   // only the pairs whose update ran (device count of k^2)
    for (int s = 0; s < nst; s++) fl_upd_sweep += 8.0 * (double)k2[s] * (2.0 * ctx->m + ctx->n);
    st->flops_update += fl_upd_sweep;
    st->flops_update_fg += fl_upd_sweep;   // F, G and Z' row tiles share one launch here
    st->launches_update_fg += (uint64_t)G * nst;
    if (timing) {
      for (size_t i = 0; i < tev.size(); i += 4) {
        float t0 = 0, t1 = 0, t2 = 0;
        GH_CUDA(cudaEventElapsedTime(&t0, tev[i], tev[i + 1]));
        GH_CUDA(cudaEventElapsedTime(&t1, tev[i + 1], tev[i + 2]));
        GH_CUDA(cudaEventElapsedTime(&t2, tev[i + 2], tev[i + 3]));
        st->t_gram += t0 * 1e-3;
        st->t_pivot += t1 * 1e-3;
        st->t_update += t2 * 1e-3;
        st->t_update_fg += t2 * 1e-3;
      }
    }
    if (sw < 64) {
      st->all_per_sweep[sw] = c.all;
      st->big_per_sweep[sw] = c.big;
    }
    st->sweeps = sw + 1;
    st->pairs_visited += pairs;
    st->transforms_all += c.all;
    st->transforms_big += c.big;
    {
      double off;   // max scaled off-diagonal measure over the block pivots' inner steps
      memcpy(&off, &c.off_bits, 8);
      st->max_offdiag_last = off;
    }
    if (c.big == 0) {
      st->converged = 1;
      break;
    }
  }
  GH_CUDA(cudaEventRecord(ctx->ev1, str));
  GH_CUDA(cudaEventSynchronize(ctx->ev1));
  destroy_events();
  float ms = 0;
  GH_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  st->seconds = ms * 1e-3;
  st->alg_flops = st->flops_gram + st->flops_update;
  st->nblocks = pl.nblk;
  st->super_blocks = pl.nsup;
  st->steps_per_sweep = pl.nst;
  st->alg_bytes = (uint64_t)((double)st->sweeps * pl.nst * 16.0 * (double)ctx->n *
                             (2.0 * ctx->m + 2.0 * (2.0 * ctx->m + ctx->n)));
  return GHSVD_OK;
}

ghsvd_status blk_sweep(Ctx* ctx, ghsvd_stats* st) {
  BlkSetup S;
  {
    ghsvd_status e = blk_setup(ctx, S);
    if (e) return e;
  }
  const bool multi = ctx->comm != nullptr;   // NCCL path (also exercised with one rank)
  const bool xch_overlap = multi && ctx->o.exchange_overlap != 0;
  {
    // one GPU: GHSVD_GROUPS=G >= 2 selects the pipelined pair-group schedule
    // (blk_sweep_groups; measured 1-2 % slower than the two-stream schedule below on
    // config 3, kept as an experiment)
    const int G = std::min(S.pl.K, ctx->o.groups);
    if (!multi && G >= 2 && ctx->o.ordering == GHSVD_ORDER_ROUND_ROBIN) return blk_sweep_groups(ctx, st, S, G);
  }
  BlkPlan& pl = S.pl;
  BlkArgs a = S.a;
  const std::vector<int>& bs_h = S.bs_h;
  const std::vector<int>& bw_h = S.bw_h;

  const int tF = S.tF, tZ = S.tZ;
  cudaStream_t str = ctx->stream;
  const uint64_t pairs = (uint64_t)ctx->n * (ctx->n - 1) / 2;
  GH_CUDA(cudaStreamSynchronize(str));
  const bool timing = ctx->o.detail_timing != 0;
  // detail_timing 2: only the F/G update spans (two events per half-step instead of four;
  // each event record costs ~3 us of stream time, 1.2 % of config 3 at four)
  const bool tfull = ctx->o.detail_timing == 1;
  // level 2 samples the update spans on every TSTRIDE-th block step (an unbiased estimate
  // of the average launch duration at 1/TSTRIDE of the event cost)
  const int tstride = tfull ? 1 : 8;
  // the sampled phase rotates with the sweep (step 0 of a sweep follows a host sync and
  // runs without a concurrent Z' update, so it must not be over-represented); with fewer
  // than 2 * TSTRIDE block steps every step is sampled
  int cur_sw = 0;
  const int nst_all = pl.nst;
  auto sampled = [&](int s) {
    return timing && (tstride == 1 || nst_all < 2 * tstride || s % tstride == cur_sw % tstride);
  };
  // The Z' update of step s (aux stream) overlaps the Gram + pivot of step s+1: Z is
  // touched by no other kernel, and Z_blk / applied are double-buffered by step parity.
  if (!ctx->aux_stream) GH_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
  if (!ctx->aux_stream2) GH_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream2, cudaStreamNonBlocking));
  // GHSVD_SERIAL=1: every kernel on the context stream, one launch per kind and step over
  // all block pairs -- the kernels run alone, so their CUDA-event durations are their
  // isolated durations (bench.py's roofline probe); same arithmetic, bitwise equal
  const bool serial = (ctx->o.schedule & GHSVD_SCHED_SERIAL) != 0;
  cudaStream_t aux = serial ? str : ctx->aux_stream;
  // the step's pairs are split in two halves on two streams so that one half's
  // latency-bound pivot kernel overlaps the other half's Gram / update kernels
  const int nh = (pl.K >= 2 && !serial) ? 2 : 1;
  const int KA = nh == 2 ? pl.K / 2 : pl.K;
  // Stream priorities steer the block scheduler (GHSVD_PRIO=0 disables, for comparison):
  //   highest  factor / pivot (latency-bound): their CTAs are placed as soon as a Gram
  //            or update CTA retires, so a half's block pivots start right after its
  //            own Grams instead of queueing behind the other half's Gram CTAs;
  //   medium   Gram and F, G update of both halves;
  //   lowest   the Z' update (aux): it has a whole step of slack and fills the SMs the
  //            latency-bound kernels leave idle.
  const bool prio = (ctx->o.schedule & GHSVD_SCHED_NO_PRIO) == 0 && !serial;
  cudaStream_t hs_st[2] = {str, ctx->aux_stream2};
  cudaStream_t fp_st[2] = {str, ctx->aux_stream2};
  if (prio) {
    int lo = 0, hi = 0;
    GH_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int i = 0; i < 2; i++) {
      // both halves at the same level (ranking half 0 above half 1 measured 2 % slower)
      const int mid = std::min(lo, hi + 1);
      if (!ctx->hi_stream[i]) GH_CUDA(cudaStreamCreateWithPriority(&ctx->hi_stream[i], cudaStreamNonBlocking, hi));
      if (!ctx->mid_stream[i])
        GH_CUDA(cudaStreamCreateWithPriority(&ctx->mid_stream[i], cudaStreamNonBlocking, mid));
      fp_st[i] = ctx->hi_stream[i];
      hs_st[i] = ctx->mid_stream[i];
    }
  } else {
    fp_st[0] = hs_st[0];
    fp_st[1] = hs_st[1];
  }
  const int h_pair0[2] = {0, KA}, h_np[2] = {KA, pl.K - KA};
  const int nst = pl.nst;
  std::vector<cudaEvent_t> ev_piv(2), ev_fg(2), ev_zdone(2), ev_gr(2), ev_bnd(2), tev;
  // GHSVD_SPLIT_BND=1 (experiment): split each half's F/G update into its boundary pair
  // and the rest, so half 0 of step s+1 may start while half 1 of step s still updates;
  // measured equal to the plain halves on config 3 (2.42 ms per block step either way)
  const bool split_bnd = !multi && nh == 2 && KA >= 2 && pl.K - KA >= 2 && (ctx->o.schedule & GHSVD_SCHED_SPLIT_BND) != 0 &&
                         ctx->o.ordering == GHSVD_ORDER_ROUND_ROBIN;
  // multi-GPU: does the exchange after step s move any block column?  (Inside an outer step
  // of a Level-3 ordering with one super pair per rank nothing moves: no exchange, and the
  // next step's Grams need not wait for this step's Z' update.)
  std::vector<char> moves(nst, 0);
  if (multi)
    for (int s = 0; s < nst; s++) moves[s] = comm_step_moves(ctx, pl.nblk, s, (s + 1) % nst) ? 1 : 0;
  cudaEvent_t ev_x;
  GH_CUDA(cudaEventCreateWithFlags(&ev_x, cudaEventDisableTiming));
  for (int i = 0; i < 2; i++) {
    GH_CUDA(cudaEventCreateWithFlags(&ev_gr[i], cudaEventDisableTiming));
    GH_CUDA(cudaEventCreateWithFlags(&ev_bnd[i], cudaEventDisableTiming));
    GH_CUDA(cudaEventCreateWithFlags(&ev_piv[i], cudaEventDisableTiming));
    GH_CUDA(cudaEventCreateWithFlags(&ev_fg[i], cudaEventDisableTiming));
    GH_CUDA(cudaEventCreateWithFlags(&ev_zdone[i], cudaEventDisableTiming));
  }
  if (timing) {
    tev.resize((size_t)nst * 8);
    for (auto& e : tev) GH_CUDA(cudaEventCreate(&e));
  }
  auto destroy_events = [&]() {
    for (auto e : ev_piv) cudaEventDestroy(e);
    for (auto e : ev_fg) cudaEventDestroy(e);
    for (auto e : ev_zdone) cudaEventDestroy(e);
    for (auto e : ev_gr) cudaEventDestroy(e);
    for (auto e : ev_bnd) cudaEventDestroy(e);
    for (auto e : tev) cudaEventDestroy(e);
    cudaEventDestroy(ev_x);
  };
  double2* zblk0 = a.zblk;
  double2* zinv0 = a.zinvT;
  int* applied0 = a.applied;
  // algorithmic flops per block step: Hermitian Grams k(k+1)/2 m each (every pair);
  // updates k^2 (2m+n) for the pairs whose update runs (device sum of k^2 per step)
  std::vector<double> fl_gram(nst, 0.0);
  std::vector<unsigned long long> k2(nst);
  for (int s = 0; s < nst; s++)
    for (int kk = pl.slot0; kk < pl.slot0 + pl.K; kk++) {
      long long bp, bq;
      blk_order_pair(a.ord, pl.nblk, pl.nsup, s, kk, &bp, &bq);
      const double kq = bw_h[bp] + bw_h[bq];
      fl_gram[s] += 8.0 * kq * (kq + 1) * ctx->m;
    }
  const char* trace_path = ctx->o.trace_path;
  std::vector<unsigned long long> trace_h;
  if (trace_path && *trace_path) {
    trace_h.assign((size_t)nst * TRACE_SLOTS * 2, 0);
    for (size_t i = 0; i < trace_h.size(); i += 2) trace_h[i] = ~0ull;
    GH_CUDA(cudaMemcpyAsync(S.trace_buf, trace_h.data(), trace_h.size() * 8, cudaMemcpyHostToDevice, str));
  }
  GH_CUDA(cudaEventRecord(ctx->ev0, str));
  for (int sw = 0; sw < ctx->o.max_sweeps; sw++) {
    cur_sw = sw;
    a.trace = (sw == 0 && !trace_h.empty()) ? S.trace_buf : nullptr;
    GH_CUDA(cudaMemsetAsync(ctx->cnt, 0, sizeof(DevCounters), str));
    GH_CUDA(cudaMemsetAsync(a.upd_k2, 0, (size_t)nst * 8, str));
    GH_CUDA(cudaEventRecord(ctx->ev2, str));
    for (int h = 0; h < nh; h++)
      if (hs_st[h] != str) GH_CUDA(cudaStreamWaitEvent(hs_st[h], ctx->ev2, 0));
    for (int s = 0; s < nst; s++) {
      const int b = s & 1;
      a.s = s;
      a.zblk = zblk0 + (size_t)b * pl.K * KM * KM;
      if (zinv0) a.zinvT = zinv0 + (size_t)b * pl.K * KM * KM;
      a.applied = applied0 + (size_t)b * pl.K;
      // The Grams of step s read block columns updated in step s-1 by their own half and,
      // through the round-robin neighbour structure (slot k of step s holds the block
      // columns of slots k-1 and k+1 of step s-1), by the other half's boundary pair only.
      if (nh == 2 && s > 0) {
        GH_CUDA(cudaStreamWaitEvent(hs_st[0], split_bnd ? ev_bnd[1] : ev_fg[1], 0));
        GH_CUDA(cudaStreamWaitEvent(hs_st[1], split_bnd ? ev_bnd[0] : ev_fg[0], 0));
      }
      // multi-GPU: the exchange after step s-1 (on str) precedes every Gram of step s
      if (multi && s > 0 && moves[s - 1])
        for (int h = 0; h < nh; h++)
          if (hs_st[h] != str) GH_CUDA(cudaStreamWaitEvent(hs_st[h], ev_x, 0));
      for (int h = 0; h < nh; h++) {
        cudaStream_t sh = hs_st[h];
        a.pair0 = h_pair0[h];
        if (tfull) GH_CUDA(cudaEventRecord(tev[8 * s + 4 * h + 0], sh));
        a.trace_id = s * TRACE_SLOTS + 0 + h;
        launch_gram(S, a, h_np[h], sh);
        if (tfull) GH_CUDA(cudaEventRecord(tev[8 * s + 4 * h + 1], sh));
        cudaStream_t fs = fp_st[h];
        if (fs != sh) {
          GH_CUDA(cudaEventRecord(ev_gr[h], sh));
          GH_CUDA(cudaStreamWaitEvent(fs, ev_gr[h], 0));
        }
        // Z_blk buffer b was last read by the Z update of step s-2
        if (s >= 2 || sw > 0) GH_CUDA(cudaStreamWaitEvent(fs, ev_zdone[b], 0));
        a.trace_id = s * TRACE_SLOTS + 2 + h;
        launch_factor(S, a, h_np[h], fs);
        a.trace_id = s * TRACE_SLOTS + 4 + h;
        launch_pivot(S, a, h_np[h], fs);
        GH_CUDA(cudaEventRecord(ev_piv[h], fs));
        if (fs != sh) GH_CUDA(cudaStreamWaitEvent(sh, ev_piv[h], 0));
        if (sampled(s)) GH_CUDA(cudaEventRecord(tev[8 * s + 4 * h + 2], sh));
        a.trace_id = s * TRACE_SLOTS + 6 + h;
        if (split_bnd) {
          // boundary pair first (the only pair of this half the other half's next-step
          // Grams read, by the round-robin neighbour structure), then the rest
          const int bp = h == 0 ? h_pair0[0] + h_np[0] - 1 : h_pair0[1];
          launch_update(S, a, bp, 1, 0, 2 * tF, 0, sh);
          GH_CUDA(cudaEventRecord(ev_bnd[h], sh));
          a.trace_id = s * TRACE_SLOTS + 10 + h;
          launch_update(S, a, h == 0 ? h_pair0[0] : h_pair0[1] + 1, h_np[h] - 1, 0, 2 * tF, 0, sh);
        } else {
          launch_update(S, a, h_pair0[h], h_np[h], 0, 2 * tF, 0, sh);
        }
        if (sampled(s)) GH_CUDA(cudaEventRecord(tev[8 * s + 4 * h + 3], sh));
        GH_CUDA(cudaEventRecord(ev_fg[h], sh));
      }
      // Z' update of all pairs of step s on the aux stream (overlaps step s+1)
      a.pair0 = 0;
      for (int h = 0; h < nh; h++) GH_CUDA(cudaStreamWaitEvent(aux, ev_piv[h], 0));
      a.trace_id = s * TRACE_SLOTS + 8;
      launch_update(S, a, 0, pl.K, 2 * tF, 2 * tF + tZ, 0, aux);
      a.trace_id = s * TRACE_SLOTS + 9;
      if (a.W) launch_update(S, a, 0, pl.K, 0, tZ, 1, aux);
      if (multi && xch_overlap && moves[s]) {
        // exchange_overlap = 1: the exchange after step s in two parts (NEXT-2, comm/compute
        // overlap): the Z', W block columns leave right after the Z' update, on the aux
        // stream and a second communicator, while the F, G block columns leave as soon as
        // the F, G updates of both halves are done -- the Grams of step s+1 need only F and
        // G, so they no longer wait for the Z' update of step s (which keeps overlapping
        // them, as on one GPU).  The next Z' update runs on the aux stream after the Z'
        // exchange.
        const int s_next = (s + 1) % nst;
        ghsvd_status e = comm_exchange(ctx, pl.nblk, s, s_next, bs_h.data(), bw_h.data(), XCH_ZW, aux);
        if (e) {
          destroy_events();
          return e;
        }
      }
      GH_CUDA(cudaEventRecord(ev_zdone[b], aux));
      GH_CUDA(cudaGetLastError());
      if (multi && moves[s]) {
        // default (exchange_overlap = 0): ONE communicator, one grouped exchange of the F, G,
        // Z' (and W) block columns on the context stream after every update of step s --
        // no two NCCL operations are ever in flight on different streams
        for (int h = 0; h < nh; h++)
          if (hs_st[h] != str) GH_CUDA(cudaStreamWaitEvent(str, ev_fg[h], 0));
        if (!xch_overlap) GH_CUDA(cudaStreamWaitEvent(str, ev_zdone[b], 0));
        const int s_next = (s + 1) % nst;
        ghsvd_status e = comm_exchange(ctx, pl.nblk, s, s_next, bs_h.data(), bw_h.data(),
                                       xch_overlap ? XCH_FG : XCH_FG | XCH_ZW, str);
        if (e) {
          destroy_events();
          return e;
        }
        GH_CUDA(cudaEventRecord(ev_x, str));
        if (hs_st[0] == str) GH_CUDA(cudaEventRecord(ev_fg[0], str));  // half 1 of step s+1 waits for it
      }
    }
    for (int h = 0; h < nh; h++)
      if (hs_st[h] != str) GH_CUDA(cudaStreamWaitEvent(str, ev_fg[h], 0));
    GH_CUDA(cudaStreamWaitEvent(str, ev_zdone[(nst - 1) & 1], 0));
    GH_CUDA(cudaEventRecord(ctx->ev3, str));
    DevCounters c;
    GH_CUDA(cudaMemcpyAsync(&c, ctx->cnt, sizeof(c), cudaMemcpyDeviceToHost, str));
    GH_CUDA(cudaMemcpyAsync(k2.data(), a.upd_k2, (size_t)nst * 8, cudaMemcpyDeviceToHost, str));
    GH_CUDA(cudaStreamSynchronize(str));
    if (multi) {
      ghsvd_status e = comm_allreduce_counters(ctx, &c);
      if (e) {
        destroy_events();
        return e;
      }
    }
    if (c.err) {
      destroy_events();
      ctx->err = c.err == -7 ? "blocked: rank-deficient block pivot (HEBPJ)"
                 : c.err == -6 ? "blocked: indefinite / singular S block pivot"
                               : "blocked: non-finite value in a block pivot";
      return c.err == -7 ? GHSVD_E_RANK_DEFICIENT : c.err == -6 ? GHSVD_E_INDEFINITE_S : GHSVD_E_NONFINITE;
    }
    if (sw == 0 && !trace_h.empty()) {
      GH_CUDA(cudaMemcpy(trace_h.data(), S.trace_buf, trace_h.size() * 8, cudaMemcpyDeviceToHost));
      if (FILE* f = fopen(trace_path, "w")) {
        static const char* names[12] = {"gram0", "gram1", "factor0", "factor1", "pivot0", "pivot1",
                                        "update0", "update1", "updateZ", "updateW", "update0b", "update1b"};
        unsigned long long t0 = ~0ull;
        for (size_t i = 0; i < trace_h.size(); i += 2) t0 = std::min(t0, trace_h[i]);
        fprintf(f, "step,kernel,start_ns,end_ns\n");
        for (int s = 0; s < nst; s++)
          for (int k = 0; k < 12; k++) {
            const unsigned long long b0 = trace_h[2 * ((size_t)s * TRACE_SLOTS + k)];
            const unsigned long long b1 = trace_h[2 * ((size_t)s * TRACE_SLOTS + k) + 1];
            if (b0 != ~0ull && b1 >= b0) fprintf(f, "%d,%s,%llu,%llu\n", s, names[k], b0 - t0, b1 - t0);
          }
        fclose(f);
      }
    }
    float kms = 0;
    GH_CUDA(cudaEventElapsedTime(&kms, ctx->ev2, ctx->ev3));
    st->kernel_seconds += kms * 1e-3;
    st->launches += (uint64_t)((S.fused ? 3 : 4) * nh + (split_bnd ? 2 : 0) + (a.W ? 2 : 1)) * nst;
    for (int s = 0; s < nst; s++) {
      st->flops_gram += fl_gram[s];
      st->flops_update += 8.0 * (double)k2[s] * (2.0 * ctx->m + ctx->n);
      // the *_update_fg figures cover the launches whose spans are recorded (all, or the
      // sampled steps under detail_timing 2; all when timing is off)
      if (!timing || sampled(s)) {
        st->flops_update_fg += 8.0 * (double)k2[s] * (2.0 * ctx->m);
        st->launches_update_fg += (uint64_t)(nh + (split_bnd ? 2 : 0));
      }
      if (sampled(s)) {
        for (int h = 0; h < nh; h++) {
          float t0 = 0, t1 = 0, t2 = 0;
          if (tfull) {
            GH_CUDA(cudaEventElapsedTime(&t0, tev[8 * s + 4 * h + 0], tev[8 * s + 4 * h + 1]));
            GH_CUDA(cudaEventElapsedTime(&t1, tev[8 * s + 4 * h + 1], tev[8 * s + 4 * h + 2]));
          }
          GH_CUDA(cudaEventElapsedTime(&t2, tev[8 * s + 4 * h + 2], tev[8 * s + 4 * h + 3]));
          st->t_gram += t0 * 1e-3;
          st->t_pivot += t1 * 1e-3;
          st->t_update += t2 * 1e-3;
          st->t_update_fg += t2 * 1e-3;
        }
      }
    }
    if (sw < 64) {
      st->all_per_sweep[sw] = c.all;
      st->big_per_sweep[sw] = c.big;
    }
    st->sweeps = sw + 1;
    st->pairs_visited += pairs;
    st->transforms_all += c.all;
    st->transforms_big += c.big;
    {
      double off;   // max scaled off-diagonal measure over the block pivots' inner steps
      memcpy(&off, &c.off_bits, 8);
      st->max_offdiag_last = off;
    }
    if (c.big == 0) {
      st->converged = 1;
      break;
    }
  }
  GH_CUDA(cudaEventRecord(ctx->ev1, str));
  GH_CUDA(cudaEventSynchronize(ctx->ev1));
  destroy_events();
  float ms = 0;
  GH_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  st->seconds = ms * 1e-3;
  // algorithmic flops of this rank: per block pair 8 [k(k+1) m + k^2 (2m + n)]
  st->alg_flops = st->flops_gram + st->flops_update;
  st->nblocks = pl.nblk;
  st->super_blocks = pl.nsup;
  st->steps_per_sweep = pl.nst;
  // HBM bytes the blocked sweep must move per block step: Grams read F, G pairs once,
  // updates read + write F, G, Z pairs once
  st->alg_bytes = (uint64_t)((double)st->sweeps * pl.nst / std::max(1, ctx->o.world_size) *
                             16.0 * (double)ctx->n * (2.0 * ctx->m + 2.0 * (2.0 * ctx->m + ctx->n)));
  return GHSVD_OK;
}

}  // namespace ghsvd
