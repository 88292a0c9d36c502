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
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "hebpj.cuh"
#include "hz2x2.cuh"
#include "internal.h"

namespace ghsvd {

namespace {

constexpr int KM = 64;          // max block-pivot order 2w
constexpr int RT = 32;          // rows per staged tile
constexpr int GS = RT + 2;      // Gram tile column stride (double2), conflict-free fragments
constexpr int ZS = KM + 4;      // Z_blk column stride in smem
constexpr int NT_G = 256, NT_P = 512, NT_U = 256;
constexpr int US = RT + 2;      // update tile column stride
constexpr int GSTAGES = 3;      // cp.async pipeline depth of the Gram kernel
constexpr int MAX_SPLIT = 16;   // max row splits of a Gram (partials summed in order)
constexpr int TRACE_SLOTS = 48; // trace launch slots per block step

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_wait_dyn(int n) {   // n in [0, 3]
  switch (n) {
    case 0: cp_wait<0>(); break;
    case 1: cp_wait<1>(); break;
    case 2: cp_wait<2>(); break;
    default: cp_wait<3>(); break;
  }
}

struct BlkArgs {
  double2* F;
  double2* G;
  double2* Z;
  long long ldm, ldn, m, n, npos;
  int nblk, s, slot0, npairs;
  int pair0;                // first local pair handled by this launch (blockIdx.x offset)
  const int* bstart;
  const int* bwidth;
  int nsplit;
  long long split_rows;     // rows per split (multiple of RT)
  double2* gpart;           // [pair][hs][split][KM*KM]
  double2* zblk;            // [pair][KM*KM]
  int* applied;             // [pair]
  double2* fhat;            // [pair][KM*KM]  F^ from HEBPJ
  double2* ghat;            // [pair][KM*KM]  G^ from pivoted Cholesky
  signed char* jhat;        // [pair][KM]     J^
  int* fact_ok;             // [pair][2]
  int* gcnt;                // [pair][2] finished Gram splits (reset by the last one)
  double2* zinvT;           // [pair][KM*KM] (Z_blk^{-1})^T if want_x, else nullptr
  double2* W;               // want_x: W^T = (Z'^{-1})^T (n rows, ld ldn)
  DevCounters* cnt;
  double eps;
  int literal;
  int inner_sweeps;
  unsigned long long* trace;  // GHSVD_TRACE: [launch id][first CTA start, last CTA end] (ns)
  int trace_id;
};

// Launch tracing (GHSVD_TRACE=<csv path>, first sweep only): thread 0 of every CTA
// folds %globaltimer into the launch's [min start, max end] with atomics.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_begin(const BlkArgs& a) {
  if (a.trace && threadIdx.x == 0) atomicMin(&a.trace[2 * a.trace_id], gtimer());
}
__device__ __forceinline__ void trace_end(const BlkArgs& a) {
  if (a.trace && threadIdx.x == 0) atomicMax(&a.trace[2 * a.trace_id + 1], gtimer());
}

__device__ __forceinline__ void pair_cols(const BlkArgs& a, int pl, int& c0p, int& wp, int& c0q, int& wq) {
  long long bp, bq;
  rr_pair(a.nblk, a.s, a.slot0 + pl, &bp, &bq);
  c0p = a.bstart[bp];
  wp = a.bwidth[bp];
  c0q = a.bstart[bq];
  wq = a.bwidth[bq];
}

// global column of pivot column c (c < wp: block p, else block q), -1 if padding
__device__ __forceinline__ long long gcol(int c, int c0p, int wp, int c0q, int wq) {
  if (c < wp) return c0p + c;
  if (c < wp + wq) return c0q + (c - wp);
  return -1;
}

// ---------------------------------------------------------------- block pivot
// blk_factor (run by the last Gram CTA of a (pair, H|S), see k_blk_gram): sum the split
// partials in fixed order; which = 0: H_blk -> HEBPJ -> F^ (and J^); which = 1: S_blk ->
// diagonally pivoted Cholesky -> G^.  F^, G^ go to L2-resident scratch.
constexpr int NT_F = 256;
__device__ void blk_factor(const BlkArgs& a, int pl, int which, double2* W) {
  __shared__ int np_sh;
  const int tid = threadIdx.x;
  int c0p, wp, c0q, wq;
  pair_cols(a, pl, c0p, wp, c0q, wq);
  const int k = wp + wq;
  // sum of split partials (lower triangle, fixed split order), full Hermitian in W;
  // L2 loads (__ldcg): the partials were written by other CTAs of this launch
  const double2* base = a.gpart + ((size_t)pl * 2 + which) * a.nsplit * (KM * KM);
  {
    const int warp = tid >> 5, lane = tid & 31;
    for (int j = warp; j < k; j += NT_F / 32) {
      for (int i = j + lane; i < k; i += 32) {
        double2 x[MAX_SPLIT];
#pragma unroll
        for (int sp = 0; sp < MAX_SPLIT; sp++)
          if (sp < a.nsplit) x[sp] = __ldcg(base + (size_t)sp * (KM * KM) + i + (size_t)j * KM);
        double2 v = make_double2(0, 0);
#pragma unroll
        for (int sp = 0; sp < MAX_SPLIT; sp++)
          if (sp < a.nsplit) {
            v.x += x[sp].x;
            v.y += x[sp].y;
          }
        if (i == j) v.y = 0.0;
        W[i + j * KM] = v;
        W[j + i * KM] = make_double2(v.x, -v.y);
      }
    }
  }
  __syncthreads();
  double2* out = (which == 0 ? a.fhat : a.ghat) + (size_t)pl * (KM * KM);
  int rc;
  if (which == 0) {
    // HEBPJ tolerance k * eps * max |H| (lower triangle), as the oracle
    double tv = 0.0;
    long long ti = 0;
    for (int e = tid; e < k * k; e += NT_F) {
      const int i = e % k, j = e / k;
      if (i >= j) hb::amax_merge(tv, ti, hb::cabs(W[i + j * KM]), 0);
    }
    hb::block_amax<NT_F>(tv, ti);
    const double tolz = __dmul_rn(__dmul_rn((double)k, 0x1p-53), tv);
    rc = hb::hebpj_dev<NT_F, KM>(W, k, KM, out, KM, a.jhat + (size_t)pl * KM, &np_sh, tolz);
  } else {
    rc = hb::pchol_dev<NT_F, KM>(W, k, KM, out, KM);
  }
  if (tid == 0) {
    a.fact_ok[pl * 2 + which] = rc == 0;
    if (rc) atomicCAS(&a.cnt->err, 0, which == 0 ? -7 : -6);
  }
}

// ---------------------------------------------------------------- Gram (DMMA)
// One CTA = one (row split, H|S, pair) (grid x = split fastest, so a pair's splits run
// together and pairs complete progressively).  The 36 lower-triangle 8x8 output tiles of the
// k x k Gram (k <= 64) are grouped by tile-row pairs {I, 7-I} (9 tiles each); warps
// 2g, 2g+1 own group g and split every 32-row stage's 8 k-steps (even / odd).  Within
// a k-step a warp loads the 8-g column fragments its 9 tiles need once (the A fragment
// of tile row I is the B fragment of tile column I) and issues 36 DMMAs (exact 4M
// complex product; J folded into the A operand).  The two k-halves are summed in a
// fixed order at the end, so the result is deterministic.
template <int GI>
__device__ __forceinline__ void gram_tiles(const double2* T, int row, double sg, double (&acc)[9][4]) {
  constexpr int IA = GI, IB = 7 - GI, NF = 8 - GI;
  const int lane = threadIdx.x & 31;
  double2 f[NF];
#pragma unroll
  for (int j = 0; j < NF; j++) f[j] = T[(8 * j + (lane >> 2)) * GS + row];
  // A operand of tile rows IA, IB: J_r conj(x): (ar, ai) with conj -> (+x.y used as -(-x.y))
  const double aar = sg * f[IA].x, aai = sg * f[IA].y;
  const double abr = sg * f[IB].x, abi = sg * f[IB].y;
#pragma unroll
  for (int t = 0; t < 9; t++) {
    const bool ra = t <= IA;
    const int J = ra ? t : t - IA - 1;
    const double ar = ra ? aar : abr, ai = ra ? aai : abi;
    const double2 y = f[J];
    // conj(x) y = (xr yr + xi yi) + i (xr yi - xi yr)
    dmma(acc[t][0], acc[t][1], ar, y.x);
    dmma(acc[t][0], acc[t][1], ai, y.y);
    dmma(acc[t][2], acc[t][3], ar, y.y);
    dmma(acc[t][2], acc[t][3], -ai, y.x);
  }
}

// 3M variant (default; GHSVD_GRAM3M=0 selects the 4M path above): of the 9 tiles of group
// g, warp 2g owns tiles 0-3 and warp 2g+1 tiles 5-8 for every k-step, and tile 4 is
// split by k-step parity (even: warp 2g, odd: warp 2g+1; its two partial sums are added
// in a fixed order at the end), so every warp does exactly 4.5 tiles per k-step.  Per
// k-step a warp loads the fragments its tiles need and issues 3 DMMAs per tile:
// P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi); Re = P1 - P2, Im = P3 - P1 - P2
// (A = J conj(X)^T, B = X).
template <int GI>
struct G3 {
  static constexpr int IA = GI, IB = 7 - GI;
  static constexpr int row(int t) { return t <= IA ? IA : IB; }
  static constexpr int col(int t) { return t <= IA ? t : t - IA - 1; }
  // tile of accumulator slot u (0..4) of warp half H; slot 4 is the shared tile 4
  static constexpr int tile(int H, int u) { return u == 4 ? 4 : (H ? 5 + u : u); }
  static constexpr bool needB(int H, bool w4, int j) {
    bool r = false;
    for (int u = 0; u < 5; u++) r = r || ((u < 4 || w4) && col(tile(H, u)) == j);
    return r;
  }
  static constexpr bool needA(int H, bool w4, int i) {
    bool r = false;
    for (int u = 0; u < 5; u++) r = r || ((u < 4 || w4) && row(tile(H, u)) == i);
    return r;
  }
};

template <int GI, int H, bool W4>
__device__ __forceinline__ void gram3_tiles(const double2* T, int row, double sg, double (&acc)[5][6]) {
  using C = G3<GI>;
  const int lane = threadIdx.x & 31;
  double2 f[8];
  double bs[8];
#pragma unroll
  for (int j = 0; j < 8; j++) {
    if (C::needB(H, W4, j) || C::needA(H, W4, j)) f[j] = T[(8 * j + (lane >> 2)) * GS + row];
    if (C::needB(H, W4, j)) bs[j] = f[j].x + f[j].y;
  }
  double ar[2] = {0, 0}, ai[2] = {0, 0}, as[2] = {0, 0};   // rows IA, IB
  if (C::needA(H, W4, C::IA)) {
    ar[0] = sg * f[C::IA].x;
    ai[0] = -(sg * f[C::IA].y);
    as[0] = ar[0] + ai[0];
  }
  if (C::needA(H, W4, C::IB)) {
    ar[1] = sg * f[C::IB].x;
    ai[1] = -(sg * f[C::IB].y);
    as[1] = ar[1] + ai[1];
  }
#pragma unroll
  for (int u = 0; u < 5; u++) {
    if (u == 4 && !W4) continue;
    const int t = C::tile(H, u);
    const int r = C::row(t) == C::IA ? 0 : 1, J = C::col(t);
    dmma(acc[u][0], acc[u][1], ar[r], f[J].x);
    dmma(acc[u][2], acc[u][3], ai[r], f[J].y);
    dmma(acc[u][4], acc[u][5], as[r], bs[J]);
  }
}

template <int GI, int H>
__device__ __forceinline__ void gram3_store(double2* out, const double (&acc)[5][6], int nslots) {
  using C = G3<GI>;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < 5; u++) {
    if (u >= nslots) continue;
    const double* c = acc[u];
    const int t = C::tile(H, u);
    const int i = 8 * C::row(t) + (lane >> 2), j = 8 * C::col(t) + 2 * (lane & 3);
    out[i + (size_t)j * KM] = make_double2(c[0] - c[2], c[4] - c[0] - c[2]);
    out[i + (size_t)(j + 1) * KM] = make_double2(c[1] - c[3], c[5] - c[1] - c[3]);
  }
}

template <bool M3>
__global__ void __launch_bounds__(NT_G, 2) k_blk_gram(BlkArgs a) {
  trace_begin(a);
  extern __shared__ __align__(128) double2 gsm[];  // [GSTAGES][KM][GS]
  const int pl = a.pair0 + blockIdx.z, hs = blockIdx.y, split = blockIdx.x;
  int c0p, wp, c0q, wq;
  pair_cols(a, pl, c0p, wp, c0q, wq);
  const double2* X = hs == 0 ? a.F : a.G;
  const long long r_begin = (long long)split * a.split_rows;
  const long long r_end = min(a.m, r_begin + a.split_rows);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gi = warp >> 1, kh = warp & 1;
  auto load_stage = [&](int st, long long r0) {
    if (r0 < r_end) {
      double2* T = gsm + (size_t)st * KM * GS;
      for (int e = tid; e < KM * RT; e += NT_G) {
        const int c = e / RT, r = e % RT;
        const long long gc = gcol(c, c0p, wp, c0q, wq);
        const long long gr = r0 + r;
        const bool ok = gc >= 0 && gr < r_end;
        cp_async16(&T[c * GS + r], ok ? (const void*)(X + gc * a.ldm + gr) : (const void*)X, ok);
      }
    }
    cp_commit();   // possibly empty: keeps one group per stage
  };
  // GSTAGES-deep cp.async pipeline over the split's 32-row stages; consume(T, r0).
  // One barrier per stage: after it every warp has finished the previous stage, whose
  // buffer is then refilled with the stage GSTAGES-1 ahead.
  auto pipeline = [&](auto&& consume) {
#pragma unroll
    for (int p = 0; p < GSTAGES - 1; p++) load_stage(p, r_begin + (long long)p * RT);
    int st = 0;
    for (long long r0 = r_begin; r0 < r_end; r0 += RT) {
      cp_wait<GSTAGES - 2>();
      __syncthreads();
      load_stage((st + GSTAGES - 1) % GSTAGES, r0 + (long long)(GSTAGES - 1) * RT);
      consume(gsm + (size_t)st * KM * GS, r0);
      st = (st + 1) % GSTAGES;
    }
    cp_wait<0>();
    __syncthreads();
  };
  double2* out = a.gpart + (((size_t)pl * 2 + hs) * a.nsplit + split) * (KM * KM);
  if constexpr (M3) {
    double acc[5][6];
#pragma unroll
    for (int t = 0; t < 5; t++)
#pragma unroll
      for (int c = 0; c < 6; c++) acc[t][c] = 0.0;
    pipeline([&](const double2* T, long long r0) {
      // not unrolled: the warp-specialized tile sets are already 16 code paths, and
      // unrolling them overflowed the instruction cache (ncu: 22 % no_inst stalls)
#pragma unroll 1
      for (int ks = 0; ks < RT / 4; ks += 2) {
        const int row0 = 4 * ks + (lane & 3), row1 = row0 + 4;
        const double sg0 = (hs == 0 && r0 + row0 >= a.npos) ? -1.0 : 1.0;
        const double sg1 = (hs == 0 && r0 + row1 >= a.npos) ? -1.0 : 1.0;
        switch (warp) {   // warp-uniform; tile 4 on even k-steps for h = 0, odd for h = 1
#define G3CASE(W, GI, H)                                       \
  case W:                                                      \
    gram3_tiles<GI, H, H == 0>(T, row0, sg0, acc);             \
    gram3_tiles<GI, H, H == 1>(T, row1, sg1, acc);             \
    break;
          G3CASE(0, 0, 0) G3CASE(1, 0, 1) G3CASE(2, 1, 0) G3CASE(3, 1, 1)
          G3CASE(4, 2, 0) G3CASE(5, 2, 1) G3CASE(6, 3, 0) default: G3CASE(7, 3, 1)
#undef G3CASE
        }
      }
    });
    // tile 4 of every group: warp 2g+1 hands its odd-k-step partial to warp 2g
    double* red = reinterpret_cast<double*>(gsm);
    if (kh) {
#pragma unroll
      for (int c = 0; c < 6; c++) red[(gi * 6 + c) * 32 + lane] = acc[4][c];
    }
    __syncthreads();
    if (!kh) {
#pragma unroll
      for (int c = 0; c < 6; c++) acc[4][c] += red[(gi * 6 + c) * 32 + lane];
    }
    const int nslots = kh ? 4 : 5;
    switch (warp) {
      case 0: gram3_store<0, 0>(out, acc, nslots); break;
      case 1: gram3_store<0, 1>(out, acc, nslots); break;
      case 2: gram3_store<1, 0>(out, acc, nslots); break;
      case 3: gram3_store<1, 1>(out, acc, nslots); break;
      case 4: gram3_store<2, 0>(out, acc, nslots); break;
      case 5: gram3_store<2, 1>(out, acc, nslots); break;
      case 6: gram3_store<3, 0>(out, acc, nslots); break;
      default: gram3_store<3, 1>(out, acc, nslots); break;
    }
  } else {
    double acc[9][4];
#pragma unroll
    for (int t = 0; t < 9; t++) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.0;
    pipeline([&](const double2* T, long long r0) {
#pragma unroll 1
      for (int ks = 0; ks < RT / 4; ks += 2) {
        const int row = 4 * (ks + kh) + (lane & 3);
        const double sg = (hs == 0 && r0 + row >= a.npos) ? -1.0 : 1.0;
        switch (gi) {   // warp-uniform
          case 0: gram_tiles<0>(T, row, sg, acc); break;
          case 1: gram_tiles<1>(T, row, sg, acc); break;
          case 2: gram_tiles<2>(T, row, sg, acc); break;
          default: gram_tiles<3>(T, row, sg, acc); break;
        }
      }
    });
    // sum the two k-halves: odd warp -> smem -> even warp (fixed order)
    double* red = reinterpret_cast<double*>(gsm);
    if (kh) {
#pragma unroll
      for (int t = 0; t < 9; t++)
#pragma unroll
        for (int c = 0; c < 4; c++) red[((gi * 9 + t) * 4 + c) * 32 + lane] = acc[t][c];
    }
    __syncthreads();
    if (!kh) {
#pragma unroll
      for (int t = 0; t < 9; t++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[t][c] += red[((gi * 9 + t) * 4 + c) * 32 + lane];
#pragma unroll
      for (int t = 0; t < 9; t++) {
        const int I = t <= gi ? gi : 7 - gi;
        const int J = t <= gi ? t : t - gi - 1;
        const int i = 8 * I + (lane >> 2), j = 8 * J + 2 * (lane & 3);
        out[i + (size_t)j * KM] = make_double2(acc[t][0], acc[t][2]);
        out[i + (size_t)(j + 1) * KM] = make_double2(acc[t][1], acc[t][3]);
      }
    }
  }
  // The last CTA of this (pair, H|S) to finish factorizes the summed Gram right away
  // (threadfence-reduction pattern): no separate launch, and a pair's block pivot is
  // formed while the Grams of later pairs are still streaming.
  __shared__ int last_sh;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int t = atomicAdd(&a.gcnt[pl * 2 + hs], 1);
    last_sh = t == a.nsplit - 1;
    if (last_sh) a.gcnt[pl * 2 + hs] = 0;   // ready for the next block step
  }
  __syncthreads();
  if (last_sh) {
    __threadfence();
    blk_factor(a, pl, hs, gsm);
  }
  trace_end(a);
}

// (Z_blk^{-1})^T for the W^T update (NEXT-1): Gauss-Jordan with partial pivoting on
// [Fh | Gh] = [Z_blk | I] (kb x kb active, ld KM, in shared memory), transposed into wo.
template <int NT>
__device__ void gj_inverse_T(double2* Fh, double2* Gh, int kb, double2* wo) {
  __shared__ int piv_sh;
  const int tid = threadIdx.x;
  __syncthreads();
  for (int c = 0; c < kb; c++) {
    if (tid == 0) {
      int pv = c;
      double best = -1.0;
      for (int i = c; i < kb; i++) {
        const double2 v = Fh[i + c * KM];
        const double av = v.x * v.x + v.y * v.y;
        if (av > best) { best = av; pv = i; }
      }
      piv_sh = pv;
    }
    __syncthreads();
    const int pv = piv_sh;
    if (pv != c) {
      for (int j = tid; j < KM; j += NT) {
        double2 t = Fh[c + j * KM]; Fh[c + j * KM] = Fh[pv + j * KM]; Fh[pv + j * KM] = t;
        t = Gh[c + j * KM]; Gh[c + j * KM] = Gh[pv + j * KM]; Gh[pv + j * KM] = t;
      }
      __syncthreads();
    }
    const double2 d = Fh[c + c * KM];
    const double dd = d.x * d.x + d.y * d.y;
    const double2 inv = make_double2(d.x / dd, -d.y / dd);
    __syncthreads();
    for (int j = tid; j < KM; j += NT) {   // scale row c
      const double2 f = Fh[c + j * KM], g = Gh[c + j * KM];
      Fh[c + j * KM] = make_double2(f.x * inv.x - f.y * inv.y, f.x * inv.y + f.y * inv.x);
      Gh[c + j * KM] = make_double2(g.x * inv.x - g.y * inv.y, g.x * inv.y + g.y * inv.x);
    }
    __syncthreads();
    for (int e = tid; e < kb * KM; e += NT) {   // eliminate column c from the other rows
      const int i = e % kb, j = e / kb;
      if (i == c) continue;
      const double2 f = Fh[i + c * KM];
      const double2 rf = Fh[c + j * KM], rg = Gh[c + j * KM];
      const double2 uf = make_double2(f.x * rf.x - f.y * rf.y, f.x * rf.y + f.y * rf.x);
      const double2 ug = make_double2(f.x * rg.x - f.y * rg.y, f.x * rg.y + f.y * rg.x);
      if (j != c) Fh[i + j * KM] = make_double2(Fh[i + j * KM].x - uf.x, Fh[i + j * KM].y - uf.y);
      Gh[i + j * KM] = make_double2(Gh[i + j * KM].x - ug.x, Gh[i + j * KM].y - ug.y);
    }
    __syncthreads();
    for (int i = tid; i < kb; i += NT)
      if (i != c) Fh[i + c * KM] = make_double2(0.0, 0.0);
    __syncthreads();
  }
  for (int e = tid; e < KM * KM; e += NT) {
    const int i = e % KM, j = e / KM;
    wo[e] = Gh[j + i * KM];   // transpose (no conjugation)
  }
}

// k_blk_pivot: one CTA per pair: F^, G^, J^ -> shared memory, border to even order
// (Sec 6.3.2), inner Level-1 sweep(s) accumulating Z_blk.
__global__ void __launch_bounds__(NT_P, 1) k_blk_pivot(BlkArgs a) {
  trace_begin(a);
  extern __shared__ __align__(128) double2 psm[];  // W0 (Z_blk) | F^ | G^  (KM*KM each)
  double2* W0 = psm;
  double2* Fh = psm + KM * KM;
  double2* Gh = psm + 2 * KM * KM;
  __shared__ signed char Jh[KM];
  __shared__ unsigned long long cnt_all, cnt_big, sweep_all;
  __shared__ int err_sh;
  const int pl = a.pair0 + blockIdx.x, tid = threadIdx.x;
  int c0p, wp, c0q, wq;
  pair_cols(a, pl, c0p, wp, c0q, wq);
  const int k = wp + wq;
  const int kb = k + (k & 1);
  if (!a.fact_ok[2 * pl] || !a.fact_ok[2 * pl + 1]) {
    if (tid == 0) a.applied[pl] = 0;
    trace_end(a);
    return;
  }
  if (tid == 0) {
    cnt_all = cnt_big = sweep_all = 0;
    err_sh = 0;
  }
  const double2* fsrc = a.fhat + (size_t)pl * (KM * KM);
  const double2* gsrc = a.ghat + (size_t)pl * (KM * KM);
  for (int e = tid; e < KM * KM; e += NT_P) {
    const int i = e % KM, j = e / KM;
    const bool in = i < k && j < k;
    Fh[e] = in ? fsrc[e] : make_double2(0, 0);
    Gh[e] = in ? gsrc[e] : make_double2(0, 0);
    W0[e] = make_double2(i == j ? 1.0 : 0.0, 0.0);   // Z_blk = I
  }
  for (int i = tid; i < KM; i += NT_P) Jh[i] = i < k ? a.jhat[(size_t)pl * KM + i] : (signed char)1;
  __syncthreads();
  // border to even order (Sec 6.3.2)
  if (tid == 0 && kb != k) {
    Fh[k + k * KM] = make_double2(1, 0);
    Gh[k + k * KM] = make_double2(1, 0);
    Jh[k] = 1;
  }
  __syncthreads();
  // inner Level-1 sweeps.  Per inner step: one HALF-warp per pivot pair forms the 8 pair
  // Gram entries (eq 6.1) -> shared memory; warp 0 then evaluates the kb/2 <= 32 2x2
  // transforms of the step one per LANE (the scalar routine runs once per pair instead
  // of once per half-warp, which cuts the step's issued instructions several-fold);
  // the half-warps then apply them to the column pairs of F^, G^ and Z_blk.
  __shared__ double gsh[KM / 2][8];
  __shared__ double zsh[KM / 2][8];
  __shared__ int ksh[KM / 2];
  __shared__ double Jd[KM];
  for (int i = tid; i < KM; i += NT_P) Jd[i] = (double)Jh[i];
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int hw = lane >> 4, hl = lane & 15;
  const unsigned hmask = hw ? 0xffff0000u : 0x0000ffffu;
  const double tol = a.eps * sqrt((double)kb);       // C-7: n = block-pivot order
  unsigned long long w0_all = 0, w0_big = 0;          // warp-0 lane counters
  double w0_off = 0.0;                                 // warp-0 lane max off-measure
  const int pr = 2 * warp + hw;                        // this half-warp's pivot pair slot
  const int b3 = (hl >> 3) & 1, b2 = (hl >> 2) & 1, b1 = (hl >> 1) & 1;
  for (int sw = 0; sw < a.inner_sweeps; sw++) {
    unsigned long long sw_all = 0, sw_big = 0;
    for (int s = 0; s < kb - 1; s++) {
      int p = 0, q = 0;
      if (pr < kb / 2) {
        rr_pair32(kb, s, pr, &p, &q);
        // rows >= kb of F^, G^ are zero, so all KM rows are summed without guards
        double g[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int t = 0; t < KM / 16; t++) {
          const int i = hl + 16 * t;
          const double2 fp = Fh[i + p * KM], fq = Fh[i + q * KM], gpp = Gh[i + p * KM], gq = Gh[i + q * KM];
          const double sg = Jd[i];
          g[0] += sg * (fp.x * fp.x + fp.y * fp.y);
          g[1] += sg * (fq.x * fq.x + fq.y * fq.y);
          g[2] += sg * (fp.x * fq.x + fp.y * fq.y);
          g[3] += sg * (fp.x * fq.y - fp.y * fq.x);
          g[4] += gpp.x * gpp.x + gpp.y * gpp.y;
          g[5] += gq.x * gq.x + gq.y * gq.y;
          g[6] += gpp.x * gq.x + gpp.y * gq.y;
          g[7] += gpp.x * gq.y - gpp.y * gq.x;
        }
        // transpose-reduce of the 8 sums over the 16 lanes: after the offsets 8, 4, 2
        // every lane keeps one value index (hl >> 1), offset 1 completes the sum
        double h4[4], h2[2];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const double snd = b3 ? g[j] : g[j + 4];
          const double kep = b3 ? g[j + 4] : g[j];
          h4[j] = kep + __shfl_xor_sync(hmask, snd, 8);
        }
#pragma unroll
        for (int j = 0; j < 2; j++) {
          const double snd = b2 ? h4[j] : h4[j + 2];
          const double kep = b2 ? h4[j + 2] : h4[j];
          h2[j] = kep + __shfl_xor_sync(hmask, snd, 4);
        }
        double w = (b1 ? h2[1] : h2[0]) + __shfl_xor_sync(hmask, b1 ? h2[0] : h2[1], 2);
        w += __shfl_xor_sync(hmask, w, 1);
        if (!(hl & 1)) gsh[pr][hl >> 1] = w;
      }
      __syncthreads();
      if (warp == 0 && lane < kb / 2) {
        const HZOut z = hz2x2_core(gsh[lane], tol, a.literal);
        zsh[lane][0] = z.z11.re; zsh[lane][1] = z.z11.im; zsh[lane][2] = z.z21.re; zsh[lane][3] = z.z21.im;
        zsh[lane][4] = z.z12.re; zsh[lane][5] = z.z12.im; zsh[lane][6] = z.z22.re; zsh[lane][7] = z.z22.im;
        ksh[lane] = z.kind;
        w0_off = fmax(w0_off, z.off);   // scaled off-diagonal measure (a5 diagnostic)
        if (z.kind < 0) atomicCAS(&err_sh, 0, z.kind);
        if (z.kind == KIND_SMALL || z.kind == KIND_BIG) {
          sw_all++;
          if (z.kind == KIND_BIG) sw_big++;
        }
      }
      __syncthreads();
      if (pr < kb / 2) {
        const int kind = ksh[pr];
        if (kind == KIND_SMALL || kind == KIND_BIG) {
          const double2 z11 = make_double2(zsh[pr][0], zsh[pr][1]), z21 = make_double2(zsh[pr][2], zsh[pr][3]);
          const double2 z12 = make_double2(zsh[pr][4], zsh[pr][5]), z22 = make_double2(zsh[pr][6], zsh[pr][7]);
          auto rot = [&](double2* M) {
#pragma unroll
            for (int t = 0; t < KM / 16; t++) {
              const int i = hl + 16 * t;
              const double2 x = M[i + p * KM], y = M[i + q * KM];
              M[i + p * KM] = make_double2(x.x * z11.x - x.y * z11.y + y.x * z21.x - y.y * z21.y,
                                           x.x * z11.y + x.y * z11.x + y.x * z21.y + y.y * z21.x);
              M[i + q * KM] = make_double2(x.x * z12.x - x.y * z12.y + y.x * z22.x - y.y * z22.y,
                                           x.x * z12.y + x.y * z12.x + y.x * z22.y + y.y * z22.x);
            }
          };
          rot(Fh);
          rot(Gh);
          rot(W0);
        }
      }
      __syncthreads();
    }
    w0_all += sw_all;
    w0_big += sw_big;
    // per-sweep totals; FB stops on a sweep without transformations (C-3)
    if (warp == 0) {
      unsigned long long t = sw_all;
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) sweep_all = t;
    }
    __syncthreads();
    const unsigned long long this_sweep = sweep_all;
    __syncthreads();
    if (this_sweep == 0) break;
  }
  if (warp == 0) {
    for (int o = 16; o > 0; o >>= 1) {
      w0_all += __shfl_xor_sync(0xffffffffu, w0_all, o);
      w0_big += __shfl_xor_sync(0xffffffffu, w0_big, o);
      w0_off = fmax(w0_off, __shfl_xor_sync(0xffffffffu, w0_off, o));
    }
    if (lane == 0) atomicMax(&a.cnt->off_bits, (unsigned long long)__double_as_longlong(w0_off));
    if (lane == 0) {
      cnt_all = w0_all;
      cnt_big = w0_big;
    }
  }
  __syncthreads();
  if (err_sh) {
    if (tid == 0) atomicCAS(&a.cnt->err, 0, err_sh);
  }
  double2* zo = a.zblk + (size_t)pl * (KM * KM);
  for (int e = tid; e < KM * KM; e += NT_P) zo[e] = W0[e];
  if (tid == 0) {
    a.applied[pl] = cnt_all > 0;
    atomicAdd(&a.cnt->all, cnt_all);
    atomicAdd(&a.cnt->big, cnt_big);
  }
  if (a.zinvT && cnt_all > 0) {
    // NEXT-1: (Z_blk^{-1})^T for the W^T update, Gauss-Jordan with partial pivoting on
    // [Fh | Gh] = [Z_blk | I] (F^, G^ are no longer needed after the inner sweep)
    __syncthreads();
    for (int e = tid; e < KM * KM; e += NT_P) {
      const int i = e % KM, j = e / KM;
      Fh[e] = W0[e];
      Gh[e] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    }
    gj_inverse_T<NT_P>(Fh, Gh, kb, a.zinvT + (size_t)pl * (KM * KM));
  }
  trace_end(a);
}

// k_blk_pivot_cl (option GHSVD_PIVOT_CL=1; default k_blk_pivot above): the
// same inner sweep on a cluster of two CTAs that split the KM rows of F^, G^ and Z_blk
// (32 rows each, 96 KB of shared memory, 256 threads), so a pivot no longer fills an SM
// alone and a Gram or update CTA can run beside it.  Per inner step each CTA forms the 8
// pair-Gram partial sums over its rows (8 lanes per pivot pair, transpose-reduce),
// writes them to both CTAs' shared memory (DSMEM, double-buffered by step parity), one
// cluster barrier, then warp 0 of each CTA sums rank 0 + rank 1 (fixed order: both CTAs
// hold bitwise the same pivot sums) and evaluates the <= 32 transforms one per lane, and
// each CTA rotates its own rows.  Measured on config 3: 266 us alone against 319 us for
// k_blk_pivot, but inside the overlapped block step the co-resident Gram / update CTAs
// share its FP64 pipe and issue slots, the pivots stretch to 370-460 us and the step
// period grows 2.43 -> 2.49 ms, so it is not the default.
constexpr int NT_PC = 256, RB = KM / 2;
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT_PC, 1) k_blk_pivot_cl(BlkArgs a) {
  trace_begin(a);
  namespace cgx = cooperative_groups;
  cgx::cluster_group cluster = cgx::this_cluster();
  const int rank = (int)cluster.block_rank();
  extern __shared__ __align__(128) double2 qsm[];   // W0 | F^ | G^ : local rows, [KM cols][RB]
  double2* W0 = qsm;
  double2* Fh = qsm + KM * RB;
  double2* Gh = qsm + 2 * KM * RB;
  __shared__ double Jd[RB];
  __shared__ double parts[2][2][KM / 2][8];   // [step parity][source rank][pair][value]
  __shared__ double zsh[KM / 2][8];
  __shared__ int ksh[KM / 2];
  __shared__ unsigned long long sweep_all_sh;
  const int pl = a.pair0 + blockIdx.x / 2, tid = threadIdx.x;
  int c0p, wp, c0q, wq;
  pair_cols(a, pl, c0p, wp, c0q, wq);
  const int k = wp + wq;
  const int kb = k + (k & 1);
  if (!a.fact_ok[2 * pl] || !a.fact_ok[2 * pl + 1]) {   // uniform over the cluster
    if (tid == 0 && rank == 0) a.applied[pl] = 0;
    trace_end(a);
    return;
  }
  const int row0 = rank * RB;
  const double2* fsrc = a.fhat + (size_t)pl * (KM * KM);
  const double2* gsrc = a.ghat + (size_t)pl * (KM * KM);
  for (int e = tid; e < KM * RB; e += NT_PC) {
    const int il = e % RB, j = e / RB, i = row0 + il;
    const bool in = i < k && j < k;
    Fh[e] = in ? fsrc[i + j * KM] : make_double2(0, 0);
    Gh[e] = in ? gsrc[i + j * KM] : make_double2(0, 0);
    W0[e] = make_double2(i == j ? 1.0 : 0.0, 0.0);   // Z_blk = I
  }
  for (int il = tid; il < RB; il += NT_PC) {
    const int i = row0 + il;
    Jd[il] = i < k ? (double)a.jhat[(size_t)pl * KM + i] : 1.0;
  }
  __syncthreads();
  // border to even order (Sec 6.3.2): row/column k in the CTA holding row k
  if (tid == 0 && kb != k && k >= row0 && k < row0 + RB) {
    Fh[(k - row0) + k * RB] = make_double2(1, 0);
    Gh[(k - row0) + k * RB] = make_double2(1, 0);
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int pr = 4 * warp + (lane >> 3);   // pivot pair slot of this 8-lane group
  const int l8 = lane & 7;
  const unsigned gmask = 0xffu << (lane & 24);
  const int b2 = (l8 >> 2) & 1, b1 = (l8 >> 1) & 1, b0 = l8 & 1;
  const double tol = a.eps * sqrt((double)kb);        // C-7: n = block-pivot order
  unsigned long long w0_all = 0, w0_big = 0;
  double w0_off = 0.0;
  int err_local = 0;
  double* peer_parts = cluster.map_shared_rank(&parts[0][0][0][0], rank ^ 1);
  int sp = 0;   // global inner-step parity
  for (int sw = 0; sw < a.inner_sweeps; sw++) {
    unsigned long long sw_all = 0, sw_big = 0;
    for (int s = 0; s < kb - 1; s++, sp ^= 1) {
      int p = 0, q = 0;
      if (pr < kb / 2) {
        rr_pair32(kb, s, pr, &p, &q);
        double g[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int t = 0; t < RB / 8; t++) {
          const int i = l8 + 8 * t;
          const double2 fp = Fh[i + p * RB], fq = Fh[i + q * RB], gpp = Gh[i + p * RB], gq = Gh[i + q * RB];
          const double sg = Jd[i];
          g[0] += sg * (fp.x * fp.x + fp.y * fp.y);
          g[1] += sg * (fq.x * fq.x + fq.y * fq.y);
          g[2] += sg * (fp.x * fq.x + fp.y * fq.y);
          g[3] += sg * (fp.x * fq.y - fp.y * fq.x);
          g[4] += gpp.x * gpp.x + gpp.y * gpp.y;
          g[5] += gq.x * gq.x + gq.y * gq.y;
          g[6] += gpp.x * gq.x + gpp.y * gq.y;
          g[7] += gpp.x * gq.y - gpp.y * gq.x;
        }
        // transpose-reduce over the 8 lanes: lane l8 ends with the sum of value l8
        double h4[4], h2[2];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const double snd = b2 ? g[j] : g[j + 4];
          const double kep = b2 ? g[j + 4] : g[j];
          h4[j] = kep + __shfl_xor_sync(gmask, snd, 4);
        }
#pragma unroll
        for (int j = 0; j < 2; j++) {
          const double snd = b1 ? h4[j] : h4[j + 2];
          const double kep = b1 ? h4[j + 2] : h4[j];
          h2[j] = kep + __shfl_xor_sync(gmask, snd, 2);
        }
        const double w = (b0 ? h2[1] : h2[0]) + __shfl_xor_sync(gmask, b0 ? h2[0] : h2[1], 1);
        parts[sp][rank][pr][l8] = w;
        peer_parts[((sp * 2 + rank) * (KM / 2) + pr) * 8 + l8] = w;
      }
      cluster.sync();   // both CTAs' partial sums of this step are in place
      if (warp == 0 && lane < kb / 2) {
        double gs[8];
#pragma unroll
        for (int c = 0; c < 8; c++) gs[c] = parts[sp][0][lane][c] + parts[sp][1][lane][c];
        const HZOut z = hz2x2_core(gs, tol, a.literal);
        zsh[lane][0] = z.z11.re; zsh[lane][1] = z.z11.im; zsh[lane][2] = z.z21.re; zsh[lane][3] = z.z21.im;
        zsh[lane][4] = z.z12.re; zsh[lane][5] = z.z12.im; zsh[lane][6] = z.z22.re; zsh[lane][7] = z.z22.im;
        ksh[lane] = z.kind;
        w0_off = fmax(w0_off, z.off);
        if (z.kind < 0 && !err_local) err_local = z.kind;
        if (z.kind == KIND_SMALL || z.kind == KIND_BIG) {
          sw_all++;
          if (z.kind == KIND_BIG) sw_big++;
        }
      }
      __syncthreads();
      if (pr < kb / 2) {
        const int kind = ksh[pr];
        if (kind == KIND_SMALL || kind == KIND_BIG) {
          const double2 z11 = make_double2(zsh[pr][0], zsh[pr][1]), z21 = make_double2(zsh[pr][2], zsh[pr][3]);
          const double2 z12 = make_double2(zsh[pr][4], zsh[pr][5]), z22 = make_double2(zsh[pr][6], zsh[pr][7]);
          auto rot = [&](double2* M) {
#pragma unroll
            for (int t = 0; t < RB / 8; t++) {
              const int i = l8 + 8 * t;
              const double2 x = M[i + p * RB], y = M[i + q * RB];
              M[i + p * RB] = make_double2(x.x * z11.x - x.y * z11.y + y.x * z21.x - y.y * z21.y,
                                           x.x * z11.y + x.y * z11.x + y.x * z21.y + y.y * z21.x);
              M[i + q * RB] = make_double2(x.x * z12.x - x.y * z12.y + y.x * z22.x - y.y * z22.y,
                                           x.x * z12.y + x.y * z12.x + y.x * z22.y + y.y * z22.x);
            }
          };
          rot(Fh);
          rot(Gh);
          rot(W0);
        }
      }
      __syncthreads();
    }
    w0_all += sw_all;
    w0_big += sw_big;
    // per-sweep totals (identical in both CTAs); FB stops on a sweep without transformations
    if (warp == 0) {
      unsigned long long t = sw_all;
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) sweep_all_sh = t;
    }
    __syncthreads();
    if (sweep_all_sh == 0) break;
  }
  double2* zo = a.zblk + (size_t)pl * (KM * KM);
  for (int e = tid; e < KM * RB; e += NT_PC) {   // zeros outside k x k (border, padding)
    const int il = e % RB, j = e / RB, i = row0 + il;
    zo[i + j * KM] = (i < k && j < k) ? W0[e] : make_double2(0.0, 0.0);
  }
  if (warp == 0 && rank == 0) {
    for (int o = 16; o > 0; o >>= 1) {
      w0_all += __shfl_xor_sync(0xffffffffu, w0_all, o);
      w0_big += __shfl_xor_sync(0xffffffffu, w0_big, o);
      w0_off = fmax(w0_off, __shfl_xor_sync(0xffffffffu, w0_off, o));
    }
    if (err_local) atomicCAS(&a.cnt->err, 0, err_local);
    if (lane == 0) {
      a.applied[pl] = w0_all > 0;
      atomicAdd(&a.cnt->all, w0_all);
      atomicAdd(&a.cnt->big, w0_big);
      atomicMax(&a.cnt->off_bits, (unsigned long long)__double_as_longlong(w0_off));
    }
  }
  cluster.sync();   // no CTA leaves while its peer may still write into its shared memory
  trace_end(a);
}

// k_blk_zinv: (Z_blk^{-1})^T of every transformed pair for the W^T update (want_x), after
// k_blk_pivot_cl has written Z_blk (zero outside k x k; the bordered and padding
// diagonal is restored to 1 so the kb x kb elimination is regular).
__global__ void __launch_bounds__(NT_P, 1) k_blk_zinv(BlkArgs a) {
  extern __shared__ __align__(128) double2 zsm2[];   // Fh | Gh (KM*KM each)
  double2* Fh = zsm2;
  double2* Gh = zsm2 + KM * KM;
  const int pl = a.pair0 + blockIdx.x, tid = threadIdx.x;
  if (!a.applied[pl]) return;
  int c0p, wp, c0q, wq;
  pair_cols(a, pl, c0p, wp, c0q, wq);
  const int k = wp + wq;
  const int kb = k + (k & 1);
  const double2* zsrc = a.zblk + (size_t)pl * (KM * KM);
  for (int e = tid; e < KM * KM; e += NT_P) {
    const int i = e % KM, j = e / KM;
    Fh[e] = (i < k && j < k) ? zsrc[e] : make_double2(i == j ? 1.0 : 0.0, 0.0);
    Gh[e] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  gj_inverse_T<NT_P>(Fh, Gh, kb, a.zinvT + (size_t)pl * (KM * KM));
}

// ---------------------------------------------------------------- update (DMMA)
// grid (pair, tile): tiles [0, tF) rows of F, [tF, 2 tF) rows of G, [2 tF, 2 tF + tZ) rows of Z.
// Measured faster than three persistent variants (Z_blk loaded once per pair, the next
// row tile prefetched, results stored from the accumulators): one CTA of 8 warps per SM
// with double-buffered 64-row tiles, two CTAs per SM walking contiguous ranges, one CTA
// of 16 warps with double-buffered 64-row tiles were 8-15 % slower.  ncu: the short-
// lived CTAs of this form keep the DMMA sub-pipe 71 % busy; in the 16-warp variant the
// (Zr + Zi) / (Xr + Xi) DADDs of the 3M scheme stall on the FP64 pipe the DMMAs occupy
// (math-pipe stalls 50 % vs 24 %).  Unrolling the k-step loop (fragment loads issued
// ahead of the previous k-step's DMMAs; bitwise the same result) was slower: config 3
// 10.78 s rolled, 10.98 s unrolled x2, 11.47 s fully unrolled.
// wmode = 1: the tiles are row tiles of W^T (n rows) and the right factor is
// (Z_blk^{-1})^T (NEXT-1 accumulation of Z'^{-1}).
template <bool M4>
__global__ void __launch_bounds__(NT_U) k_blk_update(BlkArgs a, int tF, int tile0, int tile_end, int tpc,
                                                     int wmode) {
  trace_begin(a);
  extern __shared__ __align__(128) double2 usm[];  // X tile [KM][US] | Z_blk [KM][ZS]
  const int pl = a.pair0 + blockIdx.x;
  if (!a.applied[pl]) {
    trace_end(a);
    return;
  }
  int c0p, wp, c0q, wq;
  pair_cols(a, pl, c0p, wp, c0q, wq);
  const int k = wp + wq;
  double2* Xt = usm;
  double2* Zb = usm + KM * US;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double2* zsrc = (wmode ? a.zinvT : a.zblk) + (size_t)pl * (KM * KM);
  const int I = warp & 3;          // row tile of 8 rows within the 32-row tile
  const int J0 = (warp >> 2) * 4;  // first of 4 column tiles
  const int kend = (k + 3) & ~3;
  const int tile = tile0 + blockIdx.y;
  double2* X;
  long long ld, rows, r0;
  if (wmode) {
    X = a.W; ld = a.ldn; rows = a.n; r0 = (long long)(tile - tile0) * RT;
  } else if (tile < tF) {
    X = a.F; ld = a.ldm; rows = a.m; r0 = (long long)tile * RT;
  } else if (tile < 2 * tF) {
    X = a.G; ld = a.ldm; rows = a.m; r0 = (long long)(tile - tF) * RT;
  } else {
    X = a.Z; ld = a.ldn; rows = a.n; r0 = (long long)(tile - 2 * tF) * RT;
  }
  // Loads in NPH phases (tile columns and Z_blk rows [ph*KPH, +KPH) per cp.async group)
  // would let the DMMAs over the first k-range start early; measured on config 3:
  // NPH = 1: 1472 us, 2: 1488 us, 4: 1528 us per full-step launch, so one phase.
  constexpr int NPH = 1, KPH = KM / NPH;
#pragma unroll
  for (int ph = 0; ph < NPH; ph++) {
    for (int e = tid; e < KPH * KM; e += NT_U) {
      const int i = ph * KPH + e % KPH, j = e / KPH;
      cp_async16(&Zb[j * ZS + i], zsrc + i + (size_t)j * KM, i < k && j < k);
    }
    for (int e = tid; e < KPH * RT; e += NT_U) {
      const int c = ph * KPH + e / RT, r = e % RT;
      const long long gc = gcol(c, c0p, wp, c0q, wq);
      const bool ok = gc >= 0 && r0 + r < rows;
      cp_async16(&Xt[c * US + r], ok ? (const void*)(X + gc * ld + r0 + r) : (const void*)X, ok);
    }
    cp_commit();
  }
  {
    // out (RT x KM) = Xt (RT x KM) Z_blk (KM x KM): 4 x 8 tiles of 8x8, 4 per warp.
    // Complex product by the 3M (Gauss) scheme on DMMA: P1 = Xr Zr, P2 = Xi Zi,
    // P3 = (Xr + Xi)(Zr + Zi); out = (P1 - P2) + i (P3 - P1 - P2): 3 real DMMAs per
    // 8x8x4 complex step instead of 4 (normwise error bound of the same order).
    double p1[4][2], p2[4][2], p3[4][2];
#pragma unroll
    for (int t = 0; t < 4; t++) p1[t][0] = p1[t][1] = p2[t][0] = p2[t][1] = p3[t][0] = p3[t][1] = 0.0;
#pragma unroll
    for (int ph = 0; ph < NPH; ph++) {
      cp_wait_dyn(NPH - 1 - ph);   // every phase is waited for, even past kend
      __syncthreads();
      for (int kk = ph * KPH; kk < min(kend, (ph + 1) * KPH); kk += 4) {
      const double2 x = Xt[(kk + (lane & 3)) * US + 8 * I + (lane >> 2)];  // A(i, k)
      const double xs = x.x + x.y;
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const double2 z = Zb[(8 * (J0 + t) + (lane >> 2)) * ZS + kk + (lane & 3)];  // B(k, j)
        dmma(p1[t][0], p1[t][1], x.x, z.x);
        dmma(p2[t][0], p2[t][1], x.y, z.y);
        if (M4) {   // exact 4M product: Im accumulated directly, no additions in the loop
          dmma(p3[t][0], p3[t][1], x.x, z.y);
          dmma(p3[t][0], p3[t][1], x.y, z.x);
        } else {
          dmma(p3[t][0], p3[t][1], xs, z.x + z.y);
        }
      }
    }
    }
    // accumulators -> global (each 8-lane group writes 8 consecutive rows of a column);
    // every warp has read the whole tile and the tile's rows of these columns belong to
    // this CTA alone, so no barrier is needed before the in-place stores
    const long long row = r0 + 8 * I + (lane >> 2);
    if (row < rows) {
#pragma unroll
      for (int t = 0; t < 4; t++) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int j = 8 * (J0 + t) + 2 * (lane & 3) + h;
          const long long gc = gcol(j, c0p, wp, c0q, wq);
          if (gc < 0) continue;
          X[gc * ld + row] = M4 ? make_double2(p1[t][h] - p2[t][h], p3[t][h])
                                : make_double2(p1[t][h] - p2[t][h], p3[t][h] - p1[t][h] - p2[t][h]);
        }
      }
    }
  }
  trace_end(a);
}

__global__ void k_blk_partition(int* bstart, int* bwidth, int nblk, long long n) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long w = (n + nblk - 1) / nblk;
  const long long nbig = n - (long long)nblk * (w - 1);
  long long c = 0;
  for (int b = 0; b < nblk; b++) {
    bwidth[b] = (int)(b < nbig ? w : w - 1);
    bstart[b] = (int)c;
    c += bwidth[b];
  }
}

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

// tuning knobs (experiments only; defaults are the measured best)
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

int auto_nblk(int64_t n, const ghsvd_options* o) {
  if (o->nblocks > 0) return o->nblocks;
  int64_t nb = (n + 31) / 32;      // width w <= 32 -> block pivots of order <= 64
  nb += nb & 1;
  const int64_t P = std::max(1, o->world_size);
  nb = round_up(nb, 2 * P);
  return (int)std::max<int64_t>(2, nb);
}


struct BlkPlan {
  int nblk, K, slot0, nsplit;
  long long split_rows;
};

BlkPlan make_plan(const Ctx* ctx) {
  BlkPlan p;
  p.nblk = auto_nblk(ctx->n, &ctx->o);
  const int P = std::max(1, ctx->o.world_size);
  p.K = p.nblk / 2 / P;
  p.slot0 = ctx->o.rank * p.K;
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
    const long long rows = round_up((ctx->m + ns - 1) / ns, RT);
    const int nseff = (int)((ctx->m + rows - 1) / rows);
    if (nseff != ns) continue;
    const double waves = (double)((M * ns + R - 1) / R);
    const double cost = waves * (double)(rows / RT + 3);
    if (best < 0 || cost < best_cost - 1e-9) {
      best = ns;
      best_cost = cost;
    }
  }
  p.nsplit = (int)std::max<long long>(1, best);
  if (env_int("GHSVD_NSPLIT", 0) > 0) p.nsplit = std::min(MAX_SPLIT, env_int("GHSVD_NSPLIT", 0));
  const long long rows_per = (ctx->m + p.nsplit - 1) / p.nsplit;
  p.split_rows = round_up(std::max<long long>(rows_per, 1), RT);
  p.nsplit = (int)((ctx->m + p.split_rows - 1) / p.split_rows);
  return p;
}

}  // namespace

// scratch carved by blk_setup for K block pairs per rank out of nblk block columns
static size_t blk_scratch_for(int64_t K, int64_t nb, bool want_x) {
  return al256((size_t)K * 2 * MAX_SPLIT * KM * KM * 16) + al256((size_t)2 * K * KM * KM * 16) +
         al256((size_t)2 * K * 4) + 2 * al256((size_t)(nb + 2) * 4) + 2 * al256((size_t)K * KM * KM * 16) +
         al256((size_t)K * KM) + al256((size_t)2 * K * 4) + (want_x ? al256((size_t)2 * K * KM * KM * 16) : 0) +
         al256((size_t)(nb + 2) * TRACE_SLOTS * 16) + al256((size_t)2 * K * 4) + 4096;
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
  size_t smem_g, smem_p, smem_u;
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
  S.trace_buf = (unsigned long long*)p; p += al256((size_t)(pl.nblk + 2) * TRACE_SLOTS * 16);
  a.trace = nullptr;
  a.trace_id = 0;
  k_blk_partition<<<1, 32, 0, str>>>(bstart, bwidth, pl.nblk, ctx->n);
  GH_CUDA(cudaMemsetAsync(a.gcnt, 0, (size_t)2 * pl.K * 4, str));
  GH_CUDA(cudaGetLastError());
  S.bs_h.assign(pl.nblk, 0);
  S.bw_h.assign(pl.nblk, 0);
  GH_CUDA(cudaMemcpyAsync(S.bs_h.data(), bstart, pl.nblk * 4, cudaMemcpyDeviceToHost, str));
  GH_CUDA(cudaMemcpyAsync(S.bw_h.data(), bwidth, pl.nblk * 4, cudaMemcpyDeviceToHost, str));
  GH_CUDA(cudaStreamSynchronize(str));
  ctx->blk_start = S.bs_h;
  ctx->blk_width = S.bw_h;
  a.F = ctx->F;
  a.G = ctx->G;
  a.Z = ctx->Z;
  a.ldm = ctx->ldm;
  a.ldn = ctx->ldn;
  a.m = ctx->m;
  a.n = ctx->n;
  a.npos = ctx->npos;
  a.nblk = pl.nblk;
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
  S.smem_g = (size_t)GSTAGES * KM * GS * 16;
  S.smem_p = (size_t)3 * KM * KM * 16;
  S.smem_u = (size_t)(KM * US + KM * ZS) * 16;
  GH_CUDA(cudaFuncSetAttribute(k_blk_gram<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_g));
  GH_CUDA(cudaFuncSetAttribute(k_blk_gram<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_g));
  S.gram3m = env_int("GHSVD_GRAM3M", 1) != 0;
  S.pivot_cl = env_int("GHSVD_PIVOT_CL", 0) != 0;
  S.smem_pc = (size_t)3 * KM * RB * 16;
  GH_CUDA(cudaFuncSetAttribute(k_blk_zinv, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * KM * KM * 16));
  GH_CUDA(cudaFuncSetAttribute(k_blk_pivot_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_pc));
  GH_CUDA(cudaFuncSetAttribute(k_blk_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_p));
  GH_CUDA(cudaFuncSetAttribute(k_blk_update<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_u));
  GH_CUDA(cudaFuncSetAttribute(k_blk_update<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S.smem_u));
  S.upd4m = env_int("GHSVD_UPD4M", 0) != 0;
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
  if (S.gram3m)
    k_blk_gram<true><<<dim3(S.pl.nsplit, 2, np), NT_G, S.smem_g, st>>>(a);
  else
    k_blk_gram<false><<<dim3(S.pl.nsplit, 2, np), NT_G, S.smem_g, st>>>(a);
}

// Update launch: pairs [pair0, pair0 + np), row tiles [tbeg, tend) (see k_blk_update).
static void launch_update(const BlkSetup& S, BlkArgs a, int pair0, int np, int tbeg, int tend, int wmode,
                          cudaStream_t st) {
  a.pair0 = pair0;
  if (np <= 0 || tend <= tbeg) return;
  if (S.upd4m)
    k_blk_update<true><<<dim3(np, tend - tbeg), NT_U, S.smem_u, st>>>(a, S.tF, tbeg, tend, 1, wmode);
  else
    k_blk_update<false><<<dim3(np, tend - tbeg), NT_U, S.smem_u, st>>>(a, S.tF, tbeg, tend, 1, wmode);
}

// Diagnostic: block steps [s0, s0+ns) of the first block sweep, one stream, no overlap.
ghsvd_status blk_run_steps(Ctx* ctx, int64_t s0, int64_t ns) {
  BlkSetup S;
  ghsvd_status e = blk_setup(ctx, S);
  if (e) return e;
  if (s0 < 0 || ns < 0 || s0 + ns > S.pl.nblk - 1) {
    ctx->err = "run_steps: block step range outside [0, nblk-2]";
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
  const int nst = pl.nblk - 1;
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
  double fl_gram_sweep = 0.0, fl_upd_sweep = 0.0;
  for (int s = 0; s < nst; s++)
    for (int kk = pl.slot0; kk < pl.slot0 + pl.K; kk++) {
      long long bp, bq;
      rr_pair(pl.nblk, s, kk, &bp, &bq);
      const double kq = S.bw_h[bp] + S.bw_h[bq];
      fl_gram_sweep += 8.0 * kq * (kq + 1) * ctx->m;
      fl_upd_sweep += 8.0 * kq * kq * (2.0 * ctx->m + ctx->n);
    }
  GH_CUDA(cudaEventRecord(ctx->ev0, str));
  for (int sw = 0; sw < ctx->o.max_sweeps; sw++) {
    GH_CUDA(cudaMemsetAsync(ctx->cnt, 0, sizeof(DevCounters), str));
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
    st->launches += (uint64_t)(a.W ? 4 : 3) * G * nst;
    st->flops_gram += fl_gram_sweep;
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
  st->alg_bytes = (uint64_t)((double)st->sweeps * (pl.nblk - 1) * 16.0 * (double)ctx->n *
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
  {
    // one GPU: GHSVD_GROUPS=G >= 2 selects the pipelined pair-group schedule
    // (blk_sweep_groups; measured 1-2 % slower than the two-stream schedule below on
    // config 3, kept as an experiment)
    const int G = std::min(S.pl.K, env_int("GHSVD_GROUPS", 0));
    if (!multi && G >= 2) return blk_sweep_groups(ctx, st, S, G);
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
  // The Z' update of step s (aux stream) overlaps the Gram + pivot of step s+1: Z is
  // touched by no other kernel, and Z_blk / applied are double-buffered by step parity.
  if (!ctx->aux_stream) GH_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
  if (!ctx->aux_stream2) GH_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream2, cudaStreamNonBlocking));
  // GHSVD_SERIAL=1: every kernel on the context stream, one launch per kind and step over
  // all block pairs -- the kernels run alone, so their CUDA-event durations are their
  // isolated durations (bench.py's roofline probe); same arithmetic, bitwise equal
  const bool serial = env_int("GHSVD_SERIAL", 0) != 0;
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
  const bool prio = env_int("GHSVD_PRIO", 1) != 0 && !serial;
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
  const int nst = pl.nblk - 1;
  std::vector<cudaEvent_t> ev_piv(2), ev_fg(2), ev_zdone(2), ev_gr(2), ev_bnd(2), tev;
  // GHSVD_SPLIT_BND=1 (experiment): split each half's F/G update into its boundary pair
  // and the rest, so half 0 of step s+1 may start while half 1 of step s still updates;
  // measured equal to the plain halves on config 3 (2.42 ms per block step either way)
  const bool split_bnd = !multi && nh == 2 && KA >= 2 && pl.K - KA >= 2 && env_int("GHSVD_SPLIT_BND", 0) != 0;
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
  // algorithmic flops per block step (Hermitian Grams k(k+1)/2 m each; updates k^2 (2m+n))
  std::vector<double> fl_gram(nst, 0.0), fl_upd(nst, 0.0), fl_upd_fg(nst, 0.0);
  for (int s = 0; s < nst; s++)
    for (int kk = pl.slot0; kk < pl.slot0 + pl.K; kk++) {
      long long bp, bq;
      rr_pair(pl.nblk, s, kk, &bp, &bq);
      const double kq = bw_h[bp] + bw_h[bq];
      fl_gram[s] += 8.0 * kq * (kq + 1) * ctx->m;
      fl_upd[s] += 8.0 * kq * kq * (2.0 * ctx->m + ctx->n);
      fl_upd_fg[s] += 8.0 * kq * kq * (2.0 * ctx->m);
    }
  const char* trace_path = getenv("GHSVD_TRACE");
  std::vector<unsigned long long> trace_h;
  if (trace_path && *trace_path) {
    trace_h.assign((size_t)nst * TRACE_SLOTS * 2, 0);
    for (size_t i = 0; i < trace_h.size(); i += 2) trace_h[i] = ~0ull;
    GH_CUDA(cudaMemcpyAsync(S.trace_buf, trace_h.data(), trace_h.size() * 8, cudaMemcpyHostToDevice, str));
  }
  GH_CUDA(cudaEventRecord(ctx->ev0, str));
  for (int sw = 0; sw < ctx->o.max_sweeps; sw++) {
    a.trace = (sw == 0 && !trace_h.empty()) ? S.trace_buf : nullptr;
    GH_CUDA(cudaMemsetAsync(ctx->cnt, 0, sizeof(DevCounters), str));
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
      if (multi && s > 0)
        for (int h = 0; h < nh; h++)
          if (hs_st[h] != str) GH_CUDA(cudaStreamWaitEvent(hs_st[h], ev_x, 0));
      for (int h = 0; h < nh; h++) {
        cudaStream_t sh = hs_st[h];
        a.pair0 = h_pair0[h];
        if (timing) GH_CUDA(cudaEventRecord(tev[8 * s + 4 * h + 0], sh));
        a.trace_id = s * TRACE_SLOTS + 0 + h;
        launch_gram(S, a, h_np[h], sh);
        if (timing) GH_CUDA(cudaEventRecord(tev[8 * s + 4 * h + 1], sh));
        cudaStream_t fs = fp_st[h];
        if (fs != sh) {
          GH_CUDA(cudaEventRecord(ev_gr[h], sh));
          GH_CUDA(cudaStreamWaitEvent(fs, ev_gr[h], 0));
        }
        // Z_blk buffer b was last read by the Z update of step s-2
        if (s >= 2 || sw > 0) GH_CUDA(cudaStreamWaitEvent(fs, ev_zdone[b], 0));
        a.trace_id = s * TRACE_SLOTS + 4 + h;
        launch_pivot(S, a, h_np[h], fs);
        GH_CUDA(cudaEventRecord(ev_piv[h], fs));
        if (fs != sh) GH_CUDA(cudaStreamWaitEvent(sh, ev_piv[h], 0));
        if (timing) GH_CUDA(cudaEventRecord(tev[8 * s + 4 * h + 2], sh));
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
        if (timing) GH_CUDA(cudaEventRecord(tev[8 * s + 4 * h + 3], sh));
        GH_CUDA(cudaEventRecord(ev_fg[h], sh));
      }
      // Z' update of all pairs of step s on the aux stream (overlaps step s+1)
      a.pair0 = 0;
      for (int h = 0; h < nh; h++) GH_CUDA(cudaStreamWaitEvent(aux, ev_piv[h], 0));
      a.trace_id = s * TRACE_SLOTS + 8;
      launch_update(S, a, 0, pl.K, 2 * tF, 2 * tF + tZ, 0, aux);
      a.trace_id = s * TRACE_SLOTS + 9;
      if (a.W) launch_update(S, a, 0, pl.K, 0, tZ, 1, aux);
      if (multi) {
        // The exchange after step s in two parts (NEXT-2, comm/compute overlap): the Z', W
        // block columns leave right after the Z' update, on the aux stream and a second
        // communicator, while the F, G block columns leave as soon as the F, G updates of
        // both halves are done -- the Grams of step s+1 need only F and G, so they no
        // longer wait for the Z' update of step s (which keeps overlapping them, as on one
        // GPU).  The next Z' update runs on the aux stream after the Z' exchange.
        const int s_next = (s + 1) % nst;
        ghsvd_status e = comm_exchange(ctx, pl.nblk, s, s_next, bs_h.data(), bw_h.data(), XCH_ZW, aux);
        if (e) {
          destroy_events();
          return e;
        }
      }
      GH_CUDA(cudaEventRecord(ev_zdone[b], aux));
      GH_CUDA(cudaGetLastError());
      if (multi) {
        for (int h = 0; h < nh; h++)
          if (hs_st[h] != str) GH_CUDA(cudaStreamWaitEvent(str, ev_fg[h], 0));
        const int s_next = (s + 1) % nst;
        ghsvd_status e = comm_exchange(ctx, pl.nblk, s, s_next, bs_h.data(), bw_h.data(), XCH_FG, str);
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
    st->launches += (uint64_t)(3 * nh + (split_bnd ? 2 : 0) + (a.W ? 2 : 1)) * nst;
    st->launches_update_fg += (uint64_t)(nh + (split_bnd ? 2 : 0)) * nst;
    for (int s = 0; s < nst; s++) {
      st->flops_gram += fl_gram[s];
      st->flops_update += fl_upd[s];
      st->flops_update_fg += fl_upd_fg[s];
      if (timing) {
        for (int h = 0; h < nh; h++) {
          float t0 = 0, t1 = 0, t2 = 0;
          GH_CUDA(cudaEventElapsedTime(&t0, tev[8 * s + 4 * h + 0], tev[8 * s + 4 * h + 1]));
          GH_CUDA(cudaEventElapsedTime(&t1, tev[8 * s + 4 * h + 1], tev[8 * s + 4 * h + 2]));
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
  // HBM bytes the blocked sweep must move per block step: Grams read F, G pairs once,
  // updates read + write F, G, Z pairs once
  st->alg_bytes = (uint64_t)((double)st->sweeps * (pl.nblk - 1) / std::max(1, ctx->o.world_size) *
                             16.0 * (double)ctx->n * (2.0 * ctx->m + 2.0 * (2.0 * ctx->m + ctx->n)));
  return GHSVD_OK;
}

}  // namespace ghsvd
