// blk_gram.cuh -- block Grams H_blk = F_pair^* J F_pair, S_blk = G_pair^* G_pair on
// DMMA with the fused block-pivot factorizations (HEBPJ / pivoted Cholesky) in the last
// CTA of each (pair, H|S)
// Part of blocked.cu's translation unit (included once, inside ghsvd's anonymous
// namespace context of that file); not a public header.
#pragma once
#include "blk_common.cuh"
#include "hebpj.cuh"

namespace ghsvd {
namespace {

// ---------------------------------------------------------------- block pivot
// blk_factor (run by the last Gram CTA of a (pair, H|S), see k_blk_gram): sum the split
// partials in fixed order; which = 0: H_blk -> HEBPJ -> F^ (and J^); which = 1: S_blk ->
// diagonally pivoted Cholesky -> G^.  F^, G^ go to L2-resident scratch.
constexpr int NT_F = 256;
// W: KM x KM in shared memory followed by room for the factorization scratch (no static
// shared memory: the fused Gram kernel reuses its pipeline buffers)
constexpr size_t BLK_FACTOR_SMEM = (size_t)KM * KM * 16 + sizeof(hb::HebpjScr<NT_F, KM>) + 64;
static_assert(sizeof(hb::PcholScr<KM>) <= sizeof(hb::HebpjScr<NT_F, KM>), "scratch");
static_assert(BLK_FACTOR_SMEM <= (size_t)GSTAGES * KM * GS_FUSED * 16, "fused factor scratch");
__device__ void blk_factor(const BlkArgs& a, int pl, int which, double2* W) {
  __shared__ int np_sh;
  char* scr = reinterpret_cast<char*>(W + KM * KM);
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
    auto& sc = *reinterpret_cast<hb::HebpjScr<NT_F, KM>*>(scr);
    hb::block_amax<NT_F>(tv, ti, sc.sv1, sc.si1);
    const double tolz = __dmul_rn(__dmul_rn((double)k, 0x1p-53), tv);
    rc = hb::hebpj_dev<NT_F, KM>(W, k, KM, out, KM, a.jhat + (size_t)pl * KM, &np_sh, tolz, sc);
  } else {
    rc = hb::pchol_dev<NT_F, KM>(W, k, KM, out, KM, *reinterpret_cast<hb::PcholScr<KM>*>(scr));
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
// x with its sign bit xor-ed with m (0 or 0x80000000): the J sign (+-1) applied on the
// integer pipe -- bitwise what the product by +-1 gives, without an FP64 instruction
// competing with the DMMAs for the FP64 pipe (ncu r2: the Gram's DMULs by the sign were
// 17 % of its stall samples)
__device__ __forceinline__ double sflip(double x, unsigned m) {
  return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
}

template <int GI, int TS>
__device__ __forceinline__ void gram_tiles(const double2* T, int row, unsigned sm, double (&acc)[9][4]) {
  constexpr int IA = GI, IB = 7 - GI, NF = 8 - GI;
  const int lane = threadIdx.x & 31;
  double2 f[NF];
#pragma unroll
  for (int j = 0; j < NF; j++) f[j] = T[(8 * j + (lane >> 2)) * TS + row];
  // A operand of tile rows IA, IB: J_r conj(x): (ar, ai) with conj -> (+x.y used as -(-x.y))
  const double aar = sflip(f[IA].x, sm), aai = sflip(f[IA].y, sm);
  const double abr = sflip(f[IB].x, sm), abi = sflip(f[IB].y, sm);
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

template <int GI, int H, bool W4, int TS>
__device__ __forceinline__ void gram3_tiles(const double2* T, int row, unsigned sm, double (&acc)[5][6]) {
  using C = G3<GI>;
  const int lane = threadIdx.x & 31;
  double2 f[8];
  double bs[8];
#pragma unroll
  for (int j = 0; j < 8; j++) {
    if (C::needB(H, W4, j) || C::needA(H, W4, j)) f[j] = T[(8 * j + (lane >> 2)) * TS + row];
    if (C::needB(H, W4, j)) bs[j] = f[j].x + f[j].y;
  }
  double ar[2] = {0, 0}, ai[2] = {0, 0}, as[2] = {0, 0};   // rows IA, IB
  if (C::needA(H, W4, C::IA)) {
    ar[0] = sflip(f[C::IA].x, sm);
    ai[0] = sflip(f[C::IA].y, sm ^ 0x80000000u);
    as[0] = ar[0] + ai[0];
  }
  if (C::needA(H, W4, C::IB)) {
    ar[1] = sflip(f[C::IB].x, sm);
    ai[1] = sflip(f[C::IB].y, sm ^ 0x80000000u);
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

// FUSED (default): the last CTA of each (pair, H|S) runs the block-pivot factorization
// itself, hidden behind the other pairs' Gram CTAs; with GHSVD_SCHED_SPLIT_FACTOR
// k_blk_factor does, in its own launch (measured slower: its ~310 us latency-bound span
// lands on the Gram -> pivot chain).
template <bool M3, bool FUSED>
__global__ void __launch_bounds__(NT_G, 2) k_blk_gram(BlkArgs a) {
  constexpr int TS = FUSED ? GS_FUSED : GS;
  trace_begin(a);
  extern __shared__ __align__(128) double2 gsm[];  // [GSTAGES][KM][TS]
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
      double2* T = gsm + (size_t)st * KM * TS;
      for (int e = tid; e < KM * RTG; e += NT_G) {
        const int c = e / RTG, r = e % RTG;
        const long long gc = gcol(c, c0p, wp, c0q, wq);
        const long long gr = r0 + r;
        const bool ok = gc >= 0 && gr < r_end;
        cp_async16(&T[c * TS + r], ok ? (const void*)(X + gc * a.ldm + gr) : (const void*)X, ok);
      }
    }
    cp_commit();   // possibly empty: keeps one group per stage
  };
  // GSTAGES-deep cp.async pipeline over the split's 32-row stages; consume(T, r0).
  // One barrier per stage: after it every warp has finished the previous stage, whose
  // buffer is then refilled with the stage GSTAGES-1 ahead.
  auto pipeline = [&](auto&& consume) {
#pragma unroll
    for (int p = 0; p < GSTAGES - 1; p++) load_stage(p, r_begin + (long long)p * RTG);
    int st = 0;
    for (long long r0 = r_begin; r0 < r_end; r0 += RTG) {
      cp_wait<GSTAGES - 2>();
      __syncthreads();
      load_stage((st + GSTAGES - 1) % GSTAGES, r0 + (long long)(GSTAGES - 1) * RTG);
      consume(gsm + (size_t)st * KM * TS, r0);
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
      for (int ks = 0; ks < RTG / 4; ks += 2) {
        const int row0 = 4 * ks + (lane & 3), row1 = row0 + 4;
        const unsigned sg0 = (hs == 0 && r0 + row0 >= a.npos) ? 0x80000000u : 0u;
        const unsigned sg1 = (hs == 0 && r0 + row1 >= a.npos) ? 0x80000000u : 0u;
        switch (warp) {   // warp-uniform; tile 4 on even k-steps for h = 0, odd for h = 1
#define G3CASE(W, GI, H)                                       \
  case W:                                                      \
    gram3_tiles<GI, H, H == 0, TS>(T, row0, sg0, acc);         \
    gram3_tiles<GI, H, H == 1, TS>(T, row1, sg1, acc);         \
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
      for (int ks = 0; ks < RTG / 4; ks += 2) {
        const int row = 4 * (ks + kh) + (lane & 3);
        const unsigned sg = (hs == 0 && r0 + row >= a.npos) ? 0x80000000u : 0u;
        switch (gi) {   // warp-uniform
          case 0: gram_tiles<0, TS>(T, row, sg, acc); break;
          case 1: gram_tiles<1, TS>(T, row, sg, acc); break;
          case 2: gram_tiles<2, TS>(T, row, sg, acc); break;
          default: gram_tiles<3, TS>(T, row, sg, acc); break;
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
  if constexpr (FUSED) {
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
  }
  trace_end(a);
}

// k_blk_factor: grid (H|S, pair): sum the Gram split partials and factor the block pivot
// (HEBPJ of H_blk, pivoted Cholesky of S_blk), one CTA each; W (k x k) in dynamic smem.
__global__ void __launch_bounds__(NT_F) k_blk_factor(BlkArgs a) {
  trace_begin(a);
  extern __shared__ __align__(128) double2 fsm[];   // [KM][KM]
  blk_factor(a, a.pair0 + blockIdx.y, blockIdx.x, fsm);
  trace_end(a);
}

// (Z_blk^{-1})^T for the W^T update (NEXT-1): Gauss-Jordan with partial pivoting on
// [Fh | Gh] = [Z_blk | I] (kb x kb active, ld KM, in shared memory), transposed into wo.

}  // namespace
}  // namespace ghsvd
