// blk_pivot.cuh -- the block pivot: inner Level-1 one-sided HZ sweep(s) on F^, G^ in
// shared memory accumulating Z_blk (Sec 6.4.2), and (Z_blk^{-1})^T for NEXT-1
// Part of blocked.cu's translation unit (included once, inside ghsvd's anonymous
// namespace context of that file); not a public header.
#pragma once
#include <cooperative_groups.h>

#include "blk_common.cuh"
#include "hz2x2.cuh"

namespace ghsvd {
namespace {

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
          // all loads of a matrix are issued before its first store (the compiler cannot
          // prove the stores do not alias the later loads, and the unbatched form ran one
          // load -> FMA chain -> store round trip per row: ~22 % of the kernel's samples)
          auto rot = [&](double2* M) {
            double2 x[KM / 16], y[KM / 16];
#pragma unroll
            for (int t = 0; t < KM / 16; t++) {
              x[t] = M[hl + 16 * t + p * KM];
              y[t] = M[hl + 16 * t + q * KM];
            }
#pragma unroll
            for (int t = 0; t < KM / 16; t++) {
              const int i = hl + 16 * t;
              M[i + p * KM] = make_double2(x[t].x * z11.x - x[t].y * z11.y + y[t].x * z21.x - y[t].y * z21.y,
                                           x[t].x * z11.y + x[t].y * z11.x + y[t].x * z21.y + y[t].y * z21.x);
              M[i + q * KM] = make_double2(x[t].x * z12.x - x[t].y * z12.y + y[t].x * z22.x - y[t].y * z22.y,
                                           x[t].x * z12.y + x[t].y * z12.x + y[t].x * z22.y + y[t].y * z22.x);
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
    if (cnt_all > 0) atomicAdd(&a.upd_k2[a.s], (unsigned long long)(k * k));
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
      if (w0_all > 0) atomicAdd(&a.upd_k2[a.s], (unsigned long long)(k * k));
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

}  // namespace
}  // namespace ghsvd
