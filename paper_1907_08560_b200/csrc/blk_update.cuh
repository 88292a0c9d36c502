// blk_update.cuh -- the block update [F_pair | G_pair | Z_pair] <- (.) Z_blk on DMMA
// (3M complex product), row tiles, in place (Sec 6.4.3), and the partition kernel
// Part of blocked.cu's translation unit (included once, inside ghsvd's anonymous
// namespace context of that file); not a public header.
#pragma once
#include "blk_common.cuh"

namespace ghsvd {
namespace {

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
// 10.78 s rolled, 10.98 s unrolled x2, 11.47 s fully unrolled.  Splitting the output
// columns over a 2-CTA cluster (each CTA stages half of X and of Z_blk, 70 KB, so three
// CTAs fit an SM; the peer's X half copied through DSMEM between two cluster barriers;
// bitwise the same result) was slower still: 12.64 s.
// wmode = 1: the tiles are row tiles of W^T (n rows) and the right factor is
// (Z_blk^{-1})^T (NEXT-1 accumulation of Z'^{-1}).
template <bool M4>
__global__ void __launch_bounds__(NT_U) k_blk_update(BlkArgs a, int tF, int tile0, int wmode) {
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

}  // namespace
}  // namespace ghsvd
