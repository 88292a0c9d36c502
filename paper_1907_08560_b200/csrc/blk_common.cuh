// blk_common.cuh -- constants, DMMA / cp.async helpers, the kernel argument block and
// the pair-column map shared by the blocked kernels (Sec 6.4)
// Part of blocked.cu's translation unit (included once, inside ghsvd's anonymous
// namespace context of that file); not a public header.
#pragma once
#include <cuda_runtime.h>

#include "hz2x2.cuh"
#include "internal.h"

namespace ghsvd {
namespace {

constexpr int KM = 64;          // max block-pivot order 2w
constexpr int RT = 32;          // rows per staged tile
// Gram tile column stride (double2).  A 128-bit fragment load of 8 lanes reads rows
// r..r+3 of two adjacent columns: with a stride = 4 (mod 8) slots the 8 lanes hit 8
// distinct 16-byte bank groups (stride 34 = 2 mod 8 overlapped two of them: ncu counted
// 43 % of the Gram's shared wavefronts as bank conflicts).  Two CTAs of 110.6 KB fit an
// SM because the fused factorization keeps its scratch in the same dynamic buffer.
// Gram pipeline geometry: RTG rows per stage, GSTAGES stages (compile-time; the
// -DGHSVD_GRAM_RT / -DGHSVD_GRAM_STAGES overrides exist for A/B builds only)
#ifndef GHSVD_GRAM_RT
#define GHSVD_GRAM_RT 32
#endif
#ifndef GHSVD_GRAM_STAGES
#define GHSVD_GRAM_STAGES 3
#endif
constexpr int RTG = GHSVD_GRAM_RT;
static_assert(RTG % 8 == 0 && (RTG + 4) % 8 == 4, "Gram stage rows: two k-steps per iteration, stride 4 mod 8");
constexpr int GS = RTG + 4;
constexpr int GS_FUSED = GS;
constexpr int ZS = KM + 4;      // Z_blk column stride in smem
constexpr int NT_G = 256, NT_P = 512, NT_U = 256;
constexpr int US = RT + 2;      // update tile column stride
constexpr int GSTAGES = GHSVD_GRAM_STAGES;   // cp.async pipeline depth of the Gram kernel
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
  int ord, nsup;            // block ordering (ordering.h) and its super blocks
  const int4* ptab;         // [block step][global slot] = (start p, width p, start q, width q)
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
  unsigned long long* upd_k2; // [block step] sum of k^2 over the pairs whose update runs
                              // (k = w_p + w_q; reset per sweep) -> exact update flops
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
  // the block pair of this slot and step, tabulated on the host from the ordering (ordering.h)
  const int4 t = __ldg(&a.ptab[(size_t)a.s * (a.nblk / 2) + a.slot0 + pl]);
  c0p = t.x;
  wp = t.y;
  c0q = t.z;
  wq = t.w;
}

// global column of pivot column c (c < wp: block p, else block q), -1 if padding
__device__ __forceinline__ long long gcol(int c, int c0p, int wp, int c0q, int wq) {
  if (c < wp) return c0p + c;
  if (c < wp + wq) return c0q + (c - wp);
  return -1;
}

}  // namespace
}  // namespace ghsvd
