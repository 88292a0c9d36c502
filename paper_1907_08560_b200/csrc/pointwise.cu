// pointwise.cu -- fused pointwise HZ step on sm_100a.
//
// One parallel step S_s of the round-robin ordering (Sec 6.3, Alg. 3
// PAPER.md:1758-1814) is ONE launch: n/2 thread-block clusters, one per pivot
// pair (p, q).  The C CTAs of a cluster split the m rows of the pair's four
// columns f_p, f_q, g_p, g_q into contiguous slices; each CTA
//   1. stages its slices in shared memory with TMA bulk copies
//      (cp.async.bulk global->shared, mbarrier completion) -- one HBM read,
//   2. forms its partial Grams (eq 6.1; J = diag(I_npos, -I) from the row sort),
//      reduces them warp -> CTA, then across the cluster through DSMEM in fixed
//      rank order (deterministic, identical in every CTA),
//   3. computes the 2x2 transformation Z' (hz2x2.cuh, eqs 6.2-6.12) redundantly
//      per CTA (bitwise identical inputs -> identical Z'),
//   4. if Z' is applied: updates the slices in shared memory and writes them back
//      with TMA bulk stores (one HBM write), then loads/updates/stores its slice
//      of z'_p, z'_q (n rows) the same way ("two ZVROTMs of length m and one of
//      length n").
// Counters (all, big, max off-measure) are device atomics read once per sweep
// (a5).  Per transformed pair the kernel moves the algorithmic minimum
// 128 m + 64 n bytes (read + write F, G pair columns once; Z pair read + write),
// per skipped pair 64 m bytes.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "hz2x2.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace ghsvd {

struct StepArgs {
  double2* F;
  double2* G;
  double2* Z;
  long long ldm, ldn;
  long long m, n;
  long long npos;
  long long s;
  long long cs;   // F/G rows per CTA slice
  long long zs;   // Z rows per CTA slice
  double tol;
  int literal;
  DevCounters* cnt;
  double2* W;     // want_x: W^T = (Z'^{-1})^T (n rows, ld ldn), or nullptr
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// [a b] <- [a b] Z' for one row: a' = a z11 + b z21, b' = a z12 + b z22
__device__ __forceinline__ void rot_row(double2& a, double2& b, const Cplx& z11, const Cplx& z21,
                                        const Cplx& z12, const Cplx& z22) {
  const double2 x = a, y = b;
  a.x = fma(x.x, z11.re, fma(-x.y, z11.im, fma(y.x, z21.re, -y.y * z21.im)));
  a.y = fma(x.x, z11.im, fma(x.y, z11.re, fma(y.x, z21.im, y.y * z21.re)));
  b.x = fma(x.x, z12.re, fma(-x.y, z12.im, fma(y.x, z22.re, -y.y * z22.im)));
  b.y = fma(x.x, z12.im, fma(x.y, z12.re, fma(y.x, z22.im, y.y * z22.re)));
}

template <int NT>
__global__ void __launch_bounds__(NT) k_pair_step(StepArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ double red[NT / 32][8];
  __shared__ double part[8];
  __shared__ double tot[8];
  __shared__ double zsh[8];
  __shared__ int kind_sh;

  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const long long pair = blockIdx.x / C;
  long long p, q;
  rr_pair(a.n, a.s, pair, &p, &q);

  const long long r0 = (long long)rank * a.cs;
  const long long r1 = min(a.m, r0 + a.cs);
  const long long len = r1 > r0 ? r1 - r0 : 0;
  const long long z0 = (long long)rank * a.zs;
  const long long z1 = min(a.n, z0 + a.zs);
  const long long zlen = z1 > z0 ? z1 - z0 : 0;

  double2* sFp = reinterpret_cast<double2*>(smem_raw);
  double2* sFq = sFp + a.cs;
  double2* sGp = sFq + a.cs;
  double2* sGq = sGp + a.cs;
  double2* sZp = sGq + a.cs;
  double2* sZq = sZp + a.zs;

  double2* gFp = a.F + p * a.ldm + r0;
  double2* gFq = a.F + q * a.ldm + r0;
  double2* gGp = a.G + p * a.ldm + r0;
  double2* gGq = a.G + q * a.ldm + r0;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    const unsigned bytes = (unsigned)(len * 16);
    mbar_expect_tx(&bar[0], 4u * bytes);
    if (len > 0) {
      bulk_g2s(sFp, gFp, bytes, &bar[0]);
      bulk_g2s(sFq, gFq, bytes, &bar[0]);
      bulk_g2s(sGp, gGp, bytes, &bar[0]);
      bulk_g2s(sGq, gGq, bytes, &bar[0]);
    }
  }
  mbar_wait(&bar[0], 0);

  // ---- (6.1): partial Grams over this slice (fixed per-thread row order)
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long npos_loc = a.npos - r0;  // rows i < npos_loc have J = +1
  for (long long i = tid; i < len; i += NT) {
    const double2 fp = sFp[i], fq = sFq[i], gp = sGp[i], gq = sGq[i];
    const double sgn = (i < npos_loc) ? 1.0 : -1.0;
    acc[0] = fma(sgn, fma(fp.x, fp.x, fp.y * fp.y), acc[0]);
    acc[1] = fma(sgn, fma(fq.x, fq.x, fq.y * fq.y), acc[1]);
    acc[2] = fma(sgn, fma(fp.x, fq.x, fp.y * fq.y), acc[2]);   // Re conj(fp) fq
    acc[3] = fma(sgn, fma(fp.x, fq.y, -fp.y * fq.x), acc[3]);  // Im conj(fp) fq
    acc[4] = fma(gp.x, gp.x, fma(gp.y, gp.y, acc[4]));
    acc[5] = fma(gq.x, gq.x, fma(gq.y, gq.y, acc[5]));
    acc[6] = fma(gp.x, gq.x, fma(gp.y, gq.y, acc[6]));
    acc[7] = fma(gp.x, gq.y, fma(-gp.y, gq.x, acc[7]));
  }
#pragma unroll
  for (int k = 0; k < 8; k++) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
  }
  const int warp = tid >> 5, lane = tid & 31;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 8; k++) red[warp][k] = acc[k];
  }
  __syncthreads();
  if (tid < 8) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; w++) s += red[w][tid];
    part[tid] = s;
  }
  // ---- cluster reduction through DSMEM, fixed rank order
  if (C > 1) {
    cluster.sync();
    if (tid < 8) {
      double s = 0.0;
      for (int r = 0; r < C; r++) s += *cluster.map_shared_rank(&part[tid], r);
      tot[tid] = s;
    }
    cluster_arrive_relaxed();  // remote reads done; waited on before exit
  } else {
    __syncthreads();
    if (tid < 8) tot[tid] = part[tid];
  }
  __syncthreads();
  // ---- (6.2)-(6.12): the 2x2 transformation
  if (tid == 0) {
    const HZOut z = hz2x2_dev(tot, a.tol, a.literal);
    zsh[0] = z.z11.re; zsh[1] = z.z11.im; zsh[2] = z.z21.re; zsh[3] = z.z21.im;
    zsh[4] = z.z12.re; zsh[5] = z.z12.im; zsh[6] = z.z22.re; zsh[7] = z.z22.im;
    kind_sh = z.kind;
    if (rank == 0) {
      if (z.kind < 0) atomicCAS(&a.cnt->err, 0, z.kind);
      if (z.kind == KIND_SMALL || z.kind == KIND_BIG) {
        atomicAdd(&a.cnt->all, 1ull);
        if (z.kind == KIND_BIG) atomicAdd(&a.cnt->big, 1ull);
      }
      atomicMax(&a.cnt->off_bits, (unsigned long long)__double_as_longlong(z.off));
    }
  }
  __syncthreads();
  const int kind = kind_sh;
  if (kind == KIND_SMALL || kind == KIND_BIG) {
    const Cplx z11{zsh[0], zsh[1]}, z21{zsh[2], zsh[3]}, z12{zsh[4], zsh[5]}, z22{zsh[6], zsh[7]};
    if (tid == 0) {
      const unsigned zb = (unsigned)(zlen * 16);
      mbar_expect_tx(&bar[1], 2u * zb);
      if (zlen > 0) {
        bulk_g2s(sZp, a.Z + p * a.ldn + z0, zb, &bar[1]);
        bulk_g2s(sZq, a.Z + q * a.ldn + z0, zb, &bar[1]);
      }
    }
    for (long long i = tid; i < len; i += NT) {
      double2 fp = sFp[i], fq = sFq[i], gp = sGp[i], gq = sGq[i];
      rot_row(fp, fq, z11, z21, z12, z22);
      rot_row(gp, gq, z11, z21, z12, z22);
      sFp[i] = fp; sFq[i] = fq; sGp[i] = gp; sGq[i] = gq;
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0 && len > 0) {
      const unsigned bytes = (unsigned)(len * 16);
      bulk_s2g(gFp, sFp, bytes);
      bulk_s2g(gFq, sFq, bytes);
      bulk_s2g(gGp, sGp, bytes);
      bulk_s2g(gGq, sGq, bytes);
      bulk_commit();
    }
    mbar_wait(&bar[1], 0);
    for (long long i = tid; i < zlen; i += NT) {
      double2 zp = sZp[i], zq = sZq[i];
      rot_row(zp, zq, z11, z21, z12, z22);
      sZp[i] = zp; sZq[i] = zq;
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      if (zlen > 0) {
        const unsigned zb = (unsigned)(zlen * 16);
        bulk_s2g(a.Z + p * a.ldn + z0, sZp, zb);
        bulk_s2g(a.Z + q * a.ldn + z0, sZq, zb);
        bulk_commit();
      }
      bulk_wait_all();
    }
  }
  if (C > 1) cluster_wait();
}

// Persistent, software-pipelined variant: a fixed set of clusters (as many as
// are co-resident) walks the step's pairs pair = cluster_id + it * nclusters;
// each CTA double-buffers its slices so the TMA load of pair it+1 is in flight
// while pair it is reduced, transformed, updated and stored.
template <int NT>
__global__ void __launch_bounds__(NT, 1) k_pair_step_pipe(StepArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bar[3];
  __shared__ double red[NT / 32][8];
  __shared__ double part[2][8];
  __shared__ double tot[8];
  __shared__ double zsh[8];
  __shared__ int kind_sh;

  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const long long nclusters = gridDim.x / C;
  const long long cid = blockIdx.x / C;
  const long long npairs = a.n / 2;

  const long long r0 = (long long)rank * a.cs;
  const long long r1 = min(a.m, r0 + a.cs);
  const long long len = r1 > r0 ? r1 - r0 : 0;
  const long long z0 = (long long)rank * a.zs;
  const long long z1 = min(a.n, z0 + a.zs);
  const long long zlen = z1 > z0 ? z1 - z0 : 0;
  const unsigned bytes = (unsigned)(len * 16), zb = (unsigned)(zlen * 16);

  double2* buf0 = reinterpret_cast<double2*>(smem_raw);
  double2* buf1 = buf0 + 4 * a.cs;
  double2* sZp = buf1 + 4 * a.cs;
  double2* sZq = sZp + a.zs;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue_load = [&](long long pr, double2* buf, unsigned long long* b) {
    long long p, q;
    rr_pair(a.n, a.s, pr, &p, &q);
    mbar_expect_tx(b, 4u * bytes);
    if (len > 0) {
      bulk_g2s(buf, a.F + p * a.ldm + r0, bytes, b);
      bulk_g2s(buf + a.cs, a.F + q * a.ldm + r0, bytes, b);
      bulk_g2s(buf + 2 * a.cs, a.G + p * a.ldm + r0, bytes, b);
      bulk_g2s(buf + 3 * a.cs, a.G + q * a.ldm + r0, bytes, b);
    }
  };

  if (tid == 0 && cid < npairs) issue_load(cid, buf0, &bar[0]);
  unsigned zpar = 0;
  const long long npos_loc = a.npos - r0;
  int it = 0;
  for (long long pair = cid; pair < npairs; pair += nclusters, it++) {
    const int b = it & 1;
    double2* buf = b ? buf1 : buf0;
    const long long nxt = pair + nclusters;
    if (tid == 0) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // previous stores done reading smem
      fence_proxy_async();
      if (nxt < npairs) issue_load(nxt, b ? buf0 : buf1, &bar[b ^ 1]);
    }
    mbar_wait(&bar[b], (unsigned)((it >> 1) & 1));
    long long p, q;
    rr_pair(a.n, a.s, pair, &p, &q);
    double2* sFp = buf;
    double2* sFq = buf + a.cs;
    double2* sGp = buf + 2 * a.cs;
    double2* sGq = buf + 3 * a.cs;
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (long long i = tid; i < len; i += NT) {
      const double2 fp = sFp[i], fq = sFq[i], gp = sGp[i], gq = sGq[i];
      const double sgn = (i < npos_loc) ? 1.0 : -1.0;
      acc[0] = fma(sgn, fma(fp.x, fp.x, fp.y * fp.y), acc[0]);
      acc[1] = fma(sgn, fma(fq.x, fq.x, fq.y * fq.y), acc[1]);
      acc[2] = fma(sgn, fma(fp.x, fq.x, fp.y * fq.y), acc[2]);
      acc[3] = fma(sgn, fma(fp.x, fq.y, -fp.y * fq.x), acc[3]);
      acc[4] = fma(gp.x, gp.x, fma(gp.y, gp.y, acc[4]));
      acc[5] = fma(gq.x, gq.x, fma(gq.y, gq.y, acc[5]));
      acc[6] = fma(gp.x, gq.x, fma(gp.y, gq.y, acc[6]));
      acc[7] = fma(gp.x, gq.y, fma(-gp.y, gq.x, acc[7]));
    }
#pragma unroll
    for (int k = 0; k < 8; k++) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    }
    const int warp = tid >> 5, lane = tid & 31;
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 8; k++) red[warp][k] = acc[k];
    }
    __syncthreads();
    if (tid < 8) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NT / 32; w++) s += red[w][tid];
      part[b][tid] = s;
    }
    if (C > 1) {
      cluster.sync();
      if (tid < 8) {
        double s = 0.0;
        for (int r = 0; r < C; r++) s += *cluster.map_shared_rank(&part[b][tid], r);
        tot[tid] = s;
      }
    } else {
      __syncthreads();
      if (tid < 8) tot[tid] = part[b][tid];
    }
    __syncthreads();
    if (tid == 0) {
      const HZOut z = hz2x2_dev(tot, a.tol, a.literal);
      zsh[0] = z.z11.re; zsh[1] = z.z11.im; zsh[2] = z.z21.re; zsh[3] = z.z21.im;
      zsh[4] = z.z12.re; zsh[5] = z.z12.im; zsh[6] = z.z22.re; zsh[7] = z.z22.im;
      kind_sh = z.kind;
      if (z.kind == KIND_SMALL || z.kind == KIND_BIG) {
        if (zlen > 0) {
          mbar_expect_tx(&bar[2], 2u * zb);
          bulk_g2s(sZp, a.Z + p * a.ldn + z0, zb, &bar[2]);
          bulk_g2s(sZq, a.Z + q * a.ldn + z0, zb, &bar[2]);
        } else {
          mbar_expect_tx(&bar[2], 0u);
        }
      }
      if (rank == 0) {
        if (z.kind < 0) atomicCAS(&a.cnt->err, 0, z.kind);
        if (z.kind == KIND_SMALL || z.kind == KIND_BIG) {
          atomicAdd(&a.cnt->all, 1ull);
          if (z.kind == KIND_BIG) atomicAdd(&a.cnt->big, 1ull);
        }
        atomicMax(&a.cnt->off_bits, (unsigned long long)__double_as_longlong(z.off));
      }
    }
    __syncthreads();
    const int kind = kind_sh;
    if (kind == KIND_SMALL || kind == KIND_BIG) {
      const Cplx z11{zsh[0], zsh[1]}, z21{zsh[2], zsh[3]}, z12{zsh[4], zsh[5]}, z22{zsh[6], zsh[7]};
      for (long long i = tid; i < len; i += NT) {
        double2 fp = sFp[i], fq = sFq[i], gp = sGp[i], gq = sGq[i];
        rot_row(fp, fq, z11, z21, z12, z22);
        rot_row(gp, gq, z11, z21, z12, z22);
        sFp[i] = fp; sFq[i] = fq; sGp[i] = gp; sGq[i] = gq;
      }
      fence_proxy_async();
      __syncthreads();
      if (tid == 0 && len > 0) {
        bulk_s2g(a.F + p * a.ldm + r0, sFp, bytes);
        bulk_s2g(a.F + q * a.ldm + r0, sFq, bytes);
        bulk_s2g(a.G + p * a.ldm + r0, sGp, bytes);
        bulk_s2g(a.G + q * a.ldm + r0, sGq, bytes);
        bulk_commit();
      }
      mbar_wait(&bar[2], zpar);
      zpar ^= 1u;
      for (long long i = tid; i < zlen; i += NT) {
        double2 zp = sZp[i], zq = sZq[i];
        rot_row(zp, zq, z11, z21, z12, z22);
        sZp[i] = zp; sZq[i] = zq;
      }
      fence_proxy_async();
      __syncthreads();
      if (tid == 0 && zlen > 0) {
        bulk_s2g(a.Z + p * a.ldn + z0, sZp, zb);
        bulk_s2g(a.Z + q * a.ldn + z0, sZq, zb);
        bulk_commit();
      }
    }
  }
  if (tid == 0) bulk_wait_all();
  if (C > 1) cluster.sync();  // no CTA leaves while a peer may still read its part[]
}

// Two-pass variant (no shared-memory staging): pass 1 streams the slice from HBM
// forming the Grams (loads marked L2::evict_last so the lines stay in L2), pass 2
// re-reads the slice from L2, applies Z' and streams it back.  No smem for data ->
// occupancy is bounded by registers, so more pairs are in flight per SM to hide
// the per-pair reduce -> transform latency.  HBM traffic stays 128m+64n per
// transformed pair when the in-flight slices fit in L2 (126 MB).
struct C2 {
  double2 a, b;  // two consecutive rows
};
__device__ __forceinline__ C2 ld2_keep(const double2* p) {  // 32-B load, keep in L2
  unsigned long long x0, x1, x2, x3;
  asm volatile("ld.global.L1::no_allocate.L2::evict_last.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3)
               : "l"(p));
  C2 r;
  r.a = make_double2(__longlong_as_double(x0), __longlong_as_double(x1));
  r.b = make_double2(__longlong_as_double(x2), __longlong_as_double(x3));
  return r;
}
__device__ __forceinline__ C2 ld2_last(const double2* p) {  // 32-B load, last use
  unsigned long long x0, x1, x2, x3;
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3)
               : "l"(p));
  C2 r;
  r.a = make_double2(__longlong_as_double(x0), __longlong_as_double(x1));
  r.b = make_double2(__longlong_as_double(x2), __longlong_as_double(x3));
  return r;
}
__device__ __forceinline__ void st2(double2* p, const C2& v) {
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(__double_as_longlong(v.a.x)),
               "l"(__double_as_longlong(v.a.y)), "l"(__double_as_longlong(v.b.x)), "l"(__double_as_longlong(v.b.y))
               : "memory");
}
// 32-B store whose L2 lines are marked evict-first, so the written-back rotated rows do
// not displace the evict-last rows other pairs still have to re-read in pass 2
__device__ __forceinline__ void st2_ef(double2* p, const C2& v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.b64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
               "l"(__double_as_longlong(v.a.x)), "l"(__double_as_longlong(v.a.y)), "l"(__double_as_longlong(v.b.x)),
               "l"(__double_as_longlong(v.b.y)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void gram_row(double* acc, const double2& fp, const double2& fq, const double2& gp,
                                         const double2& gq, double sgn) {
  acc[0] = fma(sgn, fma(fp.x, fp.x, fp.y * fp.y), acc[0]);
  acc[1] = fma(sgn, fma(fq.x, fq.x, fq.y * fq.y), acc[1]);
  acc[2] = fma(sgn, fma(fp.x, fq.x, fp.y * fq.y), acc[2]);
  acc[3] = fma(sgn, fma(fp.x, fq.y, -fp.y * fq.x), acc[3]);
  acc[4] = fma(gp.x, gp.x, fma(gp.y, gp.y, acc[4]));
  acc[5] = fma(gq.x, gq.x, fma(gq.y, gq.y, acc[5]));
  acc[6] = fma(gp.x, gq.x, fma(gp.y, gq.y, acc[6]));
  acc[7] = fma(gp.x, gq.y, fma(-gp.y, gq.x, acc[7]));
}

template <int NT>
__global__ void __launch_bounds__(NT) k_pair_step_2p(StepArgs a) {
  __shared__ double red[NT / 32][8];
  __shared__ double part[8];
  __shared__ double tot[8];
  __shared__ double zsh[8];
  __shared__ int kind_sh;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const long long pair = blockIdx.x / C;
  long long p, q;
  rr_pair(a.n, a.s, pair, &p, &q);
  const long long r0 = (long long)rank * a.cs;
  const long long r1 = min(a.m, r0 + a.cs);
  const long long z0 = (long long)rank * a.zs;
  const long long z1 = min(a.n, z0 + a.zs);
  double2* Fp = a.F + p * a.ldm;
  double2* Fq = a.F + q * a.ldm;
  double2* Gp = a.G + p * a.ldm;
  double2* Gq = a.G + q * a.ldm;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // rows in pairs (2i, 2i+1): r0 even (cs even), ld multiple of 16 -> 32-B aligned
  const long long h0 = r0 >> 1, h1 = (r1 + 1) >> 1;
#pragma unroll 2
  for (long long h = h0 + tid; h < h1; h += NT) {
    const C2 fp = ld2_keep(Fp + 2 * h), fq = ld2_keep(Fq + 2 * h), gp = ld2_keep(Gp + 2 * h), gq = ld2_keep(Gq + 2 * h);
    gram_row(acc, fp.a, fq.a, gp.a, gq.a, (2 * h < a.npos) ? 1.0 : -1.0);
    gram_row(acc, fp.b, fq.b, gp.b, gq.b, (2 * h + 1 < a.npos) ? 1.0 : -1.0);
  }
#pragma unroll
  for (int k = 0; k < 8; k++) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
  }
  const int warp = tid >> 5, lane = tid & 31;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 8; k++) red[warp][k] = acc[k];
  }
  __syncthreads();
  if (tid < 8) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; w++) s += red[w][tid];
    part[tid] = s;
  }
  if (C > 1) {
    cluster.sync();
    if (tid < 8) {
      double s = 0.0;
      for (int r = 0; r < C; r++) s += *cluster.map_shared_rank(&part[tid], r);
      tot[tid] = s;
    }
    cluster_arrive_relaxed();
  } else {
    __syncthreads();
    if (tid < 8) tot[tid] = part[tid];
  }
  __syncthreads();
  if (tid == 0) {
    const HZOut z = hz2x2_dev(tot, a.tol, a.literal);
    zsh[0] = z.z11.re; zsh[1] = z.z11.im; zsh[2] = z.z21.re; zsh[3] = z.z21.im;
    zsh[4] = z.z12.re; zsh[5] = z.z12.im; zsh[6] = z.z22.re; zsh[7] = z.z22.im;
    kind_sh = z.kind;
    if (rank == 0) {
      if (z.kind < 0) atomicCAS(&a.cnt->err, 0, z.kind);
      if (z.kind == KIND_SMALL || z.kind == KIND_BIG) {
        atomicAdd(&a.cnt->all, 1ull);
        if (z.kind == KIND_BIG) atomicAdd(&a.cnt->big, 1ull);
      }
      atomicMax(&a.cnt->off_bits, (unsigned long long)__double_as_longlong(z.off));
    }
  }
  __syncthreads();
  const int kind = kind_sh;
  if (kind == KIND_SMALL || kind == KIND_BIG) {
    const Cplx z11{zsh[0], zsh[1]}, z21{zsh[2], zsh[3]}, z12{zsh[4], zsh[5]}, z22{zsh[6], zsh[7]};
    // pass 2 walks the rows in reverse: the most recently loaded (most likely still in
    // L2) first; stores are marked evict-first
    const unsigned long long pol = policy_evict_first();
    const long long hl = h0 + tid + ((h1 - 1 - h0 - tid) / NT) * NT;   // this thread's last row pair
#pragma unroll 2
    for (long long h = hl; h >= h0 + tid && h < h1; h -= NT) {
      C2 fp = ld2_last(Fp + 2 * h), fq = ld2_last(Fq + 2 * h), gp = ld2_last(Gp + 2 * h), gq = ld2_last(Gq + 2 * h);
      rot_row(fp.a, fq.a, z11, z21, z12, z22);
      rot_row(fp.b, fq.b, z11, z21, z12, z22);
      rot_row(gp.a, gq.a, z11, z21, z12, z22);
      rot_row(gp.b, gq.b, z11, z21, z12, z22);
      st2_ef(Fp + 2 * h, fp, pol); st2_ef(Fq + 2 * h, fq, pol); st2_ef(Gp + 2 * h, gp, pol); st2_ef(Gq + 2 * h, gq, pol);
    }
    double2* Zp = a.Z + p * a.ldn;
    double2* Zq = a.Z + q * a.ldn;
#pragma unroll 2
    for (long long i = z0 + tid; i < z1; i += NT) {
      double2 zp = Zp[i], zq = Zq[i];
      rot_row(zp, zq, z11, z21, z12, z22);
      Zp[i] = zp; Zq[i] = zq;
    }
    if (a.W) {
      // NEXT-1: W = Z'^{-1} <- Zhat'^{-1} W on rows p, q, i.e. the
      // columns p, q of W^T times (Zhat'^{-1})^T = (1/det) [[z22, -z21], [-z12, z11]]
      const double dre = (z11.re * z22.re - z11.im * z22.im) - (z12.re * z21.re - z12.im * z21.im);
      const double dim = (z11.re * z22.im + z11.im * z22.re) - (z12.re * z21.im + z12.im * z21.re);
      const double dd = dre * dre + dim * dim;
      const Cplx idet{dre / dd, -dim / dd};
      auto cm = [](const Cplx& x, const Cplx& y) {
        return Cplx{x.re * y.re - x.im * y.im, x.re * y.im + x.im * y.re};
      };
      const Cplx i11 = cm(z22, idet), i22 = cm(z11, idet);
      const Cplx m12 = cm(z12, idet), m21 = cm(z21, idet);
      const Cplx i21{-m12.re, -m12.im}, i12{-m21.re, -m21.im};
      double2* Wp = a.W + p * a.ldn;
      double2* Wq = a.W + q * a.ldn;
      for (long long i = z0 + tid; i < z1; i += NT) {
        double2 wp = Wp[i], wq = Wq[i];
        rot_row(wp, wq, i11, i21, i12, i22);
        Wp[i] = wp; Wq[i] = wq;
      }
    }
  }
  if (C > 1) cluster_wait();
}

// ------------------------------------------------------------------ host side
typedef void (*StepKernel)(StepArgs);

static StepKernel pick_kernel(int threads, int kind) {
  if (kind == 2) {
    switch (threads) {
      case 32: return k_pair_step_2p<32>;
      case 64: return k_pair_step_2p<64>;
      case 128: return k_pair_step_2p<128>;
      case 512: return k_pair_step_2p<512>;
      default: return k_pair_step_2p<256>;
    }
  }
  if (kind == 3) {
    switch (threads) {
      case 32: return k_pair_step_pipe<32>;
      case 64: return k_pair_step_pipe<64>;
      case 128: return k_pair_step_pipe<128>;
      case 512: return k_pair_step_pipe<512>;
      default: return k_pair_step_pipe<256>;
    }
  }
  switch (threads) {
    case 32: return k_pair_step<32>;
    case 64: return k_pair_step<64>;
    case 128: return k_pair_step<128>;
    case 512: return k_pair_step<512>;
    default: return k_pair_step<256>;
  }
}

ghsvd_status pw_configure(Ctx* ctx) {
  const int64_t m = ctx->m, n = ctx->n;
  // kernel kinds (ghsvd_options.kernel): 1 = one cluster per pair (TMA staging),
  // 2 = two-pass through L2 (no staging, default), 3 = persistent pipelined TMA
  const int kk = ctx->o.kernel == 0 ? 2 : ctx->o.kernel;
  if (kk < 1 || kk > 3) {
    ctx->err = "kernel must be 0..3";
    return GHSVD_E_INVALID_ARG;
  }
  const bool pipe = kk == 3;
  if (ctx->o.want_x && kk != 2) {
    ctx->err = "want_x needs the default pointwise kernel (2)";
    return GHSVD_E_INVALID_ARG;
  }
  const int nbuf = kk == 3 ? 8 : (kk == 1 ? 4 : 0);   // F/G slice buffers (x cs) per CTA
  int C = ctx->o.cluster;
  if (C <= 0 && kk == 2) {
    // two-pass kernel: measured on config 3 (m = 10368, tools/profile_step.py, ms per
    // step): C=1/T=256 0.739, C=2/T=128 0.714, C=4/T=128 0.672, C=8/T=128 0.696; small
    // m (the pair's columns fit in L2 anyway) keeps one CTA per pair.  Capping the
    // resident CTAs per SM (so that more pass-2 reads hit L2) was slower at every cap:
    // C=4/T=128 with 9 / 6 / 4 / 3 CTAs per SM: 0.665 / 0.800 / 0.733 / 0.822 ms per step
    C = m >= 4096 ? 4 : 1;
  } else if (C <= 0) {
    // smallest power-of-two cluster whose per-CTA slices fit the smem budget
    const int64_t budget = pipe ? 200 * 1024 : 100 * 1024;
    C = 1;
    while (C < 16) {
      const int64_t cs = (m + C - 1) / C, zs = (n + C - 1) / C;
      if ((nbuf * cs + (nbuf ? 2 * zs : 0)) * 16 <= budget || (nbuf == 0 && C == 8)) break;
      C *= 2;
    }
  }
  if (C != 1 && C != 2 && C != 4 && C != 8 && C != 16) {
    ctx->err = "cluster must be 1, 2, 4, 8 or 16";
    return GHSVD_E_INVALID_ARG;
  }
  const int64_t cs = round_up((m + C - 1) / C, 2), zs = (n + C - 1) / C;
  int T = ctx->o.threads;
  if (T <= 0 && kk == 2 && m >= 4096) {
    T = 128;
  } else if (T <= 0) {
    T = 256;
    while (T > 32 && T / 2 >= cs) T /= 2;
  }
  if (T != 32 && T != 64 && T != 128 && T != 256 && T != 512) {
    ctx->err = "threads must be 32, 64, 128, 256 or 512";
    return GHSVD_E_INVALID_ARG;
  }
  const size_t smem = nbuf ? (size_t)(nbuf * cs + 2 * zs) * 16 : 0;
  if (smem > 220 * 1024) {
    ctx->err = "pointwise slices exceed shared memory; use a larger cluster";
    return GHSVD_E_INVALID_ARG;
  }
  StepKernel k = pick_kernel(T, kk);
  GH_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (C > 8) GH_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  ctx->pw_cluster = C;
  ctx->pw_threads = T;
  ctx->pw_smem = smem;
  ctx->pw_pipe = pipe;
  ctx->pw_kind = kk;
  ctx->pw_nclusters = n / 2;
  if (pipe) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n / 2 * C), 1, 1);
    cfg.blockDim = dim3(T, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    GH_CUDA(cudaOccupancyMaxActiveClusters(&ncl, k, &cfg));
    if (ncl < 1) {
      ctx->err = "pointwise: no cluster of this shape fits on the device";
      return GHSVD_E_INVALID_ARG;
    }
    ctx->pw_nclusters = std::min<int64_t>(ncl, n / 2);
  }
  return GHSVD_OK;
}

static ghsvd_status launch_step(Ctx* ctx, cudaStream_t st, int64_t s) {
  StepArgs a;
  a.F = ctx->F;
  a.G = ctx->G;
  a.Z = ctx->Z;
  a.ldm = ctx->ldm;
  a.ldn = ctx->ldn;
  a.m = ctx->m;
  a.n = ctx->n;
  a.npos = ctx->npos;
  a.s = s;
  const int C = ctx->pw_cluster;
  a.cs = round_up((ctx->m + C - 1) / C, 2);
  a.zs = (ctx->n + C - 1) / C;
  a.tol = (ctx->o.eps > 0 ? ctx->o.eps : 0x1p-53) * sqrt((double)ctx->n);
  a.literal = ctx->o.criterion == GHSVD_CRIT_LITERAL;
  a.cnt = ctx->cnt;
  a.W = ctx->o.want_x ? ctx->W : nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ctx->pw_nclusters * C), 1, 1);
  cfg.blockDim = dim3(ctx->pw_threads, 1, 1);
  cfg.dynamicSmemBytes = ctx->pw_smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GH_CUDA(cudaLaunchKernelEx(&cfg, pick_kernel(ctx->pw_threads, ctx->pw_kind), a));
  return GHSVD_OK;
}

ghsvd_status pw_run_steps(Ctx* ctx, int64_t s0, int64_t ns) {
  for (int64_t s = s0; s < s0 + ns; s++) {
    ghsvd_status e = launch_step(ctx, ctx->stream, s);
    if (e) return e;
  }
  return GHSVD_OK;
}

// Enqueue one full sweep (n-1 steps).  With use_graph the launches are
// captured once per (buffers, shape, config) and replayed as a CUDA graph.
ghsvd_status pw_sweep_launch(Ctx* ctx) {
  if (!ctx->o.use_graph) return pw_run_steps(ctx, 0, ctx->n - 1);
  const int64_t key = (int64_t)(uintptr_t)ctx->F ^ ((int64_t)ctx->n << 40) ^
                      ((int64_t)ctx->pw_cluster << 56) ^ ((int64_t)ctx->pw_threads << 48) ^ ((int64_t)ctx->pw_kind << 45) ^
                      ctx->npos * 1315423911ll ^ ctx->m * 2654435761ll;
  if (!ctx->graph || ctx->graph_key != key) {
    if (ctx->graph) {
      cudaGraphExecDestroy(ctx->graph);
      ctx->graph = nullptr;
    }
    cudaGraph_t g;
    GH_CUDA(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    for (int64_t s = 0; s < ctx->n - 1; s++) {
      ghsvd_status e = launch_step(ctx, ctx->cap_stream, s);
      if (e) {
        cudaStreamEndCapture(ctx->cap_stream, &g);
        return e;
      }
    }
    GH_CUDA(cudaStreamEndCapture(ctx->cap_stream, &g));
    GH_CUDA(cudaGraphInstantiate(&ctx->graph, g, 0));
    cudaGraphDestroy(g);
    ctx->graph_key = key;
  }
  GH_CUDA(cudaGraphLaunch(ctx->graph, ctx->stream));
  return GHSVD_OK;
}

}  // namespace ghsvd
