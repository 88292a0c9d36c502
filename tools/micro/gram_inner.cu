// The block Gram's inner loop alone (exploration tool): k_blk_gram's 3M warp-specialized
// tile code (gram3_tiles, the library's own header) over a shared-memory stage that is
// filled once -- no cp.async pipeline, no per-stage barrier, no split partials, no factor
// tail -- 8 warps per CTA, 2 CTAs per SM as in the kernel.  Compares the DMMA rate the
// instruction mix allows with the kernel's (isolated split Gram: ~79 % of ZGEMM in the
// Hermitian count, DMMA ~72 % busy).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -Iinclude -o /tmp/gram_inner tools/micro/gram_inner.cu && /tmp/gram_inner
#include <cstdio>

#include "../../paper_1907_08560_b200/csrc/blk_gram.cuh"

namespace ghsvd {
namespace {
__global__ void __launch_bounds__(NT_G, 2) k_gram_inner(double* out, int stages) {
  extern __shared__ __align__(128) double2 gsm[];
  constexpr int TS = GS;
  for (int e = threadIdx.x; e < KM * TS; e += NT_G) gsm[e] = make_double2(1e-3 * (e % 97), 1e-3 * (e % 89));
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[5][6];
#pragma unroll
  for (int t = 0; t < 5; t++)
#pragma unroll
    for (int c = 0; c < 6; c++) acc[t][c] = 0.0;
  for (int st = 0; st < stages; st++) {
    const double2* T = gsm;
#pragma unroll 1
    for (int ks = 0; ks < RTG / 4; ks += 2) {
      const int row0 = 4 * ks + (lane & 3), row1 = row0 + 4;
      const unsigned sg0 = (st & 1) ? 0x80000000u : 0u, sg1 = 0u;
      switch (warp) {
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
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 5; t++)
#pragma unroll
    for (int c = 0; c < 6; c++) s += acc[t][c];
  if (s == 1234.5) out[threadIdx.x] = s;
}
}  // namespace
}  // namespace ghsvd

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o;
  cudaMalloc(&o, 4096);
  const int smem = ghsvd::GSTAGES * ghsvd::KM * ghsvd::GS * 16;
  cudaFuncSetAttribute(ghsvd::k_gram_inner, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int stages = 512;
  ghsvd::k_gram_inner<<<2 * sms, ghsvd::NT_G, smem>>>(o, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ghsvd::k_gram_inner<<<2 * sms, ghsvd::NT_G, smem>>>(o, stages);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // per CTA and 32-row stage: 8 k-steps x 36 tiles x 3 DMMAs (8x8x4, 512 flops each)
  const double dmma_flops = 2.0 * sms * stages * (ghsvd::RTG / 4) * 36 * 3 * 512.0;
  printf("gram inner loop: %.2f TFLOP/s of DMMA (%s)\n", dmma_flops / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
