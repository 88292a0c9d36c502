// DMMA.8x8x4 issue-rate microbenchmark (exploration tool, not part of the library):
// how many independent accumulator chains per warp and warps per SM the FP64 tensor
// pipe needs on this B200 to reach its peak, with operands in registers (no loads).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_rate tools/micro/dmma_rate.cu && /tmp/dmma_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void k_rate(double* out, int iters, double seed) {
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i][0] = acc[i][1] = 0.0;
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5 + threadIdx.x * 1e-9;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
void run(int warps_per_cta, int ctas_per_sm, int sms) {
  double* d;
  cudaMalloc(&d, 1024 * sizeof(double));
  const int iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_rate<NACC><<<sms * ctas_per_sm, warps_per_cta * 32>>>(d, 16, 1.0);
  cudaEventRecord(e0);
  k_rate<NACC><<<sms * ctas_per_sm, warps_per_cta * 32>>>(d, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmmas = (double)sms * ctas_per_sm * warps_per_cta * iters * NACC;
  const double tflops = dmmas * 512.0 / (ms * 1e-3) / 1e12;
  printf("NACC %2d  warps/SM %2d  (%d CTAs x %d warps)  %.2f TFLOP/s  %.1f cycles/DMMA/SMSP @1.965GHz\n", NACC,
         warps_per_cta * ctas_per_sm, ctas_per_sm, warps_per_cta, tflops,
         (ms * 1e-3) * 1.965e9 / (dmmas / sms / 4));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  for (int w : {4, 8, 16}) {
    run<1>(w, 1, sms);
    run<2>(w, 1, sms);
    run<4>(w, 1, sms);
    run<8>(w, 1, sms);
    run<12>(w, 1, sms);
    run<16>(w, 1, sms);
    run<24>(w, 1, sms);
  }
  run<12>(8, 2, sms);
  run<15>(8, 2, sms);
  return 0;
}
