// DMMA.8x8x4 rate with the 3M scheme's side work interleaved (exploration tool): per
// iteration NACC independent DMMAs plus ND dependent-free DADDs and/or NL shared-memory
// fragment loads feeding the DMMAs, 16 warps per SM (2 CTAs x 8 warps), as in the
// blocked kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_mix tools/micro/dmma_mix.cu && /tmp/dmma_mix
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC, int ND, int NL>
__global__ void k_mix(double* out, int iters, double seed) {
  __shared__ double2 sm[64 * 36];
  for (int i = threadIdx.x; i < 64 * 36; i += blockDim.x) sm[i] = make_double2(seed + i * 1e-12, seed - i * 1e-12);
  __syncthreads();
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i][0] = acc[i][1] = 0.0;
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5 + threadIdx.x * 1e-9;
  double d[ND > 0 ? ND : 1];
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); i++) d[i] = seed * i;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; it++) {
    double2 f[NL > 0 ? NL : 1];
#pragma unroll
    for (int l = 0; l < NL; l++) f[l] = sm[(8 * l + (lane >> 2)) * 36 + (it & 7) * 4 + (lane & 3)];
#pragma unroll
    for (int i = 0; i < ND; i++) d[i] = d[i] + a;
#pragma unroll
    for (int i = 0; i < NACC; i++) {
      const double x = NL > 0 ? f[i % NL].x : a;
      const double y = NL > 0 ? f[(i + 1) % NL].y : b;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(x), "d"(y));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < ND; i++) s += d[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC, int ND, int NL>
void run(int sms) {
  double* o;
  cudaMalloc(&o, 1024 * sizeof(double));
  const int iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mix<NACC, ND, NL><<<sms * 2, 256>>>(o, 16, 1.0);
  cudaEventRecord(e0);
  k_mix<NACC, ND, NL><<<sms * 2, 256>>>(o, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmmas = (double)sms * 2 * 8 * iters * NACC;
  printf("NACC %2d  DADD %2d  LDS.128 %2d per iteration: %.2f TFLOP/s of DMMA\n", NACC, ND, NL,
         dmmas * 512.0 / (ms * 1e-3) / 1e12);
  cudaFree(o);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<12, 0, 0>(sms);
  run<12, 1, 0>(sms);
  run<12, 2, 0>(sms);
  run<12, 5, 0>(sms);
  run<12, 10, 0>(sms);
  run<12, 0, 1>(sms);
  run<12, 0, 4>(sms);
  run<12, 0, 8>(sms);
  run<12, 5, 5>(sms);
  run<27, 10, 8>(sms);
  run<24, 10, 8>(sms);
  return 0;
}
