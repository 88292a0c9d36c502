// factors.cu -- boundary data movement: the J row sort (Sec 4.5.1 n+ form),
// bordering (Sec 6.3.2), identity initialisation of Z' (Alg. 2 first line).
#include <cuda_runtime.h>

#include "internal.h"

namespace ghsvd {

__global__ void k_set_identity(double2* Z, long long ldz, long long n) {
  const long long c = blockIdx.y;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < ldz; r += (long long)gridDim.x * blockDim.x)
    Z[c * ldz + r] = make_double2(r == c ? 1.0 : 0.0, 0.0);
}

ghsvd_status launch_set_identity(Ctx* ctx, double2* Z, int64_t ldz, int64_t n) {
  if (n <= 0) return GHSVD_OK;
  dim3 grid((unsigned)((ldz + 255) / 256), (unsigned)n);
  k_set_identity<<<grid, 256, 0, ctx->stream>>>(Z, ldz, n);
  GH_CUDA(cudaGetLastError());
  return GHSVD_OK;
}

// Stable partition of the rows by sign (+ first): dest[i] = new row of row i.
// One CTA; each thread owns a contiguous chunk; block-wide exclusive scan.
// Also validates J (entries must be +-1): *npos_out = -1 on a bad entry.
__global__ void k_sort_dest(const int8_t* J, long long m, int* dest, int8_t* Jout, long long* npos_out) {
  __shared__ long long cnt[1024];
  __shared__ int bad;
  __shared__ long long npos_sh;
  const int T = blockDim.x, t = threadIdx.x;
  if (t == 0) bad = 0;
  __syncthreads();
  const long long chunk = (m + T - 1) / T;
  const long long b = min(m, t * chunk), e = min(m, b + chunk);
  long long c = 0;
  for (long long i = b; i < e; i++) {
    const int8_t j = J[i];
    if (j != 1 && j != -1) bad = 1;
    c += (j > 0);
  }
  cnt[t] = c;
  __syncthreads();
  if (t == 0) {
    long long s = 0;
    for (int k = 0; k < T; k++) {
      const long long v = cnt[k];
      cnt[k] = s;
      s += v;
    }
    *npos_out = bad ? -1 : s;
    npos_sh = s;
  }
  __syncthreads();
  const long long npos = npos_sh;
  long long pp = cnt[t];        // positives before my chunk
  long long nn = b - cnt[t];    // negatives before my chunk
  for (long long i = b; i < e; i++) {
    if (J[i] > 0) {
      dest[i] = (int)pp;
      Jout[pp] = 1;
      pp++;
    } else {
      dest[i] = (int)(npos + nn);
      Jout[npos + nn] = -1;
      nn++;
    }
  }
}

ghsvd_status launch_sort_dest(Ctx* ctx, const int8_t* Jin, int64_t m, bool, int* dest, int8_t* Jout,
                              int64_t* npos_dev) {
  k_sort_dest<<<1, 1024, 0, ctx->stream>>>(Jin, m, dest, Jout, (long long*)npos_dev);
  GH_CUDA(cudaGetLastError());
  return GHSVD_OK;
}

// dst[dest[r], c] = src[r, c]
__global__ void k_row_scatter(const double2* __restrict__ src, long long lds, double2* __restrict__ dst,
                              long long ldd, const int* __restrict__ dest, long long rows) {
  const long long c = blockIdx.y;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x)
    dst[c * ldd + dest[r]] = src[c * lds + r];
}

ghsvd_status launch_row_scatter(Ctx* ctx, const double2* src, int64_t lds, double2* dst, int64_t ldd,
                                const int* dest, int64_t rows, int64_t cols) {
  if (rows <= 0 || cols <= 0) return GHSVD_OK;
  dim3 grid((unsigned)std::min<int64_t>((rows + 255) / 256, 64), (unsigned)cols);
  k_row_scatter<<<grid, 256, 0, ctx->stream>>>(src, lds, dst, ldd, dest, rows);
  GH_CUDA(cudaGetLastError());
  return GHSVD_OK;
}

}  // namespace ghsvd
