// extract.cu -- a8: outputs of Sec 6.1.7 and eq (3.2),
// plus the device 2x2 test hook and the bordering kernel (Sec 6.3.2).
#include <cuda_runtime.h>

#include "hz2x2.cuh"
#include "internal.h"

namespace ghsvd {

// One CTA per column c: a = f_c^* J f_c, b = g_c^* g_c (J = diag(I_npos, -I)),
// lambda = a/b, Sigma'_F = |a|^1/2, Sigma'_G = b^1/2, Sigma = (Sigma'_F^2 +
// Sigma'_G^2)^1/2, sigma_f = Sigma'_F/Sigma, sigma_g = Sigma'_G/Sigma,
// Z[:, c] = Z'[:, c] / Sigma with rows un-permuted by P2 (row p2[j] <- row j).
template <int NT>
__global__ void __launch_bounds__(NT) k_extract(const double2* __restrict__ F, const double2* __restrict__ G,
                                                const double2* __restrict__ Zp, double2* __restrict__ Zout,
                                                long long ldm, long long ldn, long long m, long long n_rows,
                                                long long npos, const long long* __restrict__ p2,
                                                long long np2, double* lam, double* sf, double* sg,
                                                const double2* __restrict__ Wt, double2* __restrict__ Xout) {
  __shared__ double red[NT / 32][2];
  __shared__ double inv_sig, sig_sh;
  const long long c = blockIdx.x;
  const double2* f = F + c * ldm;
  const double2* g = G + c * ldm;
  double a = 0.0, b = 0.0;
  for (long long r = threadIdx.x; r < m; r += NT) {
    const double2 x = f[r], y = g[r];
    const double fx = fma(x.x, x.x, x.y * x.y);
    a += (r < npos) ? fx : -fx;
    b = fma(y.x, y.x, fma(y.y, y.y, b));
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5][0] = a;
    red[threadIdx.x >> 5][1] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0.0, B = 0.0;
    for (int w = 0; w < NT / 32; w++) {
      A += red[w][0];
      B += red[w][1];
    }
    const double sfp = sqrt(fabs(A)), sgp = sqrt(B);
    const double sig = sqrt(sfp * sfp + sgp * sgp);
    lam[c] = A / B;
    sf[c] = sfp / sig;
    sg[c] = sgp / sig;
    inv_sig = 1.0 / sig;
    sig_sh = sig;
  }
  __syncthreads();
  const double is = inv_sig;
  const double2* z = Zp + c * ldn;
  double2* zo = Zout + c * ldn;
  for (long long r = threadIdx.x; r < n_rows; r += NT) {
    const double2 v = z[r];
    const long long dr = (r < np2) ? p2[r] : r;
    zo[dr] = make_double2(v.x * is, v.y * is);
  }
  if (Wt) {
    // NEXT-1: X = Sigma Z'^{-1}; row c of X is Sigma_c times column c of W^T; columns
    // permuted back by P2 (X~ = X P2^T)
    const double sg_c = sig_sh;
    const double2* w = Wt + c * ldn;
    for (long long r = threadIdx.x; r < n_rows; r += NT) {
      const double2 v = w[r];
      const long long dr = (r < np2) ? p2[r] : r;
      Xout[c + dr * ldn] = make_double2(v.x * sg_c, v.y * sg_c);
    }
  }
}

ghsvd_status launch_extract(Ctx* ctx) {
  const long long np2 = ctx->have_p2 ? ctx->n_user : 0;
  k_extract<256><<<(unsigned)ctx->n, 256, 0, ctx->stream>>>(
      ctx->F, ctx->G, ctx->Z, ctx->Z2, ctx->ldm, ctx->ldn, ctx->m, ctx->n, ctx->npos,
      (const long long*)ctx->p2, np2, ctx->lam, ctx->sf, ctx->sg, ctx->o.want_x ? ctx->W : nullptr,
      ctx->o.want_x ? ctx->Xo : nullptr);
  GH_CUDA(cudaGetLastError());
  return GHSVD_OK;
}

__global__ void k_hz2x2_batch(long long count, const double* in, double tol, int literal, double* out,
                              int* kind) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= count) return;
  double g[8];
#pragma unroll
  for (int k = 0; k < 8; k++) g[k] = in[8 * i + k];
  const HZOut z = hz2x2_dev(g, tol, literal);
  double* o = out + 8 * i;
  o[0] = z.z11.re; o[1] = z.z11.im; o[2] = z.z21.re; o[3] = z.z21.im;
  o[4] = z.z12.re; o[5] = z.z12.im; o[6] = z.z22.re; o[7] = z.z22.im;
  kind[i] = z.kind;
}

ghsvd_status launch_hz2x2_batch(Ctx* ctx, int64_t count, const double* in, double tol, int criterion,
                                double* out, int* kind) {
  if (count <= 0) return GHSVD_OK;
  k_hz2x2_batch<<<(unsigned)((count + 127) / 128), 128, 0, ctx->stream>>>(
      count, in, tol, criterion == GHSVD_CRIT_LITERAL, out, kind);
  GH_CUDA(cudaGetLastError());
  return GHSVD_OK;
}

}  // namespace ghsvd
