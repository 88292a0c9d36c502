// phase1.cu -- ghsvd_factor: Phase 1 (Algorithm 1; eqs 4.1-4.3).
//
// Per atom a (one CTA each, all atoms concurrently):
//   T_a = [[T_AA, T_AB], [T_AB^*, T_BB]]  (eq 3.3; lower triangle read)
//   HEBPJ (Sec 4.2-4.3): Bunch-Parlett complete pivoting LDL^*, alpha =
//   (1+sqrt 17)/8; 2x2 pivots diagonalised by a Jacobi rotation; rows scaled
//   by |d|^1/2; Mhat = M P; rows sorted + before -.
// Then F_a = Mtilde_a [A_a; B_a] (the paper's ZGEMM, here an smem-tiled
// in-place complex product per atom and column tile), G_a = [A_a; U_a B_a]
// (ZDSCAL), and the rows of F are stably sorted by sign across atoms so the
// sweep sees J = diag(I_{n+}, -I) (Sec 4.5.1 n+ representation).
// Runs once per problem (boundary, not hot path).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "hebpj.cuh"
#include "internal.h"

namespace ghsvd {

namespace {

__device__ __forceinline__ double2 c_conj(double2 a) { return make_double2(a.x, -a.y); }

struct P1Scr {
  double2* Taa;   // NA * NL*NL staging of the T blocks
  double2* Tab;
  double2* Tbb;
  double* U;      // NA * NL
  double2* W;     // NA * r*r working matrix (L stored below the diagonal)
  double2* M;     // NA * r*r output Mtilde_a
  int* npos;      // NA
  int* info;      // NA  (0 ok, -7 rank deficient)
};

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

P1Scr carve(char* base, int64_t NA, int64_t NL) {
  const int64_t r = 2 * NL;
  P1Scr s;
  char* p = base;
  s.Taa = (double2*)p; p += al256((size_t)NA * NL * NL * 16);
  s.Tab = (double2*)p; p += al256((size_t)NA * NL * NL * 16);
  s.Tbb = (double2*)p; p += al256((size_t)NA * NL * NL * 16);
  s.U = (double*)p; p += al256((size_t)NA * NL * 8);
  s.W = (double2*)p; p += al256((size_t)NA * r * r * 16);
  s.M = (double2*)p; p += al256((size_t)NA * r * r * 16);
  s.npos = (int*)p; p += al256((size_t)NA * 4);
  s.info = (int*)p; p += al256((size_t)NA * 4);
  return s;
}

size_t carve_bytes(int64_t NA, int64_t NL) {
  const int64_t r = 2 * NL;
  return 3 * al256((size_t)NA * NL * NL * 16) + al256((size_t)NA * NL * 8) + 2 * al256((size_t)NA * r * r * 16) +
         2 * al256((size_t)NA * 4) + 256;
}

constexpr int P1T = 256;

// Build W_a (full Hermitian from the lower triangle of T_a) and the tolerance.
__global__ void __launch_bounds__(P1T) k_build_T(P1Scr s, int NL) {
  const int a = blockIdx.x, r = 2 * NL;
  const double2* taa = s.Taa + (size_t)a * NL * NL;
  const double2* tab = s.Tab + (size_t)a * NL * NL;
  const double2* tbb = s.Tbb + (size_t)a * NL * NL;
  double2* W = s.W + (size_t)a * r * r;
  for (int e = threadIdx.x; e < r * r; e += P1T) {
    const int i = e % r, j = e / r;
    const int ii = i >= j ? i : j, jj = i >= j ? j : i;  // lower-triangle source (ii >= jj)
    double2 v;
    if (ii < NL) v = taa[ii + (size_t)jj * NL];
    else if (jj >= NL) v = tbb[(ii - NL) + (size_t)(jj - NL) * NL];
    else v = c_conj(tab[jj + (size_t)(ii - NL) * NL]);  // T_BA = T_AB^*
    if (ii == jj) v.y = 0.0;
    W[i + (size_t)j * r] = (i >= j) ? v : c_conj(v);
  }
}

// HEBPJ of one T_a per CTA (in global memory, L2-resident), hebpj.cuh.
__global__ void __launch_bounds__(P1T) k_hebpj(P1Scr s, int NL) {
  const int a = blockIdx.x, r = 2 * NL;
  double2* W = s.W + (size_t)a * r * r;
  double2* M = s.M + (size_t)a * r * r;
  __shared__ signed char Jloc[512];
  __shared__ int np_sh;
  __shared__ hb::HebpjScr<P1T, 512> scr;
  // tolerance r * eps * max|T| over the lower triangle
  double tv = 0.0;
  long long ti = 0;
  for (int e = threadIdx.x; e < r * r; e += P1T) {
    const int i = e % r, j = e / r;
    if (i >= j) hb::amax_merge(tv, ti, hb::cabs(W[i + (size_t)j * r]), 0);
  }
  hb::block_amax<P1T>(tv, ti, scr.sv1, scr.si1);
  const double tolz = __dmul_rn(__dmul_rn((double)r, 0x1p-53), tv);
  const int rc = hb::hebpj_dev<P1T, 512>(W, r, r, M, r, Jloc, &np_sh, tolz, scr);
  if (threadIdx.x == 0) {
    s.info[a] = rc;
    s.npos[a] = rc ? 0 : np_sh;
  }
}

// F rows of atom a (H~_a = [A_a; B_a], r x NG at row offset a*r) <- Mtilde_a H~_a, in place.
constexpr int AM_TC = 8;  // columns per tile
__global__ void __launch_bounds__(256) k_apply_M(P1Scr s, double2* F, long long ldm, int NL, long long NG) {
  extern __shared__ double2 tile[];  // r x AM_TC
  const int a = blockIdx.y, r = 2 * NL;
  const long long c0 = (long long)blockIdx.x * AM_TC;
  const int nc = (int)min((long long)AM_TC, NG - c0);
  double2* Fa = F + (size_t)a * r;
  for (int e = threadIdx.x; e < r * nc; e += 256) {
    const int i = e % r, c = e / r;
    tile[i + c * r] = Fa[i + (c0 + c) * ldm];
  }
  __syncthreads();
  const double2* M = s.M + (size_t)a * r * r;
  for (int e = threadIdx.x; e < r * nc; e += 256) {
    const int i = e % r, c = e / r;
    double re = 0.0, im = 0.0;
    for (int l = 0; l < r; l++) {
      const double2 mv = M[i + (size_t)l * r], hv = tile[l + c * r];
      re = fma(mv.x, hv.x, fma(-mv.y, hv.y, re));
      im = fma(mv.x, hv.y, fma(mv.y, hv.x, im));
    }
    Fa[i + (c0 + c) * ldm] = make_double2(re, im);
  }
}

// Row destinations for the global sign sort and the sorted J.
__global__ void k_p1_dest(P1Scr s, int NA, int NL, int* dest, int8_t* J, long long* npos_out) {
  const int r = 2 * NL;
  __shared__ long long P[1025], Nn[1025];
  if (threadIdx.x == 0) {
    long long p = 0, q = 0;
    for (int a = 0; a < NA; a++) {
      P[a] = p;
      Nn[a] = q;
      p += s.npos[a];
      q += r - s.npos[a];
    }
    P[NA] = p;
    *npos_out = p;
  }
  __syncthreads();
  const long long np = P[NA];
  for (long long g = threadIdx.x; g < (long long)NA * r; g += blockDim.x) {
    const int a = (int)(g / r), i = (int)(g % r);
    const int npa = s.npos[a];
    const long long dd = i < npa ? P[a] + i : np + Nn[a] + (i - npa);
    dest[g] = (int)dd;
    J[dd] = i < npa ? 1 : -1;
  }
}

__global__ void k_scale_UB(double2* G, long long ldm, const double* U, int NA, int NL, long long NG) {
  const long long c = blockIdx.y;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)NA * NL;
       e += (long long)gridDim.x * blockDim.x) {
    const int a = (int)(e / NL), l = (int)(e % NL);
    double2* x = G + c * ldm + (size_t)a * 2 * NL + NL + l;
    const double u = U[e];
    *x = make_double2(x->x * u, x->y * u);
  }
}

}  // namespace

size_t phase1_scratch_bytes(int64_t m, int64_t n, int64_t nl) {
  if (nl <= 0) return 0;
  const int64_t NA = std::max<int64_t>(1, m / (2 * nl));
  return carve_bytes(NA, nl) + 2 * 256;
}

ghsvd_status phase1_factor(Ctx* ctx, int64_t NA, int64_t NL, int64_t NG, const void* A, const void* B,
                           const double* U, const void* TAA, const void* TAB, const void* TBB) {
  const int64_t r = 2 * NL, m = NA * r;
  if (r > 512 || NA > 1024) {
    ctx->err = "factor: 2*NL must be <= 512 and NA <= 1024";
    return GHSVD_E_INVALID_ARG;
  }
  if (carve_bytes(NA, NL) + 256 > ctx->L.scr_bytes) {
    ctx->err = "factor: workspace scratch too small (create with nl >= NL)";
    return GHSVD_E_WORKSPACE;
  }
  cudaStream_t st = ctx->stream;
  P1Scr s = carve(ctx->scr, NA, NL);
  long long* npos_dev = (long long*)((char*)s.info + al256((size_t)NA * 4));
  // 1. stage inputs: [A_a; B_a] into the F buffer; T blocks and U into scratch
  for (int64_t a = 0; a < NA; a++) {
    GH_CUDA(cudaMemcpy2DAsync(ctx->F + a * r, (size_t)ctx->ldm * 16, (const double2*)A + a * NL * NG,
                              (size_t)NL * 16, (size_t)NL * 16, (size_t)NG, cudaMemcpyDefault, st));
    GH_CUDA(cudaMemcpy2DAsync(ctx->F + a * r + NL, (size_t)ctx->ldm * 16, (const double2*)B + a * NL * NG,
                              (size_t)NL * 16, (size_t)NL * 16, (size_t)NG, cudaMemcpyDefault, st));
  }
  GH_CUDA(cudaMemcpyAsync(s.Taa, TAA, (size_t)NA * NL * NL * 16, cudaMemcpyDefault, st));
  GH_CUDA(cudaMemcpyAsync(s.Tab, TAB, (size_t)NA * NL * NL * 16, cudaMemcpyDefault, st));
  GH_CUDA(cudaMemcpyAsync(s.Tbb, TBB, (size_t)NA * NL * NL * 16, cudaMemcpyDefault, st));
  GH_CUDA(cudaMemcpyAsync(s.U, U, (size_t)NA * NL * 8, cudaMemcpyDefault, st));
  // 2. HEBPJ per atom
  k_build_T<<<(unsigned)NA, P1T, 0, st>>>(s, (int)NL);
  GH_CUDA(cudaGetLastError());
  k_hebpj<<<(unsigned)NA, P1T, 0, st>>>(s, (int)NL);
  GH_CUDA(cudaGetLastError());
  std::vector<int> info((size_t)NA);
  GH_CUDA(cudaMemcpyAsync(info.data(), s.info, (size_t)NA * 4, cudaMemcpyDeviceToHost, st));
  GH_CUDA(cudaStreamSynchronize(st));
  for (int64_t a = 0; a < NA; a++)
    if (info[a]) {
      ctx->err = "factor: T_a numerically singular (atom " + std::to_string(a) + ")";
      return GHSVD_E_RANK_DEFICIENT;
    }
  // 3. F_a = Mtilde_a [A_a; B_a] in place
  const size_t smem = (size_t)r * AM_TC * 16;
  GH_CUDA(cudaFuncSetAttribute(k_apply_M, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 g3((unsigned)((NG + AM_TC - 1) / AM_TC), (unsigned)NA);
  k_apply_M<<<g3, 256, smem, st>>>(s, ctx->F, ctx->ldm, (int)NL, NG);
  GH_CUDA(cudaGetLastError());
  // 4. global sign sort of F's rows: F buffer -> G buffer, then swap roles
  k_p1_dest<<<1, 256, 0, st>>>(s, (int)NA, (int)NL, ctx->rowdest, ctx->J, npos_dev);
  GH_CUDA(cudaGetLastError());
  {
    ghsvd_status e = launch_row_scatter(ctx, ctx->F, ctx->ldm, ctx->G, ctx->ldm, ctx->rowdest, m, NG);
    if (e) return e;
  }
  std::swap(ctx->F, ctx->G);
  // 5. G = [A_a; U_a B_a]
  GH_CUDA(cudaMemsetAsync(ctx->G, 0, (size_t)ctx->ldm * (ctx->n_cap + 1) * 16, st));
  for (int64_t a = 0; a < NA; a++) {
    GH_CUDA(cudaMemcpy2DAsync(ctx->G + a * r, (size_t)ctx->ldm * 16, (const double2*)A + a * NL * NG,
                              (size_t)NL * 16, (size_t)NL * 16, (size_t)NG, cudaMemcpyDefault, st));
    GH_CUDA(cudaMemcpy2DAsync(ctx->G + a * r + NL, (size_t)ctx->ldm * 16, (const double2*)B + a * NL * NG,
                              (size_t)NL * 16, (size_t)NL * 16, (size_t)NG, cudaMemcpyDefault, st));
  }
  dim3 g5((unsigned)std::min<int64_t>((NA * NL + 255) / 256, 64), (unsigned)NG);
  k_scale_UB<<<g5, 256, 0, st>>>(ctx->G, ctx->ldm, s.U, (int)NA, (int)NL, NG);
  GH_CUDA(cudaGetLastError());
  long long npos = 0;
  GH_CUDA(cudaMemcpyAsync(&npos, npos_dev, 8, cudaMemcpyDeviceToHost, st));
  GH_CUDA(cudaStreamSynchronize(st));
  ctx->npos = npos;
  return GHSVD_OK;
}

}  // namespace ghsvd
