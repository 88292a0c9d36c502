// phase2.cu -- ghsvd_reduce: optional Phase 2 (Sec 5, eq 5.1).
//
// JQR of F (m x n, J) with the paper's diagonal + partial (Bunch-Kaufman,
// alpha = (1+sqrt 17)/8) pivoting (Sec 5.2.1), hyperbolic Householder
// reflectors H(s) = I + tau s s^* J (Thm 5.1) with the
// sign-compatibility row swap, and (J,I) URV 2x2 pivots (one Jacobi rotation,
// two reflectors, rotation undone).  G is reduced by a
// Householder QR of G P2 (columns visited in P2 order instead of physically
// prepermuted, Sec 5.4.1), keeping R with a real non-negative diagonal.
// Afterwards F's rows are re-sorted so J = diag(I_{n+}, -I) again.
// Each JQR/QR step is a short sequence of kernels (column-parallel J-norms,
// dots and reflector applications across CTAs; pivot logic in one CTA); the
// 1x1 / 2x2 decision is read back once per step.  Runs once per problem.
#include <cuda_runtime.h>

#include <string>

#include "internal.h"

namespace ghsvd {

namespace {

constexpr int T2 = 256;

struct P2Scr {
  double* hd;      // n   J-norms of trailing columns
  double2* d1;     // n   h_1j
  double2* d2;     // n   h_il
  double2* s;      // m   reflector vector
  int* ctl;        // control: [0] type (1 or 2), [1] ii, [2] need2, [3] err, [4] ndiag
  double* dctl;    // [0] tau, [1..2] c1, [4..11] R (4 complex), [12] h1i
};

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

P2Scr carve(char* p, int64_t m, int64_t n) {
  P2Scr s;
  s.hd = (double*)p; p += al256((size_t)n * 8);
  s.d1 = (double2*)p; p += al256((size_t)n * 16);
  s.d2 = (double2*)p; p += al256((size_t)n * 16);
  s.s = (double2*)p; p += al256((size_t)m * 16);
  s.ctl = (int*)p; p += 256;
  s.dctl = (double*)p; p += 256;
  return s;
}

__device__ __forceinline__ double2 cmk(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) { return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return cmk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return cmk(a.x, -a.y); }
__device__ __forceinline__ double cabs_(double2 a) { return sqrt(a.x * a.x + a.y * a.y); }

// block sum of a complex value (deterministic tree); result valid in all threads
__device__ double2 block_sum2(double2 v, double2* sh) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = sh[0];
    for (int w = 1; w < T2 / 32; w++) t = cadd(t, sh[w]);
    sh[0] = t;
  }
  __syncthreads();
  const double2 r = sh[0];
  __syncthreads();
  return r;
}

// x^* J y over rows [r0, m)
__device__ double2 jdot(const double2* x, const double2* y, const int8_t* J, long long r0, long long m,
                        bool useJ, double2* sh) {
  double2 a = cmk(0, 0);
  for (long long i = r0 + threadIdx.x; i < m; i += T2) {
    const double2 u = x[i], v = y[i];
    const double j = useJ ? (double)J[i] : 1.0;
    a.x += j * (u.x * v.x + u.y * v.y);
    a.y += j * (u.x * v.y - u.y * v.x);
  }
  return block_sum2(a, sh);
}

// Block-wide argmax (largest value, smallest index on ties: the same choice as a
// sequential scan keeping the first strict maximum); result valid in every thread.
// Threads with no candidate pass v = -1 (all candidates are >= 0).
__device__ void block_argmax(double& v, long long& i) {
  __shared__ double bv[T2 / 32];
  __shared__ long long bi[T2 / 32];
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (v2 > v || (v2 == v && i2 < i)) {
      v = v2;
      i = i2;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    bv[threadIdx.x >> 5] = v;
    bi[threadIdx.x >> 5] = i;
  }
  __syncthreads();
  v = bv[0];
  i = bi[0];
  for (int w = 1; w < T2 / 32; w++)
    if (bv[w] > v || (bv[w] == v && bi[w] < i)) {
      v = bv[w];
      i = bi[w];
    }
  __syncthreads();
}

__global__ void __launch_bounds__(T2) k_jnorms(const double2* F, long long ld, const int8_t* J, long long m,
                                               long long k, P2Scr s) {
  __shared__ double2 sh[T2 / 32];
  const long long j = k + blockIdx.x;
  const double2 v = jdot(F + j * ld, F + j * ld, J, k, m, true, sh);
  if (threadIdx.x == 0) s.hd[j] = v.x;
}

__device__ void swap_cols_dev(double2* F, long long ld, long long rows, long long a, long long b) {
  if (a == b) return;
  for (long long i = threadIdx.x; i < rows; i += T2) {
    const double2 t = F[i + a * ld];
    F[i + a * ld] = F[i + b * ld];
    F[i + b * ld] = t;
  }
}

// argmax |hd| over [k, n) (first index), swap columns k <-> jm, p2, hd
__global__ void __launch_bounds__(T2) k_piv_a(double2* F, long long ld, long long m, long long n, long long k,
                                              long long* p2, P2Scr s) {
  double v = -1.0;
  long long jm = 0x7fffffffffffffffll;
  for (long long j = k + threadIdx.x; j < n; j += T2) {
    const double a = fabs(s.hd[j]);
    if (a > v) {
      v = a;
      jm = j;
    }
  }
  block_argmax(v, jm);
  if (jm == 0x7fffffffffffffffll) {   // every |hd[j]| is NaN: no candidate, flag and keep k
    if (threadIdx.x == 0) s.ctl[3] = -8;
    jm = k;
  }
  swap_cols_dev(F, ld, m, k, jm);
  if (threadIdx.x == 0 && jm != k) {
    const long long t = p2[k]; p2[k] = p2[jm]; p2[jm] = t;
    const double h = s.hd[k]; s.hd[k] = s.hd[jm]; s.hd[jm] = h;
  }
}

// out[j] = col_src^* J col_j over rows >= k, for j in [j0, n), j != skip
__global__ void __launch_bounds__(T2) k_dots(const double2* F, long long ld, const int8_t* J, long long m,
                                             long long k, long long j0, const int* ctl_src, long long src_fixed,
                                             int need_flag, P2Scr s, double2* out) {
  __shared__ double2 sh[T2 / 32];
  if (need_flag && s.ctl[2] == 0) return;
  const long long src = ctl_src ? (long long)*ctl_src : src_fixed;
  const long long j = j0 + blockIdx.x;
  const double2 v = jdot(F + src * ld, F + j * ld, J, k, m, true, sh);
  if (threadIdx.x == 0) out[j] = v;
}

__global__ void __launch_bounds__(T2) k_piv_b(long long n, long long k, P2Scr s) {
  const double alpha = (1.0 + sqrt(17.0)) / 8.0;
  long long ii = 0x7fffffffffffffffll;
  double h1i = -1.0;
  for (long long j = k + 1 + threadIdx.x; j < n; j += T2) {
    const double a = cabs_(s.d1[j]);
    if (a > h1i) { h1i = a; ii = j; }
  }
  block_argmax(h1i, ii);
  if (threadIdx.x != 0) return;
  if (ii == 0x7fffffffffffffffll) ii = k + 1;
  s.ctl[1] = (int)ii;
  const double h11 = fabs(s.hd[k]);
  s.ctl[2] = !(h11 >= alpha * h1i);
  s.ctl[0] = 1;
  s.dctl[12] = h1i;
}

__global__ void __launch_bounds__(T2) k_piv_c(double2* F, long long ld, long long m, long long n, long long k,
                                              long long* p2, P2Scr s) {
  __shared__ int act;  // 0: nothing, 1: swap k<->ii (1x1), 2: swap k+1<->ii (2x2)
  double hij = -1.0;
  if (s.ctl[2]) {   // uniform over the block
    const long long ii = s.ctl[1];
    long long li = 0x7fffffffffffffffll;
    for (long long l = k + threadIdx.x; l < n; l += T2) {
      if (l == ii) continue;
      const double a = cabs_(s.d2[l]);
      if (a > hij) { hij = a; li = l; }
    }
    block_argmax(hij, li);
  }
  if (threadIdx.x == 0) {
    act = 0;
    if (s.ctl[2]) {
      const double alpha = (1.0 + sqrt(17.0)) / 8.0;
      const long long ii = s.ctl[1];
      const double h11 = fabs(s.hd[k]), h1i = s.dctl[12];
      if (h11 * hij >= alpha * h1i * h1i) {
        act = 0;
      } else if (fabs(s.hd[ii]) >= alpha * hij) {
        act = 1;
      } else {
        act = 2;
      }
      s.ctl[0] = act == 2 ? 2 : 1;
    }
  }
  __syncthreads();
  if (act == 0) return;
  const long long ii = s.ctl[1];
  const long long a = act == 1 ? k : k + 1;
  swap_cols_dev(F, ld, m, a, ii);
  if (threadIdx.x == 0 && a != ii) {
    const long long t = p2[a]; p2[a] = p2[ii]; p2[ii] = t;
    const double h = s.hd[a]; s.hd[a] = s.hd[ii]; s.hd[ii] = h;
  }
}

// Reflector for column k (Thm 5.1): sign-compatibility row swap, s, tau, c1.
__global__ void __launch_bounds__(T2) k_refl_prep(double2* F, long long ld, int8_t* J, long long m, long long n,
                                                  long long k, P2Scr s) {
  __shared__ double2 sh[T2 / 32];
  double2* f = F + k * ld;
  const double hn = jdot(f, f, J, k, m, true, sh).x;
  if (hn == 0.0 || !isfinite(hn)) {
    if (threadIdx.x == 0 && s.ctl[3] == 0) s.ctl[3] = -7;
    return;
  }
  const int8_t sg = hn > 0.0 ? 1 : -1;
  if (J[k] != sg) {   // uniform over the block
    double bv = -1.0;
    long long best = 0x7fffffffffffffffll;
    for (long long i = k + threadIdx.x; i < m; i += T2)
      if (J[i] == sg && cabs_(f[i]) > bv) { bv = cabs_(f[i]); best = i; }
    block_argmax(bv, best);
    if (best == 0x7fffffffffffffffll) best = -1;
    if (best < 0) {
      if (threadIdx.x == 0 && s.ctl[3] == 0) s.ctl[3] = -7;
      return;
    }
    for (long long c = threadIdx.x; c < n; c += T2) {
      const double2 t = F[k + c * ld];
      F[k + c * ld] = F[best + c * ld];
      F[best + c * ld] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int8_t t = J[k]; J[k] = J[best]; J[best] = t;
    }
    __syncthreads();
  }
  const double rr = sqrt(fabs(hn));
  const double a11 = cabs_(f[k]);
  const double2 ed = a11 > 0.0 ? cmk(f[k].x / a11, f[k].y / a11) : cmk(1, 0);
  const double2 c1 = cmk(ed.x * rr, ed.y * rr);
  for (long long i = k + threadIdx.x; i < m; i += T2) s.s[i] = f[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    s.s[k] = cadd(s.s[k], c1);
    s.dctl[0] = -1.0 / (hn + rr * a11 * (double)J[k]);
    s.dctl[1] = c1.x;
    s.dctl[2] = c1.y;
  }
}

// columns j > k: x += tau s (s^* J x)   (or, for QR with useJ = 0: x += (-2/vv) v (v^* x))
__global__ void __launch_bounds__(T2) k_refl_apply(double2* F, long long ld, const int8_t* J, long long m,
                                                   long long k, long long j0, const long long* colmap, int useJ,
                                                   P2Scr s) {
  __shared__ double2 sh[T2 / 32];
  if (s.ctl[3]) return;
  const long long jj = j0 + blockIdx.x;
  const long long j = colmap ? colmap[jj] : jj;
  double2* x = F + j * ld;
  const double2 d = jdot(s.s, x, J, k, m, useJ != 0, sh);
  const double tau = s.dctl[0];
  const double2 c = cmk(d.x * tau, d.y * tau);
  for (long long i = k + threadIdx.x; i < m; i += T2) x[i] = cadd(x[i], cmul(s.s[i], c));
}

__global__ void k_refl_fin(double2* F, long long ld, long long m, long long k, P2Scr s) {
  if (s.ctl[3]) return;
  double2* f = F + k * ld;
  for (long long i = k + 1 + threadIdx.x; i < m; i += blockDim.x) f[i] = cmk(0, 0);
  if (threadIdx.x == 0) f[k] = cmk(-s.dctl[1], -s.dctl[2]);
}

// 2x2 URV pivot: Jacobi rotation of columns k, k+1 on rows >= k (dir = +1),
// or multiply rows k, k+1 back by R^* (dir = -1).
__global__ void __launch_bounds__(T2) k_rot(double2* F, long long ld, const int8_t* J, long long m, long long k,
                                            int dir, P2Scr s) {
  __shared__ double2 sh[T2 / 32];
  double2* f1 = F + k * ld;
  double2* f2 = F + (k + 1) * ld;
  double2* R = (double2*)(s.dctl + 4);  // 16-B aligned: dctl[4..11]
  if (dir > 0) {
    const double a = jdot(f1, f1, J, k, m, true, sh).x;
    const double c = jdot(f2, f2, J, k, m, true, sh).x;
    const double2 b = jdot(f1, f2, J, k, m, true, sh);
    __shared__ int bad;
    if (threadIdx.x == 0) {
      const double ab = cabs_(b);
      double l1, l2;
      if (ab == 0.0) {
        R[0] = cmk(1, 0); R[1] = cmk(0, 0); R[2] = cmk(0, 0); R[3] = cmk(1, 0);
        l1 = a; l2 = c;
      } else {
        const double2 e = cmk(b.x / ab, b.y / ab);
        const double tau = (c - a) / (2.0 * ab);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = t * cs;
        const double2 em = cconj(e);
        R[0] = cmk(cs, 0.0);
        R[1] = cmk(-em.x * sn, -em.y * sn);
        R[2] = cmk(sn, 0.0);
        R[3] = cmk(em.x * cs, em.y * cs);
        l1 = a - t * ab;
        l2 = c + t * ab;
      }
      bad = (l1 == 0.0 || l2 == 0.0);
      if (bad && s.ctl[3] == 0) s.ctl[3] = -7;
    }
    __syncthreads();
    if (bad) return;
    const double2 r0 = R[0], r1 = R[1], r2 = R[2], r3 = R[3];
    for (long long i = k + threadIdx.x; i < m; i += T2) {
      const double2 x0 = f1[i], x1 = f2[i];
      f1[i] = cadd(cmul(x0, r0), cmul(x1, r1));
      f2[i] = cadd(cmul(x0, r2), cmul(x1, r3));
    }
  } else {
    if (s.ctl[3]) return;
    if (threadIdx.x < 2) {
      const long long i = k + threadIdx.x;
      const double2 x0 = f1[i], x1 = f2[i];
      const double2 r0 = R[0], r1 = R[1], r2 = R[2], r3 = R[3];
      f1[i] = cadd(cmul(x0, cconj(r0)), cmul(x1, cconj(r2)));
      f2[i] = cadd(cmul(x0, cconj(r1)), cmul(x1, cconj(r3)));
    }
  }
}

// Householder step of the QR of G P2: column c = p2[k]; v = x - alph e_k, alph = -phase(x_k) ||x||
__global__ void __launch_bounds__(T2) k_qr_prep(double2* G, long long ld, long long m, long long k,
                                                const long long* p2, P2Scr s) {
  __shared__ double2 sh[T2 / 32];
  double2* x = G + p2[k] * ld;
  const double nrm = sqrt(jdot(x, x, nullptr, k, m, false, sh).x);
  if (nrm == 0.0) {
    if (threadIdx.x == 0 && s.ctl[3] == 0) s.ctl[3] = -7;
    return;
  }
  const double ax = cabs_(x[k]);
  const double2 ph = ax > 0.0 ? cmk(x[k].x / ax, x[k].y / ax) : cmk(1, 0);
  const double2 alph = cmk(-ph.x * nrm, -ph.y * nrm);
  for (long long i = k + threadIdx.x; i < m; i += T2) s.s[i] = x[i];
  __syncthreads();
  if (threadIdx.x == 0) s.s[k] = cmk(s.s[k].x - alph.x, s.s[k].y - alph.y);
  __syncthreads();
  const double vv = jdot(s.s, s.s, nullptr, k, m, false, sh).x;
  if (threadIdx.x == 0) {
    s.dctl[0] = -2.0 / vv;   // apply uses x += tau v (v^* x)
    x[k] = alph;             // R(k, k); entries below are never read (gather takes i <= j)
  }
}

// Column pivoting of the QR of G P2 (ZGEQP3-like, reading of the optional
// path): squared norms of rows [k, m) of the remaining columns p2[j], j >= k (recomputed
// every step: exact, no norm downdating), then the largest is swapped into position k
// in p2 (G P2 P5) and the same two columns of F are swapped (F' = F P5).
__global__ void __launch_bounds__(T2) k_qr_colnorms(const double2* G, long long ld, long long m, long long k,
                                                    const long long* p2, P2Scr s) {
  __shared__ double2 sh[T2 / 32];
  if (s.ctl[3]) return;
  const long long j = k + blockIdx.x;
  const double2* x = G + p2[j] * ld;
  const double v = jdot(x, x, nullptr, k, m, false, sh).x;
  if (threadIdx.x == 0) s.hd[j] = v;
}

__global__ void __launch_bounds__(T2) k_qr_colpiv(double2* F, long long ldf, long long mf, long long n, long long k,
                                                  long long* p2, P2Scr s) {
  __shared__ double bv[T2 / 32];
  __shared__ long long bi[T2 / 32];
  __shared__ long long piv;
  if (s.ctl[3]) return;
  double v = -1.0;
  long long idx = n;
  for (long long j = k + threadIdx.x; j < n; j += T2)
    if (s.hd[j] > v) {   // first (smallest j) maximum within the thread's strided set
      v = s.hd[j];
      idx = j;
    }
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    if (v2 > v || (v2 == v && i2 < idx)) {
      v = v2;
      idx = i2;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    bv[threadIdx.x >> 5] = v;
    bi[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bvv = bv[0];
    long long bii = bi[0];
    for (int w = 1; w < T2 / 32; w++)
      if (bv[w] > bvv || (bv[w] == bvv && bi[w] < bii)) {
        bvv = bv[w];
        bii = bi[w];
      }
    piv = bii < n ? bii : k;
    if (piv != k) {
      const long long t = p2[k];
      p2[k] = p2[piv];
      p2[piv] = t;
    }
  }
  __syncthreads();
  const long long pv = piv;
  if (pv != k) {
    double2* a = F + k * ldf;
    double2* b = F + pv * ldf;
    for (long long i = threadIdx.x; i < mf; i += T2) {
      const double2 t = a[i];
      a[i] = b[i];
      b[i] = t;
    }
  }
}

// Gs(i, j) = G(i, p2[j]) for i <= j (upper triangle), diag phases normalised.
__global__ void k_qr_gather(const double2* G, long long ld, double2* out, long long ldo, long long n,
                            const long long* p2) {
  const long long j = blockIdx.x;
  for (long long i = threadIdx.x; i < n; i += blockDim.x)
    out[i + j * ldo] = i <= j ? G[i + p2[j] * ld] : cmk(0, 0);
}

__global__ void k_qr_phase(double2* R, long long ld, long long n) {
  const long long i = blockIdx.x;
  const double2 d = R[i + i * ld];
  const double ad = cabs_(d);
  const double2 ph = ad > 0.0 ? cmk(d.x / ad, d.y / ad) : cmk(1, 0);
  const double2 cp = cconj(ph);
  for (long long j = i + threadIdx.x; j < n; j += blockDim.x) R[i + j * ld] = cmul(cp, R[i + j * ld]);
  __syncthreads();
  if (threadIdx.x == 0) R[i + i * ld].y = 0.0;
}

__global__ void k_iota(long long* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = i;
}

}  // namespace

size_t phase2_scratch_bytes(int64_t m, int64_t n) {
  return al256((size_t)n * 8) + 2 * al256((size_t)n * 16) + al256((size_t)m * 16) + 512 + 256;
}

#define P2CHK()                                    \
  do {                                             \
    cudaError_t e_ = cudaGetLastError();           \
    if (e_ != cudaSuccess) {                       \
      ctx->err = cudaGetErrorString(e_);           \
      return GHSVD_E_CUDA;                         \
    }                                              \
  } while (0)

ghsvd_status phase2_reduce(Ctx* ctx, int flags) {
  const int64_t m = ctx->m_user, n = ctx->n_user;
  const long long ld = ctx->ldm;
  cudaStream_t st = ctx->stream;
  P2Scr s = carve(ctx->scr, m, n);
  long long* p2 = (long long*)ctx->p2;
  GH_CUDA(cudaMemsetAsync(s.ctl, 0, 256, st));
  k_iota<<<8, 256, 0, st>>>(p2, n);
  P2CHK();
  int ctl[4];
  int64_t k = 0;
  while (k < n) {
    k_jnorms<<<(unsigned)(n - k), T2, 0, st>>>(ctx->F, ld, ctx->J, m, k, s);
    k_piv_a<<<1, T2, 0, st>>>(ctx->F, ld, m, n, k, p2, s);
    if (k < n - 1) {
      k_dots<<<(unsigned)(n - k - 1), T2, 0, st>>>(ctx->F, ld, ctx->J, m, k, k + 1, nullptr, k, 0, s, s.d1);
      k_piv_b<<<1, T2, 0, st>>>(n, k, s);
      k_dots<<<(unsigned)(n - k), T2, 0, st>>>(ctx->F, ld, ctx->J, m, k, k, s.ctl + 1, 0, 1, s, s.d2);
      k_piv_c<<<1, T2, 0, st>>>(ctx->F, ld, m, n, k, p2, s);
    } else {
      GH_CUDA(cudaMemsetAsync(s.ctl, 0, 16, st));
      static const int one = 1;
      GH_CUDA(cudaMemcpyAsync(s.ctl, &one, 4, cudaMemcpyHostToDevice, st));
    }
    P2CHK();
    GH_CUDA(cudaMemcpyAsync(ctl, s.ctl, 16, cudaMemcpyDeviceToHost, st));
    GH_CUDA(cudaStreamSynchronize(st));
    const int type = ctl[0];
    if (type == 2) k_rot<<<1, T2, 0, st>>>(ctx->F, ld, ctx->J, m, k, +1, s);
    for (int t = 0; t < type; t++) {
      const long long kk = k + t;
      k_refl_prep<<<1, T2, 0, st>>>(ctx->F, ld, ctx->J, m, n, kk, s);
      if (n - kk - 1 > 0)
        k_refl_apply<<<(unsigned)(n - kk - 1), T2, 0, st>>>(ctx->F, ld, ctx->J, m, kk, kk + 1, nullptr, 1, s);
      k_refl_fin<<<1, T2, 0, st>>>(ctx->F, ld, m, kk, s);
    }
    if (type == 2) k_rot<<<1, T2, 0, st>>>(ctx->F, ld, ctx->J, m, k, -1, s);
    P2CHK();
    GH_CUDA(cudaMemcpyAsync(ctl, s.ctl, 16, cudaMemcpyDeviceToHost, st));
    GH_CUDA(cudaStreamSynchronize(st));
    if (ctl[3] == -8) {
      ctx->err = "reduce: non-finite J-norms in the JQR pivot search at step " + std::to_string(k);
      return GHSVD_E_NONFINITE;
    }
    if (ctl[3]) {
      ctx->err = "reduce: degenerate JQR pivot (J-Grammian numerically singular) at step " + std::to_string(k);
      return GHSVD_E_RANK_DEFICIENT;
    }
    GH_CUDA(cudaMemsetAsync(s.ctl, 0, 16, st));
    k += type;
  }
  // Householder QR of G P2 (columns visited in P2 order); with GHSVD_REDUCE_COLPIV the
  // columns are pivoted by norm (P5), applied to p2 and to F's columns alike
  const bool colpiv = (flags & GHSVD_REDUCE_COLPIV) != 0;
  for (int64_t kk = 0; kk < n; kk++) {
    if (colpiv && kk < n - 1) {
      k_qr_colnorms<<<(unsigned)(n - kk), T2, 0, st>>>(ctx->G, ld, m, kk, p2, s);
      k_qr_colpiv<<<1, T2, 0, st>>>(ctx->F, ld, m, n, kk, p2, s);
    }
    k_qr_prep<<<1, T2, 0, st>>>(ctx->G, ld, m, kk, p2, s);
    if (n - kk - 1 > 0)
      k_refl_apply<<<(unsigned)(n - kk - 1), T2, 0, st>>>(ctx->G, ld, nullptr, m, kk, kk + 1, p2, 0, s);
    P2CHK();
  }
  GH_CUDA(cudaMemcpyAsync(ctl, s.ctl, 16, cudaMemcpyDeviceToHost, st));
  GH_CUDA(cudaStreamSynchronize(st));
  if (ctl[3]) {
    ctx->err = "reduce: G P2 numerically rank deficient";
    return GHSVD_E_RANK_DEFICIENT;
  }
  // R -> Z buffer (gather + phase normalisation) -> G (rows >= n zero)
  const long long ldz = ctx->ldn;
  k_qr_gather<<<(unsigned)n, T2, 0, st>>>(ctx->G, ld, ctx->Z, ldz, n, p2);
  k_qr_phase<<<(unsigned)n, T2, 0, st>>>(ctx->Z, ldz, n);
  P2CHK();
  GH_CUDA(cudaMemsetAsync(ctx->G, 0, (size_t)ld * (ctx->n_cap + 1) * 16, st));
  GH_CUDA(cudaMemcpy2DAsync(ctx->G, (size_t)ld * 16, ctx->Z, (size_t)ldz * 16, (size_t)n * 16, (size_t)n,
                            cudaMemcpyDeviceToDevice, st));
  // F: keep the leading n x n block, rows re-sorted by the new J (+ first)
  GH_CUDA(cudaMemcpy2DAsync(ctx->Z, (size_t)ldz * 16, ctx->F, (size_t)ld * 16, (size_t)n * 16, (size_t)n,
                            cudaMemcpyDeviceToDevice, st));
  int8_t* Jin = (int8_t*)s.s;  // reuse scratch
  GH_CUDA(cudaMemcpyAsync(Jin, ctx->J, (size_t)n, cudaMemcpyDeviceToDevice, st));
  int64_t* npos_dev = (int64_t*)s.d1;
  {
    ghsvd_status e = launch_sort_dest(ctx, Jin, n, false, ctx->rowdest, ctx->J, npos_dev);
    if (e) return e;
  }
  GH_CUDA(cudaMemsetAsync(ctx->F, 0, (size_t)ld * (ctx->n_cap + 1) * 16, st));
  {
    ghsvd_status e = launch_row_scatter(ctx, ctx->Z, ldz, ctx->F, ld, ctx->rowdest, n, n);
    if (e) return e;
  }
  long long npos = 0;
  GH_CUDA(cudaMemcpyAsync(&npos, npos_dev, 8, cudaMemcpyDeviceToHost, st));
  GH_CUDA(cudaStreamSynchronize(st));
  ctx->npos = npos;
  ctx->m_user = n;
  ctx->m = n;
  return GHSVD_OK;
}

}  // namespace ghsvd
