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
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <string>
#include <vector>

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
// blocked Phase 2: the delayed-update coefficients Y (= S^* J X) and W (= T Y) of a column
// move with it (pb entries per column; nullptr in the unblocked path)
__device__ void swap_yw(double2* Yb, double2* Wb, int pb, long long a, long long b) {
  if (!Yb || a == b) return;
  for (int i = threadIdx.x; i < pb; i += blockDim.x) {
    double2 t = Yb[i + a * pb]; Yb[i + a * pb] = Yb[i + b * pb]; Yb[i + b * pb] = t;
    t = Wb[i + a * pb]; Wb[i + a * pb] = Wb[i + b * pb]; Wb[i + b * pb] = t;
  }
}

__global__ void __launch_bounds__(T2) k_piv_a(double2* F, long long ld, long long m, long long n, long long k,
                                              long long* p2, P2Scr s, double2* Yb = nullptr,
                                              double2* Wb = nullptr, int pb = 0) {
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
  swap_yw(Yb, Wb, pb, k, jm);
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
                                              long long* p2, P2Scr s, double2* Yb = nullptr,
                                              double2* Wb = nullptr, int pb = 0) {
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
    s.ctl[6] = act;
  }
  __syncthreads();
  if (act == 0) return;
  const long long ii = s.ctl[1];
  const long long a = act == 1 ? k : k + 1;
  swap_cols_dev(F, ld, m, a, ii);
  swap_yw(Yb, Wb, pb, a, ii);
  if (threadIdx.x == 0 && a != ii) {
    const long long t = p2[a]; p2[a] = p2[ii]; p2[ii] = t;
    const double h = s.hd[a]; s.hd[a] = s.hd[ii]; s.hd[ii] = h;
  }
}

// Reflector for column k (Thm 5.1): sign-compatibility row swap, s, tau, c1; hn = the
// column's J-norm over rows >= k (uniform over the block).
__device__ void refl_prep_body(double2* F, long long ld, int8_t* J, long long m, long long n, long long k, P2Scr s,
                               double2* Sb, long long lds, int nrs, const double hn) {
  double2* f = F + k * ld;
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
    // blocked path: the panel's reflectors so far are rows of the same (delayed) transform
    for (int c = threadIdx.x; c < nrs; c += T2) {
      const double2 t = Sb[k + c * lds];
      Sb[k + c * lds] = Sb[best + c * lds];
      Sb[best + c * lds] = t;
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

__global__ void __launch_bounds__(T2) k_refl_prep(double2* F, long long ld, int8_t* J, long long m, long long n,
                                                  long long k, P2Scr s, double2* Sb = nullptr, long long lds = 0,
                                                  int nrs = 0) {
  __shared__ double2 sh[T2 / 32];
  double2* f = F + k * ld;
  const double hn = jdot(f, f, J, k, m, true, sh).x;
  refl_prep_body(F, ld, J, m, n, k, s, Sb, lds, nrs, hn);
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
  if (s.ctl[3] || s.ctl[8]) return;
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

// ------------------------------------------------------------ blocked Phase 2 (NEXT-4)
// Left-looking panels of up to PB reflectors with delayed trailing updates (the paper's
// "blocking and delaying the columns updates").  Within a panel the
// trailing columns X keep their values from the panel start; the reflectors applied so far
// are H_i = I + tau_i s_i s_i^* J (J = I for the QR of G), accumulated as
//     H_last ... H_first = I + S T S^* J,   T lower triangular,
//     T_new = [[T, 0], [tau (s^* J S) T, tau]],
// so the current value of a trailing column is x + S w with w = T y, y = S^* J x (Y, W
// keep y, w per column).  Each step forms only the pivot column(s) explicitly; the pivot
// searches use J-norms / norms downdated with the new R row (exact at every panel start,
// and a panel is cut short when a formed pivot column's exact value disagrees with its
// downdated estimate), and the Bunch-Kaufman dots of the JQR are x-dots corrected by the
// panel (u^T w).  The trailing columns are brought up to date once per panel by two plain
// ZGEMMs (W = T Y, X += S W; cuBLAS).
constexpr int PB = 33;   // max reflectors per panel (32 + one 2x2 overflow)

// out[(j - j0) * ostride] = v^* J x_j over rows [r0, m), j in [j0, j0 + gridDim.x)
__global__ void __launch_bounds__(T2) k_vdot(const double2* v, const double2* X, long long ld, const int8_t* J,
                                             long long r0, long long m, long long j0, double2* out, long long ostride) {
  __shared__ double2 sh[T2 / 32];
  const long long j = j0 + blockIdx.x;
  const double2 d = jdot(v, X + j * ld, J, r0, m, J != nullptr, sh);
  if (threadIdx.x == 0) out[(j - j0) * ostride] = d;
}

// tv[i] = s_new^* J S[:, i] (rows >= r0) for i < nr (one CTA each)
__global__ void __launch_bounds__(T2) k_sdots(const double2* snew, const double2* S, long long lds, const int8_t* J,
                                              long long r0, long long m, double2* tv) {
  __shared__ double2 sh[T2 / 32];
  const double2 d = jdot(snew, S + (size_t)blockIdx.x * lds, J, r0, m, J != nullptr, sh);
  if (threadIdx.x == 0) tv[blockIdx.x] = d;
}

// k_panel_add + k_refl_fin of the JQR in one launch (F column k: rows > k zeroed, row k = -c1)
__device__ __forceinline__ void panel_add_fin_body(double2* S, long long lds, const double2* sv, long long r0,
                                                   long long m, int nr, double2* T, const double2* tv, P2Scr s,
                                                   double2* F, long long ld) {
  const double tau = s.dctl[0];
  double2* col = S + (size_t)nr * lds;
  double2* f = F + r0 * ld;
  for (long long i = blockIdx.x * (long long)T2 + threadIdx.x; i < m; i += (long long)gridDim.x * T2) {
    col[i] = i >= r0 ? sv[i] : cmk(0, 0);
    if (i > r0) f[i] = cmk(0, 0);
  }
  if (blockIdx.x == 0) {
    for (int c = threadIdx.x; c < nr; c += T2) {
      double2 a = cmk(0, 0);
      for (int i = c; i < nr; i++) a = cadd(a, cmul(tv[i], T[i + c * PB]));   // T lower triangular
      T[nr + c * PB] = cmk(tau * a.x, tau * a.y);
    }
    if (threadIdx.x == 0) {
      T[nr + nr * PB] = cmk(tau, 0.0);
      f[r0] = cmk(-s.dctl[1], -s.dctl[2]);
    }
  }
}

__global__ void __launch_bounds__(T2) k_panel_add_fin(double2* S, long long lds, const double2* sv, long long r0,
                                                      long long m, int nr, double2* T, const double2* tv, P2Scr s,
                                                      double2* F, long long ld) {
  if (s.ctl[3] || s.ctl[8]) return;
  panel_add_fin_body(S, lds, sv, r0, m, nr, T, tv, s, F, ld);
}

// S[:, nr] = s (rows >= r0; zero above); T row nr = tau (tv^T T), T[nr][nr] = tau
__device__ __forceinline__ void panel_add_body(double2* S, long long lds, const double2* sv, long long r0, long long m,
                                               int nr, double2* T, const double2* tv, P2Scr s) {
  const double tau = s.dctl[0];
  double2* col = S + (size_t)nr * lds;
  for (long long i = blockIdx.x * (long long)T2 + threadIdx.x; i < m; i += (long long)gridDim.x * T2)
    col[i] = i >= r0 ? sv[i] : cmk(0, 0);
  if (blockIdx.x == 0) {
    for (int c = threadIdx.x; c < nr; c += T2) {
      double2 a = cmk(0, 0);
      for (int i = c; i < nr; i++) a = cadd(a, cmul(tv[i], T[i + c * PB]));   // T lower triangular
      T[nr + c * PB] = cmk(tau * a.x, tau * a.y);
    }
    if (threadIdx.x == 0) T[nr + nr * PB] = cmk(tau, 0.0);
  }
}

__global__ void __launch_bounds__(T2) k_panel_add(double2* S, long long lds, const double2* sv, long long r0,
                                                  long long m, int nr, double2* T, const double2* tv, P2Scr s) {
  if (s.ctl[3] || s.ctl[8]) return;
  panel_add_body(S, lds, sv, r0, m, nr, T, tv, s);
}

// Per trailing column j in [j0, n): w = T y (nr x nr lower triangular), then for each of the
// nnew newest reflector rows kr (rows r0, r0 + 1): r = x_j[kr] + S[kr, :] w, hd[j] -= J_kr |r|^2
// (J = nullptr: |r|^2).  One thread per column.
__global__ void k_panel_rows(const double2* X, long long ld, const int8_t* J, const double2* S, long long lds,
                             const double2* T, const double2* Y, double2* W, int nr, long long kr0, int nnew,
                             long long j0, long long n, double* hd) {
  const long long j = j0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double2* y = Y + j * PB;
  double2* w = W + j * PB;
  for (int i = 0; i < nr; i++) {
    double2 a = cmk(0, 0);
    for (int c = 0; c <= i; c++) a = cadd(a, cmul(T[i + c * PB], y[c]));
    w[i] = a;
  }
  for (int t = 0; t < nnew; t++) {
    const long long kr = kr0 + t;
    double2 r = X[kr + j * ld];
    for (int i = 0; i < nr; i++) r = cadd(r, cmul(S[kr + (size_t)i * lds], w[i]));
    const double a2 = r.x * r.x + r.y * r.y;
    hd[j] -= J ? (double)J[kr] * a2 : a2;
  }
}

// k_tw + k_form in one launch: every CTA forms w = T y (nr x nr, in shared memory), then
// out[r] = x[r] + (S w)[r] for r >= r0
__global__ void k_form_tw(const double2* x, double2* out, const double2* S, long long lds, const double2* T,
                          const double2* y, int nr, long long r0, long long m) {
  __shared__ double2 w[PB];
  if (threadIdx.x < nr) {
    const int i = threadIdx.x;
    double2 a = cmk(0, 0);
    for (int c = 0; c <= i; c++) a = cadd(a, cmul(T[i + c * PB], y[c]));
    w[i] = a;
  }
  __syncthreads();
  for (long long r = r0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < m; r += (long long)gridDim.x * blockDim.x) {
    double2 a = x[r];
    for (int i = 0; i < nr; i++) a = cadd(a, cmul(S[r + (size_t)i * lds], w[i]));
    out[r] = a;
  }
}

// out[r] = x[r] + (S w)[r] for r >= r0 (x, out may alias); rows < r0 of out untouched
__global__ void k_form(const double2* x, double2* out, const double2* S, long long lds, const double2* w, int nr,
                       long long r0, long long m) {
  for (long long r = r0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < m; r += (long long)gridDim.x * blockDim.x) {
    double2 a = x[r];
    for (int i = 0; i < nr; i++) a = cadd(a, cmul(S[r + (size_t)i * lds], w[i]));
    out[r] = a;
  }
}

__global__ void k_zero_yw(double2* Y, double2* W, long long j) {
  if (threadIdx.x < PB) {
    Y[threadIdx.x + j * PB] = cmk(0, 0);
    W[threadIdx.x + j * PB] = cmk(0, 0);
  }
}

// d[j] += u^T w_j for j in [j0, n) (the panel's correction of x-dots)
__global__ void k_dfix(double2* d, const double2* u, const double2* W, int nr, long long j0, long long n) {
  const long long j = j0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  double2 a = d[j];
  for (int i = 0; i < nr; i++) a = cadd(a, cmul(u[i], W[i + j * PB]));
  d[j] = a;
}

// exact J-norm (rows >= r0) of vector x into hd[c]; with `check`, flag (ctl[5]) when the
// downdated estimate it replaces was off by more than 1/8 of the larger magnitude
__global__ void __launch_bounds__(T2) k_exact_hd(const double2* x, const int8_t* J, long long r0, long long m,
                                                 long long c, int check, P2Scr s) {
  __shared__ double2 sh[T2 / 32];
  const double e = jdot(x, x, J, r0, m, J != nullptr, sh).x;
  if (threadIdx.x == 0) {
    const double est = s.hd[c];
    if (check && fabs(e - est) > 0.125 * fmax(fabs(e), fabs(est))) s.ctl[5] = 1;
    s.hd[c] = e;
  }
}

// yv[i] = s_i^* J x (rows >= r0) for i < nr (one CTA each): the coefficients of a column
__global__ void __launch_bounds__(T2) k_ycol(const double2* x, const double2* S, long long lds, const int8_t* J,
                                             long long r0, long long m, double2* yv) {
  __shared__ double2 sh[T2 / 32];
  const double2 d = jdot(S + (size_t)blockIdx.x * lds, x, J, r0, m, J != nullptr, sh);
  if (threadIdx.x == 0) yv[blockIdx.x] = d;
}

// w = T y for one column (T lower triangular, nr x nr)
__global__ void k_tw(const double2* T, const double2* y, double2* w, int nr) {
  const int i = threadIdx.x;
  if (i >= nr) return;
  double2 a = cmk(0, 0);
  for (int c = 0; c <= i; c++) a = cadd(a, cmul(T[i + c * PB], y[c]));
  w[i] = a;
}

// After k_piv_c (act in ctl[6]): the explicit f_ii (fx, rows >= r0) replaces the column the
// pivot moved into (k for act 1, k + 1 for act 2); its delayed coefficients become zero
__global__ void k_place_fx(double2* F, long long ld, const double2* fx, long long r0, long long m, long long k,
                           double2* Y, double2* W, P2Scr s) {
  const int act = s.ctl[6];
  if (act == 0) return;
  const long long c = act == 1 ? k : k + 1;
  for (long long r = r0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < m; r += (long long)gridDim.x * blockDim.x)
    F[r + c * ld] = fx[r];
  if (blockIdx.x == 0 && threadIdx.x < PB) {
    Y[threadIdx.x + c * PB] = cmk(0, 0);
    W[threadIdx.x + c * PB] = cmk(0, 0);
  }
}

// hd[j] = ||x_j||^2 over rows >= k (QR column pivoting)
__global__ void __launch_bounds__(T2) k_norms(const double2* X, long long ld, long long k, long long m, P2Scr s) {
  __shared__ double2 sh[T2 / 32];
  const long long j = k + blockIdx.x;
  const double v = jdot(X + j * ld, X + j * ld, nullptr, k, m, false, sh).x;
  if (threadIdx.x == 0) s.hd[j] = v;
}

// argmax of norms hd over [k, n) (QR column pivoting, blocked): swap into k with Y/W columns,
// F's columns (F' = F P5), p2
__global__ void __launch_bounds__(T2) k_qr_colpiv_blk(double2* G, long long ldg, long long mg, double2* F,
                                                      long long ldf, long long mf, long long n, long long k,
                                                      long long* p2, P2Scr s, double2* Yb, double2* Wb) {
  double v = -1.0;
  long long jm = 0x7fffffffffffffffll;
  for (long long j = k + threadIdx.x; j < n; j += T2)
    if (s.hd[j] > v) { v = s.hd[j]; jm = j; }
  block_argmax(v, jm);
  if (jm == 0x7fffffffffffffffll) jm = k;
  swap_cols_dev(G, ldg, mg, k, jm);
  swap_cols_dev(F, ldf, mf, k, jm);
  swap_yw(Yb, Wb, PB, k, jm);
  if (threadIdx.x == 0 && jm != k) {
    const long long t = p2[k]; p2[k] = p2[jm]; p2[jm] = t;
    const double h = s.hd[k]; s.hd[k] = s.hd[jm]; s.hd[jm] = h;
  }
}

// Householder vector of the (explicit) contiguous column k of the QR: v = x - alph e_k,
// tau = -2 / v^* v, x[k] = alph (R(k,k)); writes v to s.s
// pd (planned column-pivoted QR): the planned Schur diagonal, checked as in k_plan_check_qr
__global__ void __launch_bounds__(T2) k_qr_prep_c(double2* X, long long ld, long long m, long long k, P2Scr s,
                                                  const double2* pd = nullptr) {
  __shared__ double2 sh[T2 / 32];
  double2* x = X + k * ld;
  const double nn = jdot(x, x, nullptr, k, m, false, sh).x;
  if (pd && threadIdx.x == 0) {
    const double ap = pd[3 * k].x;
    if (!(nn > 0.0) || !isfinite(nn) || fabs(nn - ap) > 0.25 * fmax(nn, fabs(ap))) s.ctl[5] = 1;
  }
  const double nrm = sqrt(nn);
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
    s.dctl[0] = -2.0 / vv;
    x[k] = alph;
  }
}

// Gather G P2 (all m rows) into a contiguous buffer
__global__ void k_gather_cols(const double2* G, long long ldg, double2* out, long long ldo, long long m,
                              const long long* p2) {
  const long long j = blockIdx.y;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
    out[i + j * ldo] = G[i + p2[j] * ldg];
}

// R (upper n x n of the contiguous QR buffer) -> out with real non-negative diagonal
__global__ void k_qr_rout(const double2* X, long long ld, double2* out, long long ldo, long long n) {
  const long long i = blockIdx.x;
  const double2 d = X[i + i * ld];
  const double ad = cabs_(d);
  const double2 cp = ad > 0.0 ? cmk(d.x / ad, -d.y / ad) : cmk(1, 0);
  for (long long j = threadIdx.x; j < n; j += blockDim.x) {
    double2 v = j >= i ? cmul(cp, X[i + j * ld]) : cmk(0, 0);
    if (j == i) v = cmk(ad, 0.0);
    out[i + j * ldo] = v;
  }
}

// ------------------------------------------------ pivot plan from the J-Grammian (JQR)
// The JQR's diagonal + partial (Bunch-Kaufman) pivot decisions (Sec 5.2.1) read only the
// J-Grammian of the unreduced columns, H_k = F_k^* J_k F_k, which after each reduction step
// is the Schur complement of the previous one (a hyperbolic reflector leaves the trailing
// columns' J-products unchanged on the rows it keeps; the removed row carries exactly
// h_j1 h_11^{-1} h_1l, or the 2x2 analogue).  So the whole pivot sequence can be chosen
// first, on H = F^* J F formed once (two ZGEMMs, O(m n^2)) and reduced by symmetric rank-1
// / rank-2 Schur updates (O(n^3)) -- the "complete" use of H that PAPER.md:984-990 rules
// out only for its O(m^2 n^2) cost when recomputed from F each step -- after which the
// JQR needs no per-column pass over the trailing columns.  Every planned pivot is checked
// against the exact J-Grammian of its formed column(s) before it is used (jqr_planned).
// H is kept in the lower triangle of the trailing block (column-major, ld).
struct BkPlan {
  int* type;       // [n] 1, 2 (first column of a 2x2 pivot) or 0 (its second column)
  long long* sw1;  // [n] diagonal-pivot swap partner of position k
  long long* sw2;  // [n] second swap partner (Bunch-Kaufman), -1 if none
  int* sw2pos;     // [n] position (k or k + 1) the second swap moves into
  double2* d;      // [3 n] predicted H_kk, H_{k+1,k}, H_{k+1,k+1} at the pivot
  double* dg;      // [n] the current diagonal, contiguous (the diagonal-pivot search reads it)
  int* st;         // [0] next k, [2] k of the last step, [3] its type (0: none), [4] error
};

constexpr int TS = 1024;   // threads of the pivot-selection CTA (memory-latency bound)

// block argmax for TS threads (same tie rule as block_argmax)
__device__ void block_argmax_ts(double& v, long long& i) {
  __shared__ double bv[TS / 32];
  __shared__ long long bi[TS / 32];
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
  }
  if ((threadIdx.x & 31) == 0) { bv[threadIdx.x >> 5] = v; bi[threadIdx.x >> 5] = i; }
  __syncthreads();
  v = bv[0];
  i = bi[0];
  for (int w = 1; w < TS / 32; w++)
    if (bv[w] > v || (bv[w] == v && bi[w] < i)) { v = bv[w]; i = bi[w]; }
  __syncthreads();
}

__global__ void k_bk_diag(const double2* H, long long ld, long long n, double* dg) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
    dg[j] = H[j + j * ld].x;
}

__device__ __forceinline__ double2 hget(const double2* H, long long ld, long long j, long long l) {
  return j >= l ? H[j + l * ld] : cconj(H[l + j * ld]);
}

// symmetric interchange of indices a < b of the trailing Hermitian block [k, n) (lower storage)
__device__ void hswap(double2* H, long long ld, long long n, long long k, long long a, long long b, double* dg) {
  if (a == b) return;
  if (a > b) { const long long t = a; a = b; b = t; }
  for (long long l = k + threadIdx.x; l < a; l += blockDim.x) {
    const double2 t = H[a + l * ld]; H[a + l * ld] = H[b + l * ld]; H[b + l * ld] = t;
  }
  for (long long j = a + 1 + threadIdx.x; j < b; j += blockDim.x) {
    const double2 t = H[j + a * ld]; H[j + a * ld] = cconj(H[b + j * ld]); H[b + j * ld] = cconj(t);
  }
  for (long long j = b + 1 + threadIdx.x; j < n; j += blockDim.x) {
    const double2 t = H[j + a * ld]; H[j + a * ld] = H[j + b * ld]; H[j + b * ld] = t;
  }
  if (threadIdx.x == 0) {
    const double2 t = H[a + a * ld]; H[a + a * ld] = H[b + b * ld]; H[b + b * ld] = t;
    H[b + a * ld] = cconj(H[b + a * ld]);
    const double u = dg[a]; dg[a] = dg[b]; dg[b] = u;
  }
  __syncthreads();
}

// One pivot decision at k = st[0] (no-op once k >= n): exactly the rule of k_piv_a / k_piv_b /
// k_piv_c on the Schur complement instead of on the columns.
// diag_only: only the diagonal pivoting (the column-pivoted QR's largest remaining norm on
// the Schur complements of S = X^* X, i.e. diagonally pivoted Cholesky)
__global__ void __launch_bounds__(TS) k_bk_select(double2* H, long long ld, long long n, BkPlan pl, int diag_only) {
  const long long k = pl.st[0];
  if (k >= n) {
    if (threadIdx.x == 0) pl.st[3] = 0;
    return;
  }
  constexpr long long NONE = 0x7fffffffffffffffll;
  double v = -1.0;
  long long jm = NONE;
  for (long long j = k + threadIdx.x; j < n; j += TS) {
    const double a = fabs(pl.dg[j]);
    if (a > v) { v = a; jm = j; }
  }
  block_argmax_ts(v, jm);
  if (jm == NONE) {   // NaN diagonal
    if (threadIdx.x == 0 && pl.st[4] == 0) pl.st[4] = -8;
    jm = k;
  }
  hswap(H, ld, n, k, k, jm, pl.dg);
  int type = 1;
  long long s2 = -1;
  int s2pos = -1;
  if (k < n - 1 && !diag_only) {
    double h1i = -1.0;
    long long ii = NONE;
    for (long long j = k + 1 + threadIdx.x; j < n; j += TS) {
      const double a = cabs_(H[j + k * ld]);
      if (a > h1i) { h1i = a; ii = j; }
    }
    block_argmax_ts(h1i, ii);
    if (ii == NONE) ii = k + 1;
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    const double h11 = fabs(H[k + k * ld].x);
    if (!(h11 >= alpha * h1i)) {
      double hij = -1.0;
      long long li = NONE;
      for (long long l = k + threadIdx.x; l < n; l += TS) {
        if (l == ii) continue;
        const double a = cabs_(hget(H, ld, ii, l));
        if (a > hij) { hij = a; li = l; }
      }
      block_argmax_ts(hij, li);
      if (h11 * hij >= alpha * h1i * h1i) {
        type = 1;
      } else if (fabs(H[ii + ii * ld].x) >= alpha * hij) {
        s2 = ii; s2pos = 0;
        hswap(H, ld, n, k, k, ii, pl.dg);
      } else {
        type = 2;
        s2 = ii; s2pos = 1;
        hswap(H, ld, n, k, k + 1, ii, pl.dg);
      }
    }
  }
  if (threadIdx.x == 0) {
    pl.type[k] = type;
    pl.sw1[k] = jm;
    pl.sw2[k] = s2;
    pl.sw2pos[k] = s2pos;
    pl.d[3 * k] = H[k + k * ld];
    if (type == 2) {
      pl.d[3 * k + 1] = H[k + 1 + k * ld];
      pl.d[3 * k + 2] = H[k + 1 + (k + 1) * ld];
      pl.type[k + 1] = 0;
    }
    pl.st[2] = (int)k;
    pl.st[3] = type;
    pl.st[0] = (int)(k + type);
  }
}

// Schur update of the trailing block after the step recorded in st: lower triangle of
// [k + t, n)^2 minus H_{:,p} D^{-1} H_{p,:}, p the pivot index(es).  32 x 32 tiles.
__global__ void __launch_bounds__(256) k_bk_update(double2* H, long long ld, long long n, BkPlan pl) {
  const int t = pl.st[3];
  if (t == 0 || blockIdx.y > blockIdx.x) return;
  const long long k = pl.st[2], b0 = k + t;
  const long long j0 = b0 + 32LL * blockIdx.x, l0 = b0 + 32LL * blockIdx.y;
  if (j0 >= n) return;
  __shared__ double2 vj[32][2], ul[32][2];
  const int tid = threadIdx.x;
  if (tid < 64) {
    const int r = tid & 31;
    const bool rows = tid < 32;
    const long long x = (rows ? j0 : l0) + r;
    double2 u0 = cmk(0, 0), u1 = cmk(0, 0);
    if (x < n) {
      u0 = H[x + k * ld];
      if (t == 2) u1 = H[x + (k + 1) * ld];
    }
    if (rows) {
      if (t == 1) {
        const double d = H[k + k * ld].x;
        vj[r][0] = cmk(u0.x / d, u0.y / d);
        vj[r][1] = cmk(0, 0);
      } else {
        const double a = H[k + k * ld].x, c = H[k + 1 + (k + 1) * ld].x;
        const double2 b = H[k + 1 + k * ld];
        const double det = a * c - (b.x * b.x + b.y * b.y);
        // v = u D^{-1}, D = [[a, conj b], [b, c]]
        const double2 v0 = cadd(cmk(u0.x * c, u0.y * c), cmul(u1, cmk(-b.x, -b.y)));
        const double2 v1 = cadd(cmul(u0, cmk(-b.x, b.y)), cmk(u1.x * a, u1.y * a));
        vj[r][0] = cmk(v0.x / det, v0.y / det);
        vj[r][1] = cmk(v1.x / det, v1.y / det);
      }
    } else {
      ul[r][0] = u0;
      ul[r][1] = u1;
    }
  }
  __syncthreads();
  for (int e = tid; e < 32 * 32; e += 256) {
    const int r = e & 31, c = e >> 5;
    const long long j = j0 + r, l = l0 + c;
    if (j >= n || l >= n || l > j) continue;
    double2 a = cmul(vj[r][0], cconj(ul[c][0]));
    if (t == 2) a = cadd(a, cmul(vj[r][1], cconj(ul[c][1])));
    double2& h = H[j + l * ld];
    h = cmk(h.x - a.x, h.y - a.y);
    if (j == l) {   // the diagonal stays real (and its contiguous copy current)
      h.y = 0.0;
      pl.dg[j] = h.x;
    }
  }
}

// The planned column interchanges of position k: F columns (all m rows) and p2
__device__ __forceinline__ void plan_swaps_body(double2* F, long long ld, long long m, long long k, long long* p2,
                                                const BkPlan& pl) {
  const long long a = pl.sw1[k];
  const long long b = pl.sw2[k];
  const long long bp = k + pl.sw2pos[k];
  for (int pass = 0; pass < 2; pass++) {
    const long long x = pass == 0 ? k : bp, y = pass == 0 ? a : b;
    if (pass == 1 && b < 0) break;
    if (x == y) continue;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
      const double2 t = F[i + x * ld]; F[i + x * ld] = F[i + y * ld]; F[i + y * ld] = t;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const long long t = p2[x]; p2[x] = p2[y]; p2[y] = t;
    }
    __syncthreads();   // (the passes touch different column pairs; grid-wide order comes from
                       // each element being swapped by the same thread in both passes)
  }
}

__global__ void k_plan_swaps(double2* F, long long ld, long long m, long long k, long long* p2, BkPlan pl, P2Scr s) {
  if (s.ctl[8]) return;   // the plan was stopped at an earlier column of this panel
  plan_swaps_body(F, ld, m, k, p2, pl);
}

// k_panel_add_fin of pivot k plus the planned interchanges of the next step's position kn
// (trailing columns >= kn > k: disjoint from what the panel update touches)
__global__ void __launch_bounds__(T2) k_panel_add_fin_swap(double2* S, long long lds, const double2* sv, long long r0,
                                                           long long m, int nr, double2* T, const double2* tv,
                                                           P2Scr s, double2* F, long long ld, long long kn,
                                                           long long n, long long* p2, BkPlan pl) {
  if (s.ctl[3] || s.ctl[8]) return;
  panel_add_fin_body(S, lds, sv, r0, m, nr, T, tv, s, F, ld);
  if (kn < n) plan_swaps_body(F, ld, m, kn, p2, pl);
}

// Check a planned pivot against the exact J-Grammian of its formed column(s) fx (, fx2),
// rows >= k: off by more than a quarter (or another sign / inertia) stops the plan --
// ctl[8] = 1, ctl[9] = k, ctl[10] = reflectors in the panel before it (nr).
__device__ __forceinline__ bool plan_bad1(double a, double ap) {
  return !(a != 0.0) || !isfinite(a) || ((a > 0.0) != (ap > 0.0)) || fabs(a - ap) > 0.25 * fmax(fabs(a), fabs(ap));
}
__device__ __forceinline__ void plan_stop(P2Scr s, long long k, int nr) {
  s.ctl[8] = 1;
  s.ctl[9] = (int)k;
  s.ctl[10] = nr;
}

__global__ void __launch_bounds__(T2) k_plan_check(const double2* fx, const double2* fx2, const int8_t* J,
                                                   long long k, long long m, int type, BkPlan pl, P2Scr s, int nr) {
  __shared__ double2 sh[T2 / 32];
  if (s.ctl[8]) return;
  const double a = jdot(fx, fx, J, k, m, true, sh).x;
  double c = 0.0;
  double2 b = cmk(0, 0);
  if (type == 2) {
    c = jdot(fx2, fx2, J, k, m, true, sh).x;
    b = jdot(fx2, fx, J, k, m, true, sh);   // H_{k+1,k} = f_{k+1}^* J f_k
  }
  if (threadIdx.x != 0) return;
  const double ap = pl.d[3 * k].x;
  bool bad;
  if (type == 1) {
    bad = plan_bad1(a, ap);
  } else {
    const double cp = pl.d[3 * k + 2].x;
    const double2 bp = pl.d[3 * k + 1];
    const double da = a - ap, dc = c - cp, dbx = b.x - bp.x, dby = b.y - bp.y;
    const double diff = sqrt(da * da + dc * dc + 2.0 * (dbx * dbx + dby * dby));
    const double na = sqrt(a * a + c * c + 2.0 * (b.x * b.x + b.y * b.y));
    const double np = sqrt(ap * ap + cp * cp + 2.0 * (bp.x * bp.x + bp.y * bp.y));
    const double det = a * c - (b.x * b.x + b.y * b.y), detp = ap * cp - (bp.x * bp.x + bp.y * bp.y);
    bad = !isfinite(diff) || !(det != 0.0) || ((det > 0.0) != (detp > 0.0)) || diff > 0.25 * fmax(na, np);
  }
  if (bad) plan_stop(s, k, nr);
}

// Planned 1x1 pivot in one launch: the formed column fx is checked against the plan (a
// rejected pivot stops the plan, nothing written), copied into column k (rows >= k0) and
// turned into its reflector (refl_prep_body, the same arithmetic as k_refl_prep).
__global__ void __launch_bounds__(T2) k_refl_prep_plan(double2* F, long long ld, int8_t* J, long long m, long long n,
                                                       long long k, long long k0, const double2* fx, P2Scr s,
                                                       double2* Sb, long long lds, int nr, BkPlan pl) {
  __shared__ double2 sh[T2 / 32];
  if (s.ctl[8] || s.ctl[3]) return;
  const double hn = jdot(fx, fx, J, k, m, true, sh).x;   // uniform over the block
  if (plan_bad1(hn, pl.d[3 * k].x)) {
    if (threadIdx.x == 0) plan_stop(s, k, nr);
    return;
  }
  double2* f = F + k * ld;
  for (long long i = k0 + threadIdx.x; i < m; i += T2) f[i] = fx[i];
  __syncthreads();
  refl_prep_body(F, ld, J, m, n, k, s, Sb, lds, nr, hn);
}

// Y[i + j PB] = sum over the nb row-chunk partials part[b][i + j nr] (Kahan-compensated, in
// chunk order): the J-products of the planned JQR's flush summed in short pieces, about as
// accurate as the column search's block-reduced dots (one long GEMM accumulation over the
// m rows lost a factor 3-10 in the Grammian preservation, measured)
__global__ void k_sum_chunks(const double2* part, int nb, long long pstride, int nr, long long ncol, double2* Y) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)nr * ncol) return;
  const int i = (int)(e % nr);
  const long long j = e / nr;
  double sx = 0.0, sy = 0.0, cx = 0.0, cy = 0.0;
  for (int b = 0; b < nb; b++) {
    const double2 v = part[b * pstride + e];
    const double yx = v.x - cx, yy = v.y - cy;
    const double tx = sx + yx, ty = sy + yy;
    cx = (tx - sx) - yx;
    cy = (ty - sy) - yy;
    sx = tx;
    sy = ty;
  }
  Y[i + j * PB] = cmk(sx, sy);
}

// Planned column interchange of the column-pivoted QR at position k: X and Rf columns, p2
__device__ __forceinline__ void plan_swap_qr_body(double2* X, long long ldx, long long mx, double2* Rf, long long ldr,
                                                  long long mr, long long k, long long* p2, const BkPlan& pl) {
  const long long a = pl.sw1[k];
  if (a == k) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < mx; i += (long long)gridDim.x * blockDim.x) {
    const double2 t = X[i + k * ldx]; X[i + k * ldx] = X[i + a * ldx]; X[i + a * ldx] = t;
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < mr; i += (long long)gridDim.x * blockDim.x) {
    const double2 t = Rf[i + k * ldr]; Rf[i + k * ldr] = Rf[i + a * ldr]; Rf[i + a * ldr] = t;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t = p2[k]; p2[k] = p2[a]; p2[a] = t;
  }
}

__global__ void k_plan_swap_qr(double2* X, long long ldx, long long mx, double2* Rf, long long ldr, long long mr,
                               long long k, long long* p2, BkPlan pl) {
  plan_swap_qr_body(X, ldx, mx, Rf, ldr, mr, k, p2, pl);
}

// k_panel_add of QR pivot k plus the planned interchange of position kn > k (trailing)
__global__ void __launch_bounds__(T2) k_panel_add_swapqr(double2* S, long long lds, const double2* sv, long long r0,
                                                         long long m, int nr, double2* T, const double2* tv, P2Scr s,
                                                         double2* X, long long ldx, double2* Rf, long long ldr,
                                                         long long mr, long long kn, long long n, long long* p2,
                                                         BkPlan pl) {
  if (s.ctl[3]) return;
  panel_add_body(S, lds, sv, r0, m, nr, T, tv, s);
  if (kn < n) plan_swap_qr_body(X, ldx, m, Rf, ldr, mr, kn, p2, pl);
}

// The formed QR pivot column's squared norm (rows >= k) against the planned Schur diagonal:
// ctl[5] = 1 when off by more than a quarter
__global__ void __launch_bounds__(T2) k_plan_check_qr(const double2* x, long long k, long long m, BkPlan pl, P2Scr s) {
  __shared__ double2 sh[T2 / 32];
  const double a = jdot(x, x, nullptr, k, m, false, sh).x;
  if (threadIdx.x == 0) {
    const double ap = pl.d[3 * k].x;
    if (!(a > 0.0) || !isfinite(a) || fabs(a - ap) > 0.25 * fmax(a, fabs(ap))) s.ctl[5] = 1;
  }
}

// SJ = J S (rows [r0, m) of nr columns; ld lds)
__global__ void k_scale_j(const double2* S, double2* SJ, long long lds, const int8_t* J, long long r0, long long m,
                          int nr) {
  const long long tot = (m - r0) * (long long)nr;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long c = e / (m - r0), r = r0 + e % (m - r0);
    const double2 v = S[r + c * lds];
    SJ[r + c * lds] = J[r] > 0 ? v : cmk(-v.x, -v.y);
  }
}

}  // namespace

size_t phase2_scratch_bytes(int64_t m, int64_t n) {
  // P2Scr, then the JQR pivot plan (BkPlan: 72 bytes per column + control)
  return al256((size_t)n * 8) + 2 * al256((size_t)n * 16) + al256((size_t)m * 16) + 512 + 256 +
         2 * al256((size_t)n * 4) + 3 * al256((size_t)n * 8) + al256((size_t)3 * n * 16) + 256;
}

namespace {
// the BkPlan arrays, carved after P2Scr in the same scratch
BkPlan carve_plan(char* scr, int64_t m, int64_t n) {
  char* p = scr + al256((size_t)n * 8) + 2 * al256((size_t)n * 16) + al256((size_t)m * 16) + 512 + 256;
  BkPlan pl;
  pl.type = (int*)p; p += al256((size_t)n * 4);
  pl.sw2pos = (int*)p; p += al256((size_t)n * 4);
  pl.sw1 = (long long*)p; p += al256((size_t)n * 8);
  pl.sw2 = (long long*)p; p += al256((size_t)n * 8);
  pl.d = (double2*)p; p += al256((size_t)3 * n * 16);
  pl.dg = (double*)p; p += al256((size_t)n * 8);
  pl.st = (int*)p;
  return pl;
}
}  // namespace

#define P2CHK()                                    \
  do {                                             \
    cudaError_t e_ = cudaGetLastError();           \
    if (e_ != cudaSuccess) {                       \
      ctx->err = cudaGetErrorString(e_);           \
      return GHSVD_E_CUDA;                         \
    }                                              \
  } while (0)

// ---------------------------------------------------------------- cuBLAS (dlopen)
// Only the plain ZGEMMs of the blocked Phase 2's panel flushes use it; loaded at run time
// (torch's copy when torch is loaded), so the library keeps no link-time dependency.
namespace {
struct Cublas {
  bool tried = false, ok = false;
  cublasStatus_t (*Create)(cublasHandle_t*) = nullptr;
  cublasStatus_t (*Destroy)(cublasHandle_t) = nullptr;
  cublasStatus_t (*SetStream)(cublasHandle_t, cudaStream_t) = nullptr;
  cublasStatus_t (*Zgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const cuDoubleComplex*,
                          const cuDoubleComplex*, int, const cuDoubleComplex*, int, const cuDoubleComplex*,
                          cuDoubleComplex*, int) = nullptr;
  cublasStatus_t (*ZgemmSB)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int,
                            const cuDoubleComplex*, const cuDoubleComplex*, int, long long, const cuDoubleComplex*, int,
                            long long, const cuDoubleComplex*, cuDoubleComplex*, int, long long, int) = nullptr;
};
Cublas* cublas_lib() {
  static Cublas c;
  if (c.tried) return c.ok ? &c : nullptr;
  c.tried = true;
  const char* names[] = {"libcublas.so.12", "libcublas.so", "/usr/local/cuda/lib64/libcublas.so.12"};
  void* h = nullptr;
  for (const char* nm : names)
    if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return nullptr;
  c.Create = (decltype(c.Create))dlsym(h, "cublasCreate_v2");
  c.Destroy = (decltype(c.Destroy))dlsym(h, "cublasDestroy_v2");
  c.SetStream = (decltype(c.SetStream))dlsym(h, "cublasSetStream_v2");
  c.Zgemm = (decltype(c.Zgemm))dlsym(h, "cublasZgemm_v2");
  c.ZgemmSB = (decltype(c.ZgemmSB))dlsym(h, "cublasZgemmStridedBatched");
  c.ok = c.Create && c.Destroy && c.SetStream && c.Zgemm && c.ZgemmSB;
  return c.ok ? &c : nullptr;
}
}  // namespace

// ---------------------------------------------------------------- cuSOLVER (dlopen)
// The plain (not column-pivoted) QR of G P2 is LAPACK's ZGEQRF in the paper's own code
// ("the tall-and-skinny QR (ZGEQR from LAPACK)", Sec 5.4); here cuSOLVER's ZGEQRF,
// loaded at run time like cuBLAS.  Only R is kept.
namespace {
struct Cusolver {
  bool tried = false, ok = false;
  cusolverStatus_t (*Create)(cusolverDnHandle_t*) = nullptr;
  cusolverStatus_t (*Destroy)(cusolverDnHandle_t) = nullptr;
  cusolverStatus_t (*SetStream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
  cusolverStatus_t (*GeqrfBuf)(cusolverDnHandle_t, int, int, cuDoubleComplex*, int, int*) = nullptr;
  cusolverStatus_t (*Geqrf)(cusolverDnHandle_t, int, int, cuDoubleComplex*, int, cuDoubleComplex*, cuDoubleComplex*,
                            int, int*) = nullptr;
};
Cusolver* cusolver_lib() {
  static Cusolver c;
  if (c.tried) return c.ok ? &c : nullptr;
  c.tried = true;
  const char* names[] = {"libcusolver.so.11", "libcusolver.so", "/usr/local/cuda/lib64/libcusolver.so.11"};
  void* h = nullptr;
  for (const char* nm : names)
    if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return nullptr;
  c.Create = (decltype(c.Create))dlsym(h, "cusolverDnCreate");
  c.Destroy = (decltype(c.Destroy))dlsym(h, "cusolverDnDestroy");
  c.SetStream = (decltype(c.SetStream))dlsym(h, "cusolverDnSetStream");
  c.GeqrfBuf = (decltype(c.GeqrfBuf))dlsym(h, "cusolverDnZgeqrf_bufferSize");
  c.Geqrf = (decltype(c.Geqrf))dlsym(h, "cusolverDnZgeqrf");
  c.ok = c.Create && c.Destroy && c.SetStream && c.GeqrfBuf && c.Geqrf;
  return c.ok ? &c : nullptr;
}

// a zero R diagonal entry (G P2 numerically rank deficient) -> ctl[3] = -7
__global__ void k_qr_diag_check(const double2* X, long long ld, long long n, const int* info, P2Scr s) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const double2 d = X[k + k * ld];
    if (!(d.x != 0.0 || d.y != 0.0) || !isfinite(d.x) || !isfinite(d.y)) atomicCAS(&s.ctl[3], 0, -7);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && *info != 0) atomicCAS(&s.ctl[3], 0, -7);
}
}  // namespace

void phase2_release(Ctx* ctx) {
  if (ctx->cublas) {
    if (Cublas* c = cublas_lib()) c->Destroy((cublasHandle_t)ctx->cublas);
    ctx->cublas = nullptr;
  }
  if (ctx->cusolver) {
    if (Cusolver* c = cusolver_lib()) c->Destroy((cusolverDnHandle_t)ctx->cusolver);
    ctx->cusolver = nullptr;
  }
}

#define TRY(x)                     \
  do {                             \
    ghsvd_status s_ = (x);         \
    if (s_ != GHSVD_OK) return s_; \
  } while (0)

#define P2CUB(call)                                                   \
  do {                                                                \
    cublasStatus_t c_ = (call);                                       \
    if (c_ != CUBLAS_STATUS_SUCCESS) {                                \
      ctx->err = "reduce: cuBLAS ZGEMM failed (" + std::to_string((int)c_) + ")"; \
      return GHSVD_E_CUDA;                                            \
    }                                                                 \
  } while (0)

namespace {

struct Panel {
  double2 *S, *T, *Y, *W, *tv, *u, *fx;
  double2 *fx2, *SJ;   // planned JQR: second formed pivot column, J-scaled panel
  double2* part;       // planned JQR: row-chunk partials of the flush's J-products
  long long part_cap;  // entries available at part
  long long lds;
};

// X[r0:m, j0:n) += S[r0:m, 0:nr] W[0:nr, j0:n)  (the panel's delayed update)
ghsvd_status flush_update(Ctx* ctx, Cublas* cb, const Panel& P, double2* X, long long ld, long long r0, long long m,
                          long long j0, long long n, int nr) {
  if (nr == 0 || j0 >= n || r0 >= m) return GHSVD_OK;
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
  P2CUB(cb->Zgemm((cublasHandle_t)ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, (int)(m - r0), (int)(n - j0), nr, &one,
                  (const cuDoubleComplex*)(P.S + r0), (int)P.lds, (const cuDoubleComplex*)(P.W + j0 * PB), PB, &one,
                  (cuDoubleComplex*)(X + r0 + j0 * ld), (int)ld));
  return GHSVD_OK;
}

}  // namespace

// Blocked JQR of F (in place, like the unblocked loop of phase2_reduce), see the
// "blocked Phase 2" comment above.  Returns GHSVD_OK with s.ctl[3] clear, or an error.
static ghsvd_status jqr_blocked(Ctx* ctx, Cublas* cb, const Panel& P, P2Scr s, int64_t k_start = 0) {
  const int64_t m = ctx->m_user, n = ctx->n_user;
  const long long ld = ctx->ldm;
  cudaStream_t st = ctx->stream;
  long long* p2 = (long long*)ctx->p2;
  double2* F = ctx->F;
  int8_t* J = ctx->J;
  int ctl[8];
  auto rd = [&]() -> ghsvd_status {
    GH_CUDA(cudaMemcpyAsync(ctl, s.ctl, 32, cudaMemcpyDeviceToHost, st));
    GH_CUDA(cudaStreamSynchronize(st));
    return GHSVD_OK;
  };
  const unsigned gm = (unsigned)std::min<int64_t>(1024, (m + 255) / 256);
  int64_t k = k_start;
  while (k < n) {
    const int64_t k0 = k;
    int nr = 0, pend = 0;   // reflectors in the panel; newest ones without Y rows yet
    GH_CUDA(cudaMemsetAsync(P.T, 0, (size_t)PB * PB * 16, st));
    GH_CUDA(cudaMemsetAsync(P.Y + k * PB, 0, (size_t)PB * (n - k) * 16, st));
    GH_CUDA(cudaMemsetAsync(P.W + k * PB, 0, (size_t)PB * (n - k) * 16, st));
    k_jnorms<<<(unsigned)(n - k), T2, 0, st>>>(F, ld, J, m, k, s);   // exact J-norms at the panel start
    while (k < n && nr + 2 <= PB) {
      if (pend) {
        // Y rows of the previous step's reflectors, then w = T y and the new R rows'
        // J-norm downdate for every trailing column
        for (int t = 0; t < pend; t++)
          k_vdot<<<(unsigned)(n - k), T2, 0, st>>>(P.S + (size_t)(nr - pend + t) * P.lds, F, ld, J, k0, m, k,
                                                  P.Y + (nr - pend + t) + k * PB, PB);
        k_panel_rows<<<(unsigned)((n - k + 127) / 128), 128, 0, st>>>(F, ld, J, P.S, P.lds, P.T, P.Y, P.W, nr,
                                                                      k - pend, pend, k, n, s.hd);
        pend = 0;
      }
      GH_CUDA(cudaMemsetAsync(s.ctl, 0, 32, st));
      // 1. diagonal pivot on the (downdated) J-norms, then the pivot column made explicit
      k_piv_a<<<1, T2, 0, st>>>(F, ld, m, n, k, p2, s, P.Y, P.W, PB);
      if (nr) k_form<<<gm, 256, 0, st>>>(F + k * ld, F + k * ld, P.S, P.lds, P.W + k * PB, nr, k0, m);
      k_zero_yw<<<1, 64, 0, st>>>(P.Y, P.W, k);
      k_exact_hd<<<1, T2, 0, st>>>(F + k * ld, J, k, m, k, nr > 0, s);
      if (k < n - 1) {
        // 2. Bunch-Kaufman: h_1j = f_k^* J x_j (updated, rows >= k) = x-dot + u^T w_j
        k_vdot<<<(unsigned)(n - k - 1), T2, 0, st>>>(F + k * ld, F, ld, J, k, m, k + 1, s.d1 + (k + 1), 1);
        if (nr) {
          k_sdots<<<nr, T2, 0, st>>>(F + k * ld, P.S, P.lds, J, k, m, P.u);
          k_dfix<<<(unsigned)((n - k + 127) / 128), 128, 0, st>>>(s.d1, P.u, P.W, nr, k + 1, n);
        }
        k_piv_b<<<1, T2, 0, st>>>(n, k, s);
        TRY(rd());
        if (ctl[5]) break;    // estimate was off: flush, restart with exact J-norms
        if (ctl[2]) {
          const int64_t ii = ctl[1];
          if (nr) k_form<<<gm, 256, 0, st>>>(F + ii * ld, P.fx, P.S, P.lds, P.W + ii * PB, nr, k0, m);
          else GH_CUDA(cudaMemcpyAsync(P.fx + k0, F + ii * ld + k0, (size_t)(m - k0) * 16, cudaMemcpyDeviceToDevice, st));
          k_vdot<<<(unsigned)(n - k), T2, 0, st>>>(P.fx, F, ld, J, k, m, k, s.d2 + k, 1);
          if (nr) {
            k_sdots<<<nr, T2, 0, st>>>(P.fx, P.S, P.lds, J, k, m, P.u);
            k_dfix<<<(unsigned)((n - k + 127) / 128), 128, 0, st>>>(s.d2, P.u, P.W, nr, k, n);
          }
          k_exact_hd<<<1, T2, 0, st>>>(P.fx, J, k, m, ii, 0, s);
          k_piv_c<<<1, T2, 0, st>>>(F, ld, m, n, k, p2, s, P.Y, P.W, PB);
          k_place_fx<<<gm, 256, 0, st>>>(F, ld, P.fx, k0, m, k, P.Y, P.W, s);
        }
      } else {
        static const int one = 1;
        GH_CUDA(cudaMemcpyAsync(s.ctl, &one, 4, cudaMemcpyHostToDevice, st));
      }
      TRY(rd());
      if (ctl[3]) break;
      const int type = ctl[0];
      // 3. the reflector(s) of the pivot column(s), appended to the panel
      if (type == 2) k_rot<<<1, T2, 0, st>>>(F, ld, J, m, k, +1, s);
      for (int t = 0; t < type; t++) {
        const long long kk = k + t;
        k_refl_prep<<<1, T2, 0, st>>>(F, ld, J, m, n, kk, s, P.S, P.lds, nr);
        if (nr) k_sdots<<<nr, T2, 0, st>>>(s.s, P.S, P.lds, J, kk, m, P.tv);
        k_panel_add<<<gm, T2, 0, st>>>(P.S, P.lds, s.s, kk, m, nr, P.T, P.tv, s);
        nr++;
        if (t == 0 && type == 2) k_refl_apply<<<1, T2, 0, st>>>(F, ld, J, m, kk, kk + 1, nullptr, 1, s);
        k_refl_fin<<<1, T2, 0, st>>>(F, ld, m, kk, s);
      }
      if (type == 2) k_rot<<<1, T2, 0, st>>>(F, ld, J, m, k, -1, s);
      P2CHK();
      k += type;
      pend = type;
    }
    if (ctl[3]) break;
    // flush: the delayed update of the trailing columns [k, n)
    if (k < n && nr) {
      for (int t = 0; t < pend; t++)
        k_vdot<<<(unsigned)(n - k), T2, 0, st>>>(P.S + (size_t)(nr - pend + t) * P.lds, F, ld, J, k0, m, k,
                                                P.Y + (nr - pend + t) + k * PB, PB);
      if (pend) k_panel_rows<<<(unsigned)((n - k + 127) / 128), 128, 0, st>>>(F, ld, J, P.S, P.lds, P.T, P.Y, P.W,
                                                                             nr, k, 0, k, n, s.hd);
      TRY(flush_update(ctx, cb, P, F, ld, k0, m, k, n, nr));
      P2CHK();
    }
  }
  return GHSVD_OK;
}

// The JQR pivot plan (see BkPlan): H = F^* J F (rows J-sorted: F_+^* F_+ - F_-^* F_-, two
// ZGEMMs) into the n x n buffer Hb, then one k_bk_select + k_bk_update per step.  Fills the
// host copy of the pivot types.  p2 is not touched (the JQR applies the interchanges).
// X (m x n, ld): the first np rows carry J = +1, the rest J = -1 (np = m: the QR's S = X^* X,
// diag_only).
static ghsvd_status gram_plan(Ctx* ctx, Cublas* cb, const double2* X, long long ld, int64_t np, int diag_only,
                              double2* Hb, long long ldh, const BkPlan& pl, std::vector<int>& type_h) {
  const int64_t m = ctx->m_user, n = ctx->n_user;
  cudaStream_t st = ctx->stream;
  np = std::min<int64_t>(std::max<int64_t>(np, 0), m);
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), mone = make_cuDoubleComplex(-1.0, 0.0),
                        zero = make_cuDoubleComplex(0.0, 0.0);
  const cuDoubleComplex* Fp = (const cuDoubleComplex*)X;
  if (np > 0)
    P2CUB(cb->Zgemm((cublasHandle_t)ctx->cublas, CUBLAS_OP_C, CUBLAS_OP_N, (int)n, (int)n, (int)np, &one, Fp, (int)ld,
                    Fp, (int)ld, &zero, (cuDoubleComplex*)Hb, (int)ldh));
  if (m > np)
    P2CUB(cb->Zgemm((cublasHandle_t)ctx->cublas, CUBLAS_OP_C, CUBLAS_OP_N, (int)n, (int)n, (int)(m - np), &mone,
                    Fp + np, (int)ld, Fp + np, (int)ld, np > 0 ? &one : &zero, (cuDoubleComplex*)Hb, (int)ldh));
  GH_CUDA(cudaMemsetAsync(pl.st, 0, 32, st));
  GH_CUDA(cudaMemsetAsync(pl.type, 0, (size_t)n * 4, st));
  k_bk_diag<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Hb, ldh, n, pl.dg);
  for (int64_t i = 0; i < n; i++) {
    // the device step index k is >= i (each step advances by 1 or 2): a grid for the
    // trailing block [i + 1, n) covers it; steps past the end are no-ops
    k_bk_select<<<1, TS, 0, st>>>(Hb, ldh, n, pl, diag_only);
    const unsigned nt = (unsigned)((n - i - 1 + 31) / 32);
    if (nt) k_bk_update<<<dim3(nt, nt), 256, 0, st>>>(Hb, ldh, n, pl);
  }
  P2CHK();
  type_h.assign(n, 0);
  int stv[8];
  GH_CUDA(cudaMemcpyAsync(type_h.data(), pl.type, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
  GH_CUDA(cudaMemcpyAsync(stv, pl.st, 32, cudaMemcpyDeviceToHost, st));
  GH_CUDA(cudaStreamSynchronize(st));
  if (stv[4]) {
    ctx->err = "reduce: non-finite Grammian in the Phase-2 pivot plan";
    return GHSVD_E_NONFINITE;
  }
  return GHSVD_OK;
}

// Blocked JQR with the planned pivots: per step the planned column interchanges, the pivot
// column(s) formed from the panel (y = S^* J x, w = T y, x + S w) and CHECKED against the
// plan (k_plan_check), then the reflectors exactly as jqr_blocked; the trailing columns are
// updated once per panel by ZGEMMs (Y = (J S)^* X, W = T Y, X += S W) -- no pass over them
// per column.  A pivot the exact J-Grammian contradicts ends the plan: the panel is flushed
// and jqr_blocked (pivots searched on the columns) continues from that column.
static ghsvd_status jqr_planned(Ctx* ctx, Cublas* cb, const Panel& P, P2Scr s, const BkPlan& pl,
                                const std::vector<int>& ptype, int64_t* k_fallback) {
  const int64_t m = ctx->m_user, n = ctx->n_user;
  const long long ld = ctx->ldm;
  cudaStream_t st = ctx->stream;
  double2* F = ctx->F;
  int8_t* J = ctx->J;
  long long* p2 = (long long*)ctx->p2;
  int ctl[12];
  const unsigned gm = (unsigned)std::min<int64_t>(1024, (m + 255) / 256);
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  *k_fallback = -1;
  GH_CUDA(cudaMemsetAsync(s.ctl, 0, 48, st));
  auto rd = [&]() -> ghsvd_status {
    GH_CUDA(cudaMemcpyAsync(ctl, s.ctl, 48, cudaMemcpyDeviceToHost, st));
    GH_CUDA(cudaStreamSynchronize(st));
    return GHSVD_OK;
  };
  int64_t k = 0;
  k_plan_swaps<<<gm, 256, 0, st>>>(F, ld, m, 0, p2, pl, s);
  while (k < n) {
    const int64_t k0 = k;
    int nr = 0;
    bool stop = false;
    GH_CUDA(cudaMemsetAsync(P.T, 0, (size_t)PB * PB * 16, st));
    // The 1x1 pivots of a panel are enqueued without read-backs: a pivot the check rejects
    // stops the plan on the device (ctl[8]; the later kernels of the panel return at once)
    // and the panel's end learns where.  A 2x2 pivot reads the check back first.
    while (k < n && nr + std::max(ptype[k], 1) <= PB) {
      const int type = ptype[k] == 2 && k + 1 < n ? 2 : 1;
      // (the planned interchanges of position k ran with the previous step's last launch)
      // the pivot column(s) with the panel's delayed update, into fx (, fx2)
      for (int c = 0; c < type; c++) {
        double2* x = F + (k + c) * ld;
        double2* out = c ? P.fx2 : P.fx;
        if (nr) {
          k_ycol<<<nr, T2, 0, st>>>(x, P.S, P.lds, J, k0, m, P.u);
          k_form_tw<<<gm, 256, 0, st>>>(x, out, P.S, P.lds, P.T, P.u, nr, k0, m);
        } else {
          GH_CUDA(cudaMemcpyAsync(out + k0, x + k0, (size_t)(m - k0) * 16, cudaMemcpyDeviceToDevice, st));
        }
      }
      if (type == 1) {
        k_refl_prep_plan<<<1, T2, 0, st>>>(F, ld, J, m, n, k, k0, P.fx, s, P.S, P.lds, nr, pl);
        if (nr) k_sdots<<<nr, T2, 0, st>>>(s.s, P.S, P.lds, J, k, m, P.tv);
        k_panel_add_fin_swap<<<gm, T2, 0, st>>>(P.S, P.lds, s.s, k, m, nr, P.T, P.tv, s, F, ld, k + 1, n, p2, pl);
        nr++;
      } else {
        k_plan_check<<<1, T2, 0, st>>>(P.fx, P.fx2, J, k, m, 2, pl, s, nr);
        TRY(rd());
        if (ctl[3]) return GHSVD_OK;   // error flag: the caller reports it
        if (ctl[8]) {
          stop = true;
          break;
        }
        for (int c = 0; c < 2; c++)
          GH_CUDA(cudaMemcpyAsync(F + (k + c) * ld + k0, (c ? P.fx2 : P.fx) + k0, (size_t)(m - k0) * 16,
                                  cudaMemcpyDeviceToDevice, st));
        // the 2x2 pivot as in jqr_blocked: rotation, two reflectors, rotation undone
        k_rot<<<1, T2, 0, st>>>(F, ld, J, m, k, +1, s);
        for (int t = 0; t < 2; t++) {
          const long long kk = k + t;
          k_refl_prep<<<1, T2, 0, st>>>(F, ld, J, m, n, kk, s, P.S, P.lds, nr);
          if (nr) k_sdots<<<nr, T2, 0, st>>>(s.s, P.S, P.lds, J, kk, m, P.tv);
          k_panel_add<<<gm, T2, 0, st>>>(P.S, P.lds, s.s, kk, m, nr, P.T, P.tv, s);
          nr++;
          if (t == 0) k_refl_apply<<<1, T2, 0, st>>>(F, ld, J, m, kk, kk + 1, nullptr, 1, s);
          k_refl_fin<<<1, T2, 0, st>>>(F, ld, m, kk, s);
        }
        k_rot<<<1, T2, 0, st>>>(F, ld, J, m, k, -1, s);
        if (k + 2 < n) k_plan_swaps<<<gm, 256, 0, st>>>(F, ld, m, k + 2, p2, pl, s);
      }
      P2CHK();
      k += type;
    }
    TRY(rd());
    if (ctl[3]) return GHSVD_OK;
    int64_t kf = k;
    int nrf = nr;
    if (ctl[8]) {   // stopped at column ctl[9] with ctl[10] reflectors in the panel
      stop = true;
      kf = ctl[9];
      nrf = ctl[10];
    }
    // flush: the delayed update of the stale columns [kf, n)
    if (kf < n && nrf) {
      // Y = (J S)^* X over rows [k0, m) as partials over row chunks of 32 (strided-batched
      // ZGEMMs, column slabs sized to the free panel buffer), summed with compensation
      // (k_sum_chunks): short accumulations, as in the column search's block-reduced dots
      k_scale_j<<<gm, 256, 0, st>>>(P.S, P.SJ, P.lds, J, k0, m, nrf);
      const long long rows = m - k0, kc = 32, nb = (rows + kc - 1) / kc, full = rows / kc;
      const long long ns = std::max<long long>(1, std::min<long long>(n - kf, P.part_cap / (nb * nrf)));
      for (long long j0 = kf; j0 < n; j0 += ns) {
        const long long ncol = std::min<long long>(ns, n - j0), pstride = (long long)nrf * ncol;
        if (full > 0)
          P2CUB(cb->ZgemmSB((cublasHandle_t)ctx->cublas, CUBLAS_OP_C, CUBLAS_OP_N, nrf, (int)ncol, (int)kc, &one,
                            (const cuDoubleComplex*)(P.SJ + k0), (int)P.lds, kc,
                            (const cuDoubleComplex*)(F + k0 + j0 * ld), (int)ld, kc, &zero,
                            (cuDoubleComplex*)P.part, nrf, pstride, (int)full));
        if (full < nb)   // the ragged last chunk
          P2CUB(cb->Zgemm((cublasHandle_t)ctx->cublas, CUBLAS_OP_C, CUBLAS_OP_N, nrf, (int)ncol,
                          (int)(rows - full * kc), &one, (const cuDoubleComplex*)(P.SJ + k0 + full * kc),
                          (int)P.lds, (const cuDoubleComplex*)(F + k0 + full * kc + j0 * ld), (int)ld, &zero,
                          (cuDoubleComplex*)(P.part + full * pstride), nrf));
        k_sum_chunks<<<(unsigned)((pstride + 255) / 256), 256, 0, st>>>(P.part, (int)nb, pstride, nrf, ncol,
                                                                         P.Y + j0 * PB);
      }
      P2CUB(cb->Zgemm((cublasHandle_t)ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, nrf, (int)(n - kf), nrf, &one,
                      (const cuDoubleComplex*)P.T, PB, (const cuDoubleComplex*)(P.Y + kf * PB), PB, &zero,
                      (cuDoubleComplex*)(P.W + kf * PB), PB));
      TRY(flush_update(ctx, cb, P, F, ld, k0, m, kf, n, nrf));
      P2CHK();
    }
    if (stop) {
      *k_fallback = kf;
      GH_CUDA(cudaMemsetAsync(s.ctl, 0, 48, st));   // the column search starts clean
      return GHSVD_OK;
    }
  }
  return GHSVD_OK;
}

// Blocked Householder QR (optionally column-pivoted by norm) of the contiguous m x n
// buffer X (G P2 gathered), left-looking panels as above with J = I; the column swaps of
// the pivoted form are applied to p2 and to the n x n R_F copy Rf (F' = F P5).
static ghsvd_status qr_blocked(Ctx* ctx, Cublas* cb, const Panel& P, P2Scr s, double2* X, long long ld,
                               bool colpiv, double2* Rf, long long ldr, int64_t k_start = 0,
                               const BkPlan* plan = nullptr) {
  const int64_t m = ctx->m_user, n = ctx->n_user;
  cudaStream_t st = ctx->stream;
  long long* p2 = (long long*)ctx->p2;
  int ctl[8];
  const unsigned gm = (unsigned)std::min<int64_t>(1024, (m + 255) / 256);
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  // plan (column-pivoted form only): the planned interchanges instead of the norm search,
  // each formed pivot checked against its planned norm; after a panel with a rejected pivot
  // the search takes over (colpiv_plan off)
  bool use_plan = colpiv && plan != nullptr;
  if (use_plan) {
    GH_CUDA(cudaMemsetAsync(s.ctl + 5, 0, 4, st));
    if (k_start < n) k_plan_swap_qr<<<gm, 256, 0, st>>>(X, ld, m, Rf, ldr, n, k_start, p2, *plan);
  }
  int64_t k = k_start;
  while (k < n) {
    const int64_t k0 = k;
    int nr = 0, pend = 0;
    GH_CUDA(cudaMemsetAsync(P.T, 0, (size_t)PB * PB * 16, st));
    GH_CUDA(cudaMemsetAsync(P.Y + k * PB, 0, (size_t)PB * (n - k) * 16, st));
    GH_CUDA(cudaMemsetAsync(P.W + k * PB, 0, (size_t)PB * (n - k) * 16, st));
    const bool dyn = colpiv && !use_plan;   // pivots searched on the (downdated) norms
    if (dyn) k_norms<<<(unsigned)(n - k), T2, 0, st>>>(X, ld, k, m, s);
    while (k < n && nr + 1 <= PB) {
      if (dyn) {
        if (pend) {
          k_vdot<<<(unsigned)(n - k), T2, 0, st>>>(P.S + (size_t)(nr - 1) * P.lds, X, ld, nullptr, k0, m, k,
                                                  P.Y + (nr - 1) + k * PB, PB);
          k_panel_rows<<<(unsigned)((n - k + 127) / 128), 128, 0, st>>>(X, ld, nullptr, P.S, P.lds, P.T, P.Y, P.W,
                                                                        nr, k - 1, 1, k, n, s.hd);
          pend = 0;
        }
        GH_CUDA(cudaMemsetAsync(s.ctl + 5, 0, 4, st));
        k_qr_colpiv_blk<<<1, T2, 0, st>>>(X, ld, m, Rf, ldr, n, n, k, p2, s, P.Y, P.W);
        if (nr) k_form<<<gm, 256, 0, st>>>(X + k * ld, X + k * ld, P.S, P.lds, P.W + k * PB, nr, k0, m);
        k_zero_yw<<<1, 64, 0, st>>>(P.Y, P.W, k);
        if (nr) {
          k_exact_hd<<<1, T2, 0, st>>>(X + k * ld, nullptr, k, m, k, 1, s);
          GH_CUDA(cudaMemcpyAsync(ctl, s.ctl, 32, cudaMemcpyDeviceToHost, st));
          GH_CUDA(cudaStreamSynchronize(st));
          if (ctl[5]) break;   // downdated norm was off: flush, then exact norms again
        }
      } else {
        // (a planned interchange of position k ran with the previous column's k_panel_add)
        if (nr) {
          k_ycol<<<nr, T2, 0, st>>>(X + k * ld, P.S, P.lds, nullptr, k0, m, P.u);
          k_form_tw<<<gm, 256, 0, st>>>(X + k * ld, X + k * ld, P.S, P.lds, P.T, P.u, nr, k0, m);
        }
      }
      k_qr_prep_c<<<1, T2, 0, st>>>(X, ld, m, k, s, use_plan ? plan->d : nullptr);
      if (nr) k_sdots<<<nr, T2, 0, st>>>(s.s, P.S, P.lds, nullptr, k, m, P.tv);
      if (use_plan)
        k_panel_add_swapqr<<<gm, T2, 0, st>>>(P.S, P.lds, s.s, k, m, nr, P.T, P.tv, s, X, ld, Rf, ldr, n, k + 1, n, p2,
                                              *plan);
      else
        k_panel_add<<<gm, T2, 0, st>>>(P.S, P.lds, s.s, k, m, nr, P.T, P.tv, s);
      nr++;
      k++;
      pend = 1;
      P2CHK();
    }
    if (k < n && nr) {
      if (dyn) {
        if (pend) {
          k_vdot<<<(unsigned)(n - k), T2, 0, st>>>(P.S + (size_t)(nr - 1) * P.lds, X, ld, nullptr, k0, m, k,
                                                  P.Y + (nr - 1) + k * PB, PB);
          k_panel_rows<<<(unsigned)((n - k + 127) / 128), 128, 0, st>>>(X, ld, nullptr, P.S, P.lds, P.T, P.Y, P.W,
                                                                        nr, k, 0, k, n, s.hd);
        }
      } else {
        // Y = S^* X_t, W = T Y on the tensor cores (cuBLAS), then the update
        P2CUB(cb->Zgemm((cublasHandle_t)ctx->cublas, CUBLAS_OP_C, CUBLAS_OP_N, nr, (int)(n - k), (int)(m - k0), &one,
                        (const cuDoubleComplex*)(P.S + k0), (int)P.lds, (const cuDoubleComplex*)(X + k0 + k * ld),
                        (int)ld, &zero, (cuDoubleComplex*)(P.Y + k * PB), PB));
        P2CUB(cb->Zgemm((cublasHandle_t)ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, nr, (int)(n - k), nr, &one,
                        (const cuDoubleComplex*)P.T, PB, (const cuDoubleComplex*)(P.Y + k * PB), PB, &zero,
                        (cuDoubleComplex*)(P.W + k * PB), PB));
      }
      TRY(flush_update(ctx, cb, P, X, ld, k0, m, k, n, nr));
      P2CHK();
    }
    if (use_plan) {
      // one read-back per panel: a pivot the formed column contradicted ends the plan
      GH_CUDA(cudaMemcpyAsync(ctl, s.ctl, 32, cudaMemcpyDeviceToHost, st));
      GH_CUDA(cudaStreamSynchronize(st));
      if (ctl[3]) break;
      if (ctl[5]) {
        use_plan = false;
        if (ctx->p2_fallback_qr < 0) ctx->p2_fallback_qr = k;
      }
    }
  }
  GH_CUDA(cudaMemcpyAsync(ctl, s.ctl, 32, cudaMemcpyDeviceToHost, st));
  GH_CUDA(cudaStreamSynchronize(st));
  if (ctl[3]) {
    ctx->err = "reduce: G P2 numerically rank deficient";
    return GHSVD_E_RANK_DEFICIENT;
  }
  return GHSVD_OK;
}

static ghsvd_status phase2_reduce_blocked(Ctx* ctx, int flags, Cublas* cb) {
  const int64_t m = ctx->m_user, n = ctx->n_user;
  const long long ld = ctx->ldm;
  cudaStream_t st = ctx->stream;
  P2Scr s = carve(ctx->scr, m, n);
  long long* p2 = (long long*)ctx->p2;
  Panel P;
  P.lds = round_up(m, 16);
  P.S = ctx->Z2;   // the output-Z buffer is free until extraction
  P.T = P.S + (size_t)P.lds * PB;
  P.Y = P.T + PB * PB;
  P.W = P.Y + (size_t)PB * n;
  P.tv = P.W + (size_t)PB * n;
  P.u = P.tv + PB;
  P.fx = P.u + PB;
  P.fx2 = P.fx + P.lds;
  P.SJ = P.fx2 + P.lds;
  P.part = P.SJ + (size_t)P.lds * PB;
  P.part_cap = (long long)ctx->ldn * (ctx->n_cap + 1) - (long long)(P.part - ctx->Z2);
  GH_CUDA(cudaMemsetAsync(s.ctl, 0, 256, st));
  GH_CUDA(cudaMemsetAsync(P.S, 0, (size_t)P.lds * PB * 16, st));
  k_iota<<<8, 256, 0, st>>>(p2, n);
  P2CHK();
  if (flags & GHSVD_REDUCE_COLSEARCH) {
    TRY(jqr_blocked(ctx, cb, P, s));
  } else {
    // pivots planned on the J-Grammian (in the n x n Z buffer, free until R_F is copied
    // into it below), each checked on its formed column; the column search takes over
    // from the first pivot the check rejects
    const BkPlan pl = carve_plan(ctx->scr, m, n);
    std::vector<int> ptype;
    TRY(gram_plan(ctx, cb, ctx->F, ctx->ldm, ctx->npos, 0, ctx->Z, ctx->ldn, pl, ptype));
    int64_t kf = -1;
    TRY(jqr_planned(ctx, cb, P, s, pl, ptype, &kf));
    ctx->p2_fallback_col = kf;   // -1: every planned pivot used
    if (kf >= 0) TRY(jqr_blocked(ctx, cb, P, s, kf));
  }
  int ctl[8];
  GH_CUDA(cudaMemcpyAsync(ctl, s.ctl, 32, cudaMemcpyDeviceToHost, st));
  GH_CUDA(cudaStreamSynchronize(st));
  if (ctl[3] == -8) {
    ctx->err = "reduce: non-finite J-norms in the JQR pivot search";
    return GHSVD_E_NONFINITE;
  }
  if (ctl[3]) {
    ctx->err = "reduce: degenerate JQR pivot (J-Grammian numerically singular)";
    return GHSVD_E_RANK_DEFICIENT;
  }
  // R_F (leading n x n) -> Z; G P2 gathered into the F buffer; blocked QR there (the column
  // pivoted form swaps R_F's columns in Z alike); R_G -> G; R_F back, rows sorted by J
  const long long ldz = ctx->ldn;
  GH_CUDA(cudaMemcpy2DAsync(ctx->Z, (size_t)ldz * 16, ctx->F, (size_t)ld * 16, (size_t)n * 16, (size_t)n,
                            cudaMemcpyDeviceToDevice, st));
  k_gather_cols<<<dim3((unsigned)std::min<int64_t>(64, (m + 255) / 256), (unsigned)n), 256, 0, st>>>(
      ctx->G, ld, ctx->F, ld, m, p2);
  P2CHK();
  GH_CUDA(cudaMemsetAsync(s.ctl, 0, 256, st));
  GH_CUDA(cudaMemsetAsync(P.S, 0, (size_t)P.lds * PB * 16, st));
  if ((flags & GHSVD_REDUCE_COLPIV) && !(flags & GHSVD_REDUCE_COLSEARCH)) {
    // column pivots planned on S = (G P2)^* (G P2) (diagonally pivoted Cholesky of its Schur
    // complements = the largest remaining column norms), S in the G buffer (G P2 now lives in
    // the F buffer)
    const BkPlan pl = carve_plan(ctx->scr, m, n);
    std::vector<int> ptype;
    TRY(gram_plan(ctx, cb, ctx->F, ld, m, 1, ctx->G, ld, pl, ptype));
    TRY(qr_blocked(ctx, cb, P, s, ctx->F, ld, true, ctx->Z, ldz, 0, &pl));
  } else {
    bool done = false;
    Cusolver* cs = (flags & (GHSVD_REDUCE_COLPIV | GHSVD_REDUCE_OWN_QR)) ? nullptr : cusolver_lib();
    if (cs) {
      // the plain QR by cuSOLVER's ZGEQRF (workspace in the free n x n output-Z buffer)
      if (!ctx->cusolver) {
        cusolverDnHandle_t hs;
        if (cs->Create(&hs) != CUSOLVER_STATUS_SUCCESS) {
          ctx->err = "reduce: cusolverDnCreate failed";
          return GHSVD_E_CUDA;
        }
        ctx->cusolver = hs;
      }
      cusolverDnHandle_t hs = (cusolverDnHandle_t)ctx->cusolver;
      int lwork = 0;
      const long long cap = (long long)ctx->ldn * (ctx->n_cap + 1) - n - 16;
      if (cs->SetStream(hs, st) == CUSOLVER_STATUS_SUCCESS &&
          cs->GeqrfBuf(hs, (int)m, (int)n, (cuDoubleComplex*)ctx->F, (int)ld, &lwork) == CUSOLVER_STATUS_SUCCESS &&
          lwork <= cap) {
        cuDoubleComplex* tau = (cuDoubleComplex*)ctx->Z2;
        cuDoubleComplex* work = tau + n;
        int* info = (int*)(work + lwork);
        if (cs->Geqrf(hs, (int)m, (int)n, (cuDoubleComplex*)ctx->F, (int)ld, tau, work, lwork, info) !=
            CUSOLVER_STATUS_SUCCESS) {
          ctx->err = "reduce: cusolverDnZgeqrf failed";
          return GHSVD_E_CUDA;
        }
        k_qr_diag_check<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ctx->F, ld, n, info, s);
        P2CHK();
        int ctl4[4];
        GH_CUDA(cudaMemcpyAsync(ctl4, s.ctl, 16, cudaMemcpyDeviceToHost, st));
        GH_CUDA(cudaStreamSynchronize(st));
        if (ctl4[3]) {
          ctx->err = "reduce: G P2 numerically rank deficient";
          return GHSVD_E_RANK_DEFICIENT;
        }
        done = true;
      }
    }
    if (!done) TRY(qr_blocked(ctx, cb, P, s, ctx->F, ld, (flags & GHSVD_REDUCE_COLPIV) != 0, ctx->Z, ldz));
  }
  GH_CUDA(cudaMemsetAsync(ctx->G, 0, (size_t)ld * (ctx->n_cap + 1) * 16, st));
  k_qr_rout<<<(unsigned)n, T2, 0, st>>>(ctx->F, ld, ctx->G, ld, n);
  P2CHK();
  return GHSVD_OK;   // the caller re-sorts R_F (in Z) into F
}

// F: keep the leading n x n block (R_F, in Z), rows re-sorted by the new J (+ first)
static ghsvd_status phase2_finish(Ctx* ctx, P2Scr s) {
  const int64_t n = ctx->n_user;
  const long long ld = ctx->ldm, ldz = ctx->ldn;
  cudaStream_t st = ctx->stream;
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

ghsvd_status phase2_reduce(Ctx* ctx, int flags) {
  const int64_t m = ctx->m_user, n = ctx->n_user;
  const long long ld = ctx->ldm;
  cudaStream_t st = ctx->stream;
  P2Scr s = carve(ctx->scr, m, n);
  long long* p2 = (long long*)ctx->p2;
  // blocked (default) for large problems when cuBLAS loads and the output-Z buffer holds
  // the panel: below m n^2 ~ 2e10 the per-column launch / readback latency of the panel
  // logic outweighs the traffic it saves (config 2, 1568 x 1024: 0.26 s blocked vs 0.09 s)
  const bool big = (double)m * (double)n * (double)n >= 2e10;
  if (!(flags & GHSVD_REDUCE_UNBLOCKED) && (big || (flags & GHSVD_REDUCE_BLOCKED))) {
    // panel, its J-scaled copy, two formed columns, T, Y, W, and at least one column slab of
    // the flush's 32-row chunk partials (PB per chunk)
    const size_t need = ((size_t)round_up(m, 16) * (2 * PB + 2) + PB * PB + 2 * (size_t)PB * n + 2 * PB +
                         (size_t)((m + 31) / 32 + 1) * PB) * 16;
    const size_t have = (size_t)ctx->ldn * (ctx->n_cap + 1) * 16;
    Cublas* cb = cublas_lib();
    if (cb && need <= have) {
      if (!ctx->cublas) {
        cublasHandle_t hnd;
        if (cb->Create(&hnd) != CUBLAS_STATUS_SUCCESS) {
          ctx->err = "reduce: cublasCreate failed";
          return GHSVD_E_CUDA;
        }
        ctx->cublas = hnd;
      }
      if (cb->SetStream((cublasHandle_t)ctx->cublas, st) != CUBLAS_STATUS_SUCCESS) {
        ctx->err = "reduce: cublasSetStream failed";
        return GHSVD_E_CUDA;
      }
      TRY(phase2_reduce_blocked(ctx, flags, cb));
      return phase2_finish(ctx, s);
    }
  }
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
  return phase2_finish(ctx, s);
}

}  // namespace ghsvd
