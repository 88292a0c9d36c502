// hz2x2.cuh -- device 2x2 implicit Hari-Zimmermann transformation.
//
// PAPER.md Sec 6.1 (lines 1365-1573), eqs (6.1)-(6.12): from the unscaled
// pivot Grams h_pp, h_qq, h_pq = f_p^* J f_q and s_pp, s_qq, s_pq = g_p^* g_q
// form Z' = D0 R1 D2 R3 Phi4 (eq 6.8-6.9) in closed form (6.10)-(6.11).
//
// Arithmetic contract (reading C-8): only IEEE +, -, *, /, sqrt with
// round-to-nearest and NO contraction (every op is an explicit __d*_rn
// intrinsic), so the result is a deterministic function of the 8 inputs.
// Readings C-1 (criterion), C-2 (small = exact cos==1), C-4 (sigma = +1 at
// h = 0), C-5 (h = v = 0 closed form), C-9 (x >= 1 error), C-12, C-13 apply.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

namespace ghsvd {

enum : int { KIND_SKIP = 0, KIND_IDENTITY = 1, KIND_SMALL = 2, KIND_BIG = 3 };
enum : int { ERR_INDEF = -6, ERR_RANK = -7, ERR_NONFINITE = -8 };

struct Cplx {
  double re, im;
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }
// |z| = sqrt(re^2 + im^2)  (C-8: no hypot)
__device__ __forceinline__ double cabs_(double re, double im) {
  return dsqrt(dadd(dmul(re, re), dmul(im, im)));
}
// (a.re + i a.im)(b.re + i b.im)
__device__ __forceinline__ Cplx cmul_(Cplx a, Cplx b) {
  return Cplx{dsub(dmul(a.re, b.re), dmul(a.im, b.im)), dadd(dmul(a.re, b.im), dmul(a.im, b.re))};
}

struct HZOut {
  Cplx z11, z21, z12, z22;  // Z' (column-major 2x2)
  double off;               // scaled off-diagonal measure (diagnostic)
  int kind;                 // KIND_* or ERR_*
};

// g[8] = {hpp, hqq, hpq.re, hpq.im, spp, sqq, spq.re, spq.im}
// hz2x2_core is the inlinable body (used where one warp evaluates many pairs);
// hz2x2_dev is the same routine behind a call boundary (keeps register pressure of
// the streaming kernels low).  Both execute the identical IEEE operation sequence.
__device__ __forceinline__ HZOut hz2x2_core(const double* g, double tol, int literal) {
  HZOut o;
  o.z11 = Cplx{1.0, 0.0};
  o.z21 = Cplx{0.0, 0.0};
  o.z12 = Cplx{0.0, 0.0};
  o.z22 = Cplx{1.0, 0.0};
  o.off = 0.0;
  const double hpp = g[0], hqq = g[1], spp = g[4], sqq = g[5];
  const Cplx hpq{g[2], g[3]}, spq{g[6], g[7]};
  bool fin = true;
#pragma unroll
  for (int i = 0; i < 8; i++) fin = fin && isfinite(g[i]);
  if (!fin) { o.kind = ERR_NONFINITE; return o; }
  if (!(spp > 0.0) || !(sqq > 0.0)) { o.kind = ERR_INDEF; return o; }
  // Sec 6.1.1: pivot prescaling D0 = diag(s_pp^-1/2, s_qq^-1/2), every step.
  const double dp = ddiv(1.0, dsqrt(spp));
  const double dq = ddiv(1.0, dsqrt(sqq));
  const double Hpp = dmul(dmul(hpp, dp), dp);
  const double Hqq = dmul(dmul(hqq, dq), dq);
  const double dpq = dmul(dp, dq);
  const Cplx Hpq{dmul(hpq.re, dpq), dmul(hpq.im, dpq)};
  const Cplx Spq{dmul(spq.re, dpq), dmul(spq.im, dpq)};
  const double ah = cabs_(Hpq.re, Hpq.im);
  const double x = cabs_(Spq.re, Spq.im);
  const double aHpp = fabs(Hpp), aHqq = fabs(Hqq);
  {
    const double den = dmul(dsqrt(aHpp), dsqrt(aHqq));
    const double oh = den > 0.0 ? ddiv(ah, den) : (ah > 0.0 ? CUDART_INF : 0.0);
    o.off = oh > x ? oh : x;
  }
  // eq (6.12)
  bool doit;
  if (literal) {
    const double mx = aHpp > aHqq ? aHpp : aHqq;
    const double mn = aHpp > aHqq ? aHqq : aHpp;
    doit = (ah >= dmul(dmul(mx, tol), mn)) || (x >= tol);
  } else {
    doit = (ah >= dmul(dmul(tol, dsqrt(aHpp)), dsqrt(aHqq))) || (x >= tol);
  }
  if (!doit) { o.kind = KIND_SKIP; return o; }
  // Sec 6.1.6, first exception: both pivots already diagonal.
  if (Hpq.re == 0.0 && Hpq.im == 0.0 && Spq.re == 0.0 && Spq.im == 0.0) {
    o.kind = KIND_IDENTITY;
    return o;
  }
  if (!(x < 1.0)) { o.kind = ERR_INDEF; return o; }
  // eq (6.3): alpha_1 = arg s_pq (0 if s_pq = 0, second exception)
  const Cplx e1 = (x == 0.0) ? Cplx{1.0, 0.0} : Cplx{ddiv(Spq.re, x), ddiv(Spq.im, x)};
  // eq (6.5): u + i v = e^{-i alpha_1} h_pq
  const Cplx uv = cmul_(Cplx{e1.re, -e1.im}, Hpq);
  const double u = uv.re, v = uv.im;
  // eq (6.7): t = sqrt(1 - x^2) evaluated as sqrt((1-x)(1+x))
  const double t = dsqrt(dmul(dsub(1.0, x), dadd(1.0, x)));
  const double h = dsub(Hqq, Hpp);
  Cplx Z11, Z12, Z21, Z22;
  int kind;
  if (h == 0.0 && v == 0.0) {
    // third exception: Z = R1 D2 (reading C-5)
    const double ap = ddiv(1.0, dsqrt(dmul(2.0, dadd(1.0, x))));
    const double aq = ddiv(1.0, dsqrt(dmul(2.0, dsub(1.0, x))));
    Z11 = Cplx{ap, 0.0};
    Z12 = Cplx{dmul(e1.re, -aq), dmul(e1.im, -aq)};
    Z21 = Cplx{dmul(e1.re, ap), dmul(-e1.im, ap)};
    Z22 = Cplx{aq, 0.0};
    kind = KIND_BIG;
  } else {
    const double sigma = (h >= 0.0) ? 1.0 : -1.0;           // sigma = sgn(h), C-4
    const double v2 = dmul(2.0, v);
    const double r = dsqrt(dadd(dmul(h, h), dmul(v2, v2)));
    const double cg = ddiv(dmul(sigma, h), r);              // cos gamma, eq (6.11)
    const double sg = ddiv(dmul(sigma, v2), r);             // sin gamma
    const double N = dmul(sigma, dsub(dmul(2.0, u), dmul(dadd(Hpp, Hqq), x)));  // eq (6.7)
    const double D = dmul(t, r);
    const double rho = dsqrt(dadd(dmul(N, N), dmul(D, D)));
    const double c2 = ddiv(D, rho);                         // cos 2 theta (C-13)
    const double s2 = ddiv(N, rho);                         // sin 2 theta
    const double tcc = dmul(dmul(t, cg), c2);
    const double cphi = dsqrt(dmul(0.5, dadd(dadd(1.0, dmul(x, s2)), tcc)));  // eq (6.10)
    const double cpsi = dsqrt(dmul(0.5, dadd(dsub(1.0, dmul(x, s2)), tcc)));
    const double tsc = dmul(dmul(t, sg), c2);
    const Cplx wa = cmul_(e1, Cplx{dsub(s2, x), tsc});
    const Cplx wb = cmul_(Cplx{e1.re, -e1.im}, Cplx{dadd(s2, x), -tsc});
    const double dpsi = dmul(2.0, cpsi), dphi = dmul(2.0, cphi);
    const Cplx eas{ddiv(wa.re, dpsi), ddiv(wa.im, dpsi)};   // e^{i alpha} sin phi
    const Cplx ebs{ddiv(wb.re, dphi), ddiv(wb.im, dphi)};   // e^{-i beta} sin psi
    Z11 = Cplx{ddiv(cphi, t), 0.0};                         // eq (6.9) times Phi_4
    Z12 = Cplx{ddiv(eas.re, t), ddiv(eas.im, t)};
    Z21 = Cplx{-ddiv(ebs.re, t), -ddiv(ebs.im, t)};
    Z22 = Cplx{ddiv(cpsi, t), 0.0};
    kind = (cphi == 1.0 && cpsi == 1.0) ? KIND_SMALL : KIND_BIG;  // Sec 6.1.7, C-2
  }
  // Z' = D0 Z
  o.z11 = Cplx{dmul(Z11.re, dp), dmul(Z11.im, dp)};
  o.z21 = Cplx{dmul(Z21.re, dq), dmul(Z21.im, dq)};
  o.z12 = Cplx{dmul(Z12.re, dp), dmul(Z12.im, dp)};
  o.z22 = Cplx{dmul(Z22.re, dq), dmul(Z22.im, dq)};
  const bool zf = isfinite(o.z11.re) && isfinite(o.z11.im) && isfinite(o.z21.re) &&
                  isfinite(o.z21.im) && isfinite(o.z12.re) && isfinite(o.z12.im) &&
                  isfinite(o.z22.re) && isfinite(o.z22.im);
  o.kind = zf ? kind : ERR_NONFINITE;
  return o;
}

static __device__ __noinline__ HZOut hz2x2_dev(const double* g, double tol, int literal) {
  return hz2x2_core(g, tol, literal);
}

// Round-robin (circle) parallel ordering, reading C-11 of PAPER.md Sec 6.3:
// step s in [0, n-2], slot k in [0, n/2-1]; returns p < q.
__host__ __device__ __forceinline__ void rr_pair(long long n, long long s, long long k,
                                                 long long* p, long long* q) {
  long long a, b;
  if (k == 0) {
    a = n - 1;
    b = s;
  } else {
    const long long r = n - 1;
    a = (s + k) % r;
    b = (s - k) % r;
    if (b < 0) b += r;
  }
  *p = a < b ? a : b;
  *q = a < b ? b : a;
}

// 32-bit form of rr_pair for the in-shared-memory inner sweeps (n <= 64).
__device__ __forceinline__ void rr_pair32(int n, int s, int k, int* p, int* q) {
  int a, b;
  if (k == 0) {
    a = n - 1;
    b = s;
  } else {
    const int r = n - 1;
    a = s + k;
    if (a >= r) a -= r;
    b = s - k;
    if (b < 0) b += r;
  }
  *p = a < b ? a : b;
  *q = a < b ? b : a;
}

}  // namespace ghsvd
