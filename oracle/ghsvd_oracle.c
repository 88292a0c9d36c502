/*
 * ghsvd_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * implicit Hari-Zimmermann J-GHSVD (Novakovic, Singer, Singer, Hari;
 * arXiv:1907.08560, cited as PAPER.md:<line>).
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code with the CUDA product path.  Compiled with
 * -O2 -ffp-contract=off (no FMA contraction, SURVEY C-8) and OpenMP over the
 * disjoint pairs of a parallel step (Algorithm 3's parallel-do,
 * PAPER.md:1780-1782).  Sums run in plain sequential row order.
 *
 * Readings of the paper (listed in DESIGN.md "Readings"): C-1 relative
 * criterion by default, C-2 exact "small" test, C-3 stop on big == 0,
 * C-4 sigma = +1 at h = 0, C-5 closed form for h = v = 0, C-6 eps = 2^-53,
 * C-9 x >= 1 is an error, C-10 bordering of the factors, C-11 round-robin
 * ordering, C-12 t = sqrt((1-x)(1+x)), C-13 trig-free 2*theta.
 */
#include "ghsvd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- complex */
static orc cmk(double re, double im) { orc z; z.re = re; z.im = im; return z; }
static orc cadd(orc a, orc b) { return cmk(a.re + b.re, a.im + b.im); }
static orc csub(orc a, orc b) { return cmk(a.re - b.re, a.im - b.im); }
static orc cmul(orc a, orc b) { return cmk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
static orc cconj(orc a) { return cmk(a.re, -a.im); }
static orc cscale(orc a, double s) { return cmk(a.re * s, a.im * s); }
static double cabs2(orc a) { return a.re * a.re + a.im * a.im; }
static double cabsv(orc a) { return sqrt(a.re * a.re + a.im * a.im); }
/* conj(a) * b */
static orc cdotc1(orc a, orc b) { return cmk(a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re); }
static orc cdiv(orc a, orc b) {
  double d = b.re * b.re + b.im * b.im;
  return cmk((a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d);
}

#define EL(A, ld, i, j) (A)[(size_t)(i) + (size_t)(j) * (size_t)(ld)]

static void set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

/* ------------------------------------------------------------ ordering */
/* SURVEY C-11: circle method.  pair(s,0) = {n-1, s};
 * pair(s,k>=1) = {(s+k) mod (n-1), (s-k) mod (n-1)}, returned as p < q. */
int or_rr_pair(int64_t n, int64_t s, int64_t k, int64_t *p, int64_t *q) {
  if (n < 2 || (n & 1) || s < 0 || s > n - 2 || k < 0 || k >= n / 2) return OR_E_ARG;
  int64_t a, b;
  if (k == 0) {
    a = n - 1;
    b = s;
  } else {
    int64_t r = n - 1;
    a = (s + k) % r;
    b = ((s - k) % r + r) % r;
  }
  *p = a < b ? a : b;
  *q = a < b ? b : a;
  return OR_OK;
}

/* ----------------------------------------------- level-3 block orderings */
/* PAPER.md:1815-1824 (Sec 6.4): "a multilevel blocking principle can be applied ...
 * The same principle can be applied recursively further"; the paper builds Level 2
 * only.  Reading R2-5: nblk block columns are grouped into nsup = 2Q super
 * blocks of B = nblk / nsup consecutive block columns, and the block pairs of a block
 * sweep are ordered by super block:
 *  OR_ORDER_LEVEL3 (1): the Level-2 principle applied once more.  An outer round-robin
 *    over the 2Q super blocks (2Q - 1 outer steps t, super pair slots u < Q); a super
 *    pair is a Level-3 pivot of 2B block columns and receives ONE inner round-robin
 *    block sweep over them (2B - 1 inner steps i, slots v < B; block-oriented at Level
 *    3).  Step s = t (2B - 1) + i, slot k = u B + v.  Block pairs inside a super block
 *    are visited in every outer step (2Q - 1 times per sweep), the others once.
 *  OR_ORDER_HIER (2): every block pair exactly once per sweep, grouped by super pair:
 *    B - 1 intra steps (round-robin over the B blocks of each super block of the super
 *    pairs of outer step 0: slots v < B/2 pair inside the lower super block, the rest
 *    inside the upper one), then for every outer step t, B bipartite steps i pairing
 *    block v of the lower super block with block (v + i) mod B of the upper one.
 *    B must be even or 1.
 * LEVEL3 reduces to the Level-2 round-robin when nsup = 2 or nsup = nblk, HIER when nsup = nblk. */
static int order_args(int ord, int64_t nblk, int64_t nsup) {
  if (nblk < 2 || (nblk & 1)) return OR_E_ARG;
  if (ord == OR_ORDER_RR) return OR_OK;
  if (ord != OR_ORDER_LEVEL3 && ord != OR_ORDER_HIER) return OR_E_ARG;
  if (nsup < 2 || (nsup & 1) || nblk % nsup) return OR_E_ARG;
  int64_t B = nblk / nsup;
  if (ord == OR_ORDER_HIER && B != 1 && (B & 1)) return OR_E_ARG;
  return OR_OK;
}

int or_order_steps(int ord, int64_t nblk, int64_t nsup, int64_t *nsteps) {
  if (order_args(ord, nblk, nsup)) return OR_E_ARG;
  if (ord == OR_ORDER_RR) { *nsteps = nblk - 1; return OR_OK; }
  int64_t B = nblk / nsup;
  if (ord == OR_ORDER_LEVEL3) *nsteps = (nsup - 1) * (2 * B - 1);
  else *nsteps = (B - 1) + (nsup - 1) * B;
  return OR_OK;
}

int or_order_pair(int ord, int64_t nblk, int64_t nsup, int64_t s, int64_t k, int64_t *p, int64_t *q) {
  int64_t nst;
  if (or_order_steps(ord, nblk, nsup, &nst) || s < 0 || s >= nst || k < 0 || k >= nblk / 2)
    return OR_E_ARG;
  if (ord == OR_ORDER_RR) return or_rr_pair(nblk, s, k, p, q);
  int64_t B = nblk / nsup, u = k / B, v = k % B, P, Q, a, b;
  if (ord == OR_ORDER_LEVEL3) {
    int64_t t = s / (2 * B - 1), i = s % (2 * B - 1);
    or_rr_pair(nsup, t, u, &P, &Q);         /* outer: super pair u of outer step t */
    or_rr_pair(2 * B, i, v, &a, &b);        /* inner: local block indices in [0, 2B) */
    *p = a < B ? P * B + a : Q * B + (a - B);
    *q = b < B ? P * B + b : Q * B + (b - B);
  } else if (s < B - 1) {                   /* HIER, intra steps (outer step 0's super pairs) */
    or_rr_pair(nsup, 0, u, &P, &Q);
    int64_t half = B / 2, base = v < half ? P * B : Q * B;
    or_rr_pair(B, s, v % half, &a, &b);
    *p = base + a;
    *q = base + b;
  } else {                                  /* HIER, bipartite steps */
    int64_t s2 = s - (B - 1), t = s2 / B, i = s2 % B;
    or_rr_pair(nsup, t, u, &P, &Q);
    *p = P * B + v;
    *q = Q * B + (v + i) % B;
  }
  if (*p > *q) { int64_t x = *p; *p = *q; *q = x; }
  return OR_OK;
}

/* ------------------------------------------------------- 2x2 transform */
/* PAPER.md:1365-1573.  Exactly the sequence of Sec. 6.1.1-6.1.7:
 *   prescale by D0 (Sec 6.1.1), test (6.12), x = |s_pq|, alpha_1 = arg s_pq
 *   (6.2-6.3), u + iv (6.5), t (6.7), sigma, gamma (6.6, 6.11), 2 theta (6.7),
 *   cos phi, cos psi, e^{i alpha} sin phi, e^{-i beta} sin psi (6.10),
 *   Z = (1/t)[[c_phi, eas], [-ebs, c_psi]] (6.9 times Phi_4), Z' = D0 Z. */
int or_hz2x2(double hpp, double hqq, orc hpq, double spp, double sqq, orc spq,
             double tol, int criterion, orc z[4], double *off) {
  if (!isfinite(hpp) || !isfinite(hqq) || !isfinite(hpq.re) || !isfinite(hpq.im) ||
      !isfinite(spp) || !isfinite(sqq) || !isfinite(spq.re) || !isfinite(spq.im))
    return OR_E_NONFINITE;
  if (!(spp > 0.0) || !(sqq > 0.0)) return OR_E_INDEF;            /* C-9 */
  /* Sec 6.1.1: D0 = diag(s_pp^{-1/2}, s_qq^{-1/2}) every step */
  double dp = 1.0 / sqrt(spp);
  double dq = 1.0 / sqrt(sqq);
  double Hpp = (hpp * dp) * dp;
  double Hqq = (hqq * dq) * dq;
  double dpq = dp * dq;
  orc Hpq = cmk(hpq.re * dpq, hpq.im * dpq);
  orc Spq = cmk(spq.re * dpq, spq.im * dpq);
  double ah = cabsv(Hpq);
  double x = cabsv(Spq);
  double aHpp = fabs(Hpp), aHqq = fabs(Hqq);
  if (off) {
    double den = sqrt(aHpp) * sqrt(aHqq);
    double oh = den > 0.0 ? ah / den : (ah > 0.0 ? INFINITY : 0.0);
    *off = oh > x ? oh : x;
  }
  /* eq (6.12), C-1 */
  int doit;
  if (criterion == OR_CRIT_LITERAL) {
    double mx = aHpp > aHqq ? aHpp : aHqq;
    double mn = aHpp > aHqq ? aHqq : aHpp;
    doit = (ah >= (mx * tol) * mn) || (x >= tol);
  } else {
    doit = (ah >= (tol * sqrt(aHpp)) * sqrt(aHqq)) || (x >= tol);
  }
  if (!doit) return OR_K_SKIP;
  /* Sec 6.1.6 case 1 */
  if (Hpq.re == 0.0 && Hpq.im == 0.0 && Spq.re == 0.0 && Spq.im == 0.0) return OR_K_IDENTITY;
  if (!(x < 1.0)) return OR_E_INDEF;                                 /* C-9 */
  /* alpha_1 = arg(s_pq); case 2 of 6.1.6: x = 0 -> alpha_1 = 0 */
  orc e1 = (x == 0.0) ? cmk(1.0, 0.0) : cmk(Spq.re / x, Spq.im / x);
  /* (6.5): u + iv = e^{-i alpha_1} h_pq */
  orc uv = cmul(cconj(e1), Hpq);
  double u = uv.re, v = uv.im;
  double t = sqrt((1.0 - x) * (1.0 + x));                            /* (6.7), C-12 */
  double h = Hqq - Hpp;
  orc Z11, Z12, Z21, Z22;
  int kind;
  if (h == 0.0 && v == 0.0) {
    /* Sec 6.1.6 case 3: Z = R1 D2 (C-5) */
    double ap = 1.0 / sqrt(2.0 * (1.0 + x));
    double aq = 1.0 / sqrt(2.0 * (1.0 - x));
    Z11 = cmk(ap, 0.0);
    Z12 = cscale(e1, -aq);
    Z21 = cscale(cconj(e1), ap);
    Z22 = cmk(aq, 0.0);
    kind = OR_K_BIG;
  } else {
    double sigma = (h >= 0.0) ? 1.0 : -1.0;                          /* C-4 */
    double v2 = 2.0 * v;
    double r = sqrt(h * h + v2 * v2);
    double cg = (sigma * h) / r;                                     /* (6.11) */
    double sg = (sigma * v2) / r;
    double N = sigma * (2.0 * u - (Hpp + Hqq) * x);                  /* (6.7) numerator */
    double D = t * r;                                                /* (6.7) denominator */
    double rho = sqrt(N * N + D * D);
    double c2 = D / rho;                                             /* C-13 */
    double s2 = N / rho;
    double tcc = (t * cg) * c2;
    double cphi = sqrt(0.5 * ((1.0 + x * s2) + tcc));                /* (6.10) */
    double cpsi = sqrt(0.5 * ((1.0 - x * s2) + tcc));
    double tsc = (t * sg) * c2;
    orc wa = cmul(e1, cmk(s2 - x, tsc));
    orc wb = cmul(cconj(e1), cmk(s2 + x, -tsc));
    double dpsi = 2.0 * cpsi, dphi = 2.0 * cphi;
    orc eas = cmk(wa.re / dpsi, wa.im / dpsi);
    orc ebs = cmk(wb.re / dphi, wb.im / dphi);
    Z11 = cmk(cphi / t, 0.0);                                        /* (6.9) */
    Z12 = cmk(eas.re / t, eas.im / t);
    Z21 = cmk(-(ebs.re / t), -(ebs.im / t));
    Z22 = cmk(cpsi / t, 0.0);
    kind = (cphi == 1.0 && cpsi == 1.0) ? OR_K_SMALL : OR_K_BIG;     /* C-2 */
  }
  /* Z' = D0 Z */
  z[0] = cscale(Z11, dp);
  z[1] = cscale(Z21, dq);
  z[2] = cscale(Z12, dp);
  z[3] = cscale(Z22, dq);
  for (int i = 0; i < 4; i++)
    if (!isfinite(z[i].re) || !isfinite(z[i].im)) return OR_E_NONFINITE;
  return kind;
}

/* [x_p x_q] <- [x_p x_q] Z'  (ZVROTM, Sec 6.2.1) */
static void rot_cols(int64_t len, orc *xp, orc *xq, const orc z[4]) {
  for (int64_t i = 0; i < len; i++) {
    orc a = xp[i], b = xq[i];
    xp[i] = cadd(cmul(a, z[0]), cmul(b, z[1]));
    xq[i] = cadd(cmul(a, z[2]), cmul(b, z[3]));
  }
}

/* Optional accumulation of Z'^{-1}: when Z' <- Z' E (E = Z'hat
 * at (p, q)), Z'^{-1} <- E^{-1} Z'^{-1}, i.e. rows p and q of W = Z'^{-1} are replaced
 * by Z'hat^{-1} [w_p; w_q], Z'hat^{-1} = (1/det) [[z22, -z12], [-z21, z11]]. */
static orc *g_winv = NULL;
static int64_t g_ldw = 0, g_nw = 0;

static void rot_rows_inv(orc *W, int64_t ldw, int64_t nw, int64_t p, int64_t q, const orc z[4]) {
  /* z = {z11, z21, z12, z22} */
  orc det = csub(cmul(z[0], z[3]), cmul(z[2], z[1]));
  orc a = cdiv(z[3], det), b = cdiv(cscale(z[2], -1.0), det);
  orc c = cdiv(cscale(z[1], -1.0), det), d = cdiv(z[0], det);
  for (int64_t j = 0; j < nw; j++) {
    orc wp = EL(W, ldw, p, j), wq = EL(W, ldw, q, j);
    EL(W, ldw, p, j) = cadd(cmul(a, wp), cmul(b, wq));
    EL(W, ldw, q, j) = cadd(cmul(c, wp), cmul(d, wq));
  }
}

/* One parallel step s of the ordering (Alg. 3 body): Grams (6.1) in one pass,
 * transform, updates of F, G (m rows) and Z (nz rows). */
static int hz_step(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                   orc *G, int64_t ldg, orc *Z, int64_t ldz, int64_t nz,
                   double tol, int criterion, int64_t s, int64_t *all, int64_t *big,
                   double *offmax) {
  int64_t np = n / 2;
  int64_t a_all = 0, a_big = 0;
  double omax = 0.0;
  int err = 0;
#pragma omp parallel for schedule(static) reduction(+ : a_all, a_big) reduction(max : omax)
  for (int64_t k = 0; k < np; k++) {
    int64_t p, q;
    or_rr_pair(n, s, k, &p, &q);
    orc *fp = &EL(F, ldf, 0, p), *fq = &EL(F, ldf, 0, q);
    orc *gp = &EL(G, ldg, 0, p), *gq = &EL(G, ldg, 0, q);
    double hpp = 0.0, hqq = 0.0, spp = 0.0, sqq = 0.0;
    orc hpq = cmk(0.0, 0.0), spq = cmk(0.0, 0.0);
    for (int64_t i = 0; i < m; i++) {                 /* eq (6.1) */
      double j = (double)J[i];
      hpp += j * cabs2(fp[i]);
      hqq += j * cabs2(fq[i]);
      orc d = cdotc1(fp[i], fq[i]);
      hpq = cadd(hpq, cmk(j * d.re, j * d.im));
      spp += cabs2(gp[i]);
      sqq += cabs2(gq[i]);
      spq = cadd(spq, cdotc1(gp[i], gq[i]));
    }
    orc z[4];
    double off = 0.0;
    int kind = or_hz2x2(hpp, hqq, hpq, spp, sqq, spq, tol, criterion, z, &off);
    if (off > omax) omax = off;
    if (kind < 0) {
#pragma omp critical
      { if (err == 0) err = kind; }
      continue;
    }
    if (kind == OR_K_SKIP || kind == OR_K_IDENTITY) continue;
    rot_cols(m, fp, fq, z);
    rot_cols(m, gp, gq, z);
    rot_cols(nz, &EL(Z, ldz, 0, p), &EL(Z, ldz, 0, q), z);
    if (g_winv && nz == g_nw) rot_rows_inv(g_winv, g_ldw, g_nw, p, q, z);
    a_all += 1;
    if (kind == OR_K_BIG) a_big += 1;
  }
  *all += a_all;
  *big += a_big;
  if (offmax && omax > *offmax) *offmax = omax;
  return err;
}

int or_hz_steps(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                orc *G, int64_t ldg, orc *Z, int64_t ldz, double eps,
                int criterion, int64_t s0, int64_t ns, int nthreads,
                int64_t *all, int64_t *big) {
  if (n < 2 || (n & 1) || m < 1 || s0 < 0 || s0 + ns > n - 1) return OR_E_ARG;
  set_threads(nthreads);
  double tol = eps * sqrt((double)n);
  for (int64_t s = s0; s < s0 + ns; s++) {
    int e = hz_step(m, n, F, ldf, J, G, ldg, Z, ldz, n, tol, criterion, s, all, big, NULL);
    if (e) return e;
  }
  return OR_OK;
}

/* Sweeps on an even-order problem, Z (nz x n) updated in place.
 * stop_on_all: inner FB level (C-3) stops on all == 0, outer on big == 0. */
static int hz_sweeps_even(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                          orc *G, int64_t ldg, orc *Z, int64_t ldz, int64_t nz,
                          double tol, int criterion, int cmax, int stop_on_all,
                          or_stats *st) {
  for (int sw = 0; sw < cmax; sw++) {
    int64_t all = 0, big = 0;
    double off = 0.0;
    for (int64_t s = 0; s < n - 1; s++) {
      int e = hz_step(m, n, F, ldf, J, G, ldg, Z, ldz, nz, tol, criterion, s, &all, &big, &off);
      if (e) return e;
    }
    if (sw < OR_MAX_SWEEPS) {
      st->all_per_sweep[sw] = all;
      st->big_per_sweep[sw] = big;
      st->max_off_per_sweep[sw] = off;
    }
    st->sweeps = sw + 1;
    st->pairs_visited += (n * (n - 1)) / 2;
    st->transforms_all += all;
    st->transforms_big += big;
    if ((stop_on_all ? all : big) == 0) {
      st->converged = 1;
      break;
    }
  }
  return OR_OK;
}

int or_hz_pointwise(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                    orc *G, int64_t ldg, orc *Z, int64_t ldz, double eps,
                    int criterion, int cmax, int nthreads, or_stats *st) {
  if (m < 1 || n < 1 || ldf < m || ldg < m || ldz < n || cmax < 1) return OR_E_ARG;
  set_threads(nthreads);
  memset(st, 0, sizeof(*st));
  for (int64_t j = 0; j < n; j++)                       /* Alg. 2: Z' = I */
    for (int64_t i = 0; i < n; i++) EL(Z, ldz, i, j) = cmk(i == j ? 1.0 : 0.0, 0.0);
  if ((n & 1) == 0)
    return hz_sweeps_even(m, n, F, ldf, J, G, ldg, Z, ldz, n, eps * sqrt((double)n),
                          criterion, cmax, 0, st);
  /* Sec 6.3.2 / C-10: border with one row and one column, new element 1 */
  int64_t m1 = m + 1, n1 = n + 1;
  orc *Fb = calloc((size_t)m1 * n1, sizeof(orc));
  orc *Gb = calloc((size_t)m1 * n1, sizeof(orc));
  orc *Zb = calloc((size_t)n1 * n1, sizeof(orc));
  int8_t *Jb = malloc((size_t)m1);
  if (!Fb || !Gb || !Zb || !Jb) { free(Fb); free(Gb); free(Zb); free(Jb); return OR_E_ARG; }
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < m; i++) {
      EL(Fb, m1, i, j) = EL(F, ldf, i, j);
      EL(Gb, m1, i, j) = EL(G, ldg, i, j);
    }
  EL(Fb, m1, m, n) = cmk(1.0, 0.0);
  EL(Gb, m1, m, n) = cmk(1.0, 0.0);
  memcpy(Jb, J, (size_t)m);
  Jb[m] = 1;
  for (int64_t i = 0; i < n1; i++) EL(Zb, n1, i, i) = cmk(1.0, 0.0);
  int e = hz_sweeps_even(m1, n1, Fb, m1, Jb, Gb, m1, Zb, n1, n1, eps * sqrt((double)n1),
                         criterion, cmax, 0, st);
  for (int64_t j = 0; j < n; j++) {
    for (int64_t i = 0; i < m; i++) {
      EL(F, ldf, i, j) = EL(Fb, m1, i, j);
      EL(G, ldg, i, j) = EL(Gb, m1, i, j);
    }
    for (int64_t i = 0; i < n; i++) EL(Z, ldz, i, j) = EL(Zb, n1, i, j);
  }
  free(Fb); free(Gb); free(Zb); free(Jb);
  return e;
}

/* Algorithm 2 also accumulating W = Z'^{-1} (n even; W initialised to I). */
int or_hz_pointwise_inv(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                        orc *G, int64_t ldg, orc *Z, int64_t ldz, orc *W, int64_t ldw,
                        double eps, int criterion, int cmax, int nthreads, or_stats *st) {
  if ((n & 1) || ldw < n) return OR_E_ARG;
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < n; i++) EL(W, ldw, i, j) = cmk(i == j ? 1.0 : 0.0, 0.0);
  g_winv = W;
  g_ldw = ldw;
  g_nw = n;
  int rc = or_hz_pointwise(m, n, F, ldf, J, G, ldg, Z, ldz, eps, criterion, cmax, nthreads, st);
  g_winv = NULL;
  return rc;
}

/* ------------------------------------------------------------- extract */
int or_extract(int64_t m, int64_t n, const orc *F, int64_t ldf, const int8_t *J,
               const orc *G, int64_t ldg, const orc *Zp, int64_t ldzp,
               double *lambda, double *sigma_f, double *sigma_g, orc *Z,
               int64_t ldz) {
  for (int64_t c = 0; c < n; c++) {
    double a = 0.0, b = 0.0;
    for (int64_t i = 0; i < m; i++) {
      a += (double)J[i] * cabs2(EL(F, ldf, i, c));
      b += cabs2(EL(G, ldg, i, c));
    }
    if (!(b > 0.0)) return OR_E_INDEF;
    double sfp = sqrt(fabs(a));                       /* Sigma'_F */
    double sgp = sqrt(b);                             /* Sigma'_G */
    double sig = sqrt(sfp * sfp + sgp * sgp);         /* Sigma    */
    lambda[c] = a / b;                                /* eq (3.2), C-16 */
    if (sigma_f) sigma_f[c] = sfp / sig;
    if (sigma_g) sigma_g[c] = sgp / sig;
    if (Z)
      for (int64_t i = 0; i < n; i++) EL(Z, ldz, i, c) = cscale(EL(Zp, ldzp, i, c), 1.0 / sig);
  }
  return OR_OK;
}

/* ------------------------------------------------------ 2x2 Hermitian eig */
/* Jacobi rotation R (unitary) with R^* [[a, b],[conj b, c]] R = diag(l1, l2). */
static void herm2_jacobi(double a, orc b, double c, orc R[4], double *l1, double *l2) {
  double ab = cabsv(b);
  if (ab == 0.0) {
    R[0] = cmk(1, 0); R[1] = cmk(0, 0); R[2] = cmk(0, 0); R[3] = cmk(1, 0);
    *l1 = a; *l2 = c;
    return;
  }
  orc e = cmk(b.re / ab, b.im / ab);                  /* e^{i beta} */
  double tau = (c - a) / (2.0 * ab);
  double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
  double cs = 1.0 / sqrt(1.0 + t * t), sn = t * cs;
  /* R = diag(1, e^{-i beta}) [[cs, sn], [-sn, cs]] ; column-major R[0]=R11,R[1]=R21,R[2]=R12,R[3]=R22 */
  orc em = cconj(e);
  R[0] = cmk(cs, 0.0);
  R[1] = cscale(em, -sn);
  R[2] = cmk(sn, 0.0);
  R[3] = cscale(em, cs);
  *l1 = a - t * ab;
  *l2 = c + t * ab;
}

/* ---------------------------------------------------------------- HEBPJ */
int or_hebpj(int64_t r, const orc *T, int64_t ldt, orc *M, int64_t ldm,
             int8_t *Jr, int64_t *npos) {
  if (r < 1) return OR_E_ARG;
  const double alpha = (1.0 + sqrt(17.0)) / 8.0;
  const double eps = ldexp(1.0, -53);
  orc *W = malloc(sizeof(orc) * (size_t)r * r);
  orc *L = calloc((size_t)r * r, sizeof(orc));
  int64_t *perm = malloc(sizeof(int64_t) * (size_t)r);
  int *bsz = calloc((size_t)r, sizeof(int));
  double *d1 = calloc((size_t)r, sizeof(double));
  orc *Rk = calloc((size_t)r * 4, sizeof(orc));
  orc *Mt = calloc((size_t)r * r, sizeof(orc));
  int8_t *Js = malloc((size_t)r);
  int rc = OR_OK;
  if (!W || !L || !perm || !bsz || !d1 || !Rk || !Mt || !Js) { rc = OR_E_ARG; goto done; }
  /* Hermitian working copy from the lower triangle */
  double tmax = 0.0;
  for (int64_t j = 0; j < r; j++)
    for (int64_t i = j; i < r; i++) {
      orc v = EL(T, ldt, i, j);
      if (i == j) v.im = 0.0;
      EL(W, r, i, j) = v;
      EL(W, r, j, i) = cconj(v);
      if (cabsv(v) > tmax) tmax = cabsv(v);
    }
  for (int64_t i = 0; i < r; i++) { perm[i] = i; EL(L, r, i, i) = cmk(1, 0); }
  double tolz = (double)r * eps * tmax;
  int64_t k = 0;
  while (k < r) {
    /* Bunch-Parlett complete pivoting (Sec 4.2) */
    double mu0 = 0.0, mu1 = -1.0;
    int64_t id = k, oi = -1, oj = -1;
    for (int64_t i = k; i < r; i++) {
      double a = fabs(EL(W, r, i, i).re);
      if (a > mu1) { mu1 = a; id = i; }
    }
    /* largest off-diagonal |w_ij| found through |w_ij|^2 (same entry; where two entries'
       magnitudes round to the same double the larger square wins), then mu0 = sqrt(max)
       = the largest magnitude itself (sqrt is monotone and correctly rounded) */
    double mu0sq = 0.0;
    for (int64_t j = k; j < r; j++)
      for (int64_t i = j + 1; i < r; i++) {
        double a = cabs2(EL(W, r, i, j));
        if (a > mu0sq) { mu0sq = a; oi = i; oj = j; }
      }
    mu0 = sqrt(mu0sq);
    double mall = mu0 > mu1 ? mu0 : mu1;
    if (!(mall > tolz)) { rc = OR_E_RANK; goto done; }
    int two = !(mu1 >= alpha * mu0);
    int64_t src[2] = {id, -1};
    if (two) { src[0] = oj; src[1] = oi; }
    for (int b = 0; b < (two ? 2 : 1); b++) {
      int64_t dst = k + b, s = src[b];
      if (b == 1 && s == k) s = src[0];               /* moved by the first swap */
      if (s != dst) {
        for (int64_t c = 0; c < r; c++) { orc t = EL(W, r, dst, c); EL(W, r, dst, c) = EL(W, r, s, c); EL(W, r, s, c) = t; }
        for (int64_t c = 0; c < r; c++) { orc t = EL(W, r, c, dst); EL(W, r, c, dst) = EL(W, r, c, s); EL(W, r, c, s) = t; }
        for (int64_t c = 0; c < k; c++) { orc t = EL(L, r, dst, c); EL(L, r, dst, c) = EL(L, r, s, c); EL(L, r, s, c) = t; }
        int64_t t = perm[dst]; perm[dst] = perm[s]; perm[s] = t;
      }
    }
    if (!two) {
      double d = EL(W, r, k, k).re;
      bsz[k] = 1; d1[k] = d;
      for (int64_t i = k + 1; i < r; i++) EL(L, r, i, k) = cscale(EL(W, r, i, k), 1.0 / d);
      for (int64_t j = k + 1; j < r; j++)
        for (int64_t i = k + 1; i < r; i++)
          EL(W, r, i, j) = csub(EL(W, r, i, j), cscale(cmul(EL(W, r, i, k), cconj(EL(W, r, j, k))), 1.0 / d));
      k += 1;
    } else {
      double a = EL(W, r, k, k).re, c = EL(W, r, k + 1, k + 1).re;
      orc b = EL(W, r, k, k + 1);
      /* E^{-1} = (1/det) [[c, -b],[-conj b, a]] */
      double det = a * c - cabs2(b);
      bsz[k] = 2; bsz[k + 1] = 0;
      for (int64_t i = k + 2; i < r; i++) {
        orc w0 = EL(W, r, i, k), w1 = EL(W, r, i, k + 1);
        /* row i of C E^{-1} */
        orc l0 = cscale(csub(cscale(w0, c), cmul(w1, cconj(b))), 1.0 / det);
        orc l1 = cscale(csub(cscale(w1, a), cmul(w0, b)), 1.0 / det);
        EL(L, r, i, k) = l0;
        EL(L, r, i, k + 1) = l1;
      }
      for (int64_t j = k + 2; j < r; j++)
        for (int64_t i = k + 2; i < r; i++) {
          /* W_ij -= L_i E L_j^* expressed as l_i0 conj(w_j0) + l_i1 conj(w_j1) */
          orc t = cadd(cmul(EL(L, r, i, k), cconj(EL(W, r, j, k))),
                       cmul(EL(L, r, i, k + 1), cconj(EL(W, r, j, k + 1))));
          EL(W, r, i, j) = csub(EL(W, r, i, j), t);
        }
      double l1, l2;
      herm2_jacobi(a, b, c, &Rk[4 * k], &l1, &l2);
      d1[k] = l1; d1[k + 1] = l2;
      k += 2;
    }
  }
  /* M = L^* ; rows transformed by the D blocks (Sec 4.2) */
  for (int64_t i = 0; i < r; i++)
    for (int64_t j = 0; j < r; j++) EL(Mt, r, i, j) = cconj(EL(L, r, j, i));
  for (int64_t kk = 0; kk < r; kk++) {
    if (bsz[kk] == 1) {
      double s = sqrt(fabs(d1[kk]));
      for (int64_t j = 0; j < r; j++) EL(Mt, r, kk, j) = cscale(EL(Mt, r, kk, j), s);
      Js[kk] = d1[kk] > 0.0 ? 1 : -1;
    } else if (bsz[kk] == 2) {
      orc *R = &Rk[4 * kk];
      double s0 = sqrt(fabs(d1[kk])), s1 = sqrt(fabs(d1[kk + 1]));
      for (int64_t j = 0; j < r; j++) {
        orc x0 = EL(Mt, r, kk, j), x1 = EL(Mt, r, kk + 1, j);
        /* rows <- diag(s) R^* rows ; R^* = [[conj R11, conj R21],[conj R12, conj R22]] */
        orc y0 = cadd(cmul(cconj(R[0]), x0), cmul(cconj(R[1]), x1));
        orc y1 = cadd(cmul(cconj(R[2]), x0), cmul(cconj(R[3]), x1));
        EL(Mt, r, kk, j) = cscale(y0, s0);
        EL(Mt, r, kk + 1, j) = cscale(y1, s1);
      }
      Js[kk] = d1[kk] > 0.0 ? 1 : -1;
      Js[kk + 1] = d1[kk + 1] > 0.0 ? 1 : -1;
    }
  }
  /* Mhat = M P: column perm[l] of Mhat is column l of M; then sort rows
   * + before - (inner permutation, Sec 4.3), stable. */
  int64_t row = 0, np = 0;
  for (int pass = 0; pass < 2; pass++)
    for (int64_t i = 0; i < r; i++) {
      if ((pass == 0) != (Js[i] > 0)) continue;
      for (int64_t l = 0; l < r; l++) EL(M, ldm, row, perm[l]) = EL(Mt, r, i, l);
      Jr[row] = Js[i];
      if (Js[i] > 0) np++;
      row++;
    }
  *npos = np;
done:
  free(W); free(L); free(perm); free(bsz); free(d1); free(Rk); free(Mt); free(Js);
  return rc;
}

/* -------------------------------------------------- pivoted Cholesky */
int or_pchol(int64_t r, const orc *S, int64_t lds, orc *Gh, int64_t ldg) {
  orc *W = malloc(sizeof(orc) * (size_t)r * r);
  orc *L = calloc((size_t)r * r, sizeof(orc));
  int64_t *perm = malloc(sizeof(int64_t) * (size_t)r);
  int rc = OR_OK;
  if (!W || !L || !perm) { rc = OR_E_ARG; goto done; }
  for (int64_t j = 0; j < r; j++)
    for (int64_t i = j; i < r; i++) {
      orc v = EL(S, lds, i, j);
      if (i == j) v.im = 0.0;
      EL(W, r, i, j) = v;
      EL(W, r, j, i) = cconj(v);
    }
  for (int64_t i = 0; i < r; i++) perm[i] = i;
  for (int64_t k = 0; k < r; k++) {
    int64_t pv = k;
    for (int64_t i = k + 1; i < r; i++)
      if (EL(W, r, i, i).re > EL(W, r, pv, pv).re) pv = i;
    if (!(EL(W, r, pv, pv).re > 0.0)) { rc = OR_E_INDEF; goto done; }
    if (pv != k) {
      for (int64_t c = 0; c < r; c++) { orc t = EL(W, r, k, c); EL(W, r, k, c) = EL(W, r, pv, c); EL(W, r, pv, c) = t; }
      for (int64_t c = 0; c < r; c++) { orc t = EL(W, r, c, k); EL(W, r, c, k) = EL(W, r, c, pv); EL(W, r, c, pv) = t; }
      for (int64_t c = 0; c < k; c++) { orc t = EL(L, r, k, c); EL(L, r, k, c) = EL(L, r, pv, c); EL(L, r, pv, c) = t; }
      int64_t t = perm[k]; perm[k] = perm[pv]; perm[pv] = t;
    }
    double lkk = sqrt(EL(W, r, k, k).re);
    EL(L, r, k, k) = cmk(lkk, 0.0);
    for (int64_t i = k + 1; i < r; i++) EL(L, r, i, k) = cscale(EL(W, r, i, k), 1.0 / lkk);
    for (int64_t j = k + 1; j < r; j++)
      for (int64_t i = k + 1; i < r; i++)
        EL(W, r, i, j) = csub(EL(W, r, i, j), cmul(EL(L, r, i, k), cconj(EL(L, r, j, k))));
  }
  /* Gh = L^* P */
  for (int64_t i = 0; i < r; i++)
    for (int64_t l = 0; l < r; l++) EL(Gh, ldg, i, perm[l]) = cconj(EL(L, r, l, i));
done:
  free(W); free(L); free(perm);
  return rc;
}

/* ------------------------------------------------------------- blocked */
/* Sec 6.4.1: nblk block columns, widths w or w-1, non-increasing. */
static void block_part(int64_t n, int64_t nblk, int64_t *start, int64_t *width) {
  int64_t w = (n + nblk - 1) / nblk;
  int64_t nbig = n - nblk * (w - 1);
  int64_t c = 0;
  for (int64_t b = 0; b < nblk; b++) {
    width[b] = b < nbig ? w : w - 1;
    start[b] = c;
    c += width[b];
  }
}

/* One block pivot (Sec 6.4.2-6.4.3) for block columns bp < bq. */
static int block_pivot(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                       orc *G, int64_t ldg, orc *Z, int64_t ldz,
                       int64_t p0, int64_t wp, int64_t q0, int64_t wq,
                       int inner_sweeps, double eps, int criterion,
                       int64_t *all, int64_t *big) {
  int64_t k = wp + wq;
  int64_t kb = k + (k & 1);                  /* bordered order (Sec 6.3.2) */
  int64_t *cols = malloc(sizeof(int64_t) * (size_t)k);
  orc *Hh = calloc((size_t)k * k, sizeof(orc));
  orc *Sh = calloc((size_t)k * k, sizeof(orc));
  orc *Fh = calloc((size_t)kb * kb, sizeof(orc));
  orc *Gh = calloc((size_t)kb * kb, sizeof(orc));
  orc *Zh = calloc((size_t)kb * kb, sizeof(orc));
  orc *tmp = malloc(sizeof(orc) * (size_t)(m > n ? m : n) * k);
  int8_t *Jh = malloc((size_t)kb);
  int rc = OR_OK;
  if (!cols || !Hh || !Sh || !Fh || !Gh || !Zh || !tmp || !Jh) { rc = OR_E_ARG; goto done; }
  for (int64_t c = 0; c < wp; c++) cols[c] = p0 + c;
  for (int64_t c = 0; c < wq; c++) cols[wp + c] = q0 + c;
  /* H_blk = F_pair^* J F_pair, S_blk = G_pair^* G_pair (ZGEMM / ZHERK) */
  for (int64_t b = 0; b < k; b++)
    for (int64_t a = b; a < k; a++) {
      orc h = cmk(0, 0), s = cmk(0, 0);
      const orc *fa = &EL(F, ldf, 0, cols[a]), *fb = &EL(F, ldf, 0, cols[b]);
      const orc *ga = &EL(G, ldg, 0, cols[a]), *gb = &EL(G, ldg, 0, cols[b]);
      for (int64_t i = 0; i < m; i++) {
        orc d = cdotc1(fa[i], fb[i]);
        h = cadd(h, cscale(d, (double)J[i]));
        s = cadd(s, cdotc1(ga[i], gb[i]));
      }
      EL(Hh, k, a, b) = h;                   /* lower triangle: conj(f_a)^T f_b at (a,b) */
      EL(Sh, k, a, b) = s;
    }
  /* the (a,b) entry of F^*JF is f_a^* J f_b; we filled (a,b) for a >= b with
   * f_a^* J f_b, which is the lower triangle entry. */
  int64_t npos;
  rc = or_hebpj(k, Hh, k, Fh, kb, Jh, &npos);
  if (rc) goto done;
  rc = or_pchol(k, Sh, k, Gh, kb);
  if (rc) goto done;
  if (kb != k) { EL(Fh, kb, k, k) = cmk(1, 0); EL(Gh, kb, k, k) = cmk(1, 0); Jh[k] = 1; }
  for (int64_t i = 0; i < kb; i++) EL(Zh, kb, i, i) = cmk(1, 0);
  /* inner Level-1 sweeps on the block pivot, n in eps*sqrt(n) is kb (C-7) */
  or_stats ist;
  memset(&ist, 0, sizeof(ist));
  rc = hz_sweeps_even(kb, kb, Fh, kb, Jh, Gh, kb, Zh, kb, kb, eps * sqrt((double)kb),
                      criterion, inner_sweeps, inner_sweeps > 1, &ist);
  if (rc) goto done;
  *all += ist.transforms_all;
  *big += ist.transforms_big;
  if (ist.transforms_all == 0) goto done;    /* Sec 6.4.3: nothing applied */
  /* X_pair <- X_pair Z_blk for X in F, G (m rows) and Z (n rows) */
  orc *mats[3] = {F, G, Z};
  int64_t lds[3] = {ldf, ldg, ldz};
  int64_t rows[3] = {m, m, n};
  for (int t = 0; t < 3; t++) {
    orc *X = mats[t];
    int64_t ld = lds[t], R = rows[t];
    for (int64_t c = 0; c < k; c++)
      for (int64_t i = 0; i < R; i++) {
        orc acc = cmk(0, 0);
        for (int64_t l = 0; l < k; l++) acc = cadd(acc, cmul(EL(X, ld, i, cols[l]), EL(Zh, kb, l, c)));
        tmp[i + c * R] = acc;
      }
    for (int64_t c = 0; c < k; c++)
      for (int64_t i = 0; i < R; i++) EL(X, ld, i, cols[c]) = tmp[i + c * R];
  }
done:
  free(cols); free(Hh); free(Sh); free(Fh); free(Gh); free(Zh); free(tmp); free(Jh);
  return rc;
}

int or_block_partition(int64_t n, int64_t nblk, int64_t *start, int64_t *width) {
  if (nblk < 1 || nblk > n) return OR_E_ARG;
  block_part(n, nblk, start, width);
  return OR_OK;
}

int or_block_pair(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                  orc *G, int64_t ldg, orc *Z, int64_t ldz, int64_t p0, int64_t wp,
                  int64_t q0, int64_t wq, int inner_sweeps, double eps, int criterion,
                  int64_t *all, int64_t *big) {
  return block_pivot(m, n, F, ldf, J, G, ldg, Z, ldz, p0, wp, q0, wq, inner_sweeps, eps,
                     criterion, all, big);
}

int or_hz_blocked(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                  orc *G, int64_t ldg, orc *Z, int64_t ldz, int64_t nblk,
                  int inner_sweeps, double eps, int criterion, int cmax,
                  int nthreads, or_stats *st) {
  return or_hz_blocked_ord(m, n, F, ldf, J, G, ldg, Z, ldz, nblk, OR_ORDER_RR, 0, inner_sweeps,
                           eps, criterion, cmax, nthreads, st);
}

int or_hz_blocked_ord(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                      orc *G, int64_t ldg, orc *Z, int64_t ldz, int64_t nblk, int ord,
                      int64_t nsup, int inner_sweeps, double eps, int criterion, int cmax,
                      int nthreads, or_stats *st) {
  int64_t nst;
  if (m < 1 || n < 2 || nblk < 2 || (nblk & 1) || nblk > n || cmax < 1 || inner_sweeps < 1 ||
      or_order_steps(ord, nblk, nsup, &nst))
    return OR_E_ARG;
  set_threads(nthreads);
  memset(st, 0, sizeof(*st));
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < n; i++) EL(Z, ldz, i, j) = cmk(i == j ? 1.0 : 0.0, 0.0);
  int64_t *bs = malloc(sizeof(int64_t) * (size_t)nblk), *bw = malloc(sizeof(int64_t) * (size_t)nblk);
  if (!bs || !bw) { free(bs); free(bw); return OR_E_ARG; }
  block_part(n, nblk, bs, bw);
  int rc = OR_OK;
  for (int sw = 0; sw < cmax && rc == 0; sw++) {
    int64_t all = 0, big = 0;
    for (int64_t s = 0; s < nst && rc == 0; s++) {
      int err = 0;
      int64_t a_all = 0, a_big = 0;
#pragma omp parallel for schedule(static) reduction(+ : a_all, a_big)
      for (int64_t kk = 0; kk < nblk / 2; kk++) {
        int64_t bp, bq;
        or_order_pair(ord, nblk, nsup, s, kk, &bp, &bq);
        int64_t la = 0, lb = 0;
        int e = block_pivot(m, n, F, ldf, J, G, ldg, Z, ldz, bs[bp], bw[bp], bs[bq], bw[bq],
                            inner_sweeps, eps, criterion, &la, &lb);
        if (e) {
#pragma omp critical
          { if (err == 0) err = e; }
        }
        a_all += la;
        a_big += lb;
      }
      all += a_all;
      big += a_big;
      rc = err;
    }
    if (rc) break;
    if (sw < OR_MAX_SWEEPS) { st->all_per_sweep[sw] = all; st->big_per_sweep[sw] = big; }
    st->sweeps = sw + 1;
    st->pairs_visited += (n * (n - 1)) / 2;
    st->transforms_all += all;
    st->transforms_big += big;
    if (big == 0) { st->converged = 1; break; }
  }
  free(bs); free(bw);
  return rc;
}

/* ------------------------------------------------------------- phase 1 */
int or_factor(int64_t NA, int64_t NL, int64_t NG, const orc *A, const orc *B,
              const double *U, const orc *TAA, const orc *TAB, const orc *TBB,
              orc *F, int8_t *J, orc *G) {
  int64_t r = 2 * NL, m = 2 * NA * NL;
  int rc = OR_OK;
#pragma omp parallel for schedule(dynamic)
  for (int64_t a = 0; a < NA; a++) {
    orc *T = calloc((size_t)r * r, sizeof(orc));
    orc *M = calloc((size_t)r * r, sizeof(orc));
    int8_t *Ja = malloc((size_t)r);
    const orc *Aa = A + (size_t)a * NL * NG, *Ba = B + (size_t)a * NL * NG;
    const orc *taa = TAA + (size_t)a * NL * NL, *tab = TAB + (size_t)a * NL * NL,
              *tbb = TBB + (size_t)a * NL * NL;
    /* eq (3.3): T_a = [[T_AA, T_AB], [T_AB^*, T_BB]] (lower triangle is read) */
    for (int64_t j = 0; j < NL; j++)
      for (int64_t i = 0; i < NL; i++) {
        EL(T, r, i, j) = EL(taa, NL, i, j);
        EL(T, r, NL + i, NL + j) = EL(tbb, NL, i, j);
        EL(T, r, i, NL + j) = EL(tab, NL, i, j);
        EL(T, r, NL + j, i) = cconj(EL(tab, NL, i, j));
      }
    int64_t np;
    int e = or_hebpj(r, T, r, M, r, Ja, &np);
    if (e) {
#pragma omp critical
      { if (rc == 0) rc = e; }
    } else {
      int64_t r0 = a * r;
      /* F_a = Mtilde_a [A_a; B_a] (ZGEMM) */
      for (int64_t c = 0; c < NG; c++)
        for (int64_t i = 0; i < r; i++) {
          orc acc = cmk(0, 0);
          for (int64_t l = 0; l < NL; l++) acc = cadd(acc, cmul(EL(M, r, i, l), EL(Aa, NL, l, c)));
          for (int64_t l = 0; l < NL; l++) acc = cadd(acc, cmul(EL(M, r, i, NL + l), EL(Ba, NL, l, c)));
          EL(F, m, r0 + i, c) = acc;
        }
      /* G_a = [A_a; U_a B_a] (ZDSCAL rows) */
      for (int64_t c = 0; c < NG; c++)
        for (int64_t l = 0; l < NL; l++) {
          EL(G, m, r0 + l, c) = EL(Aa, NL, l, c);
          EL(G, m, r0 + NL + l, c) = cscale(EL(Ba, NL, l, c), U[a * NL + l]);
        }
      for (int64_t i = 0; i < r; i++) J[r0 + i] = Ja[i];
    }
    free(T); free(M); free(Ja);
  }
  return rc;
}

/* ------------------------------------------------------------- phase 2 */
static orc jdot_rows(int64_t r0, int64_t m, const orc *x, const orc *y, const int8_t *J) {
  orc s = cmk(0, 0);
  for (int64_t i = r0; i < m; i++) s = cadd(s, cscale(cdotc1(x[i], y[i]), (double)J[i]));
  return s;
}

static void swap_cols(int64_t m, orc *W, int64_t ld, int64_t a, int64_t b, int64_t *perm) {
  if (a == b) return;
  for (int64_t i = 0; i < m; i++) { orc t = EL(W, ld, i, a); EL(W, ld, i, a) = EL(W, ld, i, b); EL(W, ld, i, b) = t; }
  int64_t t = perm[a]; perm[a] = perm[b]; perm[b] = t;
}

static void swap_rows(int64_t n, orc *W, int64_t ld, int8_t *J, int64_t a, int64_t b) {
  if (a == b) return;
  for (int64_t c = 0; c < n; c++) { orc t = EL(W, ld, a, c); EL(W, ld, a, c) = EL(W, ld, b, c); EL(W, ld, b, c) = t; }
  int8_t t = J[a]; J[a] = J[b]; J[b] = t;
}

/* Hyperbolic Householder step on column k over active rows k..m-1 (Thm 5.1,
 * PAPER.md:1069-1183): row swap for sign compatibility, s = f + c1 e1,
 * tau = -1/(f^*Jf + |f^*Jf|^{1/2} |f_11| j_11), H(s) = I + tau s s^* J
 * applied to columns k+1..n-1; column k becomes -c1 e_k. */
static int jreflect(int64_t m, int64_t n, orc *W, int64_t ld, int8_t *J, int64_t k) {
  orc *f = &EL(W, ld, 0, k);
  double hn = jdot_rows(k, m, f, f, J).re;
  if (hn == 0.0 || !isfinite(hn)) return OR_E_RANK;
  int8_t sg = hn > 0.0 ? 1 : -1;
  if (J[k] != sg) {
    int64_t best = -1;
    double bv = -1.0;
    for (int64_t i = k; i < m; i++)
      if (J[i] == sg && cabsv(f[i]) > bv) { bv = cabsv(f[i]); best = i; }
    if (best < 0) return OR_E_RANK;
    swap_rows(n, W, ld, J, k, best);
  }
  double rr = sqrt(fabs(hn));
  double a11 = cabsv(f[k]);
  orc ed = a11 > 0.0 ? cmk(f[k].re / a11, f[k].im / a11) : cmk(1, 0);
  orc c1 = cscale(ed, rr);
  double tau = -1.0 / (hn + rr * a11 * (double)J[k]);
  orc *s = malloc(sizeof(orc) * (size_t)m);
  if (!s) return OR_E_ARG;
  for (int64_t i = k; i < m; i++) s[i] = f[i];
  s[k] = cadd(s[k], c1);
#pragma omp parallel for schedule(static)
  for (int64_t j = k + 1; j < n; j++) {
    orc *x = &EL(W, ld, 0, j);
    orc d = jdot_rows(k, m, s, x, J);            /* s^* J x */
    orc c = cscale(d, tau);
    for (int64_t i = k; i < m; i++) x[i] = cadd(x[i], cmul(s[i], c));
  }
  f[k] = cscale(c1, -1.0);
  for (int64_t i = k + 1; i < m; i++) f[i] = cmk(0, 0);
  free(s);
  return OR_OK;
}

int or_reduce(int64_t m, int64_t n, const orc *F, int64_t ldf, const int8_t *J,
              const orc *G, int64_t ldg, orc *Fs, int8_t *Js, orc *Gs,
              int64_t *p2, int64_t *n2x2) {
  if (m < n || n < 1) return OR_E_ARG;
  const double alpha = (1.0 + sqrt(17.0)) / 8.0;
  orc *W = malloc(sizeof(orc) * (size_t)m * n);
  int8_t *Jw = malloc((size_t)m);
  double *hd = malloc(sizeof(double) * (size_t)n);
  int rc = OR_OK;
  if (!W || !Jw || !hd) { rc = OR_E_ARG; goto done; }
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < m; i++) EL(W, m, i, j) = EL(F, ldf, i, j);
  memcpy(Jw, J, (size_t)m);
  for (int64_t j = 0; j < n; j++) p2[j] = j;
  *n2x2 = 0;
  int64_t k = 0;
  while (k < n) {
    /* Sec 5.2.1: J_k-norms of the trailing columns, largest magnitude first */
    int64_t jm = k;
    for (int64_t j = k; j < n; j++) {
      hd[j] = jdot_rows(k, m, &EL(W, m, 0, j), &EL(W, m, 0, j), Jw).re;
      if (fabs(hd[j]) > fabs(hd[jm])) jm = j;
    }
    swap_cols(m, W, m, k, jm, p2);
    { double t = hd[k]; hd[k] = hd[jm]; hd[jm] = t; }
    int two = 0;
    if (k < n - 1) {
      /* |h_1i| maximal over i > 1 */
      int64_t ii = k + 1;
      double h1i = -1.0;
      for (int64_t j = k + 1; j < n; j++) {
        double a = cabsv(jdot_rows(k, m, &EL(W, m, 0, k), &EL(W, m, 0, j), Jw));
        if (a > h1i) { h1i = a; ii = j; }
      }
      double h11 = fabs(hd[k]);
      if (!(h11 >= alpha * h1i)) {
        /* |h_ij| maximal over j != i */
        double hij = -1.0;
        for (int64_t l = k; l < n; l++) {
          if (l == ii) continue;
          double a = cabsv(jdot_rows(k, m, &EL(W, m, 0, ii), &EL(W, m, 0, l), Jw));
          if (a > hij) hij = a;
        }
        if (h11 * hij >= alpha * h1i * h1i) {
          two = 0;
        } else if (fabs(hd[ii]) >= alpha * hij) {
          swap_cols(m, W, m, k, ii, p2);
          two = 0;
        } else {
          swap_cols(m, W, m, k + 1, ii, p2);
          two = 1;
        }
      }
    }
    if (!two) {
      rc = jreflect(m, n, W, m, Jw, k);
      if (rc) goto done;
      k += 1;
    } else {
      /* (J,I) URV 2x2 pivot */
      orc *f1 = &EL(W, m, 0, k), *f2 = &EL(W, m, 0, k + 1);
      double a = jdot_rows(k, m, f1, f1, Jw).re, c = jdot_rows(k, m, f2, f2, Jw).re;
      orc b = jdot_rows(k, m, f1, f2, Jw);
      orc R[4];
      double l1, l2;
      herm2_jacobi(a, b, c, R, &l1, &l2);
      if (l1 == 0.0 || l2 == 0.0) { rc = OR_E_RANK; goto done; }
      for (int64_t i = k; i < m; i++) {           /* [f1 f2] <- [f1 f2] R on active rows */
        orc x0 = f1[i], x1 = f2[i];
        f1[i] = cadd(cmul(x0, R[0]), cmul(x1, R[1]));
        f2[i] = cadd(cmul(x0, R[2]), cmul(x1, R[3]));
      }
      rc = jreflect(m, n, W, m, Jw, k);
      if (rc) goto done;
      rc = jreflect(m, n, W, m, Jw, k + 1);
      if (rc) goto done;
      for (int64_t i = k; i < k + 2; i++) {       /* multiply back by R^* */
        orc x0 = f1[i], x1 = f2[i];
        f1[i] = cadd(cmul(x0, cconj(R[0])), cmul(x1, cconj(R[2])));
        f2[i] = cadd(cmul(x0, cconj(R[1])), cmul(x1, cconj(R[3])));
      }
      *n2x2 += 1;
      k += 2;
    }
  }
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < n; i++) EL(Fs, n, i, j) = EL(W, m, i, j);
  memcpy(Js, Jw, (size_t)n);
  /* Sec 5.4.1 prepermute G by P2, then QR of G P2 keeping R (Sec 5) */
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < m; i++) EL(W, m, i, j) = EL(G, ldg, i, p2[j]);
  for (int64_t kk = 0; kk < n; kk++) {
    orc *x = &EL(W, m, 0, kk);
    double nrm = 0.0;
    for (int64_t i = kk; i < m; i++) nrm += cabs2(x[i]);
    nrm = sqrt(nrm);
    if (nrm == 0.0) { rc = OR_E_RANK; goto done; }
    double ax = cabsv(x[kk]);
    orc ph = ax > 0.0 ? cmk(x[kk].re / ax, x[kk].im / ax) : cmk(1, 0);
    orc alph = cscale(ph, -nrm);                  /* x -> alph e1 */
    /* v = x - alph e1 ; H = I - 2 v v^* / (v^* v) */
    orc *v = malloc(sizeof(orc) * (size_t)m);
    if (!v) { rc = OR_E_ARG; goto done; }
    double vv = 0.0;
    for (int64_t i = kk; i < m; i++) v[i] = x[i];
    v[kk] = csub(v[kk], alph);
    for (int64_t i = kk; i < m; i++) vv += cabs2(v[i]);
#pragma omp parallel for schedule(static)
    for (int64_t j = kk + 1; j < n; j++) {
      orc *y = &EL(W, m, 0, j);
      orc d = cmk(0, 0);
      for (int64_t i = kk; i < m; i++) d = cadd(d, cdotc1(v[i], y[i]));
      orc c = cscale(d, -2.0 / vv);
      for (int64_t i = kk; i < m; i++) y[i] = cadd(y[i], cmul(v[i], c));
    }
    x[kk] = alph;
    for (int64_t i = kk + 1; i < m; i++) x[i] = cmk(0, 0);
    free(v);
  }
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < n; i++) EL(Gs, n, i, j) = i <= j ? EL(W, m, i, j) : cmk(0, 0);
  /* normalise R's diagonal to real >= 0: R <- diag(conj(phase)) R */
  for (int64_t i = 0; i < n; i++) {
    orc d = EL(Gs, n, i, i);
    double ad = cabsv(d);
    orc ph = ad > 0.0 ? cmk(d.re / ad, d.im / ad) : cmk(1, 0);
    for (int64_t j = i; j < n; j++) EL(Gs, n, i, j) = cmul(cconj(ph), EL(Gs, n, i, j));
    EL(Gs, n, i, i).im = 0.0;
  }
done:
  free(W); free(Jw); free(hd);
  (void)cdiv;
  return rc;
}
