/* c_demo.c -- libghsvd from plain C (no Python, no torch): the C ABI of include/ghsvd.h is
 * the product boundary.  Solves a random complex J-GHSVD problem (F, G: m x n, J with
 * about 40 % negative signs) with the pointwise and the blocked BO sweep and checks every
 * eigenpair's residual
 *     || F^* J F z - lambda G^* G z || / ((||F||_F^2 + ||G||_F^2) ||z||)  <=  1e-12 n
 * (the north star's bound), computed here in plain C from the inputs.  Inputs and
 * outputs are HOST buffers (the library copies with cudaMemcpyDefault); the workspace is
 * the caller's cudaMalloc.  Exit status 0 = all checks passed.
 *
 *   gcc -std=c99 -O2 examples/c_demo.c -Iinclude -Lpaper_1907_08560_b200 -lghsvd \
 *       -L/usr/local/cuda/lib64 -lcudart -lm -o examples/c_demo            (see build.py)
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ghsvd.h"

typedef struct { double re, im; } cplx;

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static double urand(void) { /* xorshift64*, uniform in (0, 1) */
  rng_state ^= rng_state >> 12;
  rng_state ^= rng_state << 25;
  rng_state ^= rng_state >> 27;
  return ((rng_state * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0) + 1e-300;
}
static double nrand(void) { return sqrt(-2.0 * log(urand())) * cos(6.283185307179586 * urand()); }

/* y = A x  (A: rows x cols, column-major, ld = rows) */
static void matvec(const cplx* A, int64_t rows, int64_t cols, const cplx* x, cplx* y) {
  for (int64_t i = 0; i < rows; i++) y[i].re = y[i].im = 0.0;
  for (int64_t j = 0; j < cols; j++)
    for (int64_t i = 0; i < rows; i++) {
      const cplx a = A[i + j * rows];
      y[i].re += a.re * x[j].re - a.im * x[j].im;
      y[i].im += a.re * x[j].im + a.im * x[j].re;
    }
}
/* y = A^* (s .* x)  (s = J signs or NULL) */
static void matvec_h(const cplx* A, int64_t rows, int64_t cols, const int8_t* s, const cplx* x, cplx* y) {
  for (int64_t j = 0; j < cols; j++) {
    double re = 0.0, im = 0.0;
    for (int64_t i = 0; i < rows; i++) {
      const cplx a = A[i + j * rows];
      const double sg = s ? (double)s[i] : 1.0;
      re += sg * (a.re * x[i].re + a.im * x[i].im);
      im += sg * (a.re * x[i].im - a.im * x[i].re);
    }
    y[j].re = re;
    y[j].im = im;
  }
}

static int solve_and_check(int variant, const char* name, int64_t m, int64_t n, const cplx* F, const int8_t* J,
                           const cplx* G) {
  ghsvd_options o;
  ghsvd_default_options(&o);
  o.variant = variant;
  o.max_sweeps = 60;
  const size_t bytes = ghsvd_workspace_bytes(&o, m, n, 0);
  void* ws = NULL;
  if (bytes == 0 || cudaMalloc(&ws, bytes) != cudaSuccess) {
    fprintf(stderr, "%s: workspace (%zu bytes) not available\n", name, bytes);
    return 1;
  }
  ghsvd_ctx ctx = NULL;
  ghsvd_status st = ghsvd_create(&o, m, n, 0, ws, bytes, &ctx);
  if (st != GHSVD_OK) {
    fprintf(stderr, "%s: ghsvd_create -> %d\n", name, (int)st);
    cudaFree(ws);
    return 1;
  }
  ghsvd_stats stats;
  double* lam = (double*)malloc((size_t)n * sizeof(double));
  cplx* Z = (cplx*)malloc((size_t)n * n * sizeof(cplx));
  int rc = 1;
  if ((st = ghsvd_set_factors(ctx, m, n, F, m, J, G, m)) != GHSVD_OK ||
      (st = ghsvd_sweep(ctx, &stats)) != GHSVD_OK ||
      (st = ghsvd_extract(ctx, lam, NULL, NULL, Z, n, NULL)) != GHSVD_OK) {
    fprintf(stderr, "%s: status %d: %s\n", name, (int)st, ghsvd_last_error(ctx));
  } else {
    double nf2 = 0.0;
    for (int64_t e = 0; e < m * n; e++)
      nf2 += F[e].re * F[e].re + F[e].im * F[e].im + G[e].re * G[e].re + G[e].im * G[e].im;
    cplx* t = (cplx*)malloc((size_t)m * sizeof(cplx));
    cplx* hx = (cplx*)malloc((size_t)n * sizeof(cplx));
    cplx* sx = (cplx*)malloc((size_t)n * sizeof(cplx));
    double worst = 0.0;
    for (int64_t c = 0; c < n; c++) {
      const cplx* z = Z + c * n;
      double nz = 0.0;
      for (int64_t i = 0; i < n; i++) nz += z[i].re * z[i].re + z[i].im * z[i].im;
      matvec(F, m, n, z, t);
      matvec_h(F, m, n, J, t, hx);
      matvec(G, m, n, z, t);
      matvec_h(G, m, n, NULL, t, sx);
      double r = 0.0;
      for (int64_t i = 0; i < n; i++) {
        const double dr = hx[i].re - lam[c] * sx[i].re, di = hx[i].im - lam[c] * sx[i].im;
        r += dr * dr + di * di;
      }
      const double rel = sqrt(r) / (nf2 * sqrt(nz));
      if (!(rel <= worst)) worst = rel;   /* NaN propagates */
    }
    free(t);
    free(hx);
    free(sx);
    const int ok = stats.converged && worst <= 1e-12 * (double)n;
    printf("c_demo %s: m=%lld n=%lld sweeps=%d converged=%d max residual=%.3e (bound %.1e) %s\n", name,
           (long long)m, (long long)n, stats.sweeps, stats.converged, worst, 1e-12 * (double)n,
           ok ? "OK" : "FAIL");
    rc = ok ? 0 : 1;
  }
  free(lam);
  free(Z);
  ghsvd_destroy(ctx);
  cudaFree(ws);
  return rc;
}

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 320;
  const int64_t n = argc > 2 ? atoll(argv[2]) : 192;
  cplx* F = (cplx*)malloc((size_t)m * n * sizeof(cplx));
  cplx* G = (cplx*)malloc((size_t)m * n * sizeof(cplx));
  int8_t* J = (int8_t*)malloc((size_t)m);
  for (int64_t e = 0; e < m * n; e++) {
    F[e].re = nrand() * 0.7071067811865476;
    F[e].im = nrand() * 0.7071067811865476;
    G[e].re = nrand() * 0.7071067811865476;
    G[e].im = nrand() * 0.7071067811865476;
  }
  for (int64_t i = 0; i < m; i++) J[i] = urand() < 0.4 ? -1 : 1;
  int rc = solve_and_check(GHSVD_POINTWISE, "pointwise", m, n, F, J, G);
  rc |= solve_and_check(GHSVD_BLOCKED_BO, "blocked-BO", m, n, F, J, G);
  free(F);
  free(G);
  free(J);
  return rc;
}
