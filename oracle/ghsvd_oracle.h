/*
 * ghsvd_oracle.h -- plain, slow, CPU reference ("oracle") for the implicit
 * Hari-Zimmermann J-GHSVD of Novakovic et al., arXiv:1907.08560.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_1907_08560_b200/csrc, include/ghsvd.h), and neither includes the other.
 *
 * All matrices are column-major complex128 stored as interleaved (re, im)
 * doubles; `ld` is the column stride in complex elements.  Signs J are int8 +-1.
 * Every routine returns 0 on success or a negative error code (see OR_E_*).
 */
#ifndef GHSVD_ORACLE_H
#define GHSVD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } orc;

#define OR_OK 0
#define OR_E_ARG (-1)
#define OR_E_INDEF (-6)   /* s_pp <= 0 or x >= 1: S not (numerically) definite */
#define OR_E_RANK (-7)    /* rank-deficient block pivot / T block */
#define OR_E_NONFINITE (-8)

/* kinds returned by or_hz2x2 (>= 0) */
#define OR_K_SKIP 0       /* criterion (6.12) false: nothing applied */
#define OR_K_IDENTITY 1   /* h_pq = s_pq = 0 (Sec. 6.1.6 case 1): nothing applied, not counted */
#define OR_K_SMALL 2      /* cos(phi) = cos(psi) = 1 (Sec. 6.1.7) */
#define OR_K_BIG 3

#define OR_CRIT_RELATIVE 0
#define OR_CRIT_LITERAL 1

#define OR_MAX_SWEEPS 64

typedef struct {
  int64_t sweeps;               /* sweeps performed */
  int64_t converged;            /* 1 if stopped on big == 0 */
  int64_t pairs_visited;
  int64_t transforms_all;
  int64_t transforms_big;
  int64_t all_per_sweep[OR_MAX_SWEEPS];
  int64_t big_per_sweep[OR_MAX_SWEEPS];
  double max_off_per_sweep[OR_MAX_SWEEPS];
} or_stats;

/* Round-robin (circle) parallel ordering, SURVEY C-11 reading of PAPER.md
 * Sec. 6.3 (lines 1717-1751): step s in [0, n-2], slot k in [0, n/2-1]. */
int or_rr_pair(int64_t n, int64_t s, int64_t k, int64_t *p, int64_t *q);

/* The 2x2 transformation of Sec. 6.1 (eqs 6.1-6.12). Inputs are the unscaled
 * pivot Grams (6.1); z[] = {z11, z21, z12, z22} of Z' = D0 * Z (column-major).
 * tol = eps * sqrt(n).  Returns kind >= 0 or a negative error. off receives
 * the scaled off-diagonal measure max(|H_pq|/sqrt(|H_pp||H_qq|), |S_pq|). */
int or_hz2x2(double hpp, double hqq, orc hpq, double spp, double sqq, orc spq,
             double tol, int criterion, orc z[4], double *off);

/* Pointwise Algorithm 2, Z' initialised to I, run to
 * convergence (big == 0) or cmax sweeps.  n odd is bordered (Sec. 6.3.2).
 * nthreads <= 0: OpenMP default. */
int or_hz_pointwise(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                    orc *G, int64_t ldg, orc *Z, int64_t ldz, double eps,
                    int criterion, int cmax, int nthreads, or_stats *st);

/* As or_hz_pointwise (n even) and also accumulating W = Z'^{-1} by applying each
 * 2x2 inverse to rows p, q from the left; X = Sigma W. */
int or_hz_pointwise_inv(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                        orc *G, int64_t ldg, orc *Z, int64_t ldz, orc *W, int64_t ldw,
                        double eps, int criterion, int cmax, int nthreads, or_stats *st);

/* Run only steps [s0, s0+ns) of one pointwise sweep on (F,G,Z) in place
 * (Z not reset).  n must be even.  Counters accumulated into *all, *big. */
int or_hz_steps(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                orc *G, int64_t ldg, orc *Z, int64_t ldz, double eps,
                int criterion, int64_t s0, int64_t ns, int nthreads,
                int64_t *all, int64_t *big);

/* Level-2 blocked HZ (Sec. 6.4): nblk (even) block
 * columns of width w or w-1 (Sec. 6.4.1), block pivots formed explicitly,
 * factored by HEBPJ / pivoted Cholesky, inner pointwise HZ with inner_sweeps
 * sweeps (1 = BO; >1 = FB, stopping on all == 0), update F,G,Z by Z_blk. */
int or_hz_blocked(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                  orc *G, int64_t ldg, orc *Z, int64_t ldz, int64_t nblk,
                  int inner_sweeps, double eps, int criterion, int cmax,
                  int nthreads, or_stats *st);

/* Block orderings (reading R2-5 of PAPER.md:1815-1824, Sec 6.4; see ghsvd_oracle.c):
 * OR_ORDER_RR the Level-2 round-robin (nsup ignored), OR_ORDER_LEVEL3 the recursive
 * (Level-3, block-oriented) ordering over nsup super blocks, OR_ORDER_HIER every block
 * pair once per sweep grouped by super pair.  or_order_steps: block steps per sweep;
 * or_order_pair: block pair (p < q) of slot k in step s. */
enum { OR_ORDER_RR = 0, OR_ORDER_LEVEL3 = 1, OR_ORDER_HIER = 2 };
int or_order_steps(int ord, int64_t nblk, int64_t nsup, int64_t *nsteps);
int or_order_pair(int ord, int64_t nblk, int64_t nsup, int64_t s, int64_t k, int64_t *p, int64_t *q);

/* or_hz_blocked with the block pairs of each sweep in the given ordering. */
int or_hz_blocked_ord(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                      orc *G, int64_t ldg, orc *Z, int64_t ldz, int64_t nblk, int ord,
                      int64_t nsup, int inner_sweeps, double eps, int criterion, int cmax,
                      int nthreads, or_stats *st);

/* The Sec 6.4.1 partition (widths w or w-1, non-increasing) and one block pivot
 * (Sec 6.4.2-6.4.3) of block columns [p0, p0+wp) and [q0, q0+wq), in place. */
int or_block_partition(int64_t n, int64_t nblk, int64_t *start, int64_t *width);
int or_block_pair(int64_t m, int64_t n, orc *F, int64_t ldf, const int8_t *J,
                  orc *G, int64_t ldg, orc *Z, int64_t ldz, int64_t p0, int64_t wp,
                  int64_t q0, int64_t wq, int inner_sweeps, double eps, int criterion,
                  int64_t *all, int64_t *big);

/* Outputs of Sec. 6.1.7 and eq (3.2). */
int or_extract(int64_t m, int64_t n, const orc *F, int64_t ldf, const int8_t *J,
               const orc *G, int64_t ldg, const orc *Zp, int64_t ldzp,
               double *lambda, double *sigma_f, double *sigma_g, orc *Z,
               int64_t ldz);

/* HEBPJ (Sec. 4.2-4.3): T (order r, Hermitian, only read) = M^* diag(Jr) M,
 * Bunch-Parlett complete pivoting, 2x2 pivots diagonalised by a Jacobi
 * rotation, rows scaled by |d|^(1/2), rows sorted + before -.
 * M is r x r (ldm), Jr r signs; *npos = number of + signs. */
int or_hebpj(int64_t r, const orc *T, int64_t ldt, orc *M, int64_t ldm,
             int8_t *Jr, int64_t *npos);

/* Diagonally pivoted Cholesky: S = Gh^* Gh, Gh = L^* P (Sec. 6.4.2). */
int or_pchol(int64_t r, const orc *S, int64_t lds, orc *Gh, int64_t ldg);

/* Phase 1 (Algorithm 1, eqs 4.1-4.3): per atom a, T_a = [[TAA, TAB],[TAB^*, TBB]],
 * HEBPJ, Ftilde_a = Mtilde_a [A_a; B_a], Gtilde_a = [A_a; U_a B_a].
 * A,B: NA blocks of NL x NG (block a at A + a*NL*NG, ld NL);
 * U: NA*NL reals; TAA,TAB,TBB: NA blocks of NL x NL (ld NL).
 * Outputs F, G: m x NG (m = 2 NA NL, ld m) and J (m), atom-by-atom. */
int or_factor(int64_t NA, int64_t NL, int64_t NG, const orc *A, const orc *B,
              const double *U, const orc *TAA, const orc *TAB, const orc *TBB,
              orc *F, int8_t *J, orc *G);

/* Phase 2 (Sec. 5, eq 5.1): JQR of F (m x n, J) with diagonal + partial
 * (Bunch-Kaufman) pivoting and hyperbolic Householder reflectors / 2x2 URV
 * pivots; prepermute G by P2; QR of G P2 keeping R (diag real >= 0).
 * Outputs Fs (n x n), Js (n), Gs (n x n), p2 (n: column j of the new
 * factors is column p2[j] of the old ones), *n2x2 = number of 2x2 pivots. */
int or_reduce(int64_t m, int64_t n, const orc *F, int64_t ldf, const int8_t *J,
              const orc *G, int64_t ldg, orc *Fs, int8_t *Js, orc *Gs,
              int64_t *p2, int64_t *n2x2);

#ifdef __cplusplus
}
#endif
#endif
