// hebpj.cuh -- CTA-wide Hermitian indefinite factorisation with complete pivoting
// (HEBPJ, Sec 4.2-4.3, eq 4.3) and diagonally pivoted Cholesky
// (PAPER.md:1920-1932), as __device__ routines run by one thread block on a
// matrix in global or shared memory.  Used by Phase 1 (T_a, order 2 N_L) and by
// the blocked variant's block pivots (order 2w, Sec 6.4.2).
//
// hebpj_dev: W (r x r, ld, full Hermitian; overwritten: L below the diagonal)
//   -> M (r x r, ld) with T = M^* diag(J) M, rows sorted + before - ;
//   Bunch-Parlett pivoting, alpha = (1 + sqrt 17)/8, smallest-index ties;
//   2x2 pivots diagonalised by a Jacobi rotation, rows scaled by |d|^1/2.
// pchol_dev: S (r x r, ld, full Hermitian; overwritten) -> Gh = L^* P.
#pragma once
#include <cuda_runtime.h>

namespace ghsvd {
namespace hb {

__device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ double2 add(double2 a, double2 b) { return mk(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ double2 sub(double2 a, double2 b) { return mk(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
__device__ __forceinline__ double2 mul(double2 a, double2 b) {
  return mk(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 conj(double2 a) { return mk(a.x, -a.y); }
__device__ __forceinline__ double2 scale(double2 a, double s) { return mk(__dmul_rn(a.x, s), __dmul_rn(a.y, s)); }
__device__ __forceinline__ double cabs(double2 a) { return __dsqrt_rn(__dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y))); }
__device__ __forceinline__ double cabs2(double2 a) { return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)); }

__device__ __forceinline__ void amax_merge(double& v, long long& i, double v2, long long i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}
// the Schur updates' pivot tracking of one updated entry w at (i, j): diagonal |w_ii|,
// strictly lower |w_ij|^2 with index j r + i -- the same choices as amax_merge, written as
// selects so that the diagonal crossing a warp's rows does not split it into branches
__device__ __forceinline__ void track_entry(double2 w, int i, int j, int r, double& mu1, long long& id, double& mu0,
                                            long long& oidx) {
  const double dv = fabs(w.x);
  const bool td = (i == j) && (dv > mu1 || (dv == mu1 && (long long)i < id));
  mu1 = td ? dv : mu1;
  id = td ? (long long)i : id;
  const double ov = __dadd_rn(__dmul_rn(w.x, w.x), __dmul_rn(w.y, w.y));
  const long long oi = (long long)(j * r + i);
  const bool to = (i > j) && (ov > mu0 || (ov == mu0 && oi < oidx));
  mu0 = to ? ov : mu0;
  oidx = to ? oi : oidx;
}

// Shared-memory scratch of the routines below, passed in by the caller (the blocked
// variant places it in dynamic shared memory it no longer needs, so its kernels carry no
// static shared memory; Phase 1 declares it statically).
template <int NT, int RMAX>
struct HebpjScr {
  double sv[2][2][NT / 32];
  long long si[2][2][NT / 32];
  double sv1[NT / 32];
  long long si1[NT / 32];
  double2 Rk[RMAX * 2];  // 4 per 2x2 pivot (stored at 2*k .. 2*k+3 for pivot k)
  double2 colk[2][RMAX];
  double d[RMAX];
  int perm[RMAX];
  int bsz[RMAX];
  int rowpos[RMAX];
  signed char sgn[RMAX];
  int err_sh;
};
template <int RMAX>
struct PcholScr {
  double dg[RMAX], iv[RMAX];   // l_kk and 1 / l_kk
  int perm[RMAX];
};

template <int NT>
__device__ void block_amax(double& v, long long& i, double* sv, long long* si) {
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
    amax_merge(v, i, v2, i2);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[w] = v;
    si[w] = i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < NT / 32; k++) amax_merge(sv[0], si[0], sv[k], si[k]);
  }
  __syncthreads();
  v = sv[0];
  i = si[0];
  __syncthreads();
}

// two independent (value, index) argmax reductions with one set of barriers
template <int NT>
__device__ void block_amax2(double& v, long long& i, double& u, long long& j) {
  __shared__ double sv[2][NT / 32];
  __shared__ long long si[2][NT / 32];
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
    const double u2 = __shfl_xor_sync(0xffffffffu, u, o);
    const long long j2 = __shfl_xor_sync(0xffffffffu, j, o);
    amax_merge(v, i, v2, i2);
    amax_merge(u, j, u2, j2);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[0][w] = v;
    si[0][w] = i;
    sv[1][w] = u;
    si[1][w] = j;
  }
  __syncthreads();
  v = sv[0][0];
  i = si[0][0];
  u = sv[1][0];
  j = si[1][0];
  for (int k = 1; k < NT / 32; k++) {  // every thread reduces the NT/32 partials (same order)
    amax_merge(v, i, sv[0][k], si[0][k]);
    amax_merge(u, j, sv[1][k], si[1][k]);
  }
  __syncthreads();
}

// block_amax2 with double-buffered partials (buffer `par`, alternate between calls): one
// barrier per call; a later call with the same parity is separated by the other call's
// barrier, so no reader of this buffer is left when it is rewritten.
template <int NT>
__device__ void block_amax2_db(double& v, long long& i, double& u, long long& j, int par, double (*sv)[2][NT / 32],
                               long long (*si)[2][NT / 32]) {
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
    const double u2 = __shfl_xor_sync(0xffffffffu, u, o);
    const long long j2 = __shfl_xor_sync(0xffffffffu, j, o);
    amax_merge(v, i, v2, i2);
    amax_merge(u, j, u2, j2);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[par][0][w] = v;
    si[par][0][w] = i;
    sv[par][1][w] = u;
    si[par][1][w] = j;
  }
  __syncthreads();
  v = sv[par][0][0];
  i = si[par][0][0];
  u = sv[par][1][0];
  j = si[par][1][0];
  for (int k = 1; k < NT / 32; k++) {  // every thread reduces the NT/32 partials (same order)
    amax_merge(v, i, sv[par][0][k], si[par][0][k]);
    amax_merge(u, j, sv[par][1][k], si[par][1][k]);
  }
}

// Jacobi rotation R (column-major R11, R21, R12, R22) with R^* E R = diag(l1, l2)
__device__ inline void herm2_jacobi(double a, double2 b, double c, double2* R, double* l1, double* l2) {
  const double ab = cabs(b);
  if (ab == 0.0) {
    R[0] = mk(1, 0); R[1] = mk(0, 0); R[2] = mk(0, 0); R[3] = mk(1, 0);
    *l1 = a; *l2 = c;
    return;
  }
  const double2 e = mk(__ddiv_rn(b.x, ab), __ddiv_rn(b.y, ab));
  const double tau = __ddiv_rn(__dsub_rn(c, a), __dmul_rn(2.0, ab));
  const double t = __ddiv_rn(tau >= 0.0 ? 1.0 : -1.0,
                             __dadd_rn(fabs(tau), __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(tau, tau)))));
  const double cs = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(t, t)))), sn = __dmul_rn(t, cs);
  const double2 em = conj(e);
  R[0] = mk(cs, 0.0);
  R[1] = scale(em, -sn);
  R[2] = mk(sn, 0.0);
  R[3] = scale(em, cs);
  *l1 = __dsub_rn(a, __dmul_rn(t, ab));
  *l2 = __dadd_rn(c, __dmul_rn(t, ab));
}

// Returns 0 or -7 (rank deficient).  All NT threads of the block must call it.
// tolz: pivots with max |entry| <= tolz stop the factorisation (rank deficiency).
// Loops are 2-D (warp -> column, lane -> row) with 32-bit indices: no integer
// division in the O(r^2) passes of an elimination step.
template <int NT, int RMAX>
__device__ int hebpj_dev(double2* W, int r, long long ldw, double2* M, long long ldmo, signed char* Jout,
                         int* npos_out, double tolz, HebpjScr<NT, RMAX>& sc) {
  constexpr int NW = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* perm = sc.perm;
  int* bsz = sc.bsz;
  double* d = sc.d;
  double2* Rk = sc.Rk;
  double2 (*colk)[RMAX] = sc.colk;
  int* rowpos = sc.rowpos;
  signed char* sgn = sc.sgn;
  int& err_sh = sc.err_sh;
  const double alpha = (1.0 + sqrt(17.0)) / 8.0;
  for (int i = threadIdx.x; i < r; i += NT) perm[i] = i;
  if (threadIdx.x == 0) err_sh = 0;
  __syncthreads();
  // Per-thread partial pivot searches (diagonal |w_ii|, off-diagonal |w_ij| lower
  // triangle) over the trailing matrix; after step 0 they are formed inside the previous
  // step's Schur-complement update, on exactly the values the next search would read.
  double mu1 = -1.0, mu0 = 0.0;
  long long id = 0x7fffffffffffffffll, oidx = 0x7fffffffffffffffll;
  for (int i = threadIdx.x; i < r; i += NT) amax_merge(mu1, id, fabs(W[i + i * ldw].x), i);
  // off-diagonal search on |w_ij|^2 (same entry as on |w_ij|, no square root per entry;
  // the oracle searches the same way); mu0 becomes the magnitude after the reduction
  for (int j = warp; j < r; j += NW)
    for (int i = j + 1 + lane; i < r; i += 32) amax_merge(mu0, oidx, cabs2(W[i + j * ldw]), (long long)j * r + i);
  int k = 0, par = 0;
  while (k < r) {
    block_amax2_db<NT>(mu1, id, mu0, oidx, par, sc.sv, sc.si);
    par ^= 1;
    mu0 = __dsqrt_rn(mu0);
    const double mall = mu0 > mu1 ? mu0 : mu1;
    if (!(mall > tolz)) {
      if (threadIdx.x == 0) err_sh = -7;
      __syncthreads();
      break;
    }
    const int two = !(mu1 >= __dmul_rn(alpha, mu0));
    int src0 = (int)id, src1 = -1;
    if (two) {
      src0 = (int)(oidx / r);
      src1 = (int)(oidx % r);
    }
    for (int b = 0; b < (two ? 2 : 1); b++) {
      const int dst = k + b;
      int s = b == 0 ? src0 : src1;
      if (b == 1 && s == k) s = src0;
      if (s != dst) {
        for (int c = threadIdx.x; c < r; c += NT) {
          const double2 t = W[dst + c * ldw];
          W[dst + c * ldw] = W[s + c * ldw];
          W[s + c * ldw] = t;
        }
        __syncthreads();
        for (int i = k + threadIdx.x; i < r; i += NT) {
          const double2 t = W[i + dst * ldw];
          W[i + dst * ldw] = W[i + s * ldw];
          W[i + s * ldw] = t;
        }
        if (threadIdx.x == 0) {
          const int t = perm[dst];
          perm[dst] = perm[s];
          perm[s] = t;
        }
        __syncthreads();
      }
    }
    mu1 = -1.0;
    mu0 = 0.0;
    id = oidx = 0x7fffffffffffffffll;
    if (!two) {
      // 1x1 pivot: L(:,k) = W(:,k) / d_k stays unscaled in W (scaled when M is formed);
      // the update reads column k directly, which no thread writes in this phase
      const double dk = W[k + k * ldw].x;
      const double inv = __ddiv_rn(1.0, dk);
      for (int j = k + 1 + warp; j < r; j += NW) {
        const double2 cj = conj(W[j + k * ldw]);
        for (int i = k + 1 + lane; i < r; i += 32) {
          const double2 w = sub(W[i + j * ldw], scale(mul(W[i + k * ldw], cj), inv));
          W[i + j * ldw] = w;
          track_entry(w, i, j, r, mu1, id, mu0, oidx);
        }
      }
      if (threadIdx.x == 0) {
        bsz[k] = 1;
        d[k] = dk;
      }
      k += 1;
    } else {
      const double ea = W[k + k * ldw].x, ec = W[(k + 1) + (k + 1) * ldw].x;
      const double2 eb = W[k + (k + 1) * ldw];
      const double det = __dsub_rn(__dmul_rn(ea, ec), cabs2(eb));
      const double inv = __ddiv_rn(1.0, det);
      for (int i = k + 2 + threadIdx.x; i < r; i += NT) {
        const double2 w0 = W[i + k * ldw], w1 = W[i + (k + 1) * ldw];
        colk[0][i] = w0;
        colk[1][i] = w1;
        W[i + k * ldw] = scale(sub(scale(w0, ec), mul(w1, conj(eb))), inv);
        W[i + (k + 1) * ldw] = scale(sub(scale(w1, ea), mul(w0, eb)), inv);
      }
      __syncthreads();
      for (int j = k + 2 + warp; j < r; j += NW) {
        const double2 c0 = conj(colk[0][j]), c1 = conj(colk[1][j]);
        for (int i = k + 2 + lane; i < r; i += 32) {
          const double2 t = add(mul(W[i + k * ldw], c0), mul(W[i + (k + 1) * ldw], c1));
          const double2 w = sub(W[i + j * ldw], t);
          W[i + j * ldw] = w;
          track_entry(w, i, j, r, mu1, id, mu0, oidx);
        }
      }
      if (threadIdx.x == 0) {
        double l1, l2;
        herm2_jacobi(ea, eb, ec, &Rk[2 * k], &l1, &l2);
        d[k] = l1;
        d[k + 1] = l2;
        bsz[k] = 2;
        bsz[k + 1] = 0;
        W[(k + 1) + k * ldw] = mk(0.0, 0.0);  // L's 2x2 diagonal block is I
      }
      k += 2;
    }
    // the next pivot search's barrier (block_amax2_db) orders this step's writes before
    // the next step's swaps and reads
  }
  __syncthreads();
  if (err_sh) return err_sh;
  if (threadIdx.x == 0) {
    for (int i = 0; i < r; i++) sgn[i] = d[i] > 0.0 ? 1 : -1;
    int np = 0;
    for (int i = 0; i < r; i++)
      if (sgn[i] > 0) rowpos[i] = np++;
    int q = np;
    for (int i = 0; i < r; i++)
      if (sgn[i] < 0) rowpos[i] = q++;
    *npos_out = np;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < r; i += NT) Jout[rowpos[i]] = sgn[i];
  // Mtilde(rowpos(i), perm[l]) = row i of diag(|d|^1/2) R^* L^*, column l
  for (int l = warp; l < r; l += NW) {
    for (int i = lane; i < r; i += 32) {
      auto Lh = [&](int row, int col) -> double2 {  // (L^*)(row, col) = conj(L(col, row))
        if (row == col) return mk(1.0, 0.0);
        if (col < row) return mk(0.0, 0.0);
        // L column `row` of a 1x1 pivot is stored unscaled: L = W / d (as W * (1/d))
        return conj(bsz[row] == 1 ? scale(W[col + row * ldw], __ddiv_rn(1.0, d[row])) : W[col + row * ldw]);
      };
      double2 y;
      if (bsz[i] == 1) {
        y = scale(Lh(i, l), __dsqrt_rn(fabs(d[i])));
      } else if (bsz[i] == 2) {
        const double2* R = &Rk[2 * i];
        y = scale(add(mul(conj(R[0]), Lh(i, l)), mul(conj(R[1]), Lh(i + 1, l))), __dsqrt_rn(fabs(d[i])));
      } else {
        const double2* R = &Rk[2 * (i - 1)];
        y = scale(add(mul(conj(R[2]), Lh(i - 1, l)), mul(conj(R[3]), Lh(i, l))), __dsqrt_rn(fabs(d[i])));
      }
      M[rowpos[i] + perm[l] * ldmo] = y;
    }
  }
  __syncthreads();
  return 0;
}

// Diagonally pivoted Cholesky: P S P^T = L L^*, Gh = L^* P (column perm[l] of Gh
// is column l of L^*).  S overwritten (the strictly lower part of L kept unscaled:
// L(i,k) = S(i,k) * (1/l_kk) is formed where it is used, with the same rounding as a
// stored scaled column).  Returns 0 or -6.  The pivot search (largest diagonal entry,
// smallest index on ties) is done redundantly by every warp, so no barrier is spent on
// it; one barrier per elimination step (+3 when rows are swapped).
template <int NT, int RMAX>
__device__ int pchol_dev(double2* S, int r, long long lds, double2* Gh, long long ldg, PcholScr<RMAX>& sc) {
  constexpr int NW = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* perm = sc.perm;
  double* dg = sc.dg;
  double* iv = sc.iv;
  for (int i = threadIdx.x; i < r; i += NT) perm[i] = i;
  __syncthreads();
  for (int k = 0; k < r; k++) {
    double bv = 0.0;
    int bi = 0x7fffffff;
    for (int i = k + lane; i < r; i += 32) {
      const double v = S[i + i * lds].x;
      if (bi == 0x7fffffff || v > bv) {
        bv = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (i2 != 0x7fffffff && (bi == 0x7fffffff || v2 > bv || (v2 == bv && i2 < bi))) {
        bv = v2;
        bi = i2;
      }
    }
    const int pv = bi == 0x7fffffff ? k : bi;
    if (!(S[pv + pv * lds].x > 0.0)) return -6;   // uniform across the block
    if (pv != k) {
      __syncthreads();   // every warp has finished its pivot search before rows move
      for (int c = threadIdx.x; c < r; c += NT) {
        const double2 t = S[k + c * lds];
        S[k + c * lds] = S[pv + c * lds];
        S[pv + c * lds] = t;
      }
      __syncthreads();
      for (int i = k + threadIdx.x; i < r; i += NT) {  // columns >= k hold the live matrix
        const double2 t = S[i + k * lds];
        S[i + k * lds] = S[i + pv * lds];
        S[i + pv * lds] = t;
      }
      if (threadIdx.x == 0) {
        const int t = perm[k];
        perm[k] = perm[pv];
        perm[pv] = t;
      }
      __syncthreads();
    }
    const double lkk = __dsqrt_rn(S[k + k * lds].x);
    const double inv = __ddiv_rn(1.0, lkk);
    // Schur complement with L(:,k) = S(:,k) / l_kk formed on the fly; column k and the
    // diagonal entry (k, k) are not written in this phase
    // (the lane's L(i,k) for its rows i = k+1+lane+32t are formed once, not once per j)
    constexpr int NR = (RMAX + 31) / 32;
    double2 li[NR];
#pragma unroll
    for (int t = 0; t < NR; t++) {
      const int i = k + 1 + lane + 32 * t;
      li[t] = i < r ? scale(S[i + k * lds], inv) : mk(0.0, 0.0);
    }
    for (int j = k + 1 + warp; j < r; j += NW) {
      const double2 cj = conj(scale(S[j + k * lds], inv));
#pragma unroll
      for (int t = 0; t < NR; t++) {
        const int i = k + 1 + lane + 32 * t;
        if (i < r) S[i + j * lds] = sub(S[i + j * lds], mul(li[t], cj));
      }
    }
    if (threadIdx.x == 0) {
      dg[k] = lkk;
      iv[k] = inv;
    }
    __syncthreads();
  }
  // Gh(i, perm[l]) = (L^*)(i, l) = conj(L(l, i)) for l >= i, else 0
  for (int l = warp; l < r; l += NW)
    for (int i = lane; i < r; i += 32)
      Gh[i + perm[l] * ldg] = l > i ? conj(scale(S[l + i * lds], iv[i])) : (l == i ? mk(dg[i], 0.0) : mk(0.0, 0.0));
  __syncthreads();
  return 0;
}

}  // namespace hb
}  // namespace ghsvd
