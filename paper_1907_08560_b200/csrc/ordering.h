// ordering.h -- block orderings of the blocked sweep (host and device).
//
// GHSVD_ORDER_ROUND_ROBIN: the Level-2 circle method over nblk block columns (reading
// C-11 of PAPER.md Sec 6.3, applied to block columns, Sec 6.4): nblk - 1 steps.
// The Level-3 orderings (reading R2-5 of PAPER.md:1815-1824, Sec 6.4: "a multilevel
// blocking principle ... can be applied recursively further"; the paper builds Level 2
// only) group the block columns into nsup = 2Q super blocks of B = nblk / nsup
// consecutive block columns; the block pairs of super pair u occupy slots [uB, (u+1)B):
//   GHSVD_ORDER_LEVEL3  outer circle method over the 2Q super blocks (2Q - 1 outer steps
//       t); every super pair -- a Level-3 pivot of 2B block columns -- gets one inner
//       circle-method block sweep over its 2B block columns (2B - 1 inner steps i; BO at
//       Level 3).  Step s = t (2B - 1) + i.
//   GHSVD_ORDER_HIER    every block pair once per sweep: B - 1 intra-super-block steps
//       (circle method inside each super block of outer step 0's super pairs), then for
//       every outer step t, B bipartite steps pairing block v of the lower super block
//       with block (v + i) mod B of the upper one.  B even or 1.
// With one super pair per rank, block columns move between ranks only between outer
// steps (2Q - 1 exchanges per sweep instead of nblk - 1).
#pragma once

#ifdef __CUDACC__
#define GH_HD __host__ __device__ __forceinline__
#else
#define GH_HD inline
#endif

namespace ghsvd {

// circle method over n (even) items: step s in [0, n-2], slot k in [0, n/2): {a, b}
GH_HD void ord_circle(long long n, long long s, long long k, long long* a, long long* b) {
  if (k == 0) {
    *a = n - 1;
    *b = s;
  } else {
    const long long r = n - 1;
    *a = (s + k) % r;
    long long t = (s - k) % r;
    if (t < 0) t += r;
    *b = t;
  }
}

// 0 if (ord, nblk, nsup) is a valid ordering (nsup ignored for the round-robin)
GH_HD int blk_order_check(int ord, long long nblk, long long nsup) {
  if (nblk < 2 || (nblk & 1)) return -1;
  if (ord == 0) return 0;
  if (ord != 1 && ord != 2) return -1;
  if (nsup < 2 || (nsup & 1) || nblk % nsup) return -1;
  const long long B = nblk / nsup;
  if (ord == 2 && B != 1 && (B & 1)) return -1;
  return 0;
}

// block steps per sweep
GH_HD long long blk_order_steps(int ord, long long nblk, long long nsup) {
  if (ord == 0) return nblk - 1;
  const long long B = nblk / nsup;
  return ord == 1 ? (nsup - 1) * (2 * B - 1) : (B - 1) + (nsup - 1) * B;
}

// block pair (p < q) of slot k in block step s
GH_HD void blk_order_pair(int ord, long long nblk, long long nsup, long long s, long long k, long long* p,
                          long long* q) {
  long long a, b;
  if (ord == 0) {
    ord_circle(nblk, s, k, &a, &b);
  } else {
    const long long B = nblk / nsup, u = k / B, v = k % B;
    long long P, Q;
    if (ord == 1) {
      const long long t = s / (2 * B - 1), i = s % (2 * B - 1);
      ord_circle(nsup, t, u, &P, &Q);
      if (P > Q) { const long long x = P; P = Q; Q = x; }
      long long x, y;
      ord_circle(2 * B, i, v, &x, &y);
      a = x < B ? P * B + x : Q * B + (x - B);
      b = y < B ? P * B + y : Q * B + (y - B);
    } else if (s < B - 1) {
      ord_circle(nsup, 0, u, &P, &Q);
      if (P > Q) { const long long x = P; P = Q; Q = x; }
      const long long h = B / 2, base = (v < h ? P : Q) * B;
      long long x, y;
      ord_circle(B, s, v % h, &x, &y);
      a = base + x;
      b = base + y;
    } else {
      const long long s2 = s - (B - 1), t = s2 / B, i = s2 % B;
      ord_circle(nsup, t, u, &P, &Q);
      if (P > Q) { const long long x = P; P = Q; Q = x; }
      a = P * B + v;
      b = Q * B + (v + i) % B;
    }
  }
  *p = a < b ? a : b;
  *q = a < b ? b : a;
}

}  // namespace ghsvd
