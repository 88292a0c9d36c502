"""CPU oracle for the implicit Hari-Zimmermann J-GHSVD (arXiv:1907.08560).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It wraps ``ghsvd_oracle.c`` (plain C, fp64, no FMA contraction,
OpenMP over the disjoint pairs of a step) through ctypes.  It shares no code
with ``paper_1907_08560_b200`` (the CUDA product path) and never imports it.

Parity pins for every function live in ``tests/test_oracle_*.py``; see
DESIGN.md "Oracle and pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ghsvd_oracle.c")
_LIB = os.path.join(_HERE, "libghsvd_oracle.so")

EPS = 2.0 ** -53          # SURVEY C-6 reading: unit roundoff
CRIT_RELATIVE = 0
CRIT_LITERAL = 1
K_SKIP, K_IDENTITY, K_SMALL, K_BIG = 0, 1, 2, 3
MAX_SWEEPS = 64


class OracleError(RuntimeError):
    pass


class _Orc(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class _Stats(ctypes.Structure):
    _fields_ = [
        ("sweeps", ctypes.c_int64),
        ("converged", ctypes.c_int64),
        ("pairs_visited", ctypes.c_int64),
        ("transforms_all", ctypes.c_int64),
        ("transforms_big", ctypes.c_int64),
        ("all_per_sweep", ctypes.c_int64 * MAX_SWEEPS),
        ("big_per_sweep", ctypes.c_int64 * MAX_SWEEPS),
        ("max_off_per_sweep", ctypes.c_double * MAX_SWEEPS),
    ]

    def todict(self):
        n = min(self.sweeps, MAX_SWEEPS)
        return {
            "sweeps": int(self.sweeps),
            "converged": bool(self.converged),
            "pairs_visited": int(self.pairs_visited),
            "transforms_all": int(self.transforms_all),
            "transforms_big": int(self.transforms_big),
            "all_per_sweep": [int(v) for v in self.all_per_sweep[:n]],
            "big_per_sweep": [int(v) for v in self.big_per_sweep[:n]],
            "max_off_per_sweep": [float(v) for v in self.max_off_per_sweep[:n]],
        }


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True, cwd=_HERE)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        Ci = ctypes.c_int
        L.or_rr_pair.argtypes = [I64, I64, I64, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.or_hz2x2.argtypes = [D, D, _Orc, D, D, _Orc, D, Ci, P, ctypes.POINTER(D)]
        L.or_hz_pointwise.argtypes = [I64, I64, P, I64, P, P, I64, P, I64, D, Ci, Ci, Ci,
                                      ctypes.POINTER(_Stats)]
        L.or_hz_steps.argtypes = [I64, I64, P, I64, P, P, I64, P, I64, D, Ci, I64, I64, Ci,
                                  ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.or_hz_blocked.argtypes = [I64, I64, P, I64, P, P, I64, P, I64, I64, Ci, D, Ci, Ci, Ci,
                                    ctypes.POINTER(_Stats)]
        L.or_hz_blocked_ord.argtypes = [I64, I64, P, I64, P, P, I64, P, I64, I64, Ci, I64, Ci, D, Ci,
                                        Ci, Ci, ctypes.POINTER(_Stats)]
        L.or_order_steps.argtypes = [Ci, I64, I64, ctypes.POINTER(I64)]
        L.or_order_pair.argtypes = [Ci, I64, I64, I64, I64, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.or_extract.argtypes = [I64, I64, P, I64, P, P, I64, P, I64, P, P, P, P, I64]
        L.or_block_partition.argtypes = [I64, I64, P, P]
        L.or_hz_pointwise_inv.argtypes = [I64, I64, P, I64, P, P, I64, P, I64, P, I64, D, Ci, Ci, Ci,
                                          ctypes.POINTER(_Stats)]
        L.or_block_pair.argtypes = [I64, I64, P, I64, P, P, I64, P, I64, I64, I64, I64, I64, Ci, D, Ci,
                                    ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.or_hebpj.argtypes = [I64, P, I64, P, I64, P, ctypes.POINTER(I64)]
        L.or_pchol.argtypes = [I64, P, I64, P, I64]
        L.or_factor.argtypes = [I64, I64, I64, P, P, P, P, P, P, P, P, P]
        L.or_reduce.argtypes = [I64, I64, P, I64, P, P, I64, P, P, P, P, ctypes.POINTER(I64)]
        _lib = L
    return _lib


def _cf(a):
    """complex128, Fortran order, owned copy."""
    return np.array(a, dtype=np.complex128, order="F", copy=True)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _chk(rc, what):
    if rc < 0:
        raise OracleError(f"{what}: oracle error {rc}")
    return rc


def rr_pair(n, s, k):
    p, q = ctypes.c_int64(), ctypes.c_int64()
    _chk(lib().or_rr_pair(n, s, k, ctypes.byref(p), ctypes.byref(q)), "rr_pair")
    return p.value, q.value


def hz2x2(hpp, hqq, hpq, spp, sqq, spq, n, eps=EPS, criterion=CRIT_RELATIVE):
    """Returns (kind, Z' as 2x2 complex ndarray, off) or raises on error."""
    z = np.zeros(4, dtype=np.complex128)
    off = ctypes.c_double()
    D2 = _Orc
    kind = lib().or_hz2x2(float(hpp), float(hqq), D2(complex(hpq).real, complex(hpq).imag), float(spp), float(sqq),
                          D2(complex(spq).real, complex(spq).imag), eps * np.sqrt(n), criterion, _ptr(z),
                          ctypes.byref(off))
    _chk(kind, "hz2x2")
    return kind, z.reshape(2, 2, order="F"), off.value


def hz2x2_raw(hpp, hqq, hpq, spp, sqq, spq, tol, criterion=CRIT_RELATIVE):
    """Like hz2x2 but with an explicit tol = eps*sqrt(n); returns rc instead of raising."""
    z = np.zeros(4, dtype=np.complex128)
    off = ctypes.c_double()
    D2 = _Orc
    rc = lib().or_hz2x2(float(hpp), float(hqq), D2(complex(hpq).real, complex(hpq).imag), float(spp), float(sqq),
                        D2(complex(spq).real, complex(spq).imag), tol, criterion, _ptr(z), ctypes.byref(off))
    return rc, z.reshape(2, 2, order="F"), off.value


def hz_pointwise(F, J, G, eps=EPS, criterion=CRIT_RELATIVE, cmax=30, nthreads=0):
    """Algorithm 2 to convergence.  Returns (F', G', Z', stats dict)."""
    F = _cf(F)
    G = _cf(G)
    J = np.ascontiguousarray(J, dtype=np.int8)
    m, n = F.shape
    Z = np.zeros((n, n), dtype=np.complex128, order="F")
    st = _Stats()
    _chk(lib().or_hz_pointwise(m, n, _ptr(F), m, _ptr(J), _ptr(G), m, _ptr(Z), n, eps, criterion,
                               cmax, nthreads, ctypes.byref(st)), "hz_pointwise")
    return F, G, Z, st.todict()


def hz_pointwise_inv(F, J, G, eps=EPS, criterion=CRIT_RELATIVE, cmax=30, nthreads=1):
    """Algorithm 2 also accumulating W = Z'^{-1} (n even).  Returns (F', G', Z', W, stats).
    Single-threaded: the row updates of W are not disjoint across the pairs of a step in
    memory order (they are in index space), kept sequential for clarity."""
    F = _cf(F)
    G = _cf(G)
    J = np.ascontiguousarray(J, dtype=np.int8)
    m, n = F.shape
    Z = np.zeros((n, n), dtype=np.complex128, order="F")
    W = np.zeros((n, n), dtype=np.complex128, order="F")
    st = _Stats()
    _chk(lib().or_hz_pointwise_inv(m, n, _ptr(F), m, _ptr(J), _ptr(G), m, _ptr(Z), n, _ptr(W), n, eps,
                                   criterion, cmax, nthreads, ctypes.byref(st)), "hz_pointwise_inv")
    return F, G, Z, W, st.todict()


def hz_steps(F, J, G, Z, s0, ns, eps=EPS, criterion=CRIT_RELATIVE, nthreads=0):
    """Steps [s0, s0+ns) of one sweep, in place on copies. Returns (F, G, Z, all, big)."""
    F = _cf(F)
    G = _cf(G)
    Z = _cf(Z)
    J = np.ascontiguousarray(J, dtype=np.int8)
    m, n = F.shape
    a, b = ctypes.c_int64(0), ctypes.c_int64(0)
    _chk(lib().or_hz_steps(m, n, _ptr(F), m, _ptr(J), _ptr(G), m, _ptr(Z), n, eps, criterion,
                           s0, ns, nthreads, ctypes.byref(a), ctypes.byref(b)), "hz_steps")
    return F, G, Z, a.value, b.value


ORDER_RR, ORDER_LEVEL3, ORDER_HIER = 0, 1, 2


def order_steps(ordering, nblk, nsup=0):
    """Block steps per sweep of a block ordering (or_order_steps; reading R2-5)."""
    v = ctypes.c_int64()
    _chk(lib().or_order_steps(ordering, nblk, nsup, ctypes.byref(v)), "order_steps")
    return v.value


def order_pair(ordering, nblk, nsup, s, k):
    """Block pair (p < q) of slot k in block step s (or_order_pair; reading R2-5)."""
    p, q = ctypes.c_int64(), ctypes.c_int64()
    _chk(lib().or_order_pair(ordering, nblk, nsup, s, k, ctypes.byref(p), ctypes.byref(q)), "order_pair")
    return p.value, q.value


def hz_blocked(F, J, G, nblk, inner_sweeps=1, eps=EPS, criterion=CRIT_RELATIVE, cmax=30,
               nthreads=0, ordering=ORDER_RR, nsup=0):
    F = _cf(F)
    G = _cf(G)
    J = np.ascontiguousarray(J, dtype=np.int8)
    m, n = F.shape
    Z = np.zeros((n, n), dtype=np.complex128, order="F")
    st = _Stats()
    if ordering == ORDER_RR:
        rc = lib().or_hz_blocked(m, n, _ptr(F), m, _ptr(J), _ptr(G), m, _ptr(Z), n, nblk,
                                 inner_sweeps, eps, criterion, cmax, nthreads, ctypes.byref(st))
    else:
        rc = lib().or_hz_blocked_ord(m, n, _ptr(F), m, _ptr(J), _ptr(G), m, _ptr(Z), n, nblk,
                                     ordering, nsup, inner_sweeps, eps, criterion, cmax, nthreads,
                                     ctypes.byref(st))
    _chk(rc, "hz_blocked")
    return F, G, Z, st.todict()


def block_partition(n, nblk):
    start = np.zeros(nblk, np.int64)
    width = np.zeros(nblk, np.int64)
    _chk(lib().or_block_partition(n, nblk, _ptr(start), _ptr(width)), "block_partition")
    return start, width


def block_pair(F, J, G, Z, p0, wp, q0, wq, inner_sweeps=1, eps=EPS, criterion=CRIT_RELATIVE):
    """One block pivot IN PLACE on Fortran-ordered complex128 arrays F, G (m x n), Z (n x n).
    Returns (all, big)."""
    for X in (F, G, Z):
        assert X.dtype == np.complex128 and X.flags.f_contiguous
    J = np.ascontiguousarray(J, dtype=np.int8)
    m, n = F.shape
    a, b = ctypes.c_int64(0), ctypes.c_int64(0)
    _chk(lib().or_block_pair(m, n, _ptr(F), m, _ptr(J), _ptr(G), m, _ptr(Z), n, p0, wp, q0, wq, inner_sweeps,
                             eps, criterion, ctypes.byref(a), ctypes.byref(b)), "block_pair")
    return a.value, b.value


def extract(F, J, G, Zp):
    F = _cf(F)
    G = _cf(G)
    Zp = _cf(Zp)
    J = np.ascontiguousarray(J, dtype=np.int8)
    m, n = F.shape
    lam = np.zeros(n)
    sf = np.zeros(n)
    sg = np.zeros(n)
    Z = np.zeros((n, n), dtype=np.complex128, order="F")
    _chk(lib().or_extract(m, n, _ptr(F), m, _ptr(J), _ptr(G), m, _ptr(Zp), n, _ptr(lam), _ptr(sf),
                          _ptr(sg), _ptr(Z), n), "extract")
    return lam, sf, sg, Z


def hebpj(T):
    T = _cf(T)
    r = T.shape[0]
    M = np.zeros((r, r), dtype=np.complex128, order="F")
    Jr = np.zeros(r, dtype=np.int8)
    npos = ctypes.c_int64()
    _chk(lib().or_hebpj(r, _ptr(T), r, _ptr(M), r, _ptr(Jr), ctypes.byref(npos)), "hebpj")
    return M, Jr, npos.value


def pchol(S):
    S = _cf(S)
    r = S.shape[0]
    Gh = np.zeros((r, r), dtype=np.complex128, order="F")
    _chk(lib().or_pchol(r, _ptr(S), r, _ptr(Gh), r), "pchol")
    return Gh


def factor(A, B, U, TAA, TAB, TBB):
    """Phase 1.  A, B: (NA, NL, NG); U: (NA, NL); T**: (NA, NL, NL). Returns F, J, G."""
    NA, NL, NG = A.shape
    # block a stored column-major NL x NG contiguous
    Ab = np.ascontiguousarray(np.stack([np.asfortranarray(A[a]).ravel(order="F") for a in range(NA)]),
                              dtype=np.complex128)
    Bb = np.ascontiguousarray(np.stack([np.asfortranarray(B[a]).ravel(order="F") for a in range(NA)]),
                              dtype=np.complex128)
    tb = [np.ascontiguousarray(np.stack([np.asfortranarray(T[a]).ravel(order="F") for a in range(NA)]),
                               dtype=np.complex128) for T in (TAA, TAB, TBB)]
    Uc = np.ascontiguousarray(U, dtype=np.float64)
    m = 2 * NA * NL
    F = np.zeros((m, NG), dtype=np.complex128, order="F")
    G = np.zeros((m, NG), dtype=np.complex128, order="F")
    J = np.zeros(m, dtype=np.int8)
    _chk(lib().or_factor(NA, NL, NG, _ptr(Ab), _ptr(Bb), _ptr(Uc), _ptr(tb[0]), _ptr(tb[1]),
                         _ptr(tb[2]), _ptr(F), _ptr(J), _ptr(G)), "factor")
    return F, J, G


def reduce(F, J, G):
    """Phase 2: returns (Fs, Js, Gs, p2, n2x2)."""
    F = _cf(F)
    G = _cf(G)
    J = np.ascontiguousarray(J, dtype=np.int8)
    m, n = F.shape
    Fs = np.zeros((n, n), dtype=np.complex128, order="F")
    Gs = np.zeros((n, n), dtype=np.complex128, order="F")
    Js = np.zeros(n, dtype=np.int8)
    p2 = np.zeros(n, dtype=np.int64)
    n2 = ctypes.c_int64()
    _chk(lib().or_reduce(m, n, _ptr(F), m, _ptr(J), _ptr(G), m, _ptr(Fs), _ptr(Js), _ptr(Gs),
                         _ptr(p2), ctypes.byref(n2)), "reduce")
    return Fs, Js, Gs, p2, n2.value


def pencil_eigvals(F, J, G):
    """Eigenvalues of the pencil (H, S) = (F^* J F, G^* G) by the paper's "alternative way
    forward" (Sec 4.5): H and S formed explicitly (S = G^* G, H = F^* (J F)
    with F's rows scaled by J), then a generalized Hermitian-definite solver (LAPACK ZHEGVD
    through scipy.linalg.eigh) -- the definition of the eigenvalues written out, a library
    routine as its step.  Its absolute error is ~ eps * kappa(S) * ||H||, so it is a
    reference only for WELL-CONDITIONED S (config 4, kappa(S) ~ 10), never for the
    ill-conditioned config 3, where avoiding exactly this is the paper's point
    (PAPER.md:404-407).  Returns the eigenvalues in ascending order."""
    import scipy.linalg

    F = np.asarray(F, dtype=np.complex128)
    G = np.asarray(G, dtype=np.complex128)
    Js = np.asarray(J, dtype=np.float64)
    S = G.conj().T @ G
    H = F.conj().T @ (Js[:, None] * F)
    H = 0.5 * (H + H.conj().T)
    S = 0.5 * (S + S.conj().T)
    return scipy.linalg.eigh(H, S, eigvals_only=True, driver="gvd")
