"""Thin Python binding of libghsvd.so (include/ghsvd.h) -- argument marshalling only.

Every step of the method runs inside the CUDA library; this module only
allocates the device workspace (a torch uint8 tensor), converts arrays to
pointers + leading dimensions, and raises on negative status codes.  There is
no CPU fallback: importing fails loudly if the shared library is missing.

Matrices are column-major complex128.  Accepted inputs: numpy arrays (host;
copied through the library with cudaMemcpyDefault) and torch tensors (host,
pinned or CUDA) whose first stride is 1 (i.e. column-major, e.g. ``x.t()`` of
a contiguous (n, m) tensor, or ``torch.from_numpy(np.asfortranarray(a))``).
"""
from __future__ import annotations

import ctypes
import os
import warnings
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libghsvd.so")

OK, NOT_CONVERGED = 0, 1
E_NAMES = {-1: "INVALID_ARG", -2: "STATE", -3: "CUDA", -4: "NCCL", -5: "WORKSPACE",
           -6: "INDEFINITE_S", -7: "RANK_DEFICIENT", -8: "NONFINITE"}
POINTWISE, BLOCKED_BO, BLOCKED_FB = 0, 1, 2
VARIANTS = {"pointwise": POINTWISE, "bo": BLOCKED_BO, "fb": BLOCKED_FB}
CRITERIA = {"relative": 0, "literal": 1}

# every symbol include/ghsvd.h declares (checked by tests/test_abi.py)
EXPORTS = ["ghsvd_default_options", "ghsvd_workspace_bytes", "ghsvd_create", "ghsvd_factor",
           "ghsvd_set_factors", "ghsvd_reduce", "ghsvd_get_factors", "ghsvd_sweep", "ghsvd_run_steps",
           "ghsvd_extract", "ghsvd_extract_local", "ghsvd_extract_x", "ghsvd_get_transformed", "ghsvd_get_state", "ghsvd_set_state",
           "ghsvd_hz2x2_batch", "ghsvd_last_error",
           "ghsvd_destroy", "ghsvd_version", "ghsvd_block_owner", "ghsvd_exchange_plan",
           "ghsvd_nccl_unique_id", "ghsvd_order_steps", "ghsvd_order_pair", "ghsvd_block_owner_ord",
           "ghsvd_exchange_plan_ord", "ghsvd_reduce_fallback_col"]


class GHSVDError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"ghsvd error {status} ({E_NAMES.get(status, '?')}): {msg}")
        self.status = status


SCHED_SERIAL, SCHED_NO_PRIO, SCHED_SPLIT_BND, SCHED_GRAM4M, SCHED_UPD4M, SCHED_PIVOT_CL = 1, 2, 4, 8, 16, 32
SCHED_SPLIT_FACTOR = 64
ORDER_ROUND_ROBIN, ORDER_LEVEL3, ORDER_HIER = 0, 1, 2
ORDERINGS = {"rr": ORDER_ROUND_ROBIN, "level3": ORDER_LEVEL3, "hier": ORDER_HIER}


class Options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("world_size", ctypes.c_int),
                ("rank", ctypes.c_int), ("nccl_id", ctypes.c_void_p), ("variant", ctypes.c_int),
                ("ordering", ctypes.c_int), ("nblocks", ctypes.c_int), ("max_sweeps", ctypes.c_int),
                ("criterion", ctypes.c_int), ("eps", ctypes.c_double), ("cluster", ctypes.c_int),
                ("threads", ctypes.c_int), ("use_graph", ctypes.c_int), ("kernel", ctypes.c_int),
                ("detail_timing", ctypes.c_int), ("want_x", ctypes.c_int), ("exchange_overlap", ctypes.c_int),
                ("schedule", ctypes.c_int), ("groups", ctypes.c_int), ("gram_splits", ctypes.c_int),
                ("trace_path", ctypes.c_char_p), ("super_blocks", ctypes.c_int)]


class Stats(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int), ("converged", ctypes.c_int), ("pairs_visited", ctypes.c_uint64),
                ("transforms_all", ctypes.c_uint64), ("transforms_big", ctypes.c_uint64),
                ("seconds", ctypes.c_double), ("kernel_seconds", ctypes.c_double),
                ("launches", ctypes.c_uint64), ("alg_bytes", ctypes.c_uint64),
                ("alg_flops", ctypes.c_double), ("t_gram", ctypes.c_double), ("t_pivot", ctypes.c_double),
                ("t_update", ctypes.c_double), ("t_exchange", ctypes.c_double),
                ("flops_gram", ctypes.c_double), ("flops_update", ctypes.c_double),
                ("max_offdiag_last", ctypes.c_double),
                ("all_per_sweep", ctypes.c_uint64 * 64), ("big_per_sweep", ctypes.c_uint64 * 64),
                ("launches_update_fg", ctypes.c_uint64), ("flops_update_fg", ctypes.c_double),
                ("t_update_fg", ctypes.c_double), ("nblocks", ctypes.c_int), ("super_blocks", ctypes.c_int),
                ("steps_per_sweep", ctypes.c_int)]

    def todict(self):
        k = min(self.sweeps, 64)
        return {"sweeps": self.sweeps, "converged": bool(self.converged),
                "pairs_visited": int(self.pairs_visited), "transforms_all": int(self.transforms_all),
                "transforms_big": int(self.transforms_big), "seconds": self.seconds,
                "kernel_seconds": self.kernel_seconds, "launches": int(self.launches),
                "alg_bytes": int(self.alg_bytes), "alg_flops": self.alg_flops,
                "t_gram": self.t_gram, "t_pivot": self.t_pivot, "t_update": self.t_update,
                "t_exchange": self.t_exchange, "flops_gram": self.flops_gram,
                "flops_update": self.flops_update,
                "launches_update_fg": int(self.launches_update_fg),
                "flops_update_fg": self.flops_update_fg, "t_update_fg": self.t_update_fg,
                "max_offdiag_last": self.max_offdiag_last, "nblocks": self.nblocks,
                "super_blocks": self.super_blocks, "steps_per_sweep": self.steps_per_sweep,
                "all_per_sweep": [int(v) for v in self.all_per_sweep[:k]],
                "big_per_sweep": [int(v) for v in self.big_per_sweep[:k]]}


_lib = None


def load():
    """Load libghsvd.so (build it first with ``python -m paper_1907_08560_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build the CUDA library (python -m paper_1907_08560_b200.build); "
                          "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, D, Ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    POPT = ctypes.POINTER(Options)
    L.ghsvd_default_options.argtypes = [POPT]
    L.ghsvd_default_options.restype = None
    L.ghsvd_workspace_bytes.argtypes = [POPT, I64, I64, I64]
    L.ghsvd_workspace_bytes.restype = ctypes.c_size_t
    L.ghsvd_create.argtypes = [POPT, I64, I64, I64, P, ctypes.c_size_t, ctypes.POINTER(P)]
    L.ghsvd_factor.argtypes = [P, I64, I64, I64, P, P, P, P, P, P]
    L.ghsvd_set_factors.argtypes = [P, I64, I64, P, I64, P, P, I64]
    L.ghsvd_reduce.argtypes = [P, Ci]
    L.ghsvd_get_factors.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64), P, I64, P, P, I64, P]
    L.ghsvd_sweep.argtypes = [P, ctypes.POINTER(Stats)]
    L.ghsvd_run_steps.argtypes = [P, I64, I64, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
    L.ghsvd_extract.argtypes = [P, P, P, P, P, I64, P]
    L.ghsvd_extract_local.argtypes = [P, P, P, P, P, I64, P, ctypes.POINTER(I64)]
    L.ghsvd_get_transformed.argtypes = [P, P, I64, P, I64, P, I64]
    L.ghsvd_get_state.argtypes = [P, P, I64, P, I64, P, I64, P, I64]
    L.ghsvd_set_state.argtypes = [P, P, I64, P, I64, P, I64, P, I64]
    L.ghsvd_extract_x.argtypes = [P, P, I64]
    L.ghsvd_extract_x.restype = ctypes.c_int
    L.ghsvd_hz2x2_batch.argtypes = [P, I64, P, D, Ci, P, P]
    L.ghsvd_last_error.argtypes = [P]
    L.ghsvd_last_error.restype = ctypes.c_char_p
    L.ghsvd_destroy.argtypes = [P]
    L.ghsvd_destroy.restype = None
    L.ghsvd_version.restype = ctypes.c_char_p
    L.ghsvd_block_owner.argtypes = [Ci, Ci, Ci, Ci]
    L.ghsvd_exchange_plan.argtypes = [Ci, Ci, Ci, Ci, Ci, P, P, P, P, P, P]
    L.ghsvd_reduce_fallback_col.argtypes = [P]
    L.ghsvd_reduce_fallback_col.restype = I64
    L.ghsvd_order_steps.argtypes = [Ci, Ci, Ci]
    L.ghsvd_order_steps.restype = I64
    L.ghsvd_order_pair.argtypes = [Ci, Ci, Ci, I64, I64, ctypes.POINTER(I64), ctypes.POINTER(I64)]
    L.ghsvd_block_owner_ord.argtypes = [Ci, Ci, Ci, Ci, I64, Ci]
    L.ghsvd_exchange_plan_ord.argtypes = [Ci, Ci, Ci, Ci, Ci, I64, I64, P, P, P, P, P, P]
    L.ghsvd_nccl_unique_id.argtypes = [P]
    for f in ("ghsvd_create", "ghsvd_factor", "ghsvd_set_factors", "ghsvd_reduce", "ghsvd_get_factors",
              "ghsvd_sweep", "ghsvd_run_steps", "ghsvd_extract", "ghsvd_extract_local", "ghsvd_get_transformed",
              "ghsvd_get_state",
              "ghsvd_set_state", "ghsvd_hz2x2_batch"):
        getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _as_matrix(x, rows: int, cols: int):
    """(pointer, ld, keepalive) for a column-major complex128 matrix."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if x.dtype != torch.complex128:
                raise TypeError("expected torch.complex128")
            if tuple(x.shape) != (rows, cols):
                raise ValueError(f"expected shape {(rows, cols)}, got {tuple(x.shape)}")
            if x.stride(0) != 1 and cols > 1:
                raise ValueError("torch matrix must be column-major (stride(0) == 1)")
            ld = x.stride(1) if cols > 1 else rows
            return ctypes.c_void_p(x.data_ptr()), max(ld, rows), x
    except ImportError:
        pass
    a = np.asfortranarray(np.asarray(x, dtype=np.complex128))
    if a.shape != (rows, cols):
        raise ValueError(f"expected shape {(rows, cols)}, got {a.shape}")
    return a.ctypes.data_as(ctypes.c_void_p), rows, a


def _as_vec(x, n: int, dtype):
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if x.numel() != n or not x.is_contiguous():
                raise ValueError("bad vector")
            return ctypes.c_void_p(x.data_ptr()), x
    except ImportError:
        pass
    a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
    if a.size != n:
        raise ValueError(f"expected {n} entries, got {a.size}")
    return a.ctypes.data_as(ctypes.c_void_p), a


class Context:
    """One GHSVD problem on one GPU (one rank).  See include/ghsvd.h for semantics."""

    def __init__(self, m: int, n: int, nl: int = 0, *, variant: str = "pointwise", device: int = 0,
                 stream=None, world_size: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None,
                 nblocks: int = 0, max_sweeps: int = 30, criterion: str = "relative", eps: float = 0.0,
                 cluster: int = 0, threads: int = 0, use_graph: bool = True, kernel: int = 0,
                 detail_timing=False, want_x: bool = False, exchange_overlap: bool = False,
                 schedule: Optional[int] = None, groups: Optional[int] = None, gram_splits: Optional[int] = None,
                 trace_path: Optional[str] = None, ordering="rr", super_blocks: int = 0):
        import torch
        L = load()
        self._L = L
        o = Options()
        L.ghsvd_default_options(ctypes.byref(o))
        o.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        o.stream = ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        o.world_size = world_size
        o.rank = rank
        self._nccl_id = None
        if nccl_id is not None:
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        o.variant = VARIANTS[variant] if isinstance(variant, str) else int(variant)
        o.nblocks = nblocks
        o.ordering = ORDERINGS[ordering] if isinstance(ordering, str) else int(ordering)
        o.super_blocks = super_blocks
        o.max_sweeps = max_sweeps
        o.criterion = CRITERIA[criterion] if isinstance(criterion, str) else int(criterion)
        o.eps = eps
        o.cluster = cluster
        o.threads = threads
        o.use_graph = 1 if use_graph else 0
        o.kernel = kernel
        o.detail_timing = int(detail_timing)   # bool or 0 / 1 / 2 (see ghsvd.h)
        o.want_x = 1 if want_x else 0
        o.exchange_overlap = 1 if exchange_overlap else 0
        # None keeps ghsvd_default_options' value (seeded from the GHSVD_* environment knobs)
        if schedule is not None:
            o.schedule = int(schedule)
        if groups is not None:
            o.groups = int(groups)
        if gram_splits is not None:
            o.gram_splits = int(gram_splits)
        if trace_path is not None:
            self._trace_path = trace_path.encode()
            o.trace_path = self._trace_path
        self.opts = o
        nbytes = L.ghsvd_workspace_bytes(ctypes.byref(o), m, n, nl)
        if nbytes == 0:
            raise GHSVDError(-1, "ghsvd_workspace_bytes rejected the options/sizes")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
        self.m_cap, self.n_cap = m, n
        h = ctypes.c_void_p()
        rc = L.ghsvd_create(ctypes.byref(o), m, n, nl, ctypes.c_void_p(self.workspace.data_ptr()), nbytes,
                            ctypes.byref(h))
        if rc != 0:
            raise GHSVDError(rc, "ghsvd_create failed")
        self._h = h
        self.m = self.n = None

    # ----------------------------------------------------------------- helpers
    def _check(self, rc, what):
        if rc < 0:
            raise GHSVDError(rc, f"{what}: {self._L.ghsvd_last_error(self._h).decode()}")
        if rc == NOT_CONVERGED:
            warnings.warn(f"{what}: not converged within C_max sweeps")
        return rc

    def close(self):
        if getattr(self, "_h", None):
            self._L.ghsvd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --------------------------------------------------------------------- API
    def set_factors(self, F, J, G):
        m, n = F.shape
        pf, ldf, kf = _as_matrix(F, m, n)
        pg, ldg, kg = _as_matrix(G, m, n)
        pj, kj = _as_vec(J, m, np.int8)
        self._check(self._L.ghsvd_set_factors(self._h, m, n, pf, ldf, pj, pg, ldg), "set_factors")
        self.m, self.n = m, n

    def factor(self, A, B, U, TAA, TAB, TBB):
        """Phase 1.  A, B: (NA, NL, NG) complex; U: (NA, NL); T**: (NA, NL, NL).  numpy (host) or
        torch tensors laid out as NA blocks of column-major NL x NG (see ghsvd.h)."""
        NA, NL, NG = A.shape
        keep = []

        def blocks(X, r, c):
            try:
                import torch
                if isinstance(X, torch.Tensor):
                    keep.append(X)
                    return ctypes.c_void_p(X.data_ptr())
            except ImportError:
                pass
            a = np.ascontiguousarray(np.stack([np.asfortranarray(X[i]).ravel(order="F") for i in range(NA)]),
                                     dtype=np.complex128)
            keep.append(a)
            return a.ctypes.data_as(ctypes.c_void_p)

        pa, pb = blocks(A, NL, NG), blocks(B, NL, NG)
        pu, ku = _as_vec(np.asarray(U, dtype=np.float64).reshape(-1), NA * NL, np.float64)
        ptaa, ptab, ptbb = blocks(TAA, NL, NL), blocks(TAB, NL, NL), blocks(TBB, NL, NL)
        self._check(self._L.ghsvd_factor(self._h, NA, NL, NG, pa, pb, pu, ptaa, ptab, ptbb), "factor")
        self.m, self.n = 2 * NA * NL, NG

    def reduce(self, colpiv: bool = False, unblocked: Optional[bool] = None, colsearch: bool = False,
               own_qr: bool = False):
        """Phase 2; colpiv: column-pivoted QR of G P2 (GHSVD_REDUCE_COLPIV); unblocked: True forces
        the one-reflector-per-column form (GHSVD_REDUCE_UNBLOCKED), False the blocked one
        (GHSVD_REDUCE_BLOCKED), None lets the library choose by size (see ghsvd.h); colsearch:
        the blocked JQR searches its pivots on the columns instead of planning them on the
        J-Grammian (GHSVD_REDUCE_COLSEARCH); own_qr: the blocked form's plain QR of G P2 by this
        library's kernels instead of cuSOLVER's ZGEQRF (GHSVD_REDUCE_OWN_QR)."""
        fl = (1 if colpiv else 0) | (0 if unblocked is None else (2 if unblocked else 4)) | (8 if colsearch else 0) | \
            (16 if own_qr else 0)
        self._check(self._L.ghsvd_reduce(self._h, fl), "reduce")
        self.reduce_fallback_col = int(self._L.ghsvd_reduce_fallback_col(self._h))
        self.m = self.n

    def get_factors(self):
        """-> (F, J, G, p2) numpy; F, G as the sweep starts (J-sorted rows, reduced, bordered)."""
        m, n = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._L.ghsvd_get_factors(self._h, ctypes.byref(m), ctypes.byref(n), None, 0, None, None, 0,
                                              None), "get_factors")
        m, n = m.value, n.value
        F = np.zeros((m, n), np.complex128, order="F")
        G = np.zeros((m, n), np.complex128, order="F")
        J = np.zeros(m, np.int8)
        p2 = np.zeros(self.n, np.int64)
        self._check(self._L.ghsvd_get_factors(self._h, None, None, F.ctypes.data_as(ctypes.c_void_p), m,
                                              J.ctypes.data_as(ctypes.c_void_p), G.ctypes.data_as(ctypes.c_void_p),
                                              m, p2.ctypes.data_as(ctypes.c_void_p)), "get_factors")
        return F, J, G, p2

    def export_factors(self, F, J, G):
        """Copy the starting factors into preallocated (m x n column-major) F, G and J (m int8),
        host or device (torch) buffers; returns (m, n)."""
        m, n = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._L.ghsvd_get_factors(self._h, ctypes.byref(m), ctypes.byref(n), None, 0, None, None, 0,
                                              None), "get_factors")
        pf, ldf, _ = _as_matrix(F, m.value, n.value)
        pg, ldg, _ = _as_matrix(G, m.value, n.value)
        pj, _ = _as_vec(J, m.value, np.int8)
        self._check(self._L.ghsvd_get_factors(self._h, None, None, pf, ldf, pj, pg, ldg, None), "get_factors")
        return m.value, n.value

    def factor_shape(self):
        m, n = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._L.ghsvd_get_factors(self._h, ctypes.byref(m), ctypes.byref(n), None, 0, None, None, 0,
                                              None), "get_factors")
        return m.value, n.value

    def sweep(self) -> dict:
        st = Stats()
        rc = self._check(self._L.ghsvd_sweep(self._h, ctypes.byref(st)), "sweep")
        d = st.todict()
        d["status"] = rc
        return d

    def run_steps(self, s0: int, ns: int):
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self._L.ghsvd_run_steps(self._h, s0, ns, ctypes.byref(a), ctypes.byref(b)), "run_steps")
        return a.value, b.value

    def extract(self, want_z: bool = True, out=None):
        """-> (lambda, sigma_f, sigma_g, Z) numpy (Z None if not wanted).  ``out`` may pass
        preallocated (torch/numpy) buffers (lam, sf, sg, Z)."""
        n = self.n
        if out is None:
            lam, sf, sg = np.zeros(n), np.zeros(n), np.zeros(n)
            Z = np.zeros((n, n), np.complex128, order="F") if want_z else None
        else:
            lam, sf, sg, Z = out
        pl, _ = _as_vec(lam, n, np.float64)
        ps, _ = _as_vec(sf, n, np.float64)
        pg, _ = _as_vec(sg, n, np.float64)
        if Z is not None:
            pz, ldz, _ = _as_matrix(Z, n, n)
        else:
            pz, ldz = None, n
        self._check(self._L.ghsvd_extract(self._h, pl, ps, pg, pz, ldz, None), "extract")
        return lam, sf, sg, Z

    def extract_local(self, want_z: bool = True):
        """Distributed form (ghsvd_extract_local): -> (lambda, sigma_f, sigma_g, Z_local n x ncols,
        col_ids) numpy; Z_local holds only this rank's columns, col_ids their global indices."""
        n = self.n
        lam, sf, sg = np.zeros(n), np.zeros(n), np.zeros(n)
        Z = np.zeros((n, n), np.complex128, order="F") if want_z else None
        ids = np.zeros(n, np.int64)
        nc = ctypes.c_int64()
        P = ctypes.c_void_p
        self._check(self._L.ghsvd_extract_local(self._h, lam.ctypes.data_as(P), sf.ctypes.data_as(P),
                                                sg.ctypes.data_as(P), None if Z is None else Z.ctypes.data_as(P),
                                                n, ids.ctypes.data_as(P), ctypes.byref(nc)), "extract_local")
        k = nc.value
        return lam, sf, sg, (None if Z is None else Z[:, :k].copy(order="F")), ids[:k].copy()

    def extract_x(self):
        """X = Z^{-1} (n x n numpy), requires want_x=True and a completed sweep."""
        n = self.n
        X = np.zeros((n, n), np.complex128, order="F")
        self._check(self._L.ghsvd_extract_x(self._h, X.ctypes.data_as(ctypes.c_void_p), n), "extract_x")
        return X

    def transformed(self, m: int, n: int):
        """Current F', G', Z' (bordered sizes m, n) as numpy."""
        F = np.zeros((m, n), np.complex128, order="F")
        G = np.zeros((m, n), np.complex128, order="F")
        Z = np.zeros((n, n), np.complex128, order="F")
        self._check(self._L.ghsvd_get_transformed(self._h, F.ctypes.data_as(ctypes.c_void_p), m,
                                                  G.ctypes.data_as(ctypes.c_void_p), m,
                                                  Z.ctypes.data_as(ctypes.c_void_p), n), "get_transformed")
        return F, G, Z

    def get_state(self) -> dict:
        """Checkpoint of the sweep state (numpy): F', G' (bordered m x n), Z' and, with
        want_x, W^T (n x n).  See ghsvd_get_state."""
        m, n = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._L.ghsvd_get_factors(self._h, ctypes.byref(m), ctypes.byref(n), None, 0, None, None, 0,
                                              None), "get_factors")
        m, n = m.value, n.value
        st = {"F": np.zeros((m, n), np.complex128, order="F"), "G": np.zeros((m, n), np.complex128, order="F"),
              "Z": np.zeros((n, n), np.complex128, order="F"),
              "W": np.zeros((n, n), np.complex128, order="F") if self.opts.want_x else None}
        p = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)   # noqa: E731
        self._check(self._L.ghsvd_get_state(self._h, p(st["F"]), m, p(st["G"]), m, p(st["Z"]), n, p(st["W"]), n),
                    "get_state")
        return st

    def set_state(self, st: dict):
        """Restore a get_state() checkpoint; the next sweep() resumes from it."""
        F, G, Z, W = (np.asfortranarray(st[k]) if st.get(k) is not None else None for k in ("F", "G", "Z", "W"))
        p = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)   # noqa: E731
        self._check(self._L.ghsvd_set_state(self._h, p(F), F.shape[0], p(G), G.shape[0], p(Z), Z.shape[0], p(W),
                                            Z.shape[0]), "set_state")

    def hz2x2_batch(self, pivots: np.ndarray, tol: float, criterion: int = 0):
        """Evaluate the device 2x2 transformation on (count, 8) pivots -> (Z (count, 8), kind)."""
        import torch
        x = torch.from_numpy(np.ascontiguousarray(pivots, dtype=np.float64)).cuda(self.opts.device)
        cnt = x.shape[0]
        out = torch.empty((cnt, 8), dtype=torch.float64, device=x.device)
        kind = torch.empty(cnt, dtype=torch.int32, device=x.device)
        self._check(self._L.ghsvd_hz2x2_batch(self._h, cnt, ctypes.c_void_p(x.data_ptr()), tol, criterion,
                                              ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(kind.data_ptr())),
                    "hz2x2_batch")
        return out.cpu().numpy(), kind.cpu().numpy()


def block_owner(nblk: int, world: int, s: int, b: int) -> int:
    return load().ghsvd_block_owner(nblk, world, s, b)


def order_steps(ordering, nblk: int, nsup: int = 0) -> int:
    """Block steps per sweep of a block ordering (csrc/ordering.h); -1 on bad arguments."""
    o = ORDERINGS[ordering] if isinstance(ordering, str) else int(ordering)
    return int(load().ghsvd_order_steps(o, nblk, nsup))


def order_pair(ordering, nblk: int, nsup: int, s: int, k: int):
    """Block pair (p < q) of slot k in block step s (csrc/ordering.h)."""
    o = ORDERINGS[ordering] if isinstance(ordering, str) else int(ordering)
    p, q = ctypes.c_int64(), ctypes.c_int64()
    if load().ghsvd_order_pair(o, nblk, nsup, s, k, ctypes.byref(p), ctypes.byref(q)) != 0:
        raise GHSVDError(-1, "order_pair: bad arguments")
    return p.value, q.value


def block_owner_ord(ordering, nblk: int, nsup: int, world: int, s: int, b: int) -> int:
    o = ORDERINGS[ordering] if isinstance(ordering, str) else int(ordering)
    return load().ghsvd_block_owner_ord(o, nblk, nsup, world, s, b)


def exchange_plan(nblk: int, world: int, rank: int, s: int, s_next: int, ordering="rr", nsup: int = 0):
    """-> (sends [(block, peer)], recvs [(block, peer)]) between block steps s and s_next."""
    L = load()
    o = ORDERINGS[ordering] if isinstance(ordering, str) else int(ordering)
    arr = [np.zeros(nblk, np.int64) for _ in range(4)]
    ns, nr = ctypes.c_int64(), ctypes.c_int64()
    rc = L.ghsvd_exchange_plan_ord(o, nblk, nsup, world, rank, s, s_next,
                                   *[a.ctypes.data_as(ctypes.c_void_p) for a in arr[:2]],
                                   ctypes.byref(ns), *[a.ctypes.data_as(ctypes.c_void_p) for a in arr[2:]],
                                   ctypes.byref(nr))
    if rc != 0:
        raise GHSVDError(-1, "exchange_plan: bad arguments")
    sends = list(zip(arr[0][:ns.value].tolist(), arr[1][:ns.value].tolist()))
    recvs = list(zip(arr[2][:nr.value].tolist(), arr[3][:nr.value].tolist()))
    return sends, recvs


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = load().ghsvd_nccl_unique_id(buf)
    if rc != 0:
        raise GHSVDError(rc, "ncclGetUniqueId failed (NCCL not loadable)")
    return buf.raw


def loopback_id(key: str) -> bytes:
    """128-byte id of the loopback test transport (include/ghsvd.h, nccl_id): the ranks of
    group `key` are contexts of this process on one device, each driven by its own thread."""
    k = key.encode()
    if len(k) > 112:
        raise ValueError("loopback key longer than 112 bytes")
    return b"GHSVD-LOOPBACK\0\0" + k + b"\0" * (112 - len(k))


def version() -> str:
    return load().ghsvd_version().decode()
